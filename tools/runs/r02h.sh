# round 2: evidence with the v3 kernels -- parity report, latency vs N, cfg3 (1M) bench line,
# step time vs N, config 5, reference arm
mkdir -p gpurun_out
timeout 900 python tools/parity_report.py gpurun_out/r02h_parity.json > gpurun_out/r02h_parity.log 2>&1
timeout 600 python tools/latency_bench.py gpurun_out/r02h_latency.json > gpurun_out/r02h_latency.log 2>&1
timeout 600 python bench.py --agents 1000000 --no-cpu-baseline > gpurun_out/r02h_bench_1m.json 2> gpurun_out/r02h_bench_1m.err
timeout 600 python tools/nsweep.py > gpurun_out/r02h_nsweep.jsonl 2> gpurun_out/r02h_nsweep.err
timeout 300 python tools/kscale.py 1000000 1 10 40 200 > gpurun_out/r02h_kscale_1m.json 2>&1
timeout 300 python tools/swarm_bench.py 100000 200 nccl > gpurun_out/r02h_swarm_nccl.json 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/r02h_ref.json 2> gpurun_out/r02h_ref.err
