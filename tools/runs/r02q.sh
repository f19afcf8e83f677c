# round 2 final evidence with the v9 code: headline bench, reference arm, parity report, N / K sweeps, cfg5
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02q_smi.txt
nproc >> gpurun_out/r02q_smi.txt
timeout 900 python bench.py > gpurun_out/r02q_bench.json 2> gpurun_out/r02q_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r02q_ref.json 2> gpurun_out/r02q_ref.err
timeout 900 python tools/parity_report.py gpurun_out/r02q_parity.json > gpurun_out/r02q_parity.log 2>&1
timeout 600 python tools/nsweep.py > gpurun_out/r02q_nsweep.jsonl 2> gpurun_out/r02q_nsweep.err
timeout 300 python tools/kscale.py 1000000 10 40 200 > gpurun_out/r02q_kscale_1m.json 2>&1
timeout 300 python tools/kscale.py 10000000 10 40 200 > gpurun_out/r02q_kscale_10m.json 2>&1
timeout 300 python tools/swarm_bench.py 100000 200 nccl > gpurun_out/r02q_swarm_nccl.json 2>&1
