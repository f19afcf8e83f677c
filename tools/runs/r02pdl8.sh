mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pdl8_gpu_suite.log 2>&1; tail -2 gpurun_out/pdl8_gpu_suite.log
timeout 600 python bench.py > gpurun_out/pdl8_bench.json 2>gpurun_out/pdl8_bench.err
timeout 300 python bench.py --agents 1000000 --no-cpu-baseline > gpurun_out/pdl8_bench_1m.json 2>/dev/null
timeout 600 python tools/latency_bench.py gpurun_out/pdl8_latency.json > /dev/null 2>&1
timeout 300 python tools/kscale.py 10000000 1 10 40 200 > gpurun_out/pdl8_kscale_10m.json 2>&1
timeout 300 python tools/kscale.py 1000000 1 10 40 200 > gpurun_out/pdl8_kscale_1m.json 2>&1
NSWEEP_KS=10 timeout 600 python tools/nsweep.py > gpurun_out/pdl8_nsweep.jsonl 2>&1
