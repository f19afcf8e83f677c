mkdir -p gpurun_out
timeout 600 python tools/latency_bench.py gpurun_out/pdl7_latency_on.json > /dev/null 2>gpurun_out/pdl7_latency.err
SWARMSTEP_B200_NO_OVERLAP=1 timeout 600 python tools/latency_bench.py gpurun_out/pdl7_latency_off.json > /dev/null 2>&1
