mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_overlap.py tests/test_gpu_feed.py -x -q > gpurun_out/pdl4_test.log 2>&1; echo "tests rc=$?" >> gpurun_out/pdl4_test.log
tail -3 gpurun_out/pdl4_test.log
grep -q "rc=0" gpurun_out/pdl4_test.log || exit 1
timeout 600 python tools/latency_bench.py gpurun_out/pdl4_latency_on.json > /dev/null 2>gpurun_out/pdl4_latency_on.err
SWARMSTEP_B200_NO_OVERLAP=1 timeout 600 python tools/latency_bench.py gpurun_out/pdl4_latency_off.json > /dev/null 2>&1
NSWEEP_KS=10 timeout 600 python tools/nsweep.py > gpurun_out/pdl4_nsweep_on.jsonl 2>&1
NSWEEP_KS=10 SWARMSTEP_B200_NO_OVERLAP=1 timeout 600 python tools/nsweep.py > gpurun_out/pdl4_nsweep_off.jsonl 2>&1
