mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_overlap.py tests/test_gpu_feed.py -x -q > gpurun_out/pdl6_test.log 2>&1; echo "tests rc=$?" >> gpurun_out/pdl6_test.log
tail -2 gpurun_out/pdl6_test.log
grep -q "rc=0" gpurun_out/pdl6_test.log || exit 1
timeout 600 python tools/latency_bench.py gpurun_out/pdl6_latency.json > /dev/null 2>gpurun_out/pdl6_latency.err
