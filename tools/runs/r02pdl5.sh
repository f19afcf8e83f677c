mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_overlap.py -x -q > gpurun_out/pdl5_test.log 2>&1; echo "tests rc=$?" >> gpurun_out/pdl5_test.log
tail -2 gpurun_out/pdl5_test.log
timeout 600 python tools/latency_bench.py gpurun_out/pdl5_latency.json > /dev/null 2>gpurun_out/pdl5_latency.err
