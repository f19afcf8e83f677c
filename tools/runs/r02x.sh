# round 2: fused circle launches without the per-launch fill / counter copy
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02x_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02x_gputest.log
timeout 600 python tools/latency_bench.py gpurun_out/r02x_latency.json > gpurun_out/r02x_latency.log 2>&1
