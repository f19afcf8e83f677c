# round 2: v9 = v8 + axisymmetric circle kernels; new tests (non-axisymmetric vehicle, packed low part)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02p_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02p_gputest.log
timeout 600 python tools/latency_bench.py gpurun_out/r02p_latency.json > gpurun_out/r02p_latency.log 2>&1
timeout 600 python bench.py --agents 1000000 --no-cpu-baseline > gpurun_out/r02p_bench_1m.json 2> gpurun_out/r02p_bench_1m.err
