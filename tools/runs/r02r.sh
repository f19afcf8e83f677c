# round 2: v10 = v9 + explicitly rounded (paired) sincos for the per-launch yaw terms and the circle feed
mkdir -p gpurun_out
V=tools/variants
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02r_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02r_gputest.log
for N in 10000000 1000000; do
  timeout 900 python tools/tune.py $N $V/v9.so $V/v10.so > gpurun_out/r02r_tune_$N.txt 2>&1
done
timeout 900 python bench.py > gpurun_out/r02r_bench.json 2> gpurun_out/r02r_bench.err
timeout 600 python tools/latency_bench.py gpurun_out/r02r_latency.json > gpurun_out/r02r_latency.log 2>&1
