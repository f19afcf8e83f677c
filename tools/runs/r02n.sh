# round 2: v7 = v6 + rotation-advanced fused circle feed + split translation units;
# ablations of v4's changes (v6w: FMA realized wrench, v6g: per-axis gain constants, v6y: two sincos)
mkdir -p gpurun_out
V=tools/variants
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02n_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02n_gputest.log
timeout 900 python tools/tune.py 10000000 $V/v6.so $V/v6w.so $V/v6g.so $V/v6y.so $V/v7.so > gpurun_out/r02n_tune_10000000.txt 2>&1
timeout 600 python tools/latency_bench.py gpurun_out/r02n_latency.json > gpurun_out/r02n_latency.log 2>&1
timeout 900 python bench.py > gpurun_out/r02n_bench.json 2> gpurun_out/r02n_bench.err
