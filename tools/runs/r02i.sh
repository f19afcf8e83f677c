# round 2: v3 vs v4 (axisymmetric-vehicle constants, structured realized wrench, one sincos per launch);
# per-launch overhead at 10M (ticks per launch sweep)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02i_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02i_gputest.log
V=tools/variants
for N in 10000000 1000000; do
  timeout 900 python tools/tune.py $N $V/v3.so $V/v4.so > gpurun_out/r02i_tune_$N.txt 2>&1
done
timeout 300 python tools/kscale.py 10000000 1 10 40 200 > gpurun_out/r02i_kscale_10m.json 2>&1
timeout 900 python bench.py > gpurun_out/r02i_bench.json 2> gpurun_out/r02i_bench.err
