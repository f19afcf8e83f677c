# round 2: packed lo with a per-tick snap (two forms) vs without
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02d_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02d_gputest.log
for N in 4000000 10000000; do
  timeout 900 python tools/tune.py $N tools/variants/pk2_nosnap.so tools/variants/pk2_snapA.so tools/variants/pk2_snapB.so > gpurun_out/r02d_tune_$N.txt 2>&1
done
timeout 900 python bench.py > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err
