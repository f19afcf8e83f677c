# round 2: v6 = v4 + adjacent-row pairs with 8-byte column accesses
mkdir -p gpurun_out
V=tools/variants
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02m_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02m_gputest.log
for N in 10000000 1000000; do
  timeout 900 python tools/tune.py $N $V/v3.so $V/v4.so $V/v6.so > gpurun_out/r02m_tune_$N.txt 2>&1
done
timeout 900 python bench.py > gpurun_out/r02m_bench.json 2> gpurun_out/r02m_bench.err
