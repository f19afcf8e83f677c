# round 2: persistent TMA-prefetching pair kernel (v5pf) vs v3 / v4
mkdir -p gpurun_out
V=tools/variants
for N in 10000000 1000000; do
  timeout 900 python tools/tune.py $N $V/v3.so $V/v4.so $V/v5pf.so > gpurun_out/r02j_tune_$N.txt 2>&1
done
SWARMSTEP_B200_LIB_OVERRIDE=$V/v5pf.so timeout 300 python tools/kscale.py 10000000 10 40 200 > gpurun_out/r02j_kscale_10m_pf.json 2>&1
SWARMSTEP_B200_LIB_OVERRIDE=$V/v5pf.so timeout 300 python tools/kscale.py 1000000 10 40 200 > gpurun_out/r02j_kscale_1m_pf.json 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02j_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02j_gputest.log
