# round 2: prefetching pair kernel with the max shared-memory carveout
mkdir -p gpurun_out
V=tools/variants
export SSB_DEBUG_OCC=1
for N in 10000000 1000000; do
  timeout 900 python tools/tune.py $N $V/v4.so $V/v5pf.so $V/v5pf_7.so > gpurun_out/r02k_tune_$N.txt 2>&1
done
SWARMSTEP_B200_LIB_OVERRIDE=$V/v5pf.so timeout 300 python tools/kscale.py 10000000 10 40 200 > gpurun_out/r02k_kscale_10m_pf.json 2>&1
