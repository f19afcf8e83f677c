# round 2: L2 bulk prefetch of the next round's tile in the pair kernel (distance in quarters of the resident CTAs)
mkdir -p gpurun_out
V=tools/variants
for N in 10000000 1000000; do
  timeout 900 python tools/tune.py $N $V/l2a0.so $V/l2a2.so $V/l2a4.so $V/l2a8.so > gpurun_out/r02l_tune_$N.txt 2>&1
done
for L in l2a0 l2a4; do
  SWARMSTEP_B200_LIB_OVERRIDE=$V/$L.so timeout 300 python tools/kscale.py 10000000 10 40 200 > gpurun_out/r02l_kscale_10m_$L.json 2>&1
done
