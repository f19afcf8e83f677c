# round 2: position-lo layout (float / packed) x launch-local accumulator x per-tick snap,
# and the pair kernel's setpoints in shared memory at 8/9/10 CTAs per SM
mkdir -p gpurun_out
V=tools/variants
for N in 4000000 10000000 1000000; do
  timeout 1200 python tools/tune.py $N $V/lay0.so $V/lay0acc.so $V/lay1.so $V/lay1acc.so $V/lay1snap.so $V/usm8.so $V/usm9.so $V/usm10.so > gpurun_out/r02e_tune_$N.txt 2>&1
done
