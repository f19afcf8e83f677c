# round 2: ptxas register-usage levels and 7 CTAs/SM for the paired kernel
mkdir -p gpurun_out
V=tools/variants
timeout 1200 python tools/tune.py 10000000 $V/base.so $V/rul3.so $V/rul6.so $V/rul10.so $V/minb7.so > gpurun_out/r02t_tune_10000000.txt 2>&1
