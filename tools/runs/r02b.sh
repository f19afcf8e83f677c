# round 2, session 4: parity of the restructured RK4 position update + closed-form q_des,
# and A/B of kernel variants (base = round-1 arithmetic)
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02b_smi.txt
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02b_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02b_gputest.log
for N in 4000000 1000000; do
  timeout 900 python tools/tune.py $N tools/variants/base.so tools/variants/e2.so tools/variants/e23.so tools/variants/e23p.so > gpurun_out/r02b_tune_$N.txt 2>&1
done
