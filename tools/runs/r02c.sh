# round 2: packed compensated-position word + per-tick snap + rare-case branches in the outer loop
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r02c_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02c_gputest.log
for N in 4000000 1000000; do
  timeout 900 python tools/tune.py $N tools/variants/e23.so tools/variants/pk.so tools/variants/pk_nosnap.so > gpurun_out/r02c_tune_$N.txt 2>&1
done
python tools/profile_step.py 10 2000000 > gpurun_out/r02c_prof.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quad_step -s 3 -c 1 -o gpurun_out/r02c_k10 -f python tools/profile_step.py 10 2000000 >> gpurun_out/r02c_prof.log 2>&1
python tools/profile_step.py 1 10000000 >> gpurun_out/r02c_prof.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quad_step -s 3 -c 1 -o gpurun_out/r02c_k1 -f python tools/profile_step.py 1 10000000 >> gpurun_out/r02c_prof.log 2>&1
