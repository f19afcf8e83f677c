# round 2: packed lo + launch-local position accumulator + full-rate RK4 + sparse q_err
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02f_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02f_gputest.log
timeout 900 python bench.py > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err
python tools/profile_step.py 10 2000000 > gpurun_out/r02f_prof.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quad_step -s 3 -c 1 -o gpurun_out/r02f_k10 -f python tools/profile_step.py 10 2000000 >> gpurun_out/r02f_prof.log 2>&1
python tools/profile_step.py 1 10000000 >> gpurun_out/r02f_prof.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quad_step -s 3 -c 1 -o gpurun_out/r02f_k1 -f python tools/profile_step.py 1 10000000 >> gpurun_out/r02f_prof.log 2>&1
