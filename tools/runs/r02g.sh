# round 2: v1 (committed) vs v2 (Derived constants, NaN-propagating motor clip, sign folded into the
# axis-angle factor, -z'1 computed directly) vs v3 (+ axisymmetric-inertia specialisation)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/r02g_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02g_gputest.log
V=tools/variants
for N in 10000000 1000000; do
  timeout 900 python tools/tune.py $N $V/v1.so $V/v2.so $V/v3.so > gpurun_out/r02g_tune_$N.txt 2>&1
done
timeout 900 python bench.py > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err
python tools/profile_step.py 10 2000000 > gpurun_out/r02g_prof.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quad_step -s 3 -c 1 -o gpurun_out/r02g_k10 -f python tools/profile_step.py 10 2000000 >> gpurun_out/r02g_prof.log 2>&1
