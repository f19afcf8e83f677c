# round 2: v8 = v7 with two sincos per launch; full GPU suite, bench, ncu of the K=10 and K=1 kernels, latency
mkdir -p gpurun_out
V=tools/variants
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02o_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02o_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02o_smoke.log 2>&1
timeout 900 python tools/tune.py 10000000 $V/v6.so $V/v6y.so $V/v8.so > gpurun_out/r02o_tune_10000000.txt 2>&1
timeout 900 python bench.py > gpurun_out/r02o_bench.json 2> gpurun_out/r02o_bench.err
timeout 600 python tools/latency_bench.py gpurun_out/r02o_latency.json > gpurun_out/r02o_latency.log 2>&1
python tools/profile_step.py 10 2000000 > gpurun_out/r02o_prof.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quad_step -s 3 -c 1 -o gpurun_out/r02o_k10 -f python tools/profile_step.py 10 2000000 >> gpurun_out/r02o_prof.log 2>&1
python tools/profile_step.py 1 10000000 >> gpurun_out/r02o_prof.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quad_step -s 3 -c 1 -o gpurun_out/r02o_k1 -f python tools/profile_step.py 1 10000000 >> gpurun_out/r02o_prof.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02o_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r02o_ncu_bench.log 2>&1
