# round 2, after overlapped launches: the driver's sequence, ncu launch list, ncu --set full of both step kernels
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fin2_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/fin2_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin2_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/fin2_smoke.log
timeout 900 python bench.py > gpurun_out/fin2_bench.json 2> gpurun_out/fin2_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/fin2_ref.json 2> gpurun_out/fin2_ref.err
timeout 300 python bench.py --agents 1000000 --no-cpu-baseline > gpurun_out/fin2_bench_1m.json 2>/dev/null
timeout 600 python tools/latency_bench.py gpurun_out/fin2_latency.json > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin2_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/fin2_ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quad_step -s 3 -c 1 -o gpurun_out/fin2_k10 -f python tools/profile_step.py 10 2000000 > gpurun_out/fin2_prof.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:quad_step -s 3 -c 1 -o gpurun_out/fin2_k1 -f python tools/profile_step.py 1 10000000 >> gpurun_out/fin2_prof.log 2>&1
