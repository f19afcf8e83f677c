# round 2: no per-launch fault-counter read-back (one copy per collect)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02w_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02w_gputest.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02w_bench.json 2> gpurun_out/r02w_bench.err
timeout 600 python bench.py --agents 1000000 --no-cpu-baseline > gpurun_out/r02w_bench_1m.json 2> gpurun_out/r02w_bench_1m.err
timeout 300 python tools/kscale.py 1000000 10 40 200 > gpurun_out/r02w_kscale_1m.json 2>&1
