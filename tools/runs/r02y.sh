# round 2 final: the driver's sequence -- GPU suite, smoke, bench (default), reference arm; ncu launch list
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02y_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02y_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02y_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r02y_bench.json 2> gpurun_out/r02y_bench.err
timeout 900 python bench.py --impl reference > gpurun_out/r02y_ref.json 2> gpurun_out/r02y_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02y_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/r02y_ncu_bench.log 2>&1
