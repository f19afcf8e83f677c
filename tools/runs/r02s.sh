# round 2: macro-free kernels (chosen paths only), bench with the informative device-feed e2e
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02s_gputest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02s_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02s_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r02s_bench.json 2> gpurun_out/r02s_bench.err
