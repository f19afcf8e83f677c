mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_overlap.py -x -q > gpurun_out/pdl_test.log 2>&1; echo "overlap tests rc=$?" >> gpurun_out/pdl_test.log
tail -3 gpurun_out/pdl_test.log
grep -q "rc=0" gpurun_out/pdl_test.log || exit 1
for n in 10000000 1000000; do
  timeout 300 python bench.py --agents $n --no-cpu-baseline > gpurun_out/pdl_on_$n.json 2>gpurun_out/pdl_on_$n.err
  SWARMSTEP_B200_NO_OVERLAP=1 timeout 300 python bench.py --agents $n --no-cpu-baseline > gpurun_out/pdl_off_$n.json 2>gpurun_out/pdl_off_$n.err
done
timeout 300 python tools/kscale.py 10000000 1 10 40 > gpurun_out/pdl_kscale_on.json 2>&1
SWARMSTEP_B200_NO_OVERLAP=1 timeout 300 python tools/kscale.py 10000000 1 10 40 > gpurun_out/pdl_kscale_off.json 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pdl_gpu_suite.log 2>&1; tail -3 gpurun_out/pdl_gpu_suite.log
