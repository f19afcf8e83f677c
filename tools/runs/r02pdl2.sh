mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_overlap.py tests/test_gpu_parity.py -x -q > gpurun_out/pdl2_test.log 2>&1; echo "tests rc=$?" >> gpurun_out/pdl2_test.log
tail -3 gpurun_out/pdl2_test.log
grep -q "rc=0" gpurun_out/pdl2_test.log || exit 1
timeout 600 python bench.py > gpurun_out/pdl2_bench.json 2>gpurun_out/pdl2_bench.err
for n in 1000000 100000; do
  timeout 300 python bench.py --agents $n --no-cpu-baseline > gpurun_out/pdl2_on_$n.json 2>gpurun_out/pdl2_on_$n.err
  SWARMSTEP_B200_NO_OVERLAP=1 timeout 300 python bench.py --agents $n --no-cpu-baseline > gpurun_out/pdl2_off_$n.json 2>gpurun_out/pdl2_off_$n.err
done
