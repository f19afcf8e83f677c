mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_swarm.py tests/test_gpu_multishard.py -x -q > gpurun_out/cfg5d_test.log 2>&1; echo "rc=$?" >> gpurun_out/cfg5d_test.log; tail -2 gpurun_out/cfg5d_test.log
for v in ql1 ql2 ql8; do SWARMSTEP_B200_LIB_OVERRIDE=tools/variants/$v.so timeout 300 python tools/swarm_bench.py 100000 200 nccl > gpurun_out/cfg5d_$v.json 2>&1; done
timeout 300 python tools/swarm_bench.py 100000 200 nccl > gpurun_out/cfg5d_ql4.json 2>&1
for v in ql1 ql2 ql4 ql8; do echo $v; cat gpurun_out/cfg5d_$v.json; done
