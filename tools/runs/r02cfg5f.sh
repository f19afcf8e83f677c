mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_swarm.py tests/test_gpu_multishard.py tests/test_gpu_collision.py -x -q > gpurun_out/cfg5f_test.log 2>&1; echo "rc=$?" >> gpurun_out/cfg5f_test.log; tail -2 gpurun_out/cfg5f_test.log
timeout 300 python tools/swarm_bench.py 100000 200 nccl > gpurun_out/cfg5f.json 2>&1; cat gpurun_out/cfg5f.json
timeout 300 python tools/swarm_bench.py 100000 200 p2p > gpurun_out/cfg5f_p2p.json 2>&1; cat gpurun_out/cfg5f_p2p.json
