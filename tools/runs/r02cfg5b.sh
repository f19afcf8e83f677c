mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_swarm.py tests/test_gpu_multishard.py -x -q > gpurun_out/cfg5b_test.log 2>&1; echo "rc=$?" >> gpurun_out/cfg5b_test.log; tail -2 gpurun_out/cfg5b_test.log
timeout 300 python tools/swarm_bench.py 100000 200 nccl > gpurun_out/cfg5b.json 2>&1; cat gpurun_out/cfg5b.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg5b_launches.csv python tools/swarm_bench.py 100000 20 nccl > gpurun_out/cfg5b_ncu.log 2>&1
python tools/launch_share.py gpurun_out/cfg5b_launches.csv | head -8
