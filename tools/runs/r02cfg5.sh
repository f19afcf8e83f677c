mkdir -p gpurun_out
timeout 300 python tools/swarm_bench.py 100000 200 nccl > gpurun_out/cfg5_base.json 2>&1
cat gpurun_out/cfg5_base.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg5_launches.csv python tools/swarm_bench.py 100000 20 nccl > gpurun_out/cfg5_ncu.log 2>&1
python tools/launch_share.py gpurun_out/cfg5_launches.csv | head -20
