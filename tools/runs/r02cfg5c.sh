mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:query_kernel -s 10 -c 1 -o gpurun_out/q_old -f python tools/swarm_bench.py 100000 20 nccl > gpurun_out/q_old.log 2>&1
SWARMSTEP_B200_LIB_OVERRIDE=tools/variants/q2.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:query_kernel -s 10 -c 1 -o gpurun_out/q_new -f python tools/swarm_bench.py 100000 20 nccl > gpurun_out/q_new.log 2>&1
tail -1 gpurun_out/q_old.log gpurun_out/q_new.log
