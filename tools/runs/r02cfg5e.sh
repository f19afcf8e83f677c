mkdir -p gpurun_out
for v in nb0 nb1 nb2 nb3 nb4; do SWARMSTEP_B200_LIB_OVERRIDE=tools/variants/$v.so timeout 300 python tools/swarm_bench.py 100000 200 nccl > gpurun_out/cfg5e_$v.json 2>&1; done
timeout 300 python tools/swarm_bench.py 100000 200 nccl > gpurun_out/cfg5e_full.json 2>&1
for v in nb0 nb1 nb2 nb3 nb4 full; do echo $v $(python -c "import json;d=json.loads(open('gpurun_out/cfg5e_$v.json').read().strip().splitlines()[-1]);print(d['graph_ms_per_tick']*1e3, d['device_ms_per_tick']*1e3)"); done
