mkdir -p gpurun_out
timeout 600 python tools/overlap_probe.py 1000000 > gpurun_out/r02zd_overlap_1m.json 2>&1
timeout 600 python tools/overlap_probe.py 10000000 > gpurun_out/r02zd_overlap_10m.json 2>&1
