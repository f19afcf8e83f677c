mkdir -p gpurun_out
python tools/profile_circle.py 5000 10 || exit 1
ncu --set full --clock-control none --import-source on -k regex:quad_step_pair -s 2 -c 2 -o gpurun_out/circ5k python tools/profile_circle.py 5000 10 > gpurun_out/circ5k.log 2>&1
tail -3 gpurun_out/circ5k.log
