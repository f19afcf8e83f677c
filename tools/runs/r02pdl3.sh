mkdir -p gpurun_out
for i in 1 2 3; do
  timeout 300 python bench.py --agents 1000000 --no-cpu-baseline --no-k1 > gpurun_out/pdl3_on_$i.json 2>/dev/null
  SWARMSTEP_B200_NO_OVERLAP=1 timeout 300 python bench.py --agents 1000000 --no-cpu-baseline --no-k1 > gpurun_out/pdl3_off_$i.json 2>/dev/null
done
