mkdir -p gpurun_out
for s in 4841 5987; do timeout 300 python tools/fuzz_diag.py $s > gpurun_out/r02za_diag_$s.txt 2>&1; done
