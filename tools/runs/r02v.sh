# round 2: fuzz soak with the final kernels (2000 random swarms per-step vs the oracle + kernel/fusion identity)
mkdir -p gpurun_out
SWARMSTEP_FUZZ_SEEDS=2000 timeout 2400 python -m pytest tests/test_gpu_fuzz.py -q -p no:cacheprovider > gpurun_out/r02v_fuzz_soak.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02v_fuzz_soak.txt
