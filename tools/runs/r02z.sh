# round 2: memcheck of the final kernels (if the pool allows compute-sanitizer), bigger fuzz soak
mkdir -p gpurun_out
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/r02z_memcheck.txt 2>&1
PYTORCH_NO_CUDA_MEMORY_CACHING=1 CUDA_LAUNCH_BLOCKING=1 timeout 600 python tools/sanitize_run.py > gpurun_out/r02z_nocache.txt 2>&1
echo "nocache rc=$?" >> gpurun_out/r02z_nocache.txt
echo "memcheck rc=$?" >> gpurun_out/r02z_memcheck.txt
SWARMSTEP_FUZZ_SEEDS=10000 timeout 2400 python -m pytest tests/test_gpu_fuzz.py -q -p no:cacheprovider > gpurun_out/r02z_fuzz_soak.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r02z_fuzz_soak.txt
