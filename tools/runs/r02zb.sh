# round 2: are the two soak outliers (seeds 4841, 5987) new with this round's arithmetic? run them on the
# session-start kernels (commit 2574ed1, built in tools/variants/wt_v0) and on the current ones
mkdir -p gpurun_out
cd tools/variants/wt_v0 && SWARMSTEP_FUZZ_SEEDS=6000 timeout 900 python -m pytest tests/test_gpu_fuzz.py -q -p no:cacheprovider -k "test_fuzz_per_step_against_oracle and (4841 or 5987)" > ../../../gpurun_out/r02zb_v0.txt 2>&1; cd ../../..
SWARMSTEP_FUZZ_SEEDS=6000 timeout 900 python -m pytest tests/test_gpu_fuzz.py -q -p no:cacheprovider -k "test_fuzz_per_step_against_oracle and (4841 or 5987)" > gpurun_out/r02zb_now.txt 2>&1
