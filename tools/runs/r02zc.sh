mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_layout.py -q -p no:cacheprovider > gpurun_out/r02zc.txt 2>&1
echo "rc=$?" >> gpurun_out/r02zc.txt
