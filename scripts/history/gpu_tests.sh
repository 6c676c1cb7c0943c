nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_info.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu1.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu1.log
