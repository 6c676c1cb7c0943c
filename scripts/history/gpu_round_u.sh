mkdir -p gpurun_out/ru
timeout 1800 python -m pytest tests -x -q -m gpu --timeout 900 -p no:cacheprovider > gpurun_out/ru/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/ru/pytest_gpu.log
bash scripts/gpu_ab2.sh "cur=cur pushb=pushb" "c4_grid" ru/ab.log
