mkdir -p gpurun_out/rr
timeout 1800 python -m pytest tests -x -q -m gpu --timeout 900 -p no:cacheprovider > gpurun_out/rr/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/rr/pytest_gpu.log
bash scripts/gpu_ab2.sh "cur=cur batch=batch nopf=nopf" "c4_grid" rr/ab_c4.log
