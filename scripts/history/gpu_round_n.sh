mkdir -p gpurun_out/rn
timeout 1800 python -m pytest tests -x -q -m gpu --timeout 900 -p no:cacheprovider > gpurun_out/rn/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/rn/pytest_gpu.log
bash scripts/gpu_ab2.sh "b512=cur b1024=cur:ADSB_GLOBAL_BT=1024,ADSB_GLOBAL_GRID=148" "c4_grid" rn/ab_bt.log
