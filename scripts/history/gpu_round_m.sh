mkdir -p gpurun_out/rm
bash scripts/gpu_ab2.sh "b256g444=bt b512g296=bt:ADSB_GLOBAL_BT=512,ADSB_GLOBAL_GRID=296 b512g222=bt:ADSB_GLOBAL_BT=512,ADSB_GLOBAL_GRID=222 b512g259=bt:ADSB_GLOBAL_BT=512,ADSB_GLOBAL_GRID=259" "c4_grid" rm/ab_bt.log
ADSB_GLOBAL_BT=512 ADSB_GLOBAL_GRID=296 ADSB_SAMPLER=block ADSB_NO_SMEM=1 timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu -k "holey or c3_fullsize_deterministic" -p no:cacheprovider > gpurun_out/rm/pytest_bt512.log 2>&1; echo "exit $?" >> gpurun_out/rm/pytest_bt512.log
