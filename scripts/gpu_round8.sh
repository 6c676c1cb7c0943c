timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu8.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu8.log
timeout 600 python scripts/diag_grid.py > gpurun_out/diag_grid.log 2>&1
ADSB_NO_SMEM=1 timeout 600 python scripts/diag_grid.py >> gpurun_out/diag_grid.log 2>&1
ADSB_SAMPLER=warp timeout 600 python scripts/diag_grid.py >> gpurun_out/diag_grid.log 2>&1
ADSB_TRACE=1 timeout 300 python scripts/diag_e2e.py c2_rmat18 > gpurun_out/diag_e2e.log 2>&1
for c in c2_rmat18 c3_ba; do timeout 300 python scripts/prof_one.py $c 2 >> gpurun_out/prof_one8.log 2>&1; done
