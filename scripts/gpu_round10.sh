timeout 1200 python -m pytest tests -x -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu10.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu10.log
bash scripts/gpu_variants.sh
ADSB_TRACE=1 timeout 300 python scripts/diag_e2e.py c2_rmat18 > gpurun_out/diag_e2e10.log 2>&1
timeout 900 python scripts/prof_one.py c4_grid 1 > gpurun_out/prof10_c4.log 2>&1
