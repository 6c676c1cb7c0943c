timeout 1500 python -m pytest tests -q -x -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu44.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu44.log
ADSB_TRACE=1 timeout 600 python scripts/diag_e2e.py c2_rmat18 2>&1 | grep -v "epoch .* checked\|det batch" > gpurun_out/diag_e2e44.log
ADSB_TRACE=1 timeout 600 python scripts/diag_e2e.py c3_ba 2>&1 | grep -v "epoch .* checked\|det batch" > gpurun_out/diag_e2e44_c3.log
