timeout 1500 python -m pytest tests -q -x -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu60.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu60.log
for c in c2_rmat18 c3_ba c5_rmat24 c4_grid; do ADSB_TRACE=1 timeout 600 python scripts/diag_e2e.py $c 2>&1 | grep -E "preprocess|from_csr" | tail -n 2 | sed "s/^/$c /" >> gpurun_out/e2e60.log; done
