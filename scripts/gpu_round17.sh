timeout 1200 python -m pytest tests -x -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu17.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu17.log
for c in c2_rmat18 c3_ba; do ADSB_TRACE=1 timeout 300 python scripts/prof_one.py $c 3 2>&1 | grep -v "det batch" >> gpurun_out/prof17.log; done
