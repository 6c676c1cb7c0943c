timeout 1500 python -m pytest tests -x -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu19.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu19.log
for c in c1_er c2_rmat18 c3_ba; do ADSB_TRACE=1 timeout 300 python scripts/prof_one.py $c 3 2>&1 | grep -v "det batch" >> gpurun_out/prof19.log; done
ADSB_TRACE=1 timeout 1200 python scripts/prof_one.py c4_grid 1 2>&1 | grep -v "det batch" > gpurun_out/prof19_c4.log
