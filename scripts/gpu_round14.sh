timeout 1200 python -m pytest tests -x -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu14.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu14.log
for c in c2_rmat18 c3_ba; do timeout 300 python scripts/prof_one.py $c 3 >> gpurun_out/prof14.log 2>&1; done
for c in c2_rmat18 c3_ba; do ADSB_NO_SMEM=1 timeout 300 python scripts/prof_one.py $c 2 >> gpurun_out/prof14.log 2>&1; done
timeout 900 python scripts/prof_one.py c4_grid 1 >> gpurun_out/prof14.log 2>&1
