timeout 1500 python -m pytest tests -q -x -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu48.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu48.log
for c in c2_rmat18 c3_ba; do ADSB_TRACE=1 timeout 300 python scripts/prof_one.py $c 3 2>&1 | grep -E "rep 2|arena" | tail -n 2 >> gpurun_out/prof48.log; done
ADSB_TRACE=1 timeout 900 python scripts/prof_one.py c5_rmat24 2 2>&1 | grep -E "rep|arena" >> gpurun_out/prof48.log
timeout 900 python scripts/prof_one.py c4_grid 1 2>&1 | tail -n 1 >> gpurun_out/prof48.log
