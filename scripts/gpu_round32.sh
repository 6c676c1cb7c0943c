timeout 1500 python -m pytest tests -q -x -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu32.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu32.log
ADSB_LIB_PATH=ab/libadsb_dbg.so timeout 900 python -m pytest tests -q -x -m gpu --timeout 600 -p no:cacheprovider -k "block or fused or epoch or c4 or frames" > gpurun_out/pytest_dbg32.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_dbg32.log
timeout 900 python scripts/diag_fused_repeat.py 1000 64 c1 > gpurun_out/diag32.log 2>&1
for c in c1_er c2_rmat18 c3_ba; do timeout 300 python scripts/prof_one.py $c 3 2>&1 | tail -n 1 >> gpurun_out/prof32.log; done
timeout 900 python scripts/prof_one.py c4_grid 1 >> gpurun_out/prof32.log 2>&1
