timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu7.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu7.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench7_c2.json 2> gpurun_out/bench7_c2.err
for c in c1_er c3_ba; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench7_$c.json 2> gpurun_out/bench7_$c.err; done
ADSB_TRACE=1 timeout 900 python scripts/prof_one.py c4_grid 2 > gpurun_out/prof7_c4.log 2>&1
ADSB_TRACE=1 timeout 1200 python scripts/prof_one.py c5_rmat24 2 > gpurun_out/prof7_c5.log 2>&1
