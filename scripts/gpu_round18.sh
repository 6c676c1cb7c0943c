timeout 1200 python -m pytest tests -x -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu18.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu18.log
ADSB_TRACE=1 timeout 1200 python scripts/prof_one.py c4_grid 1 2>&1 | grep -v "det batch" > gpurun_out/prof18_c4.log
for c in c1_er c2_rmat18 c3_ba; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/bench18_$c.json 2> gpurun_out/bench18_$c.err; done
timeout 1800 python bench.py --config c5_rmat24 --steps 2 --warmup 3 --no-e2e > gpurun_out/bench18_c5_rmat24.json 2> gpurun_out/bench18_c5_rmat24.err
