timeout 1200 python -m pytest tests -x -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu15.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu15.log
for c in c2_rmat18; do ADSB_TRACE=1 timeout 300 python scripts/prof_one.py $c 3 >> gpurun_out/prof15.log 2>&1; done
ADSB_NO_FUSED=1 timeout 300 python scripts/prof_one.py c2_rmat18 2 >> gpurun_out/prof15.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench15_c2.json 2> gpurun_out/bench15_c2.err
ADSB_TRACE=1 timeout 1200 python scripts/prof_one.py c5_rmat24 1 > gpurun_out/prof15_c5.log 2>&1
