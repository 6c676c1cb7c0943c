timeout 1500 python -m pytest tests -x -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu22.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu22.log
for c in c1_er c2_rmat18 c3_ba; do timeout 300 python scripts/prof_one.py $c 3 >> gpurun_out/prof22.log 2>&1; done
timeout 900 python scripts/prof_one.py c4_grid 1 >> gpurun_out/prof22.log 2>&1
