timeout 1500 python -m pytest tests -q -x -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu33.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu33.log
timeout 900 python scripts/diag_fused_repeat.py 600 64 c1 > gpurun_out/diag33.log 2>&1
for c in c1_er c2_rmat18 c3_ba; do timeout 300 python scripts/prof_one.py $c 3 2>&1 | tail -n 1 >> gpurun_out/prof33.log; done
timeout 900 python scripts/prof_one.py c4_grid 1 >> gpurun_out/prof33.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench33_c2.log 2>&1
