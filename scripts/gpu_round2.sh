timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu2.log
for c in c1_er c2_rmat18 c3_ba; do timeout 300 python scripts/prof_one.py $c 3 >> gpurun_out/prof_one.log 2>&1; done
timeout 600 python bench.py --config c2_rmat18 --steps 3 --warmup 3 > gpurun_out/bench_c2_r2.json 2> gpurun_out/bench_c2_r2.err
timeout 300 python scripts/prof_one.py c2_rmat18 2 > gpurun_out/plain.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sampler_kernel -s 6 -c 2 -o gpurun_out/prof_c2_sampler python scripts/prof_one.py c2_rmat18 2 > gpurun_out/ncu_c2.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_c2.log
