timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu6.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu6.log
for c in c1_er c2_rmat18 c3_ba; do ADSB_TRACE=1 timeout 300 python scripts/prof_one.py $c 2 >> gpurun_out/prof_one6.log 2>&1; done
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench6_c2.json 2> gpurun_out/bench6_c2.err
for c in c1_er c3_ba; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench6_$c.json 2> gpurun_out/bench6_$c.err; done
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain6.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches6_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu6_launches.log 2>&1
echo "ncu launches exit $?" >> gpurun_out/ncu6_launches.log
timeout 300 python scripts/prof_one.py c2_rmat18 2 > gpurun_out/plain6b.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sampler_cta -s 6 -c 1 -o gpurun_out/prof6_c2_cta python scripts/prof_one.py c2_rmat18 2 > gpurun_out/ncu6_full.log 2>&1
echo "ncu full exit $?" >> gpurun_out/ncu6_full.log
