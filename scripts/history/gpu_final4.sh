# Last refresh after the loop-top and level_pick threshold changes (C4's path is unchanged since final3).
mkdir -p gpurun_out/final4
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/final4/bench_c2.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final4/bench_c2_ref.log 2>&1
timeout 900 python bench.py --config c1_er --steps 10 --warmup 3 > gpurun_out/final4/bench_c1.log 2>&1
timeout 900 python bench.py --config c3_ba --steps 10 --warmup 3 > gpurun_out/final4/bench_c3.log 2>&1
timeout 1200 python bench.py --config c5_rmat24 --steps 3 --warmup 3 > gpurun_out/final4/bench_c5.log 2>&1
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/final4/plain_launches.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/final4/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/final4/ncu_launches.log 2>&1
timeout 300 python scripts/prof_one.py c2_rmat18 2 > gpurun_out/final4/plain_ncu_full.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sampler_cta_kernel -s 1 -c 1 \
  -o gpurun_out/final4/c2_fused_full python scripts/prof_one.py c2_rmat18 2 > gpurun_out/final4/ncu_full.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final4/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/final4/smoke.log
