# Final bench lines for every config, the reference arm, and the launch list of the default bench command.
mkdir -p gpurun_out/final
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/final/bench_c2.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/bench_c2_ref.log 2>&1
timeout 900 python bench.py --config c1_er --steps 10 --warmup 3 > gpurun_out/final/bench_c1.log 2>&1
timeout 900 python bench.py --config c3_ba --steps 10 --warmup 3 > gpurun_out/final/bench_c3.log 2>&1
timeout 1200 python bench.py --config c5_rmat24 --steps 3 --warmup 3 > gpurun_out/final/bench_c5.log 2>&1
timeout 1500 python bench.py --config c4_grid --steps 2 --warmup 3 --no-e2e > gpurun_out/final/bench_c4.log 2>&1
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/final/plain_launches.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/final/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/final/ncu_launches.log 2>&1
