# Session-2 final measurements: bench lines for every config + the reference arm,
# launch list of the default bench command, full ncu capture of the fused C2 kernel.
mkdir -p gpurun_out/final2
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/final2/gpu_info.txt 2>&1; nproc >> gpurun_out/final2/gpu_info.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/final2/bench_c2.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final2/bench_c2_ref.log 2>&1
timeout 900 python bench.py --config c1_er --steps 10 --warmup 3 > gpurun_out/final2/bench_c1.log 2>&1
timeout 900 python bench.py --config c3_ba --steps 10 --warmup 3 > gpurun_out/final2/bench_c3.log 2>&1
timeout 1200 python bench.py --config c5_rmat24 --steps 3 --warmup 3 > gpurun_out/final2/bench_c5.log 2>&1
timeout 1500 python bench.py --config c4_grid --steps 2 --warmup 3 --no-e2e > gpurun_out/final2/bench_c4.log 2>&1
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/final2/plain_launches.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/final2/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e \
  > gpurun_out/final2/ncu_launches.log 2>&1
timeout 300 python scripts/prof_one.py c2_rmat18 2 > gpurun_out/final2/plain_ncu_full.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sampler_cta_kernel -s 1 -c 1 \
  -o gpurun_out/final2/c2_fused_full python scripts/prof_one.py c2_rmat18 2 > gpurun_out/final2/ncu_full.log 2>&1
