mkdir -p gpurun_out/rc4b
timeout 1500 python bench.py --config c4_grid --steps 2 --warmup 3 --no-e2e > gpurun_out/rc4b/bench_c4.log 2>&1
