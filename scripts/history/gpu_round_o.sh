mkdir -p gpurun_out/ro
timeout 600 python scripts/diag_wrapper.py c3_ba > gpurun_out/ro/wrap_c3.log 2>&1
timeout 600 python scripts/diag_wrapper.py c2_rmat18 > gpurun_out/ro/wrap_c2.log 2>&1
ADSB_TRACE=1 timeout 600 python scripts/prof_one.py c3_ba 2 > gpurun_out/ro/trace_c3.log 2>&1
timeout 1500 python bench.py --config c4_grid --steps 2 --warmup 3 --no-e2e > gpurun_out/ro/bench_c4.log 2>&1
timeout 900 python bench.py --config c3_ba --steps 10 --warmup 3 > gpurun_out/ro/bench_c3.log 2>&1
