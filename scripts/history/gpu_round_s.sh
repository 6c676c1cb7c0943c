mkdir -p gpurun_out/rs
timeout 1800 python -m pytest tests -x -q -m gpu --timeout 900 -p no:cacheprovider > gpurun_out/rs/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/rs/pytest_gpu.log
bash scripts/gpu_ab2.sh "cur=cur nopf=nopf" "c4_grid c3_ba c2_rmat18" rs/ab.log
timeout 1500 python bench.py --config c4_grid --steps 2 --warmup 3 --no-e2e > gpurun_out/rs/bench_c4.log 2>&1
ADSB_TRACE=1 ADSB_LIB_PATH=ab/libadsb_cur.so timeout 600 python scripts/prof_capped.py c5_rmat24 64 2 > gpurun_out/rs/plain_c5_capped.log 2>&1 && \
ADSB_LIB_PATH=ab/libadsb_cur.so timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sampler_cta_kernel -s 1 -c 1 \
  -o gpurun_out/rs/c5_full python scripts/prof_capped.py c5_rmat24 64 2 > gpurun_out/rs/ncu_c5.log 2>&1
