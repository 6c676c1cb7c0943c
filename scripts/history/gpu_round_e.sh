mkdir -p gpurun_out/re
timeout 1500 python -m pytest tests -x -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/re/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/re/pytest_gpu.log
bash scripts/gpu_ab2.sh "hint=hint split=split" "c4_grid c3_ba c2_rmat18" re/ab.log
ADSB_LIB_PATH=ab/libadsb_split.so timeout 300 python scripts/prof_capped.py c4_grid 1184 2 > gpurun_out/re/plain_c4_capped.log 2>&1 && \
ADSB_LIB_PATH=ab/libadsb_split.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:sampler_cta_kernel -s 1 -c 1 \
  -o gpurun_out/re/c4_split_full python scripts/prof_capped.py c4_grid 1184 2 > gpurun_out/re/ncu_c4.log 2>&1
