mkdir -p gpurun_out/rq
bash scripts/gpu_ab2.sh "btpf=btpf nobtpf=nobtpf" "c2_rmat18 c3_ba c5_rmat24" rq/ab_btpf.log
ADSB_LIB_PATH=ab/libadsb_btpf.so timeout 300 python scripts/prof_capped.py c4_grid 1184 2 > gpurun_out/rq/plain_c4_capped.log 2>&1 && \
ADSB_LIB_PATH=ab/libadsb_btpf.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:sampler_cta_kernel -s 1 -c 1 \
  -o gpurun_out/rq/c4_512_full python scripts/prof_capped.py c4_grid 1184 2 > gpurun_out/rq/ncu_c4.log 2>&1
