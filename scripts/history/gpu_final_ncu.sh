mkdir -p gpurun_out/final
timeout 300 python scripts/prof_one.py c2_rmat18 2 > gpurun_out/final/plain_ncu_full.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sampler_cta_kernel -s 1 -c 1 \
  -o gpurun_out/final/c2_fused_full python scripts/prof_one.py c2_rmat18 2 > gpurun_out/final/ncu_full.log 2>&1
