mkdir -p gpurun_out/rc4n
timeout 300 python scripts/prof_capped.py c4_grid 1184 2 > gpurun_out/rc4n/plain_c4_capped.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sampler_cta_kernel -s 1 -c 1 \
  -o gpurun_out/rc4n/c4_final_full python scripts/prof_capped.py c4_grid 1184 2 > gpurun_out/rc4n/ncu_c4.log 2>&1
