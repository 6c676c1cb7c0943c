ADSB_TRACE=1 timeout 300 python scripts/diag_overhead.py c2_rmat18 > gpurun_out/diag21.log 2>&1
timeout 300 python scripts/prof_one.py c2_rmat18 2 > gpurun_out/plain21.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sampler_cta_kernel -s 1 -c 1 \
  -o gpurun_out/prof21_c2 python scripts/prof_one.py c2_rmat18 2 > gpurun_out/ncu21.log 2>&1
