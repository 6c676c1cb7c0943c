timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench31_c2.log 2>&1
timeout 300 python scripts/prof_one.py c2_rmat18 2 > gpurun_out/plain31.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sampler_cta_kernel -s 1 -c 1 \
  -o gpurun_out/prof31_c2 python scripts/prof_one.py c2_rmat18 2 > gpurun_out/ncu31.log 2>&1
