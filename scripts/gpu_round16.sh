timeout 300 python scripts/prof_one.py c2_rmat18 2 > gpurun_out/plain16.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sampler_cta -s 1 -c 1 -o gpurun_out/prof16_c2_fused python scripts/prof_one.py c2_rmat18 2 > gpurun_out/ncu16.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu16.log
