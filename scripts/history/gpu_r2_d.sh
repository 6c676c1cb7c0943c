# Round 2: GPU suite (no -x) + C5 capped ncu (full set + L2 bytes, source view).
mkdir -p gpurun_out/r2d
timeout 1800 python -m pytest tests -m gpu -q -rf --durations=20 > gpurun_out/r2d/pytest.log 2>&1
echo "pytest rc $?" >> gpurun_out/r2d/pytest.log
timeout 600 python scripts/prof_capped.py c5_rmat24 64 > gpurun_out/r2d/plain_c5.log 2>&1 && \
timeout 1500 ncu --set full --metrics lts__t_bytes.sum,lts__t_sectors.sum,lts__t_sectors_srcunit_tex.sum --clock-control none --import-source on -k regex:sampler_cta_kernel -c 1 \
  -o gpurun_out/r2d/c5_full python scripts/prof_capped.py c5_rmat24 64 > gpurun_out/r2d/ncu_c5.log 2>&1
