mkdir -p gpurun_out/rc
timeout 1500 python -m pytest tests -x -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/rc/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/rc/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rc/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/rc/smoke.log
timeout 900 python scripts/exact_bc_check.py c2_rmat18 gpurun_out/rc/exact_c2.json > gpurun_out/rc/exact_c2.log 2>&1
bash scripts/gpu_ab.sh "base new batch" "c4_grid c3_ba c2_rmat18" rc/ab.log
bash scripts/gpu_ab.sh "base new" "c5_rmat24" rc/ab_c5.log
timeout 300 python scripts/prof_capped.py c4_grid 1184 2 > gpurun_out/rc/plain_c4_capped.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sampler_cta_kernel -s 1 -c 1 \
  -o gpurun_out/rc/c4_full python scripts/prof_capped.py c4_grid 1184 2 > gpurun_out/rc/ncu_c4.log 2>&1
