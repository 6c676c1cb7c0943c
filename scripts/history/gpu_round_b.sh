mkdir -p gpurun_out/rb
timeout 1200 python -m pytest tests -x -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/rb/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/rb/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rb/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/rb/smoke.log
bash scripts/gpu_ab.sh "base new nopush tagged" "c4_grid c3_ba c2_rmat18" rb/ab.log
bash scripts/gpu_ab.sh "base new tagged" "c5_rmat24" rb/ab_c5.log
ADSB_TRACE=1 ADSB_LIB_PATH=ab/libadsb_phase.so timeout 600 python scripts/prof_one.py c4_grid 2 > gpurun_out/rb/phase_c4.log 2>&1
timeout 900 python scripts/exact_bc_check.py c2_rmat18 gpurun_out/rb/exact_c2.json > gpurun_out/rb/exact_c2.log 2>&1
