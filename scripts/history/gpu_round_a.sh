# tests with the default build, smoke, then the global-store A/B
mkdir -p gpurun_out/ra
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/ra/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/ra/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ra/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/ra/smoke.log
bash scripts/gpu_ab.sh "base clear clearcount all" "c4_grid c3_ba c2_rmat18" ra/ab.log
bash scripts/gpu_ab.sh "base all" "c5_rmat24" ra/ab_c5.log
