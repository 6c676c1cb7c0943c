mkdir -p gpurun_out/rft
timeout 1800 python -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider > gpurun_out/rft/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/rft/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rft/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/rft/smoke.log
