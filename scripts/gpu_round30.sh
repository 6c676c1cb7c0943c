timeout 1500 python scripts/diag_fused_repeat.py 3000 64 c1 > gpurun_out/diag30.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu30.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu30.log
