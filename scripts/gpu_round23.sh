timeout 600 python scripts/diag_fused_repeat.py 40 64 > gpurun_out/diag23.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu23.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu23.log
timeout 600 python scripts/diag_fused_repeat.py 40 64 >> gpurun_out/diag23.log 2>&1
