timeout 1500 python -m pytest tests -q -x -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu57.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu57.log
timeout 900 python scripts/diag_fused_repeat.py 400 64 c1 > gpurun_out/diag57.log 2>&1
bash scripts/gpu_ab.sh "l1pf rel" "c2_rmat18 c5_rmat24" ab57.log
