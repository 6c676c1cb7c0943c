mkdir -p gpurun_out/rl
timeout 1500 python -m pytest tests -x -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/rl/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/rl/pytest_gpu.log
timeout 600 python scripts/diag_e2e.py c2_rmat18 > gpurun_out/rl/diag_e2e_c2.log 2>&1
bash scripts/gpu_ab2.sh "pf1=pf1 pf2=pf2 pf3=pf3" "c2_rmat18 c3_ba c5_rmat24" rl/ab_pf.log
