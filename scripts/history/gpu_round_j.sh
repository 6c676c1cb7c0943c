mkdir -p gpurun_out/rj
timeout 1500 python -m pytest tests -x -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/rj/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/rj/pytest_gpu.log
bash scripts/gpu_ab2.sh "filt=filt nofilt=nofilt" "c5_rmat24 c3_ba c2_rmat18" rj/ab_filt.log
timeout 600 python scripts/diag_e2e.py c2_rmat18 > gpurun_out/rj/diag_e2e_c2.log 2>&1
