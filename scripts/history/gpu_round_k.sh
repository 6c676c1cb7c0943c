mkdir -p gpurun_out/rk
timeout 1500 python -m pytest tests -x -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/rk/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/rk/pytest_gpu.log
timeout 600 python scripts/diag_e2e.py c2_rmat18 > gpurun_out/rk/diag_e2e_c2.log 2>&1
ADSB_NO_EAGER_UPLOAD=1 timeout 600 python scripts/diag_e2e.py c2_rmat18 > gpurun_out/rk/diag_e2e_c2_lazy.log 2>&1
timeout 900 python bench.py > gpurun_out/rk/bench_c2.log 2>&1
