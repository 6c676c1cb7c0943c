# tests (default build + debug-checks build), smoke, bench lines for every config
mkdir -p gpurun_out/rh
timeout 1500 python -m pytest tests -x -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/rh/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/rh/pytest_gpu.log
ADSB_LIB_PATH=ab/libadsb_dbg.so timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -m gpu --timeout 900 -p no:cacheprovider > gpurun_out/rh/pytest_gpu_debugchecks.log 2>&1
echo "pytest exit $?" >> gpurun_out/rh/pytest_gpu_debugchecks.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rh/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/rh/smoke.log
timeout 900 python bench.py > gpurun_out/rh/bench_c2.log 2>&1
timeout 900 python bench.py --config c1_er --steps 10 > gpurun_out/rh/bench_c1.log 2>&1
timeout 900 python bench.py --config c3_ba --steps 10 > gpurun_out/rh/bench_c3.log 2>&1
timeout 1200 python bench.py --config c5_rmat24 --steps 3 > gpurun_out/rh/bench_c5.log 2>&1
timeout 1500 python bench.py --config c4_grid --steps 2 --no-e2e > gpurun_out/rh/bench_c4.log 2>&1
