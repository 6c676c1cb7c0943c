mkdir -p gpurun_out/rw
timeout 1800 python -m pytest tests -x -q -m gpu --timeout 900 -p no:cacheprovider > gpurun_out/rw/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/rw/pytest_gpu.log
ADSB_LIB_PATH=ab/libadsb_kary.so timeout 1200 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -x -q -m gpu --timeout 900 -p no:cacheprovider -k "c3_fullsize or block_teams_frames_ba or sampler_variants" > gpurun_out/rw/pytest_kary.log 2>&1
echo "pytest exit $?" >> gpurun_out/rw/pytest_kary.log
