mkdir -p gpurun_out/rc4
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu --timeout 900 -p no:cacheprovider -k "c4_fullsize" > gpurun_out/rc4/pytest.log 2>&1; echo "exit $?" >> gpurun_out/rc4/pytest.log
