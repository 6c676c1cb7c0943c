mkdir -p gpurun_out/rsp
bash scripts/gpu_ab2.sh "spec=spec nospec=nospec" "c4_grid c3_ba c5_rmat24" rsp/ab.log
ADSB_LIB_PATH=ab/libadsb_spec.so timeout 1500 python -m pytest tests -x -q -m gpu --timeout 900 -p no:cacheprovider > gpurun_out/rsp/pytest.log 2>&1; echo "exit $?" >> gpurun_out/rsp/pytest.log
