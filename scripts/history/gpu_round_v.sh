mkdir -p gpurun_out/rv
timeout 1800 python -m pytest tests -x -q -m gpu --timeout 900 -p no:cacheprovider > gpurun_out/rv/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/rv/pytest_gpu.log
bash scripts/gpu_ab2.sh "kary=kary nokary=nokary" "c2_rmat18 c3_ba c5_rmat24 c4_grid" rv/ab.log
for v in kary nokary; do for i in 1 2 3; do ADSB_LIB_PATH=ab/libadsb_$v.so timeout 300 python scripts/diag_wrapper.py c2_rmat18 2>&1 | tail -3 | sed "s/^/$v /" >> gpurun_out/rv/c2_fine.log; done; done
