mkdir -p gpurun_out/raa
for r in 1 2; do
bash scripts/gpu_ab2.sh "base=base pair=pair" "c2_rmat18 c5_rmat24" raa/ab.log scripts/prof_one.py 4
done
ADSB_LIB_PATH=ab/libadsb_pair.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -m gpu --timeout 900 -p no:cacheprovider -k "epoch or fused or c2_fullsize or c5_fullsize" > gpurun_out/raa/pytest_pair.log 2>&1
echo "pytest exit $?" >> gpurun_out/raa/pytest_pair.log
