mkdir -p gpurun_out/ri
timeout 1500 python -m pytest tests -x -q -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/ri/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/ri/pytest_gpu.log
bash scripts/gpu_ab2.sh "lp=lp nolp=nolp" "c5_rmat24 c3_ba c2_rmat18" ri/ab_lp.log
for c in c2_rmat18 c3_ba c5_rmat24; do
  ADSB_TRACE=1 ADSB_LIB_PATH=ab/libadsb_lpphase.so timeout 600 python scripts/prof_one.py $c 2 2>&1 | grep -E "phase|sample cycles|for_edges|rep 1" | tail -n 4 >> gpurun_out/ri/phase.log
done
