timeout 1500 python -m pytest tests -q -x -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu54.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu54.log
ADSB_LIB_PATH=ab/libadsb_dbg.so timeout 900 python -m pytest tests -q -x -m gpu --timeout 600 -p no:cacheprovider -k "block or fused or epoch or c4 or frames" > gpurun_out/pytest_dbg54.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_dbg54.log
for cap in 2944 3200 3392; do
  for c in c3_ba c2_rmat18; do
    ADSB_TRACE=1 ADSB_HASH_CAP=$cap timeout 300 python scripts/prof_one.py $c 3 2>&1 | grep -E "arena|rep 2" | tail -n 2 | tr '\n' ' ' | sed "s/^/cap=$cap /" >> gpurun_out/cap54.log; echo >> gpurun_out/cap54.log
  done
done
for cap in 2944 3392; do
  ADSB_TRACE=1 ADSB_HASH_CAP=$cap timeout 600 python scripts/prof_one.py c5_rmat24 2 2>&1 | grep -E "arena|rep 1" | tail -n 2 | tr '\n' ' ' | sed "s/^/cap=$cap /" >> gpurun_out/cap54.log; echo >> gpurun_out/cap54.log
done
