timeout 1500 python -m pytest tests -q -x -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu35.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu35.log
for v in b1 b2 b4 b8; do
  for c in c2_rmat18 c3_ba; do
    ADSB_LIB_PATH=ab/libadsb_$v.so timeout 300 python scripts/prof_one.py $c 3 2>&1 | tail -n 1 | sed "s/^/$v /" >> gpurun_out/ab35.log
  done
done
for v in b1 b4; do ADSB_LIB_PATH=ab/libadsb_$v.so timeout 600 python scripts/prof_one.py c4_grid 1 2>&1 | tail -n 1 | sed "s/^/$v /" >> gpurun_out/ab35.log; done
