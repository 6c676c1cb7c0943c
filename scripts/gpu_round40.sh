timeout 1500 python -m pytest tests -q -x -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu40.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu40.log
for round in 1 2; do
for v in r1 n1 n2 n4; do
  for c in c2_rmat18 c3_ba; do
    ADSB_LIB_PATH=ab/libadsb_$v.so timeout 300 python scripts/prof_one.py $c 3 2>&1 | tail -n 1 | sed "s/^/$v /" >> gpurun_out/ab40.log
  done
done
done
for v in r1 n1 n2; do ADSB_LIB_PATH=ab/libadsb_$v.so timeout 600 python scripts/prof_one.py c4_grid 1 2>&1 | tail -n 1 | sed "s/^/$v /" >> gpurun_out/ab40.log; done
