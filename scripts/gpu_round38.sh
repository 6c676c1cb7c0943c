timeout 1500 python -m pytest tests -q -x -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu38.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu38.log
timeout 900 python scripts/diag_fused_repeat.py 600 64 c1 > gpurun_out/diag38.log 2>&1
for round in 1 2; do
for v in agg rec; do
  for c in c2_rmat18 c3_ba c1_er; do
    ADSB_SAMPLER=block ADSB_LIB_PATH=ab/libadsb_$v.so timeout 300 python scripts/prof_one.py $c 3 2>&1 | tail -n 1 | sed "s/^/$v /" >> gpurun_out/ab38.log
  done
done
done
