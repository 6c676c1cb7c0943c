for round in 1 2; do
for v in b1m4 b2m3 b4m3 b4m2 b1m3; do
  for c in c2_rmat18 c3_ba; do
    ADSB_LIB_PATH=ab/libadsb_$v.so timeout 300 python scripts/prof_one.py $c 3 2>&1 | tail -n 1 | sed "s/^/$v /" >> gpurun_out/ab45.log
  done
done
done
