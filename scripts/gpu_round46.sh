for round in 1 2; do
for v in b1m4 b1m5 b1m6; do
  for c in c2_rmat18 c3_ba; do
    ADSB_TRACE=1 ADSB_LIB_PATH=ab/libadsb_$v.so timeout 300 python scripts/prof_one.py $c 3 2>&1 | grep -E "rep 2|arena" | tail -n 2 | sed "s/^/$v /" >> gpurun_out/ab46.log
  done
done
done
