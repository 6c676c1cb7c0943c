for cap in 2048 2176 2304 2432 2560 2816 3072; do
  for c in c3_ba c2_rmat18; do
    ADSB_TRACE=1 ADSB_HASH_CAP=$cap timeout 300 python scripts/prof_one.py $c 3 2>&1 | grep -E "arena|rep 2" | tail -n 2 | tr '\n' ' ' | sed "s/^/cap=$cap /" >> gpurun_out/cap52.log; echo >> gpurun_out/cap52.log
  done
done
for cap in 2048 2304 2816; do
  ADSB_TRACE=1 ADSB_HASH_CAP=$cap timeout 600 python scripts/prof_one.py c5_rmat24 2 2>&1 | grep -E "arena|rep 1" | tail -n 2 | tr '\n' ' ' | sed "s/^/cap=$cap /" >> gpurun_out/cap52.log; echo >> gpurun_out/cap52.log
done
