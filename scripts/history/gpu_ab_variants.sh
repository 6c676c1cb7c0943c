# A/B of kernel variants built into ab/ (ADSB_LIB_PATH), interleaved
for round in 1 2; do
  for v in head cur cub nopf; do
    for c in c2_rmat18 c3_ba; do
      ADSB_LIB_PATH=ab/libadsb_$v.so timeout 300 python scripts/prof_one.py $c 3 2>&1 | tail -n 1 | sed "s/^/$v /" >> gpurun_out/ab_variants.log
    done
  done
done
for v in head cur nopf; do
  ADSB_LIB_PATH=ab/libadsb_$v.so timeout 300 python scripts/prof_one.py c4_grid 1 2>&1 | tail -n 1 | sed "s/^/$v /" >> gpurun_out/ab_variants.log
done
