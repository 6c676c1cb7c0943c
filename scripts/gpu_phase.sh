# per-phase cycle breakdown (diagnostic build ab/libadsb_phase.so)
for c in c2_rmat18 c3_ba c1_er; do
  ADSB_SAMPLER=block ADSB_TRACE=1 ADSB_LIB_PATH=ab/libadsb_phase.so timeout 300 python scripts/prof_one.py $c 2 2>&1 | grep -E "phase|rep 1" | tail -n 2 >> gpurun_out/phase.log
done
ADSB_TRACE=1 ADSB_LIB_PATH=ab/libadsb_phase.so timeout 600 python scripts/prof_one.py c4_grid 1 2>&1 | grep -E "phase|rep 0" >> gpurun_out/phase.log
