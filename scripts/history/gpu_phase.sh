# per-phase cycle breakdown (diagnostic build ab/libadsb_phase.so, -DADSB_PHASE_TIMING)
for c in ${1:-c2_rmat18 c3_ba}; do
  ADSB_TRACE=1 ADSB_LIB_PATH=ab/libadsb_phase.so timeout 600 python scripts/prof_one.py $c 2 2>&1 | grep -E "phase|sample cycles|for_edges|rep 1" | tail -n 4 >> gpurun_out/phase.log
done
