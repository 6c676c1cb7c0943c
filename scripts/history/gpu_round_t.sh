mkdir -p gpurun_out/rt
ADSB_TRACE=1 ADSB_LIB_PATH=ab/libadsb_phase.so timeout 600 python scripts/prof_one.py c4_grid 2 2>&1 | grep -E "phase|sample cycles|for_edges|rep 1" | tail -n 4 > gpurun_out/rt/phase_c4.log
bash scripts/gpu_ab2.sh "g296=cur g259=cur:ADSB_GLOBAL_GRID=259 g222=cur:ADSB_GLOBAL_GRID=222 g148x1024=cur:ADSB_GLOBAL_BT=1024,ADSB_GLOBAL_GRID=148" "c4_grid" rt/ab_grid.log
