# Round 2 o: C4 phase breakdown (phase-timing build) on a capped run.
mkdir -p gpurun_out/r2o; rm -f gpurun_out/r2o/*
export ADSB_GRAPH_CACHE=build/gcache
ADSB_LIB_PATH=ab/libadsb_phase.so ADSB_TRACE=1 timeout 600 python scripts/prof_capped.py c4_grid 2368 2 > gpurun_out/r2o/phase_c4.log 2>&1
ADSB_LIB_PATH=ab/libadsb_phase.so ADSB_TRACE=1 timeout 600 python scripts/prof_one.py c3_ba 2 > gpurun_out/r2o/phase_c3.log 2>&1
ADSB_LIB_PATH=ab/libadsb_phase.so ADSB_TRACE=1 timeout 600 python scripts/prof_one.py c2_rmat18 2 > gpurun_out/r2o/phase_c2.log 2>&1
