mkdir -p gpurun_out/rf
bash scripts/gpu_ab2.sh "g592=cur g444=cur:ADSB_GLOBAL_GRID=444 g296=cur:ADSB_GLOBAL_GRID=296 g888=cur:ADSB_GLOBAL_GRID=888" "c4_grid" rf/ab_grid.log
ADSB_TRACE=1 ADSB_LIB_PATH=ab/libadsb_phase.so timeout 600 python scripts/prof_one.py c5_rmat24 2 > gpurun_out/rf/phase_c5.log 2>&1
ADSB_LIB_PATH=ab/libadsb_cur.so timeout 600 python scripts/prof_capped.py c5_rmat24 64 2 > gpurun_out/rf/plain_c5_capped.log 2>&1 && \
ADSB_LIB_PATH=ab/libadsb_cur.so timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sampler_cta_kernel -s 1 -c 1 \
  -o gpurun_out/rf/c5_full python scripts/prof_capped.py c5_rmat24 64 2 > gpurun_out/rf/ncu_c5.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_small.py > gpurun_out/rf/memcheck.log 2>&1; echo "exit $?" >> gpurun_out/rf/memcheck.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize_small.py > gpurun_out/rf/racecheck.log 2>&1; echo "exit $?" >> gpurun_out/rf/racecheck.log
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python scripts/sanitize_small.py > gpurun_out/rf/synccheck.log 2>&1; echo "exit $?" >> gpurun_out/rf/synccheck.log
