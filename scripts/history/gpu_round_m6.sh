mkdir -p gpurun_out/rm6
bash scripts/gpu_ab2.sh "cur=cur m6g444=m6:ADSB_GLOBAL_GRID=444 m6g370=m6:ADSB_GLOBAL_GRID=370" "c4_grid" rm6/ab.log
