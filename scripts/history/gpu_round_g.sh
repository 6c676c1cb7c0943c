mkdir -p gpurun_out/rg
bash scripts/gpu_ab2.sh "k8=cur k16=cur:ADSB_RING_K=16 k32=cur:ADSB_RING_K=32 k64=cur:ADSB_RING_K=64" "c5_rmat24 c2_rmat18" rg/ab_ring.log
bash scripts/gpu_ab2.sh "g592=cur g518=cur:ADSB_GLOBAL_GRID=518 g444=cur:ADSB_GLOBAL_GRID=444 g407=cur:ADSB_GLOBAL_GRID=407 g370=cur:ADSB_GLOBAL_GRID=370" "c4_grid" rg/ab_grid.log
