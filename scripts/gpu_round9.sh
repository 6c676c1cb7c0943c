timeout 900 python scripts/diag_c4.py > gpurun_out/diag_c4.log 2>&1
ADSB_NO_SMEM=1 timeout 900 python scripts/diag_c4.py > gpurun_out/diag_c4_nosmem.log 2>&1
ADSB_SAMPLER=warp timeout 900 python scripts/diag_c4.py > gpurun_out/diag_c4_warp.log 2>&1
