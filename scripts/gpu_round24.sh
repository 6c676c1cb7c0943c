ADSB_LIB_PATH=ab/libadsb_head.so timeout 900 python scripts/diag_fused_repeat.py 100 64 > gpurun_out/diag24_head.log 2>&1
timeout 900 python scripts/diag_fused_repeat.py 100 64 > gpurun_out/diag24_new.log 2>&1
