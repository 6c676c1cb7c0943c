ADSB_LIB_PATH=ab/libadsb_dbg.so timeout 900 python scripts/diag_fused_repeat.py 200 16 > gpurun_out/diag26_b16.log 2>&1
ADSB_LIB_PATH=ab/libadsb_dbg.so timeout 900 python scripts/diag_fused_repeat.py 200 64 > gpurun_out/diag26_b64.log 2>&1
