timeout 1000 python scripts/diag_fused_repeat.py 250 16 > gpurun_out/diag27_b16.log 2>&1
timeout 1000 python scripts/diag_fused_repeat.py 250 64 > gpurun_out/diag27_b64.log 2>&1
