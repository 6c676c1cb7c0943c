timeout 900 python scripts/diag_fused_repeat.py 150 16 > gpurun_out/diag25_b16.log 2>&1
timeout 900 python scripts/diag_fused_repeat.py 150 64 > gpurun_out/diag25_b64.log 2>&1
