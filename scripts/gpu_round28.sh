timeout 1200 python scripts/diag_fused_repeat.py 400 64 > gpurun_out/diag28_b64.log 2>&1
