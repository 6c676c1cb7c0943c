timeout 1500 python scripts/diag_fused_repeat.py 3000 64 c1 > gpurun_out/diag29.log 2>&1
