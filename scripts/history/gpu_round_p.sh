mkdir -p gpurun_out/rp
timeout 600 python scripts/diag_e2e.py c3_ba > gpurun_out/rp/diag_e2e_c3.log 2>&1
ADSB_TRACE=1 timeout 600 python scripts/diag_e2e.py c3_ba 2>&1 | grep -E "preprocess|from_csr" > gpurun_out/rp/diag_e2e_c3_trace.log
bash scripts/gpu_ab2.sh "h0=cur h1=cur:ADSB_CSR_HINT=1" "c3_ba" rp/ab_hint_c3.log
