ADSB_NO_SMEM=1 timeout 900 python scripts/diag_ba.py > gpurun_out/diag_ba.log 2>&1
timeout 900 python scripts/diag_ba.py >> gpurun_out/diag_ba.log 2>&1
ADSB_NO_SMEM=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/diag_ba.py 16384 > gpurun_out/sanitizer_ba.log 2>&1
echo "sanitizer exit $?" >> gpurun_out/sanitizer_ba.log
