# GPU suite on the debug-check build (-DADSB_DEBUG_CHECKS: device bounds checks and invariant asserts; compute-sanitizer
# is closed on the pool) + a capped C5 run and full C2/C3 runs under it.
mkdir -p gpurun_out/r3q; rm -f gpurun_out/r3q/*
export ADSB_GRAPH_CACHE=build/gcache ADSB_LIB_PATH=ab/libadsb_dbg.so
timeout 2400 python -m pytest tests -q -m gpu --timeout 900 -p no:cacheprovider -rf > gpurun_out/r3q/pytest_dbg.log 2>&1
echo "pytest exit $?" >> gpurun_out/r3q/pytest_dbg.log
for c in c2_rmat18 c3_ba; do timeout 600 python scripts/prof_one.py $c 1 > gpurun_out/r3q/dbg_$c.log 2>&1; echo "exit $?" >> gpurun_out/r3q/dbg_$c.log; done
timeout 900 python scripts/prof_capped.py c5_rmat24 256 > gpurun_out/r3q/dbg_c5.log 2>&1; echo "exit $?" >> gpurun_out/r3q/dbg_c5.log
