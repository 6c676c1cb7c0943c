# deterministic pipeline trace (batches) on C1 and C3
mkdir -p gpurun_out/r3p; rm -f gpurun_out/r3p/*
export ADSB_GRAPH_CACHE=build/gcache
for c in c1_er c3_ba; do ADSB_TRACE=1 timeout 300 python scripts/prof_one.py $c 3 > gpurun_out/r3p/trace_$c.log 2>&1; done
