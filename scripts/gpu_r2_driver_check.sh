# What the driver runs at round end, on a box with no graph cache: smoke, the default bench and the reference arm (timed).
mkdir -p gpurun_out/r2h; rm -f gpurun_out/r2h/*
unset ADSB_GRAPH_CACHE
( time timeout 600 python -c "import __graft_entry__ as g; g.smoke()" ) > gpurun_out/r2h/smoke.log 2>&1
( time timeout 1500 python bench.py ) > gpurun_out/r2h/bench_default.log 2>&1
( time timeout 1500 python bench.py --impl reference ) > gpurun_out/r2h/bench_reference.log 2>&1
