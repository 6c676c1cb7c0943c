# Round 2: the new default bench line (C5) and the libadsb-free reference arm.
mkdir -p gpurun_out/r2b
( time timeout 1500 python bench.py --steps 5 --warmup 3 ) > gpurun_out/r2b/bench_c5.log 2>&1
( time timeout 1500 python bench.py --impl reference --steps 5 --warmup 3 ) > gpurun_out/r2b/ref_c5.log 2>&1
( time timeout 600 python bench.py --config c1_er --steps 5 --warmup 3 ) > gpurun_out/r2b/bench_c1.log 2>&1
