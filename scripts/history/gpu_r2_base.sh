# Round 2 baseline on HEAD: GPU suite, C5 bench (the new default workload), smoke.
mkdir -p gpurun_out/r2a
nproc > gpurun_out/r2a/nproc.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2a/pytest.log 2>&1
timeout 1200 python bench.py --config c5_rmat24 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2a/bench_c5.log 2>&1
timeout 900 python bench.py --config c4_grid --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/r2a/bench_c4.log 2>&1
