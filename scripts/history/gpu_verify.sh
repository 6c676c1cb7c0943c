# Re-entry check: GPU parity suite, smoke and the default bench line.
mkdir -p gpurun_out/verify
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/verify/gpu_info.txt 2>&1
nproc >> gpurun_out/verify/gpu_info.txt
timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/verify/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/verify/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/verify/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/verify/smoke.log
timeout 900 python bench.py > gpurun_out/verify/bench_default.log 2>&1
echo "bench exit $?" >> gpurun_out/verify/bench_default.log
timeout 900 python bench.py --config c4_grid --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/verify/bench_c4.log 2>&1
