#!/bin/bash
# Full GPU suite + smoke on HEAD (round 2 re-entry check).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu_info.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -rf --durations=25 > gpurun_out/pytest_gpu_r2.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_r2.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_r2.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke_r2.log
