# Round 2: full GPU suite on the current tree + smoke.
mkdir -p gpurun_out/r2c
timeout 1800 python -m pytest tests -m gpu -q -x -rf --durations=15 > gpurun_out/r2c/pytest.log 2>&1
echo "pytest rc $?" >> gpurun_out/r2c/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c/smoke.log 2>&1
