# Round 2 g: suite on the kVec-template build; C5 CSR L2-hint sweep; C1/C3 det traces.
mkdir -p gpurun_out/r2g; rm -f gpurun_out/r2g/*
export ADSB_GRAPH_CACHE=build/gcache
timeout 1800 python -m pytest tests -m gpu -q -rf --durations=10 > gpurun_out/r2g/pytest.log 2>&1
echo "pytest rc $?" >> gpurun_out/r2g/pytest.log
bash scripts/gpu_ab_env.sh "ADSB_VEC4=1|ADSB_VEC4=0|ADSB_CSR_HINT=0.25|ADSB_CSR_HINT=0.5|ADSB_CSR_HINT=1" "c5_rmat24" r2g/env_c5.log
ADSB_TRACE=1 timeout 300 python scripts/prof_one.py c1_er 3 > gpurun_out/r2g/trace_c1.log 2>&1
ADSB_TRACE=1 timeout 300 python scripts/prof_one.py c3_ba 3 > gpurun_out/r2g/trace_c3.log 2>&1
