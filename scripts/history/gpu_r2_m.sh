# Round 2 m: fused deterministic frames (one launch, device-side ordered cutoff) - suite + A/B vs batches.
mkdir -p gpurun_out/r2m; rm -f gpurun_out/r2m/*
export ADSB_GRAPH_CACHE=build/gcache
for c in c5_rmat24 c2_rmat18 c3_ba c1_er; do timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('$c')" ; done
timeout 1800 python -m pytest tests -m gpu -q -rf -x --durations=5 > gpurun_out/r2m/pytest.log 2>&1
echo "pytest rc $?" >> gpurun_out/r2m/pytest.log
bash scripts/gpu_ab_env.sh "ADSB_NO_FUSED_DET=1|ADSB_NO_FUSED_DET=|ADSB_SAMPLER=block" "c3_ba c1_er" r2m/env.log
ADSB_TRACE=1 timeout 300 python scripts/prof_one.py c3_ba 3 > gpurun_out/r2m/trace_c3.log 2>&1
