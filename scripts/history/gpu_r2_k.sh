# Round 2 k: migrate overflowing samples to a global region instead of redoing them; suite + A/B.
mkdir -p gpurun_out/r2k; rm -f gpurun_out/r2k/*
export ADSB_GRAPH_CACHE=build/gcache
for c in c5_rmat24 c2_rmat18 c3_ba; do timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('$c')" ; done
timeout 1800 python -m pytest tests -m gpu -q -rf -x --durations=5 > gpurun_out/r2k/pytest.log 2>&1
echo "pytest rc $?" >> gpurun_out/r2k/pytest.log
bash scripts/gpu_ab.sh "nomig mig" "c5_rmat24 c2_rmat18 c3_ba" r2k/ab.log
