# Round 2 i: hub probes by binary search of the other side's level list.
mkdir -p gpurun_out/r2i; rm -f gpurun_out/r2i/*
export ADSB_GRAPH_CACHE=build/gcache
for c in c5_rmat24 c2_rmat18 c3_ba; do timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('$c')" ; done
bash scripts/gpu_ab.sh "nohub hub" "c5_rmat24 c2_rmat18 c3_ba" r2i/ab.log
timeout 1800 python -m pytest tests -m gpu -q -rf --durations=10 > gpurun_out/r2i/pytest.log 2>&1
echo "pytest rc $?" >> gpurun_out/r2i/pytest.log
