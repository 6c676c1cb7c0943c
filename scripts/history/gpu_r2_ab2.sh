# Round 2 A/B 2: vectorised (16-byte) flattened adjacency reads; GPU suite on the default (vec4) build.
mkdir -p gpurun_out/r2f
export ADSB_GRAPH_CACHE=build/gcache
for c in c5_rmat24 c2_rmat18 c3_ba; do timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('$c')" ; done
bash scripts/gpu_ab.sh "w0 w1 w2" "c5_rmat24 c2_rmat18 c3_ba" r2f/ab2.log
timeout 1800 python -m pytest tests -m gpu -q -rf --durations=10 > gpurun_out/r2f/pytest.log 2>&1
echo "pytest rc $?" >> gpurun_out/r2f/pytest.log
