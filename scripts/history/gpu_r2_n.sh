# Round 2 n: fused det v2 (parallel path recording, spf 1) vs the previous build.
mkdir -p gpurun_out/r2n; rm -f gpurun_out/r2n/*
export ADSB_GRAPH_CACHE=build/gcache
for c in c5_rmat24 c2_rmat18 c3_ba; do timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('$c')" ; done
bash scripts/gpu_ab.sh "base fdet2" "c5_rmat24 c2_rmat18 c3_ba" r2n/ab.log
ADSB_LIB_PATH=ab/libadsb_fdet2.so ADSB_TRACE=1 timeout 300 python scripts/prof_one.py c3_ba 3 > gpurun_out/r2n/trace_c3.log 2>&1
ADSB_LIB_PATH=ab/libadsb_fdet2.so ADSB_SAMPLER=block timeout 300 python scripts/prof_one.py c1_er 3 > gpurun_out/r2n/c1_block.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rf -x --durations=5 > gpurun_out/r2n/pytest.log 2>&1
echo "pytest rc $?" >> gpurun_out/r2n/pytest.log
