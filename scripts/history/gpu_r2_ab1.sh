# Round 2 A/B 1: CSR policy hoist, lean edge loop, shared-memory membership filter (C5, C2, C3), + phase breakdown.
mkdir -p gpurun_out/r2e
export ADSB_GRAPH_CACHE=build/gcache
for c in c5_rmat24 c2_rmat18 c3_ba; do timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('$c')" ; done
ADSB_LIB_PATH=ab/libadsb_phase.so ADSB_TRACE=1 timeout 300 python scripts/prof_one.py c5_rmat24 2 > gpurun_out/r2e/phase_c5.log 2>&1
ADSB_LIB_PATH=ab/libadsb_phase.so ADSB_TRACE=1 timeout 300 python scripts/prof_one.py c2_rmat18 2 > gpurun_out/r2e/phase_c2.log 2>&1
bash scripts/gpu_ab.sh "v0 v1 v2 v3 v4" "c5_rmat24 c2_rmat18 c3_ba" r2e/ab1.log
