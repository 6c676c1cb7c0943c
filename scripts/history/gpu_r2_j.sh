# Round 2 j: hub search threshold sweep.
mkdir -p gpurun_out/r2j; rm -f gpurun_out/r2j/*
export ADSB_GRAPH_CACHE=build/gcache
for c in c5_rmat24 c2_rmat18 c3_ba; do timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('$c')" ; done
bash scripts/gpu_ab_env.sh "ADSB_HUB_FACTOR=0|ADSB_HUB_FACTOR=1|ADSB_HUB_FACTOR=2|ADSB_HUB_FACTOR=4|ADSB_HUB_FACTOR=8|ADSB_HUB_FACTOR=16" "c5_rmat24 c2_rmat18 c3_ba" r2j/env.log
