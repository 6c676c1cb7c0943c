# Round 2 l: table size vs blocks per SM (fallback share changed with hub probes); hub factor in quarters.
mkdir -p gpurun_out/r2l; rm -f gpurun_out/r2l/*
export ADSB_GRAPH_CACHE=build/gcache
for c in c5_rmat24 c2_rmat18 c3_ba; do timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('$c')" ; done
bash scripts/gpu_ab_env.sh "ADSB_HASH_CAP=2944|ADSB_HASH_CAP=4608|ADSB_HASH_CAP=7296|ADSB_HUB_FACTOR=2|ADSB_HUB_FACTOR=8" "c5_rmat24 c2_rmat18 c3_ba" r2l/env.log
