# e2e breakdown on C5 with and without the hub search trees (fresh graph handle per step).
mkdir -p gpurun_out/r3k; rm -f gpurun_out/r3k/*
export ADSB_GRAPH_CACHE=build/gcache
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('c5_rmat24')"
ADSB_TRACE=1 timeout 600 python scripts/diag_e2e.py c5_rmat24 > gpurun_out/r3k/e2e_trees.log 2>&1
ADSB_NO_HUB_TREES=1 ADSB_TRACE=1 timeout 600 python scripts/diag_e2e.py c5_rmat24 > gpurun_out/r3k/e2e_notrees.log 2>&1
