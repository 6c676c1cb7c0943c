# Round 2 (session 4) o: C4: fraction of CSR reads marked L2 evict_last (the 77 MB CSR exceeds half of L2, so the default is 0).
mkdir -p gpurun_out/r3o; rm -f gpurun_out/r3o/*
export ADSB_GRAPH_CACHE=build/gcache
timeout 600 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('c4_grid')"
for i in 1 2; do
for h in 0 0.25 0.5 0.75 1.0; do
  echo "== c4 ADSB_CSR_HINT=$h" >> gpurun_out/r3o/ab.log
  ADSB_CSR_HINT=$h timeout 600 python scripts/prof_capped.py c4_grid 2368 2 2>&1 | tail -1 >> gpurun_out/r3o/ab.log
done; done
