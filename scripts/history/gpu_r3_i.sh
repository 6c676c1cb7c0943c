# Round 2 (session 4) i: C4: offsets prefetch at claim time on the low-degree path (cpflow) vs the default build.
mkdir -p gpurun_out/r3i; rm -f gpurun_out/r3i/*
export ADSB_GRAPH_CACHE=build/gcache
timeout 600 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('c4_grid')"
for i in 1 2; do
for v in nocpf cpflow; do
  echo "== c4 $v" >> gpurun_out/r3i/ab.log
  ADSB_LIB_PATH=ab/libadsb_$v.so timeout 600 python scripts/prof_capped.py c4_grid 2368 2 2>&1 | tail -1 >> gpurun_out/r3i/ab.log
done; done
