# Round 2 q: low-degree frontier vertices two at a time (overlapped round trips) on C4.
mkdir -p gpurun_out/r2q; rm -f gpurun_out/r2q/*
export ADSB_GRAPH_CACHE=build/gcache
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('c4_grid')"
for v in nopair pair nopair pair; do ADSB_LIB_PATH=ab/libadsb_$v.so timeout 600 python scripts/prof_capped.py c4_grid 2368 2 2>&1 | tail -1 | sed "s/^/$v /" >> gpurun_out/r2q/ab.log; done
ADSB_LIB_PATH=ab/libadsb_pair.so timeout 900 python -m pytest tests -m gpu -q -rf -x -k "c4 or lattice or grid or sigma_wrap or degenerate" > gpurun_out/r2q/pytest.log 2>&1
echo "pytest rc $?" >> gpurun_out/r2q/pytest.log
