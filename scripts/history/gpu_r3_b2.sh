# C5 ncu --set full with sources; the report comes back in gpurun_out/r3b.
mkdir -p gpurun_out/r3b
export ADSB_GRAPH_CACHE=build/gcache
M="--metrics lts__t_bytes.sum,lts__t_sectors.sum,lts__t_sector_hit_rate.pct"
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('c5_rmat24')"
timeout 600 python scripts/prof_capped.py c5_rmat24 64 > gpurun_out/r3b/plain_c5_capped.log 2>&1 && \
timeout 1500 ncu --set full $M --clock-control none --import-source on -k regex:sampler_cta_kernel -c 1 \
  -o gpurun_out/r3b/c5_full python scripts/prof_capped.py c5_rmat24 64 > gpurun_out/r3b/ncu_c5.log 2>&1
ls -la gpurun_out/r3b > gpurun_out/r3b/ls.txt
