# Round 2 (session 4) b: C5 profile with join levels: phase build (if present), ncu --set full + source hot lines, bench lines.
mkdir -p gpurun_out/r3b /tmp/ncu; rm -f gpurun_out/r3b/*
export ADSB_GRAPH_CACHE=build/gcache
M="--metrics lts__t_bytes.sum,lts__t_sectors.sum,lts__t_sector_hit_rate.pct"
for c in c5_rmat24 c2_rmat18 c3_ba; do timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('$c')" ; done
if [ -f ab/libadsb_phase.so ]; then
  ADSB_LIB_PATH=ab/libadsb_phase.so ADSB_TRACE=1 timeout 300 python scripts/prof_one.py c5_rmat24 2 > gpurun_out/r3b/phase_c5.log 2>&1
  ADSB_LIB_PATH=ab/libadsb_phase.so ADSB_TRACE=1 timeout 300 python scripts/prof_one.py c2_rmat18 2 > gpurun_out/r3b/phase_c2.log 2>&1
fi
for c in c5_rmat24 c2_rmat18 c3_ba; do ADSB_TRACE=1 timeout 300 python scripts/prof_one.py $c 3 > gpurun_out/r3b/plain_$c.log 2>&1; done
timeout 600 python scripts/prof_capped.py c5_rmat24 64 > gpurun_out/r3b/plain_c5_capped.log 2>&1 && \
timeout 1500 ncu --set full $M --clock-control none --import-source on -k regex:sampler_cta_kernel -c 1 \
  -o /tmp/ncu/c5_full python scripts/prof_capped.py c5_rmat24 64 > gpurun_out/r3b/ncu_c5.log 2>&1
if [ -f /tmp/ncu/c5_full.ncu-rep ]; then
  python scripts/ncu_summary.py /tmp/ncu/c5_full.ncu-rep > gpurun_out/r3b/c5_full.json 2>&1
  ncu -i /tmp/ncu/c5_full.ncu-rep --page source --csv --print-source cuda > /tmp/ncu/c5_source.csv 2>/dev/null
  python scripts/ncu_lines.py /tmp/ncu/c5_source.csv 60 > gpurun_out/r3b/c5_hot_lines.txt 2>&1
fi
