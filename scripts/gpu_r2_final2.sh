# Round 2 final (after the probe-prefetch commit): C5 bench line + reference arm, launch list, ncu --set full of the C5
# sampler (sources imported), e2e breakdown, the GPU suite and smoke on HEAD.
mkdir -p gpurun_out/r2g /tmp/ncu; rm -f gpurun_out/r2g/*
export ADSB_GRAPH_CACHE=build/gcache
M="--metrics lts__t_bytes.sum,lts__t_sectors.sum,lts__t_sector_hit_rate.pct"
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('c5_rmat24')"
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/r2g/bench_c5.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2g/bench_c5_reference.log 2>&1
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2g/plain_launches.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
  --log-file gpurun_out/r2g/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2g/ncu_launches.log 2>&1
timeout 600 python scripts/prof_capped.py c5_rmat24 64 > gpurun_out/r2g/plain_c5.log 2>&1 && \
timeout 1500 ncu --set full $M --clock-control none --import-source on -k regex:sampler_cta_kernel -c 1 \
  -o gpurun_out/r2g/c5_full python scripts/prof_capped.py c5_rmat24 64 > gpurun_out/r2g/ncu_c5.log 2>&1
python scripts/ncu_summary.py gpurun_out/r2g/c5_full.ncu-rep > gpurun_out/r2g/c5_full.json 2>&1
ADSB_TRACE=1 timeout 600 python scripts/diag_e2e.py c5_rmat24 > gpurun_out/r2g/e2e_c5.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -rf --durations=15 > gpurun_out/r2g/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2g/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/r2g/smoke.log
