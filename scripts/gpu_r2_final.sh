# Round 2 final measurements on HEAD: bench lines (C5 default + C1..C4), the reference arm, launch list of the default
# bench, ncu --set full (+ L2 bytes) of the sampler kernel on every config, the GPU suite and smoke.
# Each ncu command follows the same plain command (exit 0) with &&. Reports go to /tmp/ncu (gpurun_out is capped at
# 64 MiB); their summaries and the C5 report (sources imported, for the hot-line listing) come back.
mkdir -p gpurun_out/r2f /tmp/ncu; rm -f gpurun_out/r2f/*
export ADSB_GRAPH_CACHE=build/gcache
M="--metrics lts__t_bytes.sum,lts__t_sectors.sum,lts__t_sector_hit_rate.pct"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/r2f/gpu_info.txt 2>&1
for c in c5_rmat24 c2_rmat18 c3_ba c4_grid c1_er; do timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('$c')" ; done
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/r2f/bench_c5.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2f/bench_c5_reference.log 2>&1
for c in c1_er c2_rmat18 c3_ba; do timeout 900 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/r2f/bench_$c.log 2>&1; done
timeout 900 python bench.py --config c4_grid --steps 2 --warmup 3 > gpurun_out/r2f/bench_c4_grid.log 2>&1
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2f/plain_launches.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
  --log-file gpurun_out/r2f/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2f/ncu_launches.log 2>&1
timeout 600 python scripts/prof_capped.py c5_rmat24 64 > gpurun_out/r2f/plain_c5.log 2>&1 && \
timeout 1500 ncu --set full $M --clock-control none --import-source on -k regex:sampler_cta_kernel -c 1 \
  -o gpurun_out/r2f/c5_full python scripts/prof_capped.py c5_rmat24 64 > gpurun_out/r2f/ncu_c5.log 2>&1
timeout 300 python scripts/prof_one.py c2_rmat18 2 > gpurun_out/r2f/plain_c2.log 2>&1 && \
timeout 900 ncu --set full $M --clock-control none -k regex:sampler_cta_kernel -s 1 -c 1 \
  -o /tmp/ncu/c2_full python scripts/prof_one.py c2_rmat18 2 > gpurun_out/r2f/ncu_c2.log 2>&1
timeout 300 python scripts/prof_one.py c3_ba 1 > gpurun_out/r2f/plain_c3.log 2>&1 && \
timeout 900 ncu --set full $M --clock-control none -k regex:sampler_cta_kernel -s 2 -c 1 \
  -o /tmp/ncu/c3_full python scripts/prof_one.py c3_ba 1 > gpurun_out/r2f/ncu_c3.log 2>&1
timeout 300 python scripts/prof_one.py c1_er 1 > gpurun_out/r2f/plain_c1.log 2>&1 && \
timeout 900 ncu --set full $M --clock-control none -k regex:sampler_kernel -c 1 \
  -o /tmp/ncu/c1_full python scripts/prof_one.py c1_er 1 > gpurun_out/r2f/ncu_c1.log 2>&1
timeout 600 python scripts/prof_capped.py c4_grid 1184 > gpurun_out/r2f/plain_c4.log 2>&1 && \
timeout 1500 ncu --set full $M --clock-control none -k regex:sampler_cta_kernel -c 1 \
  -o /tmp/ncu/c4_full python scripts/prof_capped.py c4_grid 1184 > gpurun_out/r2f/ncu_c4.log 2>&1
python scripts/ncu_summary.py gpurun_out/r2f/c5_full.ncu-rep > gpurun_out/r2f/c5_full.json 2>&1
for c in c1 c2 c3 c4; do
  [ -f /tmp/ncu/${c}_full.ncu-rep ] && python scripts/ncu_summary.py /tmp/ncu/${c}_full.ncu-rep > gpurun_out/r2f/${c}_full.json 2>&1
done
timeout 1800 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -rf --durations=15 > gpurun_out/r2f/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2f/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2f/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/r2f/smoke.log
du -sh gpurun_out/r2f > gpurun_out/r2f/du.txt
