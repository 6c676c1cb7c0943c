# A/B: predicted det batch sizes; low-degree expansion on C4; bench with reference_equivalent
for c in c1_er c3_ba; do timeout 300 python scripts/prof_one.py $c 3 >> gpurun_out/prof20.log 2>&1; done
for c in c1_er c3_ba; do ADSB_DET_PIPELINE=1 timeout 300 python scripts/prof_one.py $c 2 2>&1 | sed 's/^/pipe /' >> gpurun_out/prof20.log; done
timeout 900 python scripts/prof_one.py c4_grid 1 > gpurun_out/prof20_c4.log 2>&1
ADSB_NO_LOWDEG=1 timeout 900 python scripts/prof_one.py c4_grid 1 2>&1 | sed 's/^/nolowdeg /' >> gpurun_out/prof20_c4.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench20_c2.log 2>&1
timeout 600 python bench.py --config c3_ba --steps 5 --warmup 3 > gpurun_out/bench20_c3.log 2>&1
