timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu4.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu4.log
for c in c1_er c2_rmat18 c3_ba; do timeout 300 python scripts/prof_one.py $c 3 >> gpurun_out/prof_one4.log 2>&1; done
for c in c1_er c2_rmat18 c3_ba; do ADSB_SAMPLER=warp timeout 300 python scripts/prof_one.py $c 2 >> gpurun_out/prof_one4_warp.log 2>&1; done
for h in 1024 2048 8192; do ADSB_HASH_CAP=$h timeout 300 python scripts/prof_one.py c2_rmat18 2 >> gpurun_out/prof_one4_hash.log 2>&1; ADSB_HASH_CAP=$h timeout 300 python scripts/prof_one.py c3_ba 2 >> gpurun_out/prof_one4_hash.log 2>&1; done
timeout 300 python scripts/prof_one.py c2_rmat18 2 > gpurun_out/plain4.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sampler_cta -s 6 -c 1 -o gpurun_out/prof4_c2_cta python scripts/prof_one.py c2_rmat18 2 > gpurun_out/ncu4_c2.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu4_c2.log
