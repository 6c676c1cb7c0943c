timeout 900 python -m pytest tests -x -q -m gpu --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu5.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu5.log
for cfg in "2048 256" "2048 128" "1024 128" "1024 256" "4096 256" "512 128"; do
  set -- $cfg
  for c in c1_er c2_rmat18 c3_ba; do
    echo "H=$1 BT=$2 $(ADSB_HASH_CAP=$1 ADSB_BLOCK=$2 timeout 300 python scripts/prof_one.py $c 2 2>&1 | tail -1)" >> gpurun_out/prof_one5.log
  done
done
