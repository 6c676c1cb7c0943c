# Round 2 (session 4) h: offsets / row-head prefetch at claims (nocpf = off), adjacency L1 prefetch distance 2 (pfd2), ring and table sizes.
mkdir -p gpurun_out/r3h; rm -f gpurun_out/r3h/*
export ADSB_GRAPH_CACHE=build/gcache
for c in c5_rmat24 c2_rmat18 c3_ba; do timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('$c')" ; done
run() { # config, env...
  c=$1; shift
  echo "== $c $*" >> gpurun_out/r3h/ab.log
  env "$@" ADSB_TRACE=1 timeout 300 python scripts/prof_one.py $c 4 2>&1 | grep -E "rep [123]|Error|error" | tail -3 >> gpurun_out/r3h/ab.log
}
for i in 1 2; do
  for c in c5_rmat24 c2_rmat18 c3_ba; do
    run $c ADSB_LIB_PATH=ab/libadsb_nocpf.so; run $c X=1; run $c ADSB_LIB_PATH=ab/libadsb_pfd2.so
  done
done
run c5_rmat24 ADSB_RING_K=64
run c5_rmat24 ADSB_HASH_CAP=2560
run c5_rmat24 ADSB_HASH_CAP=3200
run c5_rmat24 ADSB_HUB_FACTOR=8
run c5_rmat24 ADSB_HUB_FACTOR=16
run c2_rmat18 ADSB_HASH_CAP=2560
run c2_rmat18 ADSB_HASH_CAP=3200
run c3_ba ADSB_HASH_CAP=2560
run c3_ba ADSB_HASH_CAP=3200
timeout 900 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -rf -x -k "tree or variants or frames or small or block_teams" > gpurun_out/r3h/pytest_quick.log 2>&1
echo "pytest exit $?" >> gpurun_out/r3h/pytest_quick.log
