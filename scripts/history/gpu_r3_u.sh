# env-only re-sweep on the final build: hub threshold factor (quarters) and ring size on C5, hub factor on C2
mkdir -p gpurun_out/r3u; rm -f gpurun_out/r3u/*
export ADSB_GRAPH_CACHE=build/gcache
for c in c5_rmat24 c2_rmat18; do timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('$c')" ; done
run() { c=$1; shift
  echo "== $c $*" >> gpurun_out/r3u/ab.log
  env "$@" timeout 300 python scripts/prof_one.py $c 4 2>&1 | grep -E "rep [123]|Error|error" | tail -3 >> gpurun_out/r3u/ab.log
}
for i in 1 2; do
  run c5_rmat24 X=1
  for f in 8 10 14 16 24; do run c5_rmat24 ADSB_HUB_FACTOR=$f; done
  run c5_rmat24 ADSB_RING_K=16
  run c5_rmat24 ADSB_RING_K=48
  run c2_rmat18 X=1
  for f in 2 3 6 8; do run c2_rmat18 ADSB_HUB_FACTOR=$f; done
done
