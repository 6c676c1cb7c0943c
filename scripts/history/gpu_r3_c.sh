# Round 2 (session 4) c: hub search trees x bulk L2 prefetch of scanned rows x join levels, A/B on C5/C2/C3; then the GPU suite.
mkdir -p gpurun_out/r3c; rm -f gpurun_out/r3c/*
export ADSB_GRAPH_CACHE=build/gcache
for c in c5_rmat24 c2_rmat18 c3_ba; do timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('$c')" ; done
run() { # config, env...
  c=$1; shift
  echo "== $c $*" >> gpurun_out/r3c/ab.log
  env "$@" ADSB_TRACE=1 timeout 300 python scripts/prof_one.py $c 3 2>&1 | grep -E "rep [12]|join levels|Error|error" | tail -3 >> gpurun_out/r3c/ab.log
}
T0="ADSB_NO_HUB_TREES=1"; T1="ADSB_HUB_TREES=1"
run c5_rmat24 $T0 ADSB_BULK_MIN=0 ADSB_JOIN=0
run c5_rmat24 $T1 ADSB_BULK_MIN=0 ADSB_JOIN=0
run c5_rmat24 $T0 ADSB_BULK_MIN=64 ADSB_JOIN=0
run c5_rmat24 $T1 ADSB_BULK_MIN=64 ADSB_JOIN=0
run c5_rmat24 $T1 ADSB_BULK_MIN=64 ADSB_JOIN=1
run c5_rmat24 $T1 ADSB_BULK_MIN=256 ADSB_JOIN=0
run c5_rmat24 $T1 ADSB_BULK_MIN=2048 ADSB_JOIN=0
run c5_rmat24 $T1 ADSB_BULK_MIN=64 ADSB_JOIN=0 ADSB_HUB_FACTOR=2
run c5_rmat24 $T1 ADSB_BULK_MIN=64 ADSB_JOIN=0 ADSB_HUB_FACTOR=1
run c5_rmat24 $T1 ADSB_BULK_MIN=64 ADSB_JOIN=0 ADSB_HUB_FACTOR=8
run c5_rmat24 $T0 ADSB_BULK_MIN=0 ADSB_JOIN=0
run c5_rmat24 $T1 ADSB_BULK_MIN=64 ADSB_JOIN=0
for c in c2_rmat18 c3_ba; do
  run $c $T0 ADSB_BULK_MIN=0 ADSB_JOIN=0
  run $c $T1 ADSB_BULK_MIN=0 ADSB_JOIN=0
  run $c $T1 ADSB_BULK_MIN=64 ADSB_JOIN=0
  run $c $T1 ADSB_BULK_MIN=0 ADSB_JOIN=1
  run $c $T1 ADSB_BULK_MIN=0 ADSB_JOIN=0 ADSB_HUB_FACTOR=2
  run $c $T1 ADSB_BULK_MIN=0 ADSB_JOIN=0 ADSB_HUB_FACTOR=1
  run $c $T0 ADSB_BULK_MIN=0 ADSB_JOIN=0
  run $c $T1 ADSB_BULK_MIN=0 ADSB_JOIN=0
done
timeout 1800 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -rf -x > gpurun_out/r3c/pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r3c/pytest.log
