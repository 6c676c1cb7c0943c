# Round 2 (session 4) d: hub search trees in the vector kernels only: base build (round-2 HEAD) vs this build, on C5/C2/C3; tree tests.
mkdir -p gpurun_out/r3d; rm -f gpurun_out/r3d/*
export ADSB_GRAPH_CACHE=build/gcache
for c in c5_rmat24 c2_rmat18 c3_ba; do timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('$c')" ; done
run() { # config, env...
  c=$1; shift
  echo "== $c $*" >> gpurun_out/r3d/ab.log
  env "$@" ADSB_TRACE=1 timeout 300 python scripts/prof_one.py $c 4 2>&1 | grep -E "rep [123]|Error|error" | tail -3 >> gpurun_out/r3d/ab.log
}
B="ADSB_LIB_PATH=ab/libadsb_base.so"
for i in 1 2; do
  run c5_rmat24 $B
  run c5_rmat24 X=1
  run c5_rmat24 ADSB_HUB_FACTOR=6
  run c5_rmat24 ADSB_HUB_FACTOR=12
  run c5_rmat24 ADSB_HUB_FACTOR=16
  run c5_rmat24 ADSB_NO_HUB_TREES=1
done
for c in c2_rmat18 c3_ba; do for i in 1 2; do run $c $B; run $c X=1; done; done
timeout 900 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -rf -x -k "tree or variants or c5 or frames_match" > gpurun_out/r3d/pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r3d/pytest.log
