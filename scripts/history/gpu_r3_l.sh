# Round 2 (session 4) l: state-word prefetch of filter hits in the fallback samples' probe passes (default build) vs HEAD (head).
mkdir -p gpurun_out/r3l; rm -f gpurun_out/r3l/*
export ADSB_GRAPH_CACHE=build/gcache
for c in c5_rmat24; do timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('$c')" ; done
run() { # config, env...
  c=$1; shift
  echo "== $c $*" >> gpurun_out/r3l/ab.log
  env "$@" ADSB_TRACE=1 timeout 300 python scripts/prof_one.py $c 4 2>&1 | grep -E "rep [123]|Error|error" | tail -3 >> gpurun_out/r3l/ab.log
}
for i in 1 2 3; do run c5_rmat24 ADSB_LIB_PATH=ab/libadsb_head.so; run c5_rmat24 X=1; done
timeout 900 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -rf -x -k "tree or variants or c5 or frames_match" > gpurun_out/r3l/pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r3l/pytest.log
