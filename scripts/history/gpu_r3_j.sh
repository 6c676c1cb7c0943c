# Round 2 (session 4) j: fused epochs record a sample's path once, in parallel (recpath), vs per step by thread 0 (default build).
mkdir -p gpurun_out/r3j; rm -f gpurun_out/r3j/*
export ADSB_GRAPH_CACHE=build/gcache
for c in c5_rmat24 c2_rmat18; do timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('$c')" ; done
run() { # config, env...
  c=$1; shift
  echo "== $c $*" >> gpurun_out/r3j/ab.log
  env "$@" ADSB_TRACE=1 timeout 300 python scripts/prof_one.py $c 4 2>&1 | grep -E "rep [123]|Error|error" | tail -3 >> gpurun_out/r3j/ab.log
}
for i in 1 2 3; do for c in c5_rmat24 c2_rmat18; do run $c X=1; run $c ADSB_LIB_PATH=ab/libadsb_recpath.so; run $c ADSB_LIB_PATH=ab/libadsb_recpath2.so; done; done
ADSB_LIB_PATH=ab/libadsb_recpath.so timeout 1800 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -rf -x > gpurun_out/r3j/pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r3j/pytest.log
