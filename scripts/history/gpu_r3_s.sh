# predicted-migration factor 1 / 2 (default) / 3
mkdir -p gpurun_out/r3s; rm -f gpurun_out/r3s/*
export ADSB_GRAPH_CACHE=build/gcache
for c in c5_rmat24 c2_rmat18 c3_ba; do timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('$c')" ; done
run() { c=$1; shift
  echo "== $c $*" >> gpurun_out/r3s/ab.log
  env "$@" timeout 300 python scripts/prof_one.py $c 4 2>&1 | grep -E "rep [123]|Error|error" | tail -3 >> gpurun_out/r3s/ab.log
}
for i in 1 2; do for c in c5_rmat24 c2_rmat18 c3_ba; do run $c X=1; run $c ADSB_LIB_PATH=ab/libadsb_pf1.so; run $c ADSB_LIB_PATH=ab/libadsb_pf3.so; done; done
