# predicted-migration threshold: 1.0 (default build) / 0.5 (pq2) / 0.75 (pq3) x the table's room; then the GPU suite on the default build
mkdir -p gpurun_out/r3t; rm -f gpurun_out/r3t/*
export ADSB_GRAPH_CACHE=build/gcache
for c in c5_rmat24 c2_rmat18 c3_ba; do timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('$c')" ; done
run() { c=$1; shift
  echo "== $c $*" >> gpurun_out/r3t/ab.log
  env "$@" timeout 300 python scripts/prof_one.py $c 4 2>&1 | grep -E "rep [123]|Error|error" | tail -3 >> gpurun_out/r3t/ab.log
}
for i in 1 2; do for c in c5_rmat24 c2_rmat18 c3_ba; do run $c X=1; run $c ADSB_LIB_PATH=ab/libadsb_pq2.so; run $c ADSB_LIB_PATH=ab/libadsb_pq3.so; done; done
timeout 1800 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -rf -x > gpurun_out/r3t/pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r3t/pytest.log
