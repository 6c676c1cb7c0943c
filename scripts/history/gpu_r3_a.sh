# Round 2 (session 4) a: join levels. A/B on C5/C2/C3 (join off, overflow-only, prediction factors), then the GPU suite.
mkdir -p gpurun_out/r3a; rm -f gpurun_out/r3a/*
export ADSB_GRAPH_CACHE=build/gcache
for c in c5_rmat24 c2_rmat18 c3_ba; do timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('$c')" ; done
for c in c5_rmat24 c2_rmat18 c3_ba; do
  for v in "ADSB_JOIN=0" "ADSB_JOIN_FACTOR=0" "ADSB_JOIN_FACTOR=2" "ADSB_JOIN_FACTOR=4" "ADSB_JOIN_FACTOR=8" "ADSB_JOIN_FACTOR=16" "ADSB_JOIN=0" "ADSB_JOIN_FACTOR=4"; do
    echo "== $c $v" >> gpurun_out/r3a/ab.log
    env $v ADSB_TRACE=1 timeout 300 python scripts/prof_one.py $c 3 2>&1 | grep -E "rep [12]|join levels" | tail -3 >> gpurun_out/r3a/ab.log
  done
done
timeout 1800 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -rf -x > gpurun_out/r3a/pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r3a/pytest.log
