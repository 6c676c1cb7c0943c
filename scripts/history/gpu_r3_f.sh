# Round 2 (session 4) f: lazy level degree sums; predicted-migration factor 2 / 4 / 8. x128 = previous build (no lazy sums).
mkdir -p gpurun_out/r3f; rm -f gpurun_out/r3f/*
export ADSB_GRAPH_CACHE=build/gcache
for c in c5_rmat24 c2_rmat18 c3_ba; do timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('$c')" ; done
run() { # config, env...
  c=$1; shift
  echo "== $c $*" >> gpurun_out/r3f/ab.log
  env "$@" ADSB_TRACE=1 timeout 300 python scripts/prof_one.py $c 4 2>&1 | grep -E "rep [123]|Error|error" | tail -3 >> gpurun_out/r3f/ab.log
}
timeout 900 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -rf -x -k "tree or variants or frames or small or block_teams" > gpurun_out/r3f/pytest_quick.log 2>&1
echo "pytest exit $?" >> gpurun_out/r3f/pytest_quick.log
for i in 1 2; do
  for c in c5_rmat24 c2_rmat18 c3_ba; do
    run $c ADSB_LIB_PATH=ab/libadsb_x128.so; run $c X=1; run $c ADSB_LIB_PATH=ab/libadsb_predict2.so; run $c ADSB_LIB_PATH=ab/libadsb_predict8.so
  done
done
timeout 1800 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -rf -x > gpurun_out/r3f/pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r3f/pytest.log
