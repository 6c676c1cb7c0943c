# Round 2 (session 4) e: 16-byte tagged claims (one-pass fallback levels) + predicted migration: base build vs this build.
mkdir -p gpurun_out/r3e; rm -f gpurun_out/r3e/*
export ADSB_GRAPH_CACHE=build/gcache
for c in c5_rmat24 c2_rmat18 c3_ba; do timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('$c')" ; done
run() { # config, env...
  c=$1; shift
  echo "== $c $*" >> gpurun_out/r3e/ab.log
  env "$@" ADSB_TRACE=1 timeout 300 python scripts/prof_one.py $c 4 2>&1 | grep -E "rep [123]|Error|error" | tail -3 >> gpurun_out/r3e/ab.log
}
B="ADSB_LIB_PATH=ab/libadsb_base.so"
timeout 900 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -rf -x -k "tree or variants or frames or small or block_teams" > gpurun_out/r3e/pytest_quick.log 2>&1
echo "pytest exit $?" >> gpurun_out/r3e/pytest_quick.log
for i in 1 2; do
  for c in c5_rmat24 c2_rmat18 c3_ba; do run $c $B; run $c X=1; [ -f ab/libadsb_nopredict.so ] && run $c ADSB_LIB_PATH=ab/libadsb_nopredict.so; done
done
run c5_rmat24 ADSB_NO_SMEM=1 $B
run c5_rmat24 ADSB_NO_SMEM=1
timeout 1800 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -rf -x > gpurun_out/r3e/pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r3e/pytest.log
