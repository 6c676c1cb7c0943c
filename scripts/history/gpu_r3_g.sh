# Round 2 (session 4) g: fallback samples of the vector kernels: 16-byte adjacency reads (novf = off) + state prefetch in claim passes (nopf = off);
# x128 = previous build (predict factor 4, scalar fallback). Phase breakdown of C5 from the phase build.
mkdir -p gpurun_out/r3g; rm -f gpurun_out/r3g/*
export ADSB_GRAPH_CACHE=build/gcache
for c in c5_rmat24 c2_rmat18 c3_ba; do timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1903_09422_b200 import datasets; datasets.graph('$c')" ; done
run() { # config, env...
  c=$1; shift
  echo "== $c $*" >> gpurun_out/r3g/ab.log
  env "$@" ADSB_TRACE=1 timeout 300 python scripts/prof_one.py $c 4 2>&1 | grep -E "rep [123]|Error|error" | tail -3 >> gpurun_out/r3g/ab.log
}
timeout 900 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -rf -x -k "tree or variants or frames or small or block_teams" > gpurun_out/r3g/pytest_quick.log 2>&1
echo "pytest exit $?" >> gpurun_out/r3g/pytest_quick.log
for i in 1 2; do
  for c in c5_rmat24 c2_rmat18 c3_ba; do
    run $c ADSB_LIB_PATH=ab/libadsb_x128.so; run $c X=1; run $c ADSB_LIB_PATH=ab/libadsb_novf.so; run $c ADSB_LIB_PATH=ab/libadsb_nopf.so
  done
done
ADSB_LIB_PATH=ab/libadsb_phase.so ADSB_TRACE=1 timeout 300 python scripts/prof_one.py c5_rmat24 2 > gpurun_out/r3g/phase_c5.log 2>&1
timeout 1800 python -m pytest tests -q -m gpu --timeout 600 -p no:cacheprovider -rf -x > gpurun_out/r3g/pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r3g/pytest.log
