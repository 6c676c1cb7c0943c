# A/B of libadsb builds in ab/ (ADSB_LIB_PATH), interleaved; usage: bash scripts/gpu_ab.sh "v1 v2 ..." "cfg1 cfg2 ..." out.log [tests]
VARIANTS="$1"; CONFIGS="$2"; OUT="gpurun_out/$3"
if [ "$4" = "tests" ]; then
  timeout 1500 python -m pytest tests -q -x -m gpu --timeout 600 -p no:cacheprovider > gpurun_out/pytest_ab.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_ab.log
fi
for round in 1 2; do
  for v in $VARIANTS; do
    for c in $CONFIGS; do
      ADSB_LIB_PATH=ab/libadsb_$v.so timeout 600 python scripts/prof_one.py $c 3 2>&1 | tail -n 1 | sed "s/^/$v /" >> $OUT
    done
  done
done
