# A/B of the block sampler's unroll factor and register budget: each variant is
# built in a scratch copy of the repo, then timed on C2 and C3.
set -u
ROOT=$(pwd)
for v in "1 4" "2 3" "2 4" "4 2" "4 3"; do
  set -- $v
  D=/tmp/var_u$1_m$2
  rm -rf $D; mkdir -p $D
  cp -r paper_1903_09422_b200 include scripts tests oracle $D/ 2>/dev/null
  (cd $D && ADSB_NVCC_EXTRA="-DADSB_UNROLL=$1 -DADSB_MINB_PER_256=$2" python -m paper_1903_09422_b200.build --force > build.log 2>&1)
  for c in c2_rmat18 c3_ba; do
    echo "U=$1 MINB=$2 $( (cd $D && timeout 300 python scripts/prof_one.py $c 2 2>&1 | tail -1) )" >> $ROOT/gpurun_out/variants.log
  done
done
