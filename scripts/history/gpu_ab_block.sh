# A/B: block size and hash capacity of the block-team sampler (C2 fused epochs, C3 deterministic)
for cfg in "256 2048" "256 1024" "128 2048" "128 1024" "128 512"; do
  set -- $cfg
  for c in c2_rmat18 c3_ba; do
    ADSB_BLOCK=$1 ADSB_HASH_CAP=$2 timeout 300 python scripts/prof_one.py $c 3 2>&1 | tail -n 1 | sed "s/^/bt=$1 H=$2 /" >> gpurun_out/ab_block.log
  done
done
