set -x
nproc > gpurun_out/nproc.txt
for c in c1_er c2_rmat18 c3_ba; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c exit $?" >> gpurun_out/bench_status.txt
done
