mkdir -p gpurun_out/ry
for r in 1 2; do
bash scripts/gpu_ab2.sh "lp2=tk lp4=lp4 lp8=lp8" "c2_rmat18 c5_rmat24 c3_ba" ry/ab.log scripts/prof_one.py 4
done
timeout 1800 python -m pytest tests -x -q -m gpu --timeout 900 -p no:cacheprovider > gpurun_out/ry/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/ry/pytest_gpu.log
