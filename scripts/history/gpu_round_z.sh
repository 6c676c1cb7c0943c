mkdir -p gpurun_out/rz
for r in 1 2; do
bash scripts/gpu_ab2.sh "lp8=lp8 lp16=lp16 lp32=lp32" "c2_rmat18 c5_rmat24 c3_ba" rz/ab.log scripts/prof_one.py 4
done
