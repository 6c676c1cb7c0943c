mkdir -p gpurun_out/rx
for r in 1 2 3; do
bash scripts/gpu_ab2.sh "tk=tk notk=notk" "c2_rmat18 c5_rmat24" rx/ab.log scripts/prof_one.py 4
done
