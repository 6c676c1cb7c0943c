# A/B of environment settings on the current build; usage: bash scripts/gpu_ab_env.sh "ENV1=a ENV2=b|ENV1=c" "cfg..." out.log
IFS='|' read -ra SETTINGS <<< "$1"; CONFIGS="$2"; OUT="gpurun_out/$3"
for round in 1 2; do
  for st in "${SETTINGS[@]}"; do
    for c in $CONFIGS; do
      env $st timeout 600 python scripts/prof_one.py $c 3 2>&1 | tail -n 1 | sed "s/^/[$st] /" >> $OUT
    done
  done
done
