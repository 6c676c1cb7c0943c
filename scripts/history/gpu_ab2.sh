# A/B of (lib, env) variants, interleaved over 2 rounds.
# usage: bash scripts/gpu_ab2.sh "name=lib[:VAR=val,...] ..." "cfg1 cfg2" out.log [script args]
VARIANTS="$1"; CONFIGS="$2"; OUT="gpurun_out/$3"; SCRIPT=${4:-"scripts/prof_one.py"}; SARGS=${5:-3}
for round in 1 2; do
  for spec in $VARIANTS; do
    name=${spec%%=*}; rest=${spec#*=}; lib=${rest%%:*}; envs=""
    [ "$rest" != "$lib" ] && envs=$(echo ${rest#*:} | tr ',' ' ')
    for c in $CONFIGS; do
      env $envs ADSB_LIB_PATH=ab/libadsb_$lib.so timeout 900 python $SCRIPT $c $SARGS 2>&1 | tail -n 1 | sed "s/^/$name /" >> $OUT
    done
  done
done
