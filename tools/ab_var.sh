#!/bin/bash
# Interleaved A/B timing of attention / library variants on one box (the power-capped clock drifts between boxes, so
# only runs interleaved in one gpurun call are compared).  Each argument is "name:ENV=VAL[,ENV=VAL...]"; the default
# compares the two attention pipelines that remain switchable.  Writes gpurun_out/ab_<name>_<rep>.log and prints
#   name_rep  ms_per_call  attention_ms  sm_mhz
# Examples:  bash tools/ab_var.sh v2:SVG2_ATTN_VARIANT=2 v3:SVG2_ATTN_VARIANT=3
#            bash tools/ab_var.sh base:SVG2_LIBRARY=build/a.so new:SVG2_LIBRARY=build/b.so
#            bash tools/ab_var.sh poly0:SVG2_EXP_POLY=0 poly4:SVG2_EXP_POLY=4
set -u
specs=("$@")
[ ${#specs[@]} -eq 0 ] && specs=("v2:SVG2_ATTN_VARIANT=2" "v3:SVG2_ATTN_VARIANT=3")
reps=${AB_REPS:-2}
for r in $(seq 1 "$reps"); do
  for spec in "${specs[@]}"; do
    name=${spec%%:*}
    envs=${spec#*:}
    env ${envs//,/ } timeout 300 python bench.py --steps 10 --no-cpu --no-e2e --no-dense > "gpurun_out/ab_${name}_${r}.log" 2>&1
  done
done
for spec in "${specs[@]}"; do
  name=${spec%%:*}
  for r in $(seq 1 "$reps"); do
    echo -n "${name}_${r} "
    tail -1 "gpurun_out/ab_${name}_${r}.log" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), round(d['stages_ms']['attention'],2), d['clocks']['sm_mhz'])" 2>&1 | tail -1
  done
done
