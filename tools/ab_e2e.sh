#!/bin/bash
# Interleaved A/B of the host-buffer (e2e) path: each argument "name:ENV=VAL[,ENV=VAL...]"; prints
#   name_rep  ms_per_call  e2e_ms  sm_mhz
set -u
reps=${AB_REPS:-2}
for r in $(seq 1 "$reps"); do
  for spec in "$@"; do
    name=${spec%%:*}; envs=${spec#*:}
    env ${envs//,/ } timeout 300 python bench.py --steps 10 --no-cpu --no-dense > "gpurun_out/abe_${name}_${r}.log" 2>&1
  done
done
for spec in "$@"; do
  name=${spec%%:*}
  for r in $(seq 1 "$reps"); do
    echo -n "${name}_${r} "
    tail -1 "gpurun_out/abe_${name}_${r}.log" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2), d['clocks']['sm_mhz'])" 2>&1 | tail -1
  done
done
