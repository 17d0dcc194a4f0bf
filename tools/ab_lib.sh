#!/bin/bash
# Interleaved A/B timing of library builds on one box (the power-capped clock drifts between boxes, so only runs
# interleaved in one gpurun call are compared).  Each argument is "name:path/to/libsvg2.so"; extra bench flags in
# AB_FLAGS.  Writes gpurun_out/ab_<name>_<rep>.log and prints  name_rep ms_per_call attention_ms sm_mhz.
set -u
reps=${AB_REPS:-2}
flags=${AB_FLAGS:-"--steps 10 --no-cpu --no-e2e --no-dense"}
for r in $(seq 1 "$reps"); do
  for spec in "$@"; do
    name=${spec%%:*}
    lib=${spec#*:}
    SVG2_LIBRARY=$lib timeout 300 python bench.py $flags > "gpurun_out/ab_${name}_${r}.log" 2>&1
  done
done
for spec in "$@"; do
  name=${spec%%:*}
  for r in $(seq 1 "$reps"); do
    echo -n "${name}_${r} "
    tail -1 "gpurun_out/ab_${name}_${r}.log" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), round(d['stages_ms']['attention'],2), d['clocks']['sm_mhz'], round(d['roofline']['frac'],3), round(d['density'],4), 'kmeans', round(d['stages_ms']['kmeans_k']+d['stages_ms']['kmeans_q'],3))" 2>&1 | tail -1
  done
done
