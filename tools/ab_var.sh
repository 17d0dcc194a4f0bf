#!/bin/bash
# Interleaved A/B of attention options (timing only) -> gpurun_out/ab_var_<name>.log, summary on stdout
run() { name=$1; shift; env "$@" timeout 300 python bench.py --steps 10 --no-cpu --no-e2e --no-dense > gpurun_out/ab_var_$name.log 2>&1; }
for r in a b; do for k in 4 6 8 10; do run p${k}_$r SVG2_EXP_POLY=$k; done; done
for f in gpurun_out/ab_var_*.log; do echo -n "$f "; tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), round(d['stages_ms']['attention'],2), d['clocks']['sm_mhz'])" 2>&1 | tail -1; done
