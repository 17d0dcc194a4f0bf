#!/bin/bash
# Timing runs (no A/B switch) -> gpurun_out/ab_var_<name>.log, summary on stdout
run() { name=$1; shift; env "$@" timeout 300 python bench.py --steps 10 --no-cpu --no-e2e --no-dense > gpurun_out/ab_var_$name.log 2>&1; }
for r in a b; do run cur_$r; done
for f in gpurun_out/ab_var_*.log; do echo -n "$f "; tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); st=d['stages_ms']; print(round(d['ms_per_step'],2), {k: round(v,3) for k,v in st.items()}, d['clocks']['sm_mhz'])" 2>&1 | tail -1; done
