#!/bin/bash
# A/B of the softmax switches (timing only) -> gpurun_out/ab_spec_<name>.log, summary on stdout
run() { name=$1; shift; env "$@" timeout 300 python bench.py --steps 10 --no-cpu --no-e2e --no-dense > gpurun_out/ab_spec_$name.log 2>&1; }
run s0 SVG2_SPECULATIVE_EXP=0
run s1 SVG2_SPECULATIVE_EXP=1
run s0b SVG2_SPECULATIVE_EXP=0
run s1b SVG2_SPECULATIVE_EXP=1
for f in gpurun_out/ab_spec_*.log; do echo -n "$f "; tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), round(d['stages_ms']['attention'],2), d['clocks']['sm_mhz'])"; done
