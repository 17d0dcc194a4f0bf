#!/bin/bash
# A/B of two library builds (timing only)
run() { name=$1; shift; env "$@" timeout 300 python bench.py --steps 10 --no-cpu --no-e2e --no-dense > gpurun_out/ab_lib_$name.log 2>&1; }
for r in a b c; do run base_$r SVG2_LIBRARY=build/libsvg2_base.so; run lpt_$r SVG2_LIBRARY=build/libsvg2_lpt.so; done
for f in gpurun_out/ab_lib_*.log; do echo -n "$f "; tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), round(d['stages_ms']['attention'],2), d['clocks']['sm_mhz'])" 2>&1 | tail -1; done
