#!/bin/bash
run() { name=$1; shift; timeout 300 python bench.py --steps 10 --no-cpu --no-e2e --no-dense "$@" > gpurun_out/ab_fp8_$name.log 2>&1; }
for r in a b; do run bf16_$r; run fp8_$r --fp8; done
for f in gpurun_out/ab_fp8_*.log; do echo -n "$f "; tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), round(d['stages_ms']['attention'],2), round(d['stages_ms']['permute'],3), d['clocks']['sm_mhz'])" 2>&1 | tail -1; done
