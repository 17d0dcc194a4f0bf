#!/bin/bash
# e2e host-pipeline chunking A/B -> gpurun_out/ab_host_<name>.log
run() { name=$1; shift; env "$@" timeout 300 python bench.py --steps 5 --no-cpu --no-dense > gpurun_out/ab_host_$name.log 2>&1; }
for c in 2 3 4 6; do run r1_c$c SVG2_HOST_RAMP=1 SVG2_HOST_CHUNKS=$c; done
run r0_c6 SVG2_HOST_RAMP=0 SVG2_HOST_CHUNKS=6
for f in gpurun_out/ab_host_*.log; do echo -n "$f "; tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2))" 2>&1 | tail -1; done
