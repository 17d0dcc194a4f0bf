#!/bin/bash
# A/B runs of the attention-kernel switches (timing only): writes gpurun_out/ab_<name>.log
run() { name=$1; shift; env "$@" timeout 300 python bench.py --steps 10 --no-cpu --no-e2e --no-dense > gpurun_out/ab_$name.log 2>&1; }
run base
run split SVG2_SPLIT_P=1
run nosm SVG2_DEBUG_MODE=1
