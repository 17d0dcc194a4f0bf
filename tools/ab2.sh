#!/bin/bash
# A/B of the attention pipeline designs (v2: 128-key S, v3: double-buffered 64-key S), timing only
run() { name=$1; shift; env "$@" timeout 300 python bench.py --steps 10 --no-cpu --no-e2e --no-dense > gpurun_out/ab_$name.log 2>&1; }
run v2 SVG2_ATTN_VARIANT=2
run v3 SVG2_ATTN_VARIANT=3
run v2nosm SVG2_ATTN_VARIANT=2 SVG2_DEBUG_MODE=1
run v2p8 SVG2_ATTN_VARIANT=2 SVG2_EXP_POLY_STRIDE=8
run v3p8 SVG2_ATTN_VARIANT=3 SVG2_EXP_POLY_STRIDE=8
