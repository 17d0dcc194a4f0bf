#!/bin/bash
# A/B of the exp2 MUFU/FMA split: bench (attention stage) per SVG2_EXP_POLY_STRIDE
for s in 0 8 4 2; do
  SVG2_EXP_POLY_STRIDE=$s timeout 300 python bench.py --steps 5 --no-cpu --no-e2e --no-dense > gpurun_out/bench_poly$s.log 2>&1
done
