#!/bin/bash
# Run on the GPU box (gpurun): launch list + one `ncu --set full` capture per hot kernel.
# Usage: bash tools/profile.sh [workload]
set -u
WL=${1:-hunyuan720p}
OUT=gpurun_out
mkdir -p $OUT
# 1) every launch of one warm bench step, device time each (cold cache, serialised: compare shares)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$WL.csv \
  python bench.py --workload $WL --profile-once > $OUT/ncu_launches_stdout.log 2>&1
# 2) full sections of the attention kernel (skip the cold call's launch)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_varblock_attn -s 1 -c 1 \
  -o $OUT/prof_attn_$WL -f python bench.py --workload $WL --profile-once > $OUT/ncu_attn_stdout.log 2>&1
# 3) the k-means assign kernel
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_assign_tc -s 10 -c 1 \
  -o $OUT/prof_assign_$WL -f python bench.py --workload $WL --profile-once > $OUT/ncu_assign_stdout.log 2>&1
ls -la $OUT
