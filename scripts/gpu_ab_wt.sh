#!/bin/bash
# same-box A/B: scratch/wt (a git worktree of the previous commit, built
# in place) against the working tree, config 3 alternately
mkdir -p gpurun_out
for i in 1 2; do
  (cd scratch/wt && timeout 300 python bench.py --no-cpu-baseline) > gpurun_out/abwt_A_$i.json 2>/dev/null
  timeout 300 python bench.py --no-cpu-baseline > gpurun_out/abwt_B_$i.json 2>/dev/null
done
