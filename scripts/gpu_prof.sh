#!/bin/bash
# ncu --set full of selected kernels of one config-3 step.
# Usage: bash scripts/gpu_prof.sh <tag> <kernel regex> [bench args...]
tag=$1; shift; kre=$1; shift
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$kre" -s 6 -c 4 \
  -o gpurun_out/prof_$tag python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph "$@" > gpurun_out/prof_$tag.log 2>&1
echo "ncu rc=$?"
