#!/bin/bash
# ncu --set full of one pass-A launch (config 3) with source correlation;
# the stall columns are read here with scripts/ncu_sass_hot.py.
tag=${1:-s}
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_pxa" -s 3 -c 1 \
  -o gpurun_out/prof_pxa_$tag python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/prof_pxa_$tag.log 2>&1
echo "rc=$?" >> gpurun_out/prof_pxa_$tag.log
