#!/bin/bash
# Tensor-pipe activity of pass B (k_pxb) for configs 3 and 5: one ncu capture
# of one launch each (ComputeWorkloadAnalysis section + tensor pipe metrics).
# Usage: bash scripts/gpu_tc_pipe.sh TAG
tag=${1:-tc}
mkdir -p gpurun_out
for c in c3 c5; do
  timeout 600 ncu --clock-control none -k regex:k_pxb -s 3 -c 1 \
    --section ComputeWorkloadAnalysis --section SpeedOfLight \
    --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.max.pct_of_peak_sustained_active,gpu__time_duration.sum,sm__cycles_active.avg \
    --csv --page raw --log-file gpurun_out/tcpipe_${c}_$tag.csv \
    python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/tcpipe_${c}_$tag.log 2>&1
  echo "$c rc=$?" >> gpurun_out/tcpipe_${c}_$tag.log
done
