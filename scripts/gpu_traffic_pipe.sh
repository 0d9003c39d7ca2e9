#!/bin/bash
# In-pipeline DRAM traffic per kernel: ncu with --cache-control none (L2 is
# not flushed between kernels, so each kernel sees the L2 state its
# predecessor left, as in the timed graph; the bench's own 256 MiB flush
# still runs between steps).  One metric pass per kernel.
tag=${1:-tp}
mkdir -p gpurun_out
python -m paper_2511_22793_b200.build > /dev/null 2>&1
for cfg in c3 c1 c5; do
  timeout 600 ncu --cache-control none --clock-control none \
    --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    -k regex:"k_(px|tile_sort|preprocess|mlp)" -s 25 -c 100 --csv --log-file gpurun_out/traffic_pipe_${cfg}_$tag.csv \
    python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
done
ls -la gpurun_out/traffic_pipe_*_$tag.csv
