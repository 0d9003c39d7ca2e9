#!/bin/bash
# ncu --set full captures of the final build's benched kernels (c3, c1, c2,
# c5) + the in-pipeline DRAM traffic run.  Outputs under gpurun_out/.
tag=${1:-f}
mkdir -p gpurun_out
python -m paper_2511_22793_b200.build > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_(px|tile_sort|preprocess|mlp)" -s 12 -c 5 \
  -o gpurun_out/prof_c3_$tag python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/prof_c3_$tag.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_(px|tile_sort|preprocess|mlp)" -s 8 -c 4 \
  -o gpurun_out/prof_c1_$tag python bench.py --config c1 --steps 2 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/prof_c1_$tag.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_(raster_bwd|gauss_bwd|adam|loss_band)" -s 6 -c 6 \
  -o gpurun_out/prof_c2_$tag python bench.py --config c2 --steps 2 --warmup 1 --no-cpu-baseline --no-graph > gpurun_out/prof_c2_$tag.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(pxb|tile_sort)" -s 2 -c 2 \
  -o gpurun_out/prof_c5_$tag python bench.py --config c5 --steps 1 --warmup 1 --no-cpu-baseline --no-graph > gpurun_out/prof_c5_$tag.log 2>&1
bash scripts/gpu_traffic_pipe.sh $tag
ls -la gpurun_out/prof_*_$tag.ncu-rep
