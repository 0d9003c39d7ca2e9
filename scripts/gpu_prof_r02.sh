#!/bin/bash
# ncu --set full captures of the benched kernels (c3 render, c1 render,
# c2 train backward) + the e2e diagnostic.  Outputs under gpurun_out/.
tag=${1:-p}
mkdir -p gpurun_out
timeout 300 python scripts/diag_e2e.py c3 > gpurun_out/diag_e2e_c3_$tag.txt 2>&1
timeout 300 python scripts/diag_e2e.py c1 > gpurun_out/diag_e2e_c1_$tag.txt 2>&1
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3_$tag.json 2> gpurun_out/bench_c3_$tag.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_(px|tile_sort|preprocess|mlp)" -s 12 -c 5 \
  -o gpurun_out/prof_c3_$tag python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/prof_c3_$tag.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_(px|tile_sort|preprocess|mlp)" -s 8 -c 4 \
  -o gpurun_out/prof_c1_$tag python bench.py --config c1 --steps 2 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/prof_c1_$tag.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_(raster_bwd|gauss_bwd|adam)" -s 3 -c 3 \
  -o gpurun_out/prof_c2_$tag python bench.py --config c2 --steps 2 --warmup 1 --no-cpu-baseline --no-graph > gpurun_out/prof_c2_$tag.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
  --log-file gpurun_out/launches_c2_$tag.csv python bench.py --config c2 --steps 5 --warmup 2 --no-cpu-baseline > /dev/null 2>&1
echo done
