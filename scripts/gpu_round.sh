#!/bin/bash
# One gpurun call: GPU parity tests, smoke, benches, ncu launch list and a
# full capture of the top kernels.  Outputs under gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 300 python bench.py --config c1 --no-cpu-baseline > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 300 python bench.py --config c2 --steps 50 > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 300 python bench.py --config c2 --steps 50 --deterministic > gpurun_out/bench_c2det.json 2> gpurun_out/bench_c2det.err
timeout 300 python bench.py --config c5 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 300 python scripts/timeline_c3.py > gpurun_out/timeline_c3.txt 2>&1
timeout 300 python scripts/dbg_prep.py > gpurun_out/dbg_prep.txt 2>&1
timeout 400 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_(px|tile_sort|bin|preprocess|mlp)" -s 10 -c 5 \
  -o gpurun_out/prof_c3 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/prof_c3.log 2>&1
ls -la gpurun_out
