#!/bin/bash
# Quick GPU iteration: parity tests, smoke, config-3/1/2 bench (no CPU leg),
# per-kernel launch list.  Usage: bash scripts/gpu_quick.sh [tag]
tag=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -q -m gpu --maxfail=15 -p no:cacheprovider > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$tag.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_c3_$tag.json 2> gpurun_out/bench_c3_$tag.err
timeout 300 python bench.py --config c1 --no-cpu-baseline > gpurun_out/bench_c1_$tag.json 2> gpurun_out/bench_c1_$tag.err
timeout 300 python bench.py --config c2 --steps 30 > gpurun_out/bench_c2_$tag.json 2> gpurun_out/bench_c2_$tag.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none -c 200 --csv \
  --log-file gpurun_out/launches_$tag.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo done
