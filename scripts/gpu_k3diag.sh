#!/bin/bash
# K3 per-phase clocks (experiments build), then the normal build: forward /
# scale parity tests and a config-3 bench (outputs under gpurun_out/)
tag=${1:-k3}
mkdir -p gpurun_out
python -m paper_2511_22793_b200.build --experiments --force > gpurun_out/build_$tag.log 2>&1 || { tail -30 gpurun_out/build_$tag.log; exit 1; }
timeout 300 python scripts/dbg_sort.py > gpurun_out/dbg_sort_$tag.txt 2>&1
[ -n "$C5" ] && timeout 300 python scripts/dbg_sort_c5.py > gpurun_out/dbg_sort_c5_$tag.txt 2>&1 && cat gpurun_out/dbg_sort_c5_$tag.txt
[ -n "$TIMELINE" ] && timeout 300 python scripts/timeline_c3.py > gpurun_out/timeline_$tag.txt 2>&1
python -m paper_2511_22793_b200.build --force > gpurun_out/build2_$tag.log 2>&1 || { tail -30 gpurun_out/build2_$tag.log; exit 1; }
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_forward.py tests/test_gpu_scale.py > gpurun_out/pytest_$tag.log 2>&1
tail -3 gpurun_out/pytest_$tag.log
timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline > gpurun_out/bench_c3_$tag.json 2> gpurun_out/bench_c3_$tag.err
cat gpurun_out/dbg_sort_$tag.txt | head -30
[ -n "$TIMELINE" ] && head -12 gpurun_out/timeline_$tag.txt
python -c "import json;d=json.load(open('gpurun_out/bench_c3_$tag.json'));print('c3', d['value'], d['ms_per_step'], d.get('latency_ms') or {k:v for k,v in d.items() if 'p50' in k or 'p99' in k})"
