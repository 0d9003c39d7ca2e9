#!/bin/bash
# forward/scale parity tests + config-3 and config-5 benches
tag=${1:-fb}
mkdir -p gpurun_out
python -m paper_2511_22793_b200.build > gpurun_out/build_$tag.log 2>&1 || { tail -20 gpurun_out/build_$tag.log; exit 1; }
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_forward.py tests/test_gpu_scale.py > gpurun_out/pytest_$tag.log 2>&1
tail -2 gpurun_out/pytest_$tag.log
timeout 300 python bench.py --steps 200 --warmup 20 --no-cpu-baseline > gpurun_out/bench_c3_$tag.json 2> gpurun_out/bench_c3_$tag.err
timeout 300 python bench.py --config c5 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c5_$tag.json 2> gpurun_out/bench_c5_$tag.err
timeout 300 python bench.py --config c1 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c1_$tag.json 2> gpurun_out/bench_c1_$tag.err
for c in c3 c5 c1; do python -c "import json;d=json.load(open('gpurun_out/bench_${c}_$tag.json'));print('$c', round(d['value'],1), 'p50', d['p50_ms'], 'p99', d['p99_ms'], {k: round(v,1) for k,v in d['stages_us'].items()})"; done
