#!/bin/bash
# training parity tests + config-2 / config-4 benches
tag=${1:-tb}
mkdir -p gpurun_out
python -m paper_2511_22793_b200.build > gpurun_out/build_$tag.log 2>&1 || { tail -20 gpurun_out/build_$tag.log; exit 1; }
timeout 900 python -m pytest -q -x -m gpu tests/test_gpu_train.py tests/test_gpu_backward.py tests/test_gpu_dp.py > gpurun_out/pytest_$tag.log 2>&1
tail -1 gpurun_out/pytest_$tag.log
for c in c2 c4; do
  timeout 400 python bench.py --config $c --steps 50 --no-cpu-baseline > gpurun_out/bench_${c}_$tag.json 2> gpurun_out/bench_${c}_$tag.err
  python -c "import json;d=json.load(open('gpurun_out/bench_${c}_$tag.json'));print('$c', round(d['value'],1), round(d['e2e']['value'],1), {k: round(v,1) for k,v in d['stages_us'].items()})"
done
