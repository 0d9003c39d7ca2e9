#!/bin/bash
# config-5 bench + wide-channel parity tests (+ optional A/B env)
tag=${1:-c5}
mkdir -p gpurun_out
python -m paper_2511_22793_b200.build > /dev/null 2>&1
timeout 600 python -m pytest -q -x -m gpu tests/test_gpu_scale.py -k "config5 or wide" tests/test_gpu_forward.py > gpurun_out/pytest_$tag.log 2>&1
tail -2 gpurun_out/pytest_$tag.log
timeout 300 python bench.py --config c5 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c5_$tag.json 2> gpurun_out/bench_c5_$tag.err
python -c "import json;d=json.load(open('gpurun_out/bench_c5_$tag.json'));print('c5', d['value'], d['ms_per_step'], d.get('stages_us'))"
if [ -n "$AB" ]; then
  python -m paper_2511_22793_b200.build --experiments --force > /dev/null 2>&1
  for v in 0 1; do GSPARC_PXB_TMAJ=$v timeout 300 python bench.py --config c5 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys;d=json.loads(sys.stdin.read());print('TMAJ=$v', d['value'], d.get('stages_us'))"; done
fi
