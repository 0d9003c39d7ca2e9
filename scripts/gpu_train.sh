#!/bin/bash
# training-path iteration: train/backward/loss parity tests + c2 bench + launch list
tag=${1:-t}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_backward.py tests/test_gpu_dp.py::test_dp_two_ranks_on_one_gpu "tests/test_gpu_scale.py::test_config2_train_step_parity" tests/test_rfsim.py -q -x -p no:cacheprovider -m gpu > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$tag.log
timeout 300 python bench.py --config c2 --steps 50 --no-cpu-baseline > gpurun_out/bench_c2_$tag.json 2> gpurun_out/bench_c2_$tag.err
timeout 300 python bench.py --config c2 --steps 50 --no-cpu-baseline --deterministic > gpurun_out/bench_c2det_$tag.json 2> gpurun_out/bench_c2det_$tag.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
  --log-file gpurun_out/launches_c2_$tag.csv python bench.py --config c2 --steps 5 --warmup 2 --no-cpu-baseline > /dev/null 2>&1
echo done
