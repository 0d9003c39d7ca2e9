#!/bin/bash
# same-box A/B of the training step: scratch/wt (previous commit) vs the
# working tree, config 2 alternately, then the training parity tests on B
mkdir -p gpurun_out
for i in 1 2; do
  (cd scratch/wt && timeout 300 python bench.py --config c2 --steps 50 --no-cpu-baseline) > gpurun_out/abwt2_A_$i.json 2>/dev/null
  timeout 300 python bench.py --config c2 --steps 50 --no-cpu-baseline > gpurun_out/abwt2_B_$i.json 2>/dev/null
done
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_backward.py tests/test_gpu_dp.py tests/test_gpu_reference_suite.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest_abwt2.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_abwt2.log
