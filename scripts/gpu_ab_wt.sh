#!/bin/bash
# same-box A/B: scratch/wt (a git worktree of the previous commit, built
# in place) against the working tree, config 3 and config 1 alternately;
# then the forward parity tests on the working tree
mkdir -p gpurun_out
for i in 1 2; do
  (cd scratch/wt && timeout 300 python bench.py --no-cpu-baseline) > gpurun_out/abwt_A_$i.json 2>/dev/null
  timeout 300 python bench.py --no-cpu-baseline > gpurun_out/abwt_B_$i.json 2>/dev/null
done
(cd scratch/wt && timeout 300 python bench.py --config c1 --no-cpu-baseline) > gpurun_out/abwt_A_c1.json 2>/dev/null
timeout 300 python bench.py --config c1 --no-cpu-baseline > gpurun_out/abwt_B_c1.json 2>/dev/null
timeout 300 python bench.py --config c2 --steps 50 --no-cpu-baseline > gpurun_out/abwt_B_c2.json 2>/dev/null
timeout 900 python -m pytest tests/test_gpu_forward.py tests/test_gpu_scale.py tests/test_gpu_overlap.py -q -m gpu -p no:cacheprovider > gpurun_out/pytest_abwt.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_abwt.log
