#!/bin/bash
# A/B iteration: forward/train parity tests, then config-3/1/2/5 benches
# without the CPU leg.  Usage: bash scripts/gpu_ab.sh TAG [tests...]
tag=${1:-ab}; shift
tests=${@:-tests/test_gpu_forward.py tests/test_gpu_train.py}
mkdir -p gpurun_out
timeout 900 python -m pytest $tests -q -m gpu -x -p no:cacheprovider > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$tag.log
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_c3_${tag}_$i.json 2> gpurun_out/bench_c3_$tag.err
done
timeout 300 python bench.py --config c1 --no-cpu-baseline > gpurun_out/bench_c1_$tag.json 2> gpurun_out/bench_c1_$tag.err
timeout 300 python bench.py --config c2 --steps 30 --no-cpu-baseline > gpurun_out/bench_c2_$tag.json 2> gpurun_out/bench_c2_$tag.err
timeout 300 python bench.py --config c5 > gpurun_out/bench_c5_$tag.json 2> gpurun_out/bench_c5_$tag.err
echo done
