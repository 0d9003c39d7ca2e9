#!/bin/bash
# forward-path iteration: forward parity tests + c3/c1/c5 benches
tag=${1:-f}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_forward.py tests/test_gpu_overlap.py tests/test_gpu_scale.py -q -x -p no:cacheprovider -m gpu > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$tag.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_c3_$tag.json 2> gpurun_out/bench_c3_$tag.err
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_c3b_$tag.json 2> gpurun_out/bench_c3b_$tag.err
timeout 300 python bench.py --config c1 --no-cpu-baseline > gpurun_out/bench_c1_$tag.json 2> gpurun_out/bench_c1_$tag.err
timeout 300 python bench.py --config c5 --steps 30 > gpurun_out/bench_c5_$tag.json 2> gpurun_out/bench_c5_$tag.err
echo done
