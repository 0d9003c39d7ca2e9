#!/bin/bash
# Round-2 GPU pass: parity tests, smoke, benches of every config (incl. the
# self-launched 2-rank path), per-kernel launch list.  Usage:
#   bash scripts/gpu_r02.sh TAG [tests|bench|all]
tag=${1:-q}; what=${2:-all}
mkdir -p gpurun_out
lscpu > gpurun_out/lscpu.txt 2>&1
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
if [ "$what" != bench ]; then
timeout 1500 python -m pytest tests/ -q -m gpu --maxfail=20 -p no:cacheprovider -rs > gpurun_out/pytest_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_$tag.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$tag.log
fi
if [ "$what" != tests ]; then
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3_$tag.json 2> gpurun_out/bench_c3_$tag.err
timeout 300 python bench.py --config c1 > gpurun_out/bench_c1_$tag.json 2> gpurun_out/bench_c1_$tag.err
timeout 400 python bench.py --config c2 --steps 50 > gpurun_out/bench_c2_$tag.json 2> gpurun_out/bench_c2_$tag.err
timeout 300 python bench.py --config c4 --steps 50 --no-cpu-baseline > gpurun_out/bench_c4_$tag.json 2> gpurun_out/bench_c4_$tag.err
timeout 300 python bench.py --config c4 --gpus 2 --steps 30 --no-cpu-baseline > gpurun_out/bench_c4g2_$tag.json 2> gpurun_out/bench_c4g2_$tag.err
timeout 300 python bench.py --config c5 > gpurun_out/bench_c5_$tag.json 2> gpurun_out/bench_c5_$tag.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file gpurun_out/launches_$tag.csv python bench.py --steps 10 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
fi
echo done
