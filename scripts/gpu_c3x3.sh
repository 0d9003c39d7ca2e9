mkdir -p gpurun_out
for i in 1 2 3; do timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_c3_ab10_$i.json 2>/dev/null; done
timeout 300 python bench.py --config c5 > gpurun_out/bench_c5_ab10.json 2>/dev/null
