for v in 48 32 40 64 1073741824 48 32 40 64 1073741824; do
  GSPARC_BIN_SMALL=$v timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], round(d['stages_us']['preprocess'],1))" >> gpurun_out/ab3.txt
done
