# bench c3 twice, printing ms_per_step and the per-stage event times
for i in 1 2; do
  timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], {k: round(v,1) for k,v in d['stages_us'].items()})" >> gpurun_out/ab.txt
done
