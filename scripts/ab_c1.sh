for c in c1 c3 c1 c3 c2; do
  timeout 300 python bench.py --config $c --no-cpu-baseline --steps 50 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['value'], d['ms_per_step'], d.get('p50_ms'))" >> gpurun_out/ab12.txt
done
