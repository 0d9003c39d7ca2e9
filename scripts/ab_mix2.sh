for c in c5 c1 c3; do for v in "GSPARC_PXB_MIX=1" "GSPARC_PXB_MIX=0"; do
  env $v timeout 300 python bench.py --config $c --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $v', d['value'], d['ms_per_step'], d['p50_ms'])" >> gpurun_out/ab6.txt
done; done
