for v in "GSPARC_PXA_MIX=1" "GSPARC_PXA_MIX=0" "GSPARC_PXA_MIX=1" "GSPARC_PXA_MIX=0"; do
  env $v timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['p50_ms'])" >> gpurun_out/ab7.txt
done
GSPARC_PXA_MIX=1 python scripts/timeline_c3.py > gpurun_out/tl_ma.txt 2>&1
