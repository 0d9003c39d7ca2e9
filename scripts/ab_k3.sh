for v in "GSPARC_X=1" "GSPARC_NO_PDL_K3=1" "GSPARC_X=1" "GSPARC_NO_PDL_K3=1"; do
  env $v timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['p50_ms'])" >> gpurun_out/ab8.txt
done
python scripts/timeline_c3.py > gpurun_out/tl_k3.txt 2>&1
