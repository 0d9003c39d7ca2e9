for v in "GSPARC_X=1" "GSPARC_NO_PDL_K2=1" "GSPARC_X=1" "GSPARC_NO_PDL_K2=1"; do
  env $v timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['p50_ms'], d['gpu_launches'])" >> gpurun_out/ab9.txt
done
