for v in "GSPARC_X=1" "GSPARC_NO_PDL_B=1" "GSPARC_X=1" "GSPARC_NO_PDL_B=1"; do
  r=$(env $v timeout 300 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])")
  echo "$v $r" >> gpurun_out/ab.txt
done
