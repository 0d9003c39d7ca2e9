#!/bin/bash
# A/B experiments in one gpurun call: run bench.py once per environment
# setting and append "setting ms_per_step p50_ms" to gpurun_out/ab.txt.
#   bash scripts/ab_env.sh [--config c3] "GSPARC_NO_PDL=1" "GSPARC_X=1" ...
# (needs the experiments build: python -m paper_2511_22793_b200.build --experiments;
#  switches read by the library: GSPARC_NO_PDL, GSPARC_NO_PDL_K2/_K3/_B,
#  GSPARC_PXA_SMEM, GSPARC_PXB_MIX, GSPARC_BIN_SMALL, GSPARC_MLP_SBLOCKS)
cfg=c3
if [ "$1" = "--config" ]; then cfg=$2; shift 2; fi
mkdir -p gpurun_out
for v in "$@"; do
  env $v timeout 300 python bench.py --config $cfg --no-cpu-baseline 2>/dev/null | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg $v', d['ms_per_step'], d.get('p50_ms'))" \
    >> gpurun_out/ab.txt
done
