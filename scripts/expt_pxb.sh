# pass-B timing experiments (GSPARC_PXB_EXPT bits: 1 no coef loads, 2 no
# weights, 4 no MMAs, 8 cp.async producer); results are NOT images
for m in 0 8 1 3 7 4 6; do
  GSPARC_PXB_EXPT=$m timeout 300 python bench.py --no-cpu-baseline --steps 100 > gpurun_out/expt_$m.json 2>/dev/null
done
