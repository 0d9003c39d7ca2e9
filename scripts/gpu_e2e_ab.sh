mkdir -p gpurun_out
for nb in 2 3 4; do
timeout 300 python bench.py --no-cpu-baseline --e2e-buffers $nb > gpurun_out/e2e_nb$nb.json 2> gpurun_out/e2e_nb$nb.err
done
timeout 300 python bench.py --config c1 --no-cpu-baseline --e2e-buffers 2 > gpurun_out/e2e_c1_nb2.json 2> gpurun_out/e2e_c1.err
timeout 300 python bench.py --config c1 --no-cpu-baseline --e2e-buffers 3 > gpurun_out/e2e_c1_nb3.json 2>> gpurun_out/e2e_c1.err
