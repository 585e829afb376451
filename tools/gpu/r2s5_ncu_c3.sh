# ncu --set full of one C3 lean CSR step launch (256-replica slab), source counters; timing first without ncu
timeout 200 python tools/configs_bench.py --only C3 --steps 20 2>&1 | grep -o '"us_per_step": [0-9.]*'
timeout 600 ncu --set full --import-source on --clock-control none -k regex:csr_step_lean --launch-skip 30 -c 1 \
  -o gpurun_out/r2s5_c3_lean python tools/configs_bench.py --only C3 --steps 20 > gpurun_out/ncu_c3_lean.log 2>&1; echo "ncu rc=$?"
