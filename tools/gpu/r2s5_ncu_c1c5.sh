# ncu --set full of the C1 planes pair kernel (20-step launch) and the C5 single-GPU e2m1 streaming pair kernel (4-step launch)
timeout 300 python tools/configs_bench.py --only C1 --steps 20 2>&1 | grep -o '"us_per_step": [0-9.]*'
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gsb_multistep_pair_kernel --launch-skip 1 -c 1 \
  -o gpurun_out/r2s5_c1_full python tools/configs_bench.py --only C1 --steps 20 > gpurun_out/ncu_c1.log 2>&1; echo "ncu c1 rc=$?"
timeout 300 python tools/c5_bench.py --steps 4 2>&1 | tail -1 | cut -c1-160
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:gsb_multistep_pair_kernel --launch-skip 1 -c 1 \
  -o gpurun_out/r2s5_c5_full python tools/c5_bench.py --steps 4 > gpurun_out/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
