# one ncu --set full capture (source counters) of the C2 TS kernel, 20-step launch
timeout 300 python tools/step_driver.py --steps 20 > gpurun_out/ncu_ts_plain.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gsb_resident_ts --launch-skip 1 -c 1 \
  -o gpurun_out/r2s2_ts_full python tools/step_driver.py --steps 20 > gpurun_out/ncu_ts.log 2>&1; echo "ncu rc=$?"
tail -3 gpurun_out/ncu_ts.log
