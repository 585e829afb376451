# Closing measurements of the last session (hook-free library): smoke, ncu launch lists -> traffic, bench (20 and 200 steps),
# reference arm, ncu --set full of the TS kernel (20-step launch)
set -u
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/fin_smoke.log
for K in 20 200; do
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size \
  --clock-control none --csv --log-file gpurun_out/r2_traffic_$K.csv \
  python bench.py --steps $K --warmup 5 --no-tts --no-cpu-baseline > gpurun_out/fin_ncu_$K.log 2>&1; echo "ncu $K rc=$?"
done
python tools/traffic_from_ncu.py gpurun_out/r2_traffic_20.csv gpurun_out/r2_traffic_200.csv > /dev/null && cp profiles/r02_traffic.json gpurun_out/r02_traffic.json; echo "traffic rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/fin_bench.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --steps 200 --warmup 5 --no-tts --no-cpu-baseline > gpurun_out/fin_bench200.log 2>&1; echo "bench200 rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/fin_ref.log 2>&1; echo "ref rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gsb_resident_ts --launch-skip 1 -c 1 \
  -o gpurun_out/r2s5_ts_full python tools/step_driver.py --steps 20 > gpurun_out/ncu_ts.log 2>&1; echo "ncu ts rc=$?"
