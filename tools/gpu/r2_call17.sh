for K in 20 200; do
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/r2_traffic_$K.csv python bench.py --steps $K --warmup 5 --no-tts --no-cpu-baseline > gpurun_out/r2_traffic_$K.log 2>&1
echo "K=$K rc=$?"
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gsb_resident_ts -s 1 -c 1 -o gpurun_out/r2_ts_full python bench.py --steps 20 --warmup 5 --no-tts --no-cpu-baseline --no-configs > gpurun_out/r2_ts_ncu.log 2>&1
echo "full rc=$?"
