for K in 20 200; do
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/r2_traffic_$K.csv python bench.py --steps $K --warmup 5 --no-tts --no-cpu-baseline > gpurun_out/r2_traffic_$K.log 2>&1
echo "K=$K rc=$?"
done
ls -la gpurun_out/
