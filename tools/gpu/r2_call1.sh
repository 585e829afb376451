set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python bench.py --steps 20 --warmup 5 --no-tts --no-cpu-baseline > gpurun_out/r2_bench20.log 2>&1
python bench.py --steps 200 --warmup 5 --no-tts --no-cpu-baseline > gpurun_out/r2_bench200.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gsb_resident_parts -s 1 -c 1 -o gpurun_out/r2_res_full python bench.py --steps 20 --warmup 5 --no-tts --no-cpu-baseline > gpurun_out/r2_ncu.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputests.log 2>&1
tail -3 gpurun_out/r2_gputests.log
