SBG_RES_GTRACE=1 timeout 300 python bench.py --steps 20 --warmup 5 --no-tts --no-cpu-baseline > gpurun_out/r2c3_bench20.log 2>&1
ls gpurun_out/
