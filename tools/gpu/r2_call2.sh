set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "resident or e2m1 or c2_shape or pipelined or p2" > gpurun_out/r2c2_tests.log 2>&1
tail -3 gpurun_out/r2c2_tests.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-tts --no-cpu-baseline > gpurun_out/r2c2_bench20.log 2>&1
timeout 300 python bench.py --steps 200 --warmup 5 --no-tts --no-cpu-baseline > gpurun_out/r2c2_bench200.log 2>&1
grep -o '"ms_per_step": [0-9.e-]*' gpurun_out/r2c2_bench*.log
