timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "ts_kernel or c2_shape" > gpurun_out/r2c20_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r2c20_tests.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-tts --no-cpu-baseline --no-configs > gpurun_out/r2c20_b20.log 2>&1
timeout 300 python bench.py --steps 200 --warmup 5 --no-tts --no-cpu-baseline --no-configs > gpurun_out/r2c20_b200.log 2>&1
grep -o '"ms_per_step": [0-9.e-]*' gpurun_out/r2c20_b*.log
SBG_RES_TRACE=1 timeout 300 python tools/step_driver.py --steps 60 > gpurun_out/r2c20_t.log 2>&1
