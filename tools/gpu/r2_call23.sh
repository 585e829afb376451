timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ts_kernel or resident or e2m1 or c2_shape or pipelined or p2" > gpurun_out/r2c23_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r2c23_tests.log
for pkb in 1 0; do
SBG_RES_PKB=$pkb timeout 300 python bench.py --steps 20 --warmup 5 --no-tts --no-cpu-baseline --no-configs > gpurun_out/r2c23_b20_$pkb.log 2>&1
SBG_RES_PKB=$pkb timeout 300 python bench.py --steps 200 --warmup 5 --no-tts --no-cpu-baseline --no-configs > gpurun_out/r2c23_b200_$pkb.log 2>&1
done
grep -o '"ms_per_step": [0-9.e-]*' gpurun_out/r2c23_b*.log
SBG_RES_TRACE=1 timeout 300 python tools/step_driver.py --steps 60 > gpurun_out/r2c23_t.log 2>&1
