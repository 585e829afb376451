timeout 600 python -m pytest tests/test_gpu_p3_scale.py tests/test_gpu_rowshard.py -x -q > gpurun_out/r2c6_a.log 2>&1; tail -5 gpurun_out/r2c6_a.log
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "dt_sweep or reused" > gpurun_out/r2c6_b.log 2>&1; tail -5 gpurun_out/r2c6_b.log
timeout 300 python -m pytest tests/test_gpu_rowshard_ipc.py -x -q > gpurun_out/r2c6_c.log 2>&1; tail -15 gpurun_out/r2c6_c.log
