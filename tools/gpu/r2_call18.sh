timeout 900 python -m pytest tests/test_gpu_statistics.py -q -rs > gpurun_out/r2c18.log 2>&1; echo rc=$?; tail -15 gpurun_out/r2c18.log
