timeout 900 python -m pytest tests/test_gpu_acceptance.py -q -k "criterion_5 or criterion_6" > gpurun_out/r2c21.log 2>&1; echo rc=$?; tail -15 gpurun_out/r2c21.log
