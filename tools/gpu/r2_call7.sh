timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2c7_bench.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/r2c7_bench.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2c7_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/r2c7_tests.log
