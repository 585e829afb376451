# fused multi-step row-shard emulation: the row-shard tests; C5 N=100000 fused timing at G = 2, 4, 8
timeout 600 python -m pytest tests/test_gpu_rowshard.py -q -x > gpurun_out/fused_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/fused_tests.log
