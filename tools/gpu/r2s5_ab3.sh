timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "ts_kernel or resident or c2_shape or run_pipelined or run_best or p2_ or map_cache" > gpurun_out/s5_ab3_tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -2 gpurun_out/s5_ab3_tests.log
[ $rc -eq 0 ] || exit 1
bash tools/gpu/r2s5_ab.sh
