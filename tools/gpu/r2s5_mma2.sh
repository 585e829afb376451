export SBG_LIB_OVERRIDE=$PWD/tools/ab/mma2.so
timeout 100 python tools/step_driver.py --steps 20 --warm 20 2>&1 | tail -1
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "ts_kernel or resident_kernel_equals or c2_shape or e2m1_resident or run_pipelined" > gpurun_out/s5_mma2_tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/s5_mma2_tests.log
unset SBG_LIB_OVERRIDE
[ $rc -eq 0 ] || exit 1
AB="base mma2" bash tools/gpu/r2s5_ab.sh
