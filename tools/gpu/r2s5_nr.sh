# resident kernel choice when NR = 160 and NR = 128 need the same number of groups: TS (new) vs 128-wide (old rule)
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "ts_kernel or resident or e2m1 or c2_shape or run_pipelined or run_best or p2_" > gpurun_out/s5_nr_tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/s5_nr_tests.log
for R in 1000 1440 2304 4320 8192; do for rule in 0 1; do
SBG_RES_NR_TS=$rule timeout 120 python tools/step_driver.py --steps 200 --warm 600 --R $R 2>&1 | tail -1 | sed "s/^/nr_ts=$rule /"
done; done
