SBG_RES_GTRACE=1 timeout 120 python tools/step_driver.py --steps 20 > gpurun_out/s5_gtrace.log 2>&1; tail -1 gpurun_out/s5_gtrace.log
python tools/dev/gtrace_groups.py gpurun_out/res_gtrace_20.txt
