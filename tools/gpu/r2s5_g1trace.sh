export SBG_LIB_OVERRIDE=$PWD/paper_2508_17655_b200/libsbgpu_dev.so
SBG_RES_TRACE=2 timeout 120 python tools/step_driver.py --steps 20 --warm 900 > gpurun_out/s5_g1.log 2>&1; tail -1 gpurun_out/s5_g1.log
python tools/dev/trace_group_steps.py gpurun_out/res_trace.txt
