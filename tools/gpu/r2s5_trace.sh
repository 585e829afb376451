SBG_RES_TRACE=1 timeout 120 python tools/step_driver.py --steps 60 > gpurun_out/s5_trace.log 2>&1; tail -1 gpurun_out/s5_trace.log
python tools/dev/trace_parts4.py gpurun_out/res_trace.txt
