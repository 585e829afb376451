SBG_RES_TRACE=1 timeout 300 python tools/step_driver.py --steps 60 > gpurun_out/r2c9a.log 2>&1; cp gpurun_out/res_trace.txt gpurun_out/res_trace_base.txt
SBG_STEP_DBG=3 SBG_RES_TRACE=1 timeout 300 python tools/step_driver.py --steps 60 > gpurun_out/r2c9b.log 2>&1; cp gpurun_out/res_trace.txt gpurun_out/res_trace_dbg3.txt
SBG_STEP_DBG=3 timeout 300 python tools/step_driver.py --steps 200 > gpurun_out/r2c9c.log 2>&1
timeout 300 python tools/step_driver.py --steps 200 > gpurun_out/r2c9d.log 2>&1
cat gpurun_out/r2c9*.log
