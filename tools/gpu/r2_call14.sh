for d in 0 6; do
SBG_STEP_DBG=$d SBG_RES_TRACE=1 timeout 300 python tools/step_driver.py --steps 60 > gpurun_out/r2c14_$d.log 2>&1; cp gpurun_out/res_trace.txt gpurun_out/res_trace_d$d.txt
SBG_STEP_DBG=$d timeout 300 python tools/step_driver.py --steps 200 >> gpurun_out/r2c14_$d.log 2>&1
cat gpurun_out/r2c14_$d.log
done
