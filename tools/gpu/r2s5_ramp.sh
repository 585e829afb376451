for R in 1440 4320; do
SBG_RES_TRACE=1 timeout 120 python tools/step_driver.py --steps 60 --warm 900 --R $R > gpurun_out/s5_ramp.log 2>&1; tail -1 gpurun_out/s5_ramp.log
python tools/dev/trace_parts4.py gpurun_out/res_trace.txt
done
