# epilogue bound probe: period with the phase math (6) / the math and x, y traffic (7) taken out
for d in 0 6 7; do
SBG_STEP_DBG=$d timeout 300 python tools/step_driver.py --steps 200 2>&1 | tail -1 | sed "s/^/dbg=$d /"
SBG_STEP_DBG=$d SBG_RES_TRACE=1 timeout 300 python tools/step_driver.py --steps 60 > /dev/null 2>&1
python tools/dev/trace_parts.py gpurun_out/res_trace.txt 2>/dev/null | sed "s/^/dbg=$d /"
done
