# C2 TS kernel timelines: per-(CTA, group) stamps at 20 and 200 steps, the per-step part trace at 60
for st in 20 200; do
SBG_RES_GTRACE=1 timeout 300 python tools/step_driver.py --steps $st 2>&1 | tail -1
done
SBG_RES_TRACE=1 timeout 300 python tools/step_driver.py --steps 60 2>&1 | tail -1
python tools/dev/trace_parts.py gpurun_out/res_trace.txt
