# A/B of builds of libsbgpu.so on the C2 step loop: tools/ab/<name>.so for each name in $AB
for rep in 1 2; do
for v in $AB; do
export SBG_LIB_OVERRIDE=$PWD/tools/ab/$v.so
for st in 20 200; do
timeout 300 python tools/step_driver.py --steps $st 2>&1 | tail -1 | sed "s/^/$v st=$st /"
done; done; done
for v in $AB; do
export SBG_LIB_OVERRIDE=$PWD/tools/ab/$v.so
SBG_RES_TRACE=1 timeout 300 python tools/step_driver.py --steps 60 > /dev/null 2>&1
python tools/dev/trace_parts.py gpurun_out/res_trace.txt 2>/dev/null | sed "s/^/$v /"
done
