SBG_RES_GTRACE=1 timeout 300 python tools/step_driver.py --steps 60 > gpurun_out/r2c16_g.log 2>&1; cat gpurun_out/r2c16_g.log
