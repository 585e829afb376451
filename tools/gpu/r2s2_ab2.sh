# A/B of the in-tree build (tools/ab/base.so) against tools/ab/$V.so on the C2 bench leg + parity of $V
SBG_LIB_OVERRIDE=$PWD/tools/ab/$V.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ts_kernel or resident or e2m1 or c2_shape or p2 or run" > gpurun_out/ab2_tests.log 2>&1; echo "tests($V) rc=$?"; tail -1 gpurun_out/ab2_tests.log
for rep in 1 2; do for v in base $V; do for st in 20 200; do
SBG_LIB_OVERRIDE=$PWD/tools/ab/$v.so timeout 300 python bench.py --steps $st --warmup 5 --no-tts --no-cpu-baseline --no-configs 2>/dev/null | grep -o '"ms_per_step": [0-9.e-]*' | sed "s/^/$v st=$st /"
done; done; done
