# TS launch host overhead: parity tests of the resident kernels, bench line at 20 / 200 steps (headline leg only)
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ts_kernel or resident or e2m1 or c2_shape or p2 or run" > gpurun_out/ts20_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/ts20_tests.log
for st in 20 200; do for r in 1 2; do
timeout 300 python bench.py --steps $st --warmup 5 --no-tts --no-cpu-baseline --no-configs 2>/dev/null | grep -o '"ms_per_step": [0-9.e-]*' | sed "s/^/steps=$st /"
done; done
