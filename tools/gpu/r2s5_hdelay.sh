# TS kernel: G_0 helper of the next group delayed by SBG_TS_HDELAY steps; bitwise test then A/B at 20 steps
SBG_TS_HDELAY=8 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "ts_kernel_edge or c2_shape or resident_kernel_equals" > gpurun_out/s5_hd_tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -2 gpurun_out/s5_hd_tests.log
[ $rc -eq 0 ] || exit 1
for rep in 1 2 3; do for hd in 0 4 8 12; do
SBG_TS_HDELAY=$hd timeout 120 python bench.py --steps 20 --warmup 5 --no-tts --no-cpu-baseline --no-configs 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('hdelay=$hd steps=20', round(d['ms_per_step']*1e3,2), d['clocks']['sm_mhz'])"
done; done
