# TS kernel: one publisher warp per part (SBG_TS_MPUB=1), bitwise tests then A/B at 20 and 200 steps
timeout 240 python -m pytest tests/test_gpu_parity.py -q -x -k "ts_kernel and mpub" > gpurun_out/s5_mpub_tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/s5_mpub_tests.log
[ $rc -eq 0 ] || exit 1
for rep in 1 2; do for steps in 20 200; do for cfg in "0 4" "1 4" "0 5" "1 5"; do set -- $cfg
SBG_TS_MPUB=$1 SBG_RES_PARTS=$2 timeout 120 python bench.py --steps $steps --warmup 5 --no-tts --no-cpu-baseline --no-configs 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('mpub=$1 parts=$2 steps=$steps', round(d['ms_per_step']*1e3,2), d['clocks']['sm_mhz'])"
done; done; done
