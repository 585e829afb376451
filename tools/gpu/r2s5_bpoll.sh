# TS kernel: batched dependency observation in the producer (SBG_TS_BPOLL, default on) x publisher warps x parts
timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "ts_kernel or resident or c2_shape" > gpurun_out/s5_bpoll_tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/s5_bpoll_tests.log
[ $rc -eq 0 ] || exit 1
for rep in 1 2; do for steps in 20 200; do for cfg in "0 0 4" "1 0 4" "1 1 4" "1 0 5" "1 1 5"; do set -- $cfg
SBG_TS_BPOLL=$1 SBG_TS_MPUB=$2 SBG_RES_PARTS=$3 timeout 120 python bench.py --steps $steps --warmup 5 --no-tts --no-cpu-baseline --no-configs 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('bpoll=$1 mpub=$2 parts=$3 steps=$steps', round(d['ms_per_step']*1e3,2), d['clocks']['sm_mhz'])"
done; done; done
