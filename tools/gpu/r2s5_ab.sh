# same-box A/B of library builds (tools/ab/*.so, names in $AB) on the C2 bench leg at 20 and 200 steps
for rep in 1 2 3; do for steps in 20 200; do for v in $AB; do
SBG_LIB_OVERRIDE=$PWD/tools/ab/$v.so timeout 120 python bench.py --steps $steps --warmup 5 --no-tts --no-cpu-baseline --no-configs 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$v steps=$steps', round(d['ms_per_step']*1e3,2), d['clocks']['sm_mhz'])"
done; done; done
