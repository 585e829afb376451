# timing-only A/B of tools/ab/*.so builds on the C2 bench leg, with SM clocks
for rep in 1 2 3; do for v in $AB; do
SBG_LIB_OVERRIDE=$PWD/tools/ab/$v.so timeout 300 python bench.py --steps 20 --warmup 5 --no-tts --no-cpu-baseline --no-configs 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$v', round(d['ms_per_step']*1e3,2), d['clocks'])"
done; done
