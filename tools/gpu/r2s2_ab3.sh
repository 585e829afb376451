# timing-only A/B (no parity: the probe changes the op order): tools/ab/base.so vs tools/ab/$V.so
for rep in 1 2; do for v in base $V; do for st in 20 200; do
SBG_LIB_OVERRIDE=$PWD/tools/ab/$v.so timeout 300 python bench.py --steps $st --warmup 5 --no-tts --no-cpu-baseline --no-configs 2>/dev/null | grep -o '"ms_per_step": [0-9.e-]*' | sed "s/^/$v st=$st /"
done; done; done
