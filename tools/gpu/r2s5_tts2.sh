for rule in 1 0 1; do
SBG_RES_NR_TS=$rule timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-configs 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][-1])
for k in ('tts99','tts99_gdsb'):
    t=d[k]; print('nr_ts=$rule',k,'t_batch_s',round(t['t_batch_s'],4),'device_ms',round(t['device_ms_batch'],1),'tts99_run_ms',round(t['tts99_run_ms'],1))
"
done
