for rule in 0 1; do
SBG_RES_NR_TS=$rule timeout 200 python tools/dev/tts_leg_time.py gdsb 21500 1000 2>&1 | tail -4 | cut -c1-200 | sed "s/^/nr_ts=$rule /"
done
