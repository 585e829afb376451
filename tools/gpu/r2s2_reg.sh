# regression check: C1 / C4 / C5 with the build of 7fdacde vs now
for r in 1 2; do for v in o7f base; do
SBG_LIB_OVERRIDE=$PWD/tools/ab/$v.so timeout 600 python tools/configs_bench.py --only C1,C4 --steps 20 2>&1 | grep -o '"us_per_step": [0-9.]*' | tr '\n' ' ' | sed "s/^/$v /"; echo
done; done
