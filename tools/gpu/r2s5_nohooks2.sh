for rep in 1 2; do for v in trace1 nohooks; do
SBG_LIB_OVERRIDE=$PWD/tools/ab/$v.so timeout 300 python tools/configs_bench.py --only C1,C4 --steps 20 2>/dev/null | tr -d '\n' | grep -o '"C[0-9][^"]*": {[^}]*"us_per_step": [0-9.]*' | sed 's/{.*"us_per_step"/us_per_step/' | sed "s/^/$v /"
done; done
