# C3: x, y, p L2 policy A/B (evict_first / normal / last), with and without 128-replica slabs
for r in 1 2; do for v in base pol1 pol2; do for slab in 0 128; do
SBG_CSR_SLAB=$slab SBG_LIB_OVERRIDE=$PWD/tools/ab/$v.so timeout 300 python tools/configs_bench.py --only C3 --steps 20 2>&1 | grep -o '"us_per_step": [0-9.]*' | sed "s/^/$v slab=$slab /"
done; done; done
