# C3: slab width x grid size of the lean CSR step (tasks per warp made integral), 100 steps
for cfg in "256 0" "256 1000" "256 834" "256 715" "128 0" "128 834" "128 1000" "128 625" "512 0" "512 1000" "512 1112"; do set -- $cfg
SBG_CSR_SLAB=$1 SBG_CSR_BLOCKS=$2 timeout 200 python tools/configs_bench.py --only C3 --steps 100 2>&1 | grep -o '"us_per_step": [0-9.]*' | sed "s/^/slab=$1 blocks=$2 /"
done
