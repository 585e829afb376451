# C5 row shards at G = 8 (lockstep on one GPU): per-rank step with and without the K split
for ks in 1 2 3; do
SBG_KSPLIT=$ks timeout 600 python tools/c5_shard_bench.py --world 8 --steps 4 2>&1 | grep -o '"us_per_step_per_rank": [0-9.]*\|"hbm_frac": [0-9.]*' | tr '\n' ' ' | sed "s/^/ks=$ks /"; echo
done
