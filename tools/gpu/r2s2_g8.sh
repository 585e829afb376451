# C5 row shards at G = 8 / 4 / 2 (lockstep) with uniform K split 1..4 after the early drain
for G in 8 4 2; do for ks in 1 2 3 4; do
SBG_KSPLIT=$ks timeout 600 python tools/c5_shard_bench.py --world $G --steps 4 2>&1 | grep -o '"us_per_step_per_rank": [0-9.]*' | sed "s/^/G=$G ks=$ks /"
done; done
