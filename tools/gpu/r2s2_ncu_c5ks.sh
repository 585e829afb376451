# ncu --set full of one row-shard step launch at G = 8 with SBG_KSPLIT=3 and without
for ks in 3 1; do
SBG_KSPLIT=$ks timeout 900 ncu --set full --import-source on --clock-control none -k regex:gsb_multistep_pair_kernel --launch-skip 24 -c 1 \
  -o gpurun_out/r2s2_c5_ks$ks python tools/c5_shard_bench.py --world 8 --steps 4 > gpurun_out/ncu_c5ks$ks.log 2>&1; echo "ncu ks=$ks rc=$?"
done
