# tail-only K split: bitwise tests (new + K split + row shards), C5 single-GPU timing with / without, G=4 shards
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "tail_split or k_split" > gpurun_out/kt_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/kt_tests.log
timeout 900 python -m pytest tests/test_gpu_rowshard.py -q -x > gpurun_out/kt_rs.log 2>&1; echo "rowshard rc=$?"; tail -1 gpurun_out/kt_rs.log
for r in 1 2; do for kt in 1 0; do
SBG_KTAIL=$kt timeout 600 python tools/c5_bench.py 2>&1 | grep -o '"us_per_step[a-z_]*": [0-9.]*' | head -2 | tr '\n' ' ' | sed "s/^/ktail=$kt /"; echo
done; done
for kt in 1 0; do SBG_KTAIL=$kt timeout 600 python tools/c5_shard_bench.py --world 4 --steps 4 2>&1 | grep -o '"us_per_step_per_rank": [0-9.]*' | sed "s/^/G4 ktail=$kt /"; done
