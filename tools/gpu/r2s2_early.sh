# C5: early accumulator drain (e2m1 pair kernel) A/B + its parity
SBG_LIB_OVERRIDE=$PWD/tools/ab/early.so timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rowshard.py -q -x -k "tail_split or k_split or stream or shard" > gpurun_out/early_t.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/early_t.log
for r in 1 2; do for v in base early; do
SBG_LIB_OVERRIDE=$PWD/tools/ab/$v.so timeout 600 python tools/c5_bench.py 2>&1 | grep -o '"us_per_step": [0-9.]*' | sed "s/^/$v /"
done; done
SBG_LIB_OVERRIDE=$PWD/tools/ab/early.so SBG_PAIR_TRACE=1 timeout 300 python tools/c5_bench.py --steps 3 > /dev/null 2>&1; python tools/dev/utrace_summary.py gpurun_out/pair_utrace.txt 2>/dev/null | head -5
for v in base early; do SBG_LIB_OVERRIDE=$PWD/tools/ab/$v.so timeout 600 python tools/c5_shard_bench.py --world 4 --steps 4 2>&1 | grep -o '"us_per_step_per_rank": [0-9.]*' | sed "s/^/G4 $v /"; done
