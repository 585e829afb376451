# C5: tile-state L2 prefetch A/B (with / without), tail split on, + unit trace with the prefetch
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tail_split or k_split or stream" > gpurun_out/pf_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/pf_tests.log
for r in 1 2; do for v in base nopf; do
SBG_LIB_OVERRIDE=$PWD/tools/ab/$v.so timeout 600 python tools/c5_bench.py 2>&1 | grep -o '"us_per_step": [0-9.]*' | sed "s/^/$v /"
done; done
SBG_LIB_OVERRIDE=$PWD/tools/ab/base.so SBG_PAIR_TRACE=1 timeout 300 python tools/c5_bench.py --steps 3 > /dev/null 2>&1; python tools/dev/utrace_summary.py gpurun_out/pair_utrace.txt | head -5
