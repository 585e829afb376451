# C5 (stages, state buffers) alternatives of the e2m1 streaming pair kernel
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tail_split" > gpurun_out/c5cfg_t.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/c5cfg_t.log
for cfg in 0 43 34; do for r in 1 2; do
SBG_C5_CFG=$cfg timeout 600 python tools/c5_bench.py 2>&1 | grep -o '"us_per_step": [0-9.]*' | sed "s/^/cfg=$cfg /"
done; done
SBG_C5_CFG=43 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "tail_split" > gpurun_out/c5cfg_t2.log 2>&1; echo "tests43 rc=$?"; tail -1 gpurun_out/c5cfg_t2.log
SBG_C5_CFG=43 SBG_PAIR_TRACE=1 timeout 300 python tools/c5_bench.py --steps 3 > /dev/null 2>&1; python tools/dev/utrace_summary.py gpurun_out/pair_utrace.txt 2>/dev/null | head -5
