# C4 (real J): SK tests (bitwise vs the mirror), P3 at N=4096, on the default (pair) and single-CTA kernels; timing
timeout 900 python -m pytest tests/test_gpu_sk.py tests/test_gpu_p3_scale.py tests/test_gpu_graph.py -q -x > gpurun_out/c4_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c4_tests.log
SBG_FX_PAIR=0 timeout 900 python -m pytest tests/test_gpu_sk.py -q -x > gpurun_out/c4_tests0.log 2>&1; echo "tests(single) rc=$?"; tail -1 gpurun_out/c4_tests0.log
for k in 1 0; do SBG_FX_PAIR=$k timeout 300 python tools/configs_bench.py --only C4 --steps 20 2>&1 | grep -o '"us_per_step": [0-9.]*' | sed "s/^/pair=$k /"; done
timeout 300 python tools/configs_bench.py --only C4 --steps 20 2>&1 | grep -o '"us_per_step": [0-9.]*' | sed "s/^/default /"
timeout 900 python -m pytest tests/test_gpu_statistics.py -q -x -k "sk or c4 or 4096" > gpurun_out/c4_stat.log 2>&1; echo "stat rc=$?"; tail -1 gpurun_out/c4_stat.log
