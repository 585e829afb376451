# library without dev hooks (default build) vs with (tools/ab/trace1.so): full GPU suite on the new default, then A/B
timeout 1700 python -m pytest tests -m gpu -q -x > gpurun_out/s5_nohooks_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/s5_nohooks_tests.log
for rep in 1 2; do for v in trace1 nohooks; do
SBG_LIB_OVERRIDE=$PWD/tools/ab/$v.so timeout 300 python tools/configs_bench.py --only C1,C4 --steps 20 2>/dev/null | grep -o '"C[0-9]"[^}]*"us_per_step": [0-9.]*' | sed "s/^/$v /" | cut -c1-160
SBG_LIB_OVERRIDE=$PWD/tools/ab/$v.so timeout 300 python tools/c5_bench.py 2>/dev/null | tail -2 | cut -c1-200 | sed "s/^/$v C5 /"
done; done
