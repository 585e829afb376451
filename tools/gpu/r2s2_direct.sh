# direct-state epilogue (continuous variants in the pair kernel): parity with it, C1 / C4 timing A/B
SBG_LIB_OVERRIDE=$PWD/tools/ab/direct.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sk.py tests/test_gpu_p3_scale.py -q -x > gpurun_out/direct_t.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/direct_t.log
for r in 1 2; do for v in base direct; do
SBG_LIB_OVERRIDE=$PWD/tools/ab/$v.so timeout 600 python tools/configs_bench.py --only C1,C4 --steps 20 2>&1 | grep -o '"us_per_step": [0-9.]*' | tr '\n' ' ' | sed "s/^/$v /"; echo
done; done
