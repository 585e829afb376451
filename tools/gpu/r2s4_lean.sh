# C3: lean CSR kernel A/B (SBG_CSR_LEAN = -1 round-1 kernel, 1 / 2 / 4 gathers per round), bitwise tests first
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "csr" > gpurun_out/s4_lean_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s4_lean_tests.log
for rep in 1 2; do for lean in -1 1 2 4; do for slab in 0 512; do for steps in 20 100; do
SBG_CSR_LEAN=$lean SBG_CSR_SLAB=$slab timeout 300 python tools/configs_bench.py --only C3 --steps $steps 2>&1 | grep -o '"us_per_step": [0-9.]*' | sed "s/^/lean=$lean slab=$slab steps=$steps /"
done; done; done; done
