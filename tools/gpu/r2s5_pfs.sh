# C3: lean CSR step with the task's x, y, p prefetched into shared memory by cp.async (SBG_CSR_PFS=1)
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "csr" > gpurun_out/s5_pfs_tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -2 gpurun_out/s5_pfs_tests.log
[ $rc -eq 0 ] || exit 1
for rep in 1 2; do for cfg in "0 2" "1 2" "1 4" "0 4"; do set -- $cfg; for steps in 20 100; do
SBG_CSR_PFS=$1 SBG_CSR_LEAN=$2 timeout 200 python tools/configs_bench.py --only C3 --steps $steps 2>&1 | grep -o '"us_per_step": [0-9.]*' | sed "s/^/pfs=$1 lean=$2 steps=$steps /"
done; done; done
