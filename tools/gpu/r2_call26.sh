timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "csr" > gpurun_out/r2c26_t.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r2c26_t.log
for pf in 0 6 7; do
for rep in 1 2; do
SBG_CSR_PF=$pf timeout 300 python tools/configs_bench.py --only C3 --steps 50 2>/dev/null | grep us_per_step | sed "s/^/pf=$pf /"
done; done
