timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2s2_full_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2s2_full_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2s2_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r2s2_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2s2_bench_full.log 2>&1; echo "bench rc=$?"
tail -c 2500 gpurun_out/r2s2_bench_full.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2s2_bench_ref.log 2>&1; echo "ref rc=$?"; tail -c 600 gpurun_out/r2s2_bench_ref.log
