# Session 5 opening: full GPU suite, smoke, bench (20 steps) on HEAD after the container was re-created
set -u
timeout 1700 python -m pytest tests -m gpu -q -x > gpurun_out/s5_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/s5_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/s5_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/s5_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/s5_bench.log | cut -c1-600
