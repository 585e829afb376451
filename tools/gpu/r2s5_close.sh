# last closing run: full GPU suite, smoke, bench (20 steps, all legs), bench 200
set -u
timeout 1700 python -m pytest tests -m gpu -q -x > gpurun_out/close_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/close_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/close_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/close_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/close_bench.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --steps 200 --warmup 5 --no-tts --no-cpu-baseline > gpurun_out/close_bench200.log 2>&1; echo "bench200 rc=$?"
timeout 900 python bench.py > gpurun_out/close_bench_default.log 2>&1; echo "bench default rc=$?"
