timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py tests/test_gpu_cli.py tests/test_gpu_edge_cases.py -x -q -k "csr or graph or gset or cli or edge or CSR" > gpurun_out/r2c22.log 2>&1; echo rc=$?; tail -3 gpurun_out/r2c22.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-tts --no-cpu-baseline > gpurun_out/r2c22_b.log 2>&1
python -c "
import json
for l in open('gpurun_out/r2c22_b.log'):
    if l.startswith('{'): d=json.loads(l)
print(d['configs']['C3']['us_per_step'], d['configs']['C3']['roofline']['frac'])"
