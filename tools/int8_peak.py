"""Measured dense int8 tensor throughput on this B200 ('int8 is not measured; the
builder must measure it the same way'): torch._int_mm (cuBLASLt int8 GEMM) at 8192^3,
best of 10 (burst) and back to back for ~4 s (sustained), 2*N^3 ops per GEMM."""
import json
import time

import torch

n = 8192
a = torch.randint(-127, 127, (n, n), dtype=torch.int8, device="cuda")
b = torch.randint(-127, 127, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
for _ in range(3):
    torch._int_mm(a, b)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    torch._int_mm(a, b)
    e.record()
    torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e) / 1e3)
t0 = time.time()
k = 0
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
while time.time() - t0 < 4.0:
    for _ in range(20):
        torch._int_mm(a, b)
    k += 20
    torch.cuda.synchronize()
e.record()
torch.cuda.synchronize()
sus = s.elapsed_time(e) / 1e3 / k
ops = 2.0 * n ** 3
out = {"int8_tops_burst": ops / best / 1e12, "int8_tops_sustained": ops / sus / 1e12, "n": n,
       "how": "torch._int_mm (cuBLASLt) int8 x int8 -> int32, 8192^3, best of 10 / back to back 4 s, CUDA events",
       "gpu": torch.cuda.get_device_name()}
print(json.dumps(out))
