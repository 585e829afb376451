import torch, time
x = torch.empty(131*2**20//4, dtype=torch.float32).pin_memory()
d = torch.empty_like(x, device="cuda")
for _ in range(3): d.copy_(x, non_blocking=True)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record(); d.copy_(x, non_blocking=True); e.record(); torch.cuda.synchronize()
print("H2D pinned 131 MB: %.2f ms = %.1f GB/s" % (s.elapsed_time(e), 131*2**20/s.elapsed_time(e)/1e6))
