"""Measured dense FP4 (e2m1) tensor throughput on this B200 -- the ceiling of the kind::mxf4
resident kernel -- measured like tools/int8_peak.py with a library block-scaled FP4 GEMM at
8192^3: burst = best of 5 runs of 10 queued calls, sustained = back to back for ~4 s;
2*N^3 ops per GEMM. Tries torch._scaled_mm (cuBLASLt, MX block-32 E8M0 scales) first,
then flashinfer's mm_fp4 (NVFP4)."""
import json
import time

import torch

n = 8192


def timed(fn):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):  # burst: 10 queued calls (host launch overhead hidden), best of 5
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            fn()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3 / 10)
    t0 = time.time()
    k = 0
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    while time.time() - t0 < 4.0:
        for _ in range(20):
            fn()
        k += 20
        torch.cuda.synchronize()
    e.record()
    torch.cuda.synchronize()
    return best, s.elapsed_time(e) / 1e3 / k


def scaled_mm():
    fp4 = torch.float4_e2m1fn_x2
    a = torch.randint(0, 256, (n, n // 2), dtype=torch.uint8, device="cuda").view(fp4)
    b = torch.randint(0, 256, (n, n // 2), dtype=torch.uint8, device="cuda").view(fp4)
    # MX scales: one E8M0 per 32 K elements, in the 128x4 swizzled blocks cuBLASLt expects
    sa = torch.full((n * (n // 32),), 127, dtype=torch.uint8, device="cuda").view(torch.float8_e8m0fnu)
    sb = torch.full((n * (n // 32),), 127, dtype=torch.uint8, device="cuda").view(torch.float8_e8m0fnu)
    fn = lambda: torch._scaled_mm(a, b.t(), sa, sb, out_dtype=torch.bfloat16)  # noqa: E731
    fn()
    return fn, "torch._scaled_mm (cuBLASLt) float4_e2m1fn_x2 x float4_e2m1fn_x2, MX block-32 E8M0 scales -> bf16"


def scaled_mm_nvfp4():
    fp4 = torch.float4_e2m1fn_x2
    a = torch.randint(0, 256, (n, n // 2), dtype=torch.uint8, device="cuda").view(fp4)
    b = torch.randint(0, 256, (n, n // 2), dtype=torch.uint8, device="cuda").view(fp4)
    sa = torch.full((n * (n // 16),), 0x38, dtype=torch.uint8, device="cuda").view(torch.float8_e4m3fn)
    sb = torch.full((n * (n // 16),), 0x38, dtype=torch.uint8, device="cuda").view(torch.float8_e4m3fn)
    fn = lambda: torch._scaled_mm(a, b.t(), sa, sb, out_dtype=torch.bfloat16)  # noqa: E731
    fn()
    return fn, "torch._scaled_mm (cuBLASLt) float4_e2m1fn_x2, NVFP4 block-16 E4M3 scales -> bf16"


def flashinfer_fp4():
    import flashinfer

    a = torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
    gs = torch.tensor([1.0], device="cuda")
    a4, asf = flashinfer.fp4_quantize(a, gs, 16, False)
    b4, bsf = flashinfer.fp4_quantize(b, gs, 16, False)
    alpha = torch.tensor([1.0], device="cuda")
    fn = lambda: flashinfer.mm_fp4(a4, b4.t(), asf, bsf.t(), alpha, torch.bfloat16)  # noqa: E731
    fn()
    return fn, "flashinfer.mm_fp4 (NVFP4 block-16 scales) -> bf16"


out = {"n": n, "gpu": torch.cuda.get_device_name()}
errs, runs = [], []
for make in (scaled_mm, scaled_mm_nvfp4, flashinfer_fp4):
    try:
        fn, how = make()
        best, sus = timed(fn)
        ops = 2.0 * n ** 3
        runs.append({"fp4_tops_burst": ops / best / 1e12, "fp4_tops_sustained": ops / sus / 1e12, "how": how})
    except Exception as e:  # report and try the next library
        errs.append(f"{make.__name__}: {type(e).__name__}: {str(e)[:400]}")
if runs:  # the fastest library is the measured peak
    out.update(max(runs, key=lambda r: r["fp4_tops_burst"]))
out["all"] = runs
out["errors"] = errs
print(json.dumps(out))
