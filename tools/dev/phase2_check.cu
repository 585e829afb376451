// Dev check: gsb_phase2 (packed f32x2) vs gsb_phase (scalar) bitwise on random inputs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2508_17655_b200/csrc/gsb_phase.cuh"
using namespace sbg;
__global__ void k(const float* in, uint32_t* out, int n, PhaseConsts kc, PhaseIdent id) {
  int i = (blockIdx.x * blockDim.x + threadIdx.x) * 2;
  if (i + 1 >= n) return;
  float F0 = in[4 * i], x0 = in[4 * i + 1], y0 = in[4 * i + 2], p0 = in[4 * i + 3];
  float F1 = in[4 * i + 4], x1 = in[4 * i + 5], y1 = in[4 * i + 6], p1 = in[4 * i + 7];
  float a0 = x0, b0 = y0, c0 = p0, a1 = x1, b1 = y1, c1 = p1;
  gsb_phase(F0, a0, b0, c0, kc);
  gsb_phase(F1, a1, b1, c1, kc);
  PhaseConsts2 k2(kc, id);
  gsb_phase2(F0, F1, x0, x1, y0, y1, p0, p1, k2, k2.a);
  out[3 * i] = __float_as_uint(a0) ^ __float_as_uint(x0);
  out[3 * i + 1] = __float_as_uint(b0) ^ __float_as_uint(y0);
  out[3 * i + 2] = __float_as_uint(c0) ^ __float_as_uint(p0);
  out[3 * i + 3] = __float_as_uint(a1) ^ __float_as_uint(x1);
  out[3 * i + 4] = __float_as_uint(b1) ^ __float_as_uint(y1);
  out[3 * i + 5] = __float_as_uint(c1) ^ __float_as_uint(p1);
}
int main() {
  const int n = 1 << 20;
  float* h = new float[4 * n];
  uint64_t s = 12345;
  for (int i = 0; i < 4 * n; ++i) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    float u = float((s >> 40) & 0xFFFFFF) / 16777216.0f * 2.f - 1.f;
    int f = i % 4;
    h[i] = f == 0 ? float(int(u * 500)) : (f == 3 ? 0.5f + 0.5f * u : u);
  }
  float* d; uint32_t* o;
  cudaMalloc(&d, 16 * n); cudaMalloc(&o, 12 * n);
  cudaMemcpy(d, h, 16 * n, cudaMemcpyHostToDevice);
  PhaseConsts kc{0.2f, 0.0111803f, 1.25f, 1.0f / 997.0f};
  k<<<n / 512, 256>>>(d, o, n, kc, PhaseIdent{-0.0f, 1.0f, -1.0f});
  uint32_t* r = new uint32_t[3 * n];
  cudaMemcpy(r, o, 12 * n, cudaMemcpyDeviceToHost);
  long bad = 0; int shown = 0;
  for (int i = 0; i < 3 * n; ++i) if (r[i]) { ++bad; if (shown++ < 5) printf("diff at %d (elem %d comp %d): xor %08x\n", i, i / 3, i % 3, r[i]); }
  printf("mismatches: %ld of %d (%s)\n", bad, 3 * n, cudaGetErrorString(cudaGetLastError()));
  return bad != 0;
}
