// Dev probe: L2 -> SM throughput on the B200, the bound of the CSR step (C3), whose
// 512 B gathers of the ping-pong operand and the state stream are served from L2.
//  (a) stream: every warp reads consecutive 512 B rows of an L2-resident buffer (LDG.128);
//  (b) gather: every warp reads 512 B rows at pseudo-random row indices (the C3 pattern:
//      one row = 128 replicas x 4 B of the gathered operand), rows from a 41 MB buffer.
// Reported as bytes delivered to the SMs per second (CUDA events, best of 5).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_probe l2_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void probe(const int4* __restrict__ buf, int64_t rows, int iters, int gather, int4* out) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  int4 acc = make_int4(0, 0, 0, 0);
  uint32_t h = uint32_t(warp) * 2654435761u + 12345u;
  for (int it = 0; it < iters; ++it) {
    int64_t row;
    if (gather) {
      h = h * 1664525u + 1013904223u;
      row = int64_t(h % uint32_t(rows));
    } else {
      row = (warp + int64_t(it) * nwarps) % rows;
    }
    const int4 v = buf[row * 32 + lane];  // 512 B per warp
    acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
  }
  if (acc.x == 0x7fffffff) out[0] = acc;
}

int main() {
  const int64_t rows = 41 * 1024 * 1024 / 512;  // 41 MB: the C3 operand (20000 x 512 x 4 B)
  int4* buf;
  int4* out;
  cudaMalloc(&buf, rows * 512);
  cudaMalloc(&out, 16);
  cudaMemset(buf, 1, rows * 512);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int gather = 0; gather < 2; ++gather)
    for (int wps : {16, 32, 64}) {  // warps per SM
      const int threads = 256, blocks = sms * wps / 8, iters = 2000;
      float best = 1e30f;
      for (int rep = 0; rep < 6; ++rep) {
        cudaEventRecord(a);
        probe<<<blocks, threads>>>(buf, rows, iters, gather, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep > 0 && ms < best) best = ms;
      }
      const double bytes = double(blocks) * threads / 32 * iters * 512;
      printf("%s warps/SM %2d: %.0f GB/s (%s)\n", gather ? "gather" : "stream", wps, bytes / (best * 1e-3) / 1e9,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
