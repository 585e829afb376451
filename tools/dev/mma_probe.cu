// Dev probe: throughput of back-to-back tcgen05.mma.cta_group::2.kind::i8 (M=256, N=64/128/256, K=32)
// from fixed shared-memory operands (no loads), timed per CTA pair with clock64.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2508_17655_b200/csrc/ptx.cuh"
using namespace sbg;
template <int N, int FENCE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) probe(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t base = (ptx::smem_u32(sm) + 1023u) & ~1023u;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 65536 + 1024);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 4);
  const int warp = threadIdx.x >> 5;
  const uint32_t cr = ptx::cluster_ctarank();
  for (int i = threadIdx.x; i < 65536; i += blockDim.x) sm[(base - ptx::smem_u32(sm)) + i] = uint8_t(i * 7);
  if (threadIdx.x == 0) { ptx::mbar_init(ptx::smem_u32(bar), 1); ptx::mbar_init(ptx::smem_u32(bar + 1), 1); ptx::fence_mbar_init(); }
  if (warp == 2) { ptx::tmem_alloc_pair(ptx::smem_u32(slot), 256); ptx::tmem_relinquish_pair(); }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  ptx::cluster_sync_all();
  ptx::tc_fence_after();
  const uint32_t tmem = *slot;
  if (cr == 0 && warp == 1) {
    constexpr uint32_t idesc = ptx::idesc_i8(256, N, true, true);
    const uint64_t adesc = ptx::smem_desc_k_sw128(base);
    const uint64_t bdesc = ptx::smem_desc_k_sw128(base + 32768);
    unsigned long long t0 = clock64();
    if (ptx::elect_one()) {
      for (int i = 0; i < iters; ++i) {
        if (FENCE == 1 && (i & 3) == 0) ptx::tc_fence_after();
        if (FENCE == 2 && (i & 3) == 0) ptx::mma_commit_pair_mc(ptx::smem_u32(bar + 1), 0x3);
        ptx::mma_i8_pair(tmem, adesc + 2 * (i & 3), bdesc + 2 * (i & 3), idesc, i != 0);
      }
      ptx::mma_commit_pair_mc(ptx::smem_u32(bar), 0x3);
    }
    __syncwarp();
    ptx::mbar_wait(ptx::smem_u32(bar), 0);
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 32) out[0] = t1 - t0;
  } else if (cr == 1 && warp == 1) {
    ptx::mbar_wait(ptx::smem_u32(bar), 0);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync_all();
  if (warp == 2) ptx::tmem_dealloc_pair(tmem, 256);
}
template <int N, int FENCE>
void run(int grid) {
  unsigned long long* d; cudaMalloc(&d, 8);
  const int smem = 65536 + 1024 + 64;
  cudaFuncSetAttribute(probe<N, FENCE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  probe<N, FENCE><<<grid, 128, smem>>>(iters, d);
  cudaDeviceSynchronize();
  unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double macs = 256.0 * N * 32;  // per pair
  printf("fence %d N=%3d grid %3d: %.1f cycles per MMA, %.0f int8 MAC/cycle/SM (%s)\n", FENCE, N, grid, double(h) / iters,
         macs / (double(h) / iters) / 2, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  for (int g : {148}) { run<64, 0>(g); run<128, 0>(g); run<64, 1>(g); run<128, 1>(g); run<64, 2>(g); run<128, 2>(g); }
  return 0;
}
