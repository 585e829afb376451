// Dev probe: the operand-ring handshake of the pair kernels without data movement.
// Both CTAs' producers wait empty[s] and arrive on the leader's full[s] (count 2, like the
// TMA expect_tx arrivals); the leader's MMA warp waits full[s], issues MPS MMAs and commits
// empty[s] to both CTAs. Cycles per MMA vs the back-to-back rate (43 / 64 cycles, N=64/128).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2508_17655_b200/csrc/ptx.cuh"
using namespace sbg;
template <int N, int ST, int MPS, int GRP = 1>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) pipe(int stages_total, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t base = (ptx::smem_u32(sm) + 1023u) & ~1023u;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + 65536 + 1024);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bars + 2 * ST + 2);
  auto full = [&](int s) { return ptx::smem_u32(bars + s); };
  auto empty = [&](int s) { return ptx::smem_u32(bars + ST + s); };
  const uint32_t done = ptx::smem_u32(bars + 2 * ST);
  const int warp = threadIdx.x >> 5;
  const uint32_t cr = ptx::cluster_ctarank();
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) { ptx::mbar_init(full(s), 2); ptx::mbar_init(empty(s), 1); }
    ptx::mbar_init(done, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) { ptx::tmem_alloc_pair(ptx::smem_u32(slot), 256); ptx::tmem_relinquish_pair(); }
  ptx::tc_fence_before();
  ptx::cluster_sync_all();
  ptx::tc_fence_after();
  const uint32_t tmem = *slot;
  unsigned long long t0 = clock64();
  if (warp == 0) {
    int stage = 0; uint32_t ph = 0;
    for (int i = 0; i < stages_total; ++i) {
      ptx::mbar_wait(empty(stage), ph ^ 1u);
      if (ptx::elect_one()) ptx::mbar_arrive_cluster(ptx::mapa(full(stage), 0));
      __syncwarp();
      if (++stage == ST) { stage = 0; ph ^= 1u; }
    }
  } else if (warp == 1 && cr == 0) {
    constexpr uint32_t idesc = ptx::idesc_i8(256, N, true, true);
    const uint64_t adesc = ptx::smem_desc_k_sw128(base);
    const uint64_t bdesc = ptx::smem_desc_k_sw128(base + 32768);
    int stage = 0; uint32_t ph = 0;
    for (int i = 0; i < stages_total; i += GRP) {
      int st[GRP];
#pragma unroll
      for (int g = 0; g < GRP; ++g) {
        ptx::mbar_wait(full(stage), ph);
        st[g] = stage;
        if (++stage == ST) { stage = 0; ph ^= 1u; }
      }
      ptx::tc_fence_after();
      if (ptx::elect_one()) {
#pragma unroll
        for (int g = 0; g < GRP; ++g) {
          for (int k = 0; k < MPS; ++k) ptx::mma_i8_pair(tmem, adesc + 2 * (k & 3), bdesc + 2 * (k & 3), idesc, (i | k | g) != 0);
          ptx::mma_commit_pair_mc(empty(st[g]), 0x3);
        }
      }
      __syncwarp();
    }
    if (ptx::elect_one()) ptx::mma_commit_pair_mc(done, 0x3);
    __syncwarp();
    ptx::mbar_wait(done, 0);
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0 && threadIdx.x == 32) out[0] = t1 - t0;
  } else if (warp == 1) {
    ptx::mbar_wait(done, 0);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync_all();
  if (warp == 2) ptx::tmem_dealloc_pair(tmem, 256);
}
template <int N, int ST, int MPS, int GRP = 1>
void run() {
  unsigned long long* d; cudaMalloc(&d, 8);
  const int smem = 65536 + 1024 + 1024;
  cudaFuncSetAttribute(pipe<N, ST, MPS, GRP>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int total = 2048;
  pipe<N, ST, MPS, GRP><<<148, 128, smem>>>(total, d);
  cudaDeviceSynchronize();
  unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("grp %d N=%3d stages %d, %d MMAs/stage: %.1f cycles per MMA (%s)\n", GRP, N, ST, MPS, double(h) / (total * MPS),
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  run<64, 8, 4>(); run<128, 8, 4>(); run<64, 8, 4, 2>(); run<128, 8, 4, 2>(); run<64, 8, 4, 4>(); run<128, 8, 4, 4>();
  return 0;
}
