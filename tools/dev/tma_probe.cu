// Dev probe: latency of TMA loads of G-like tiles from L2-resident data, one CTA per SM,
// all SMs at once (the resident kernel's per-step G fetch): (a) one 40-row x 128 B box,
// (b) eight such boxes issued back to back (8 K blocks), (c) one 3D box {128 B, 40 rows,
// 8 K blocks} covering the same 40 KB. Cycles from the first issue to the mbarrier phase.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>
#include "../../paper_2508_17655_b200/csrc/ptx.cuh"
using namespace sbg;

__device__ __forceinline__ void tma3(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma2(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
          "r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}

__global__ void probe(const __grid_constant__ CUtensorMap m2, const __grid_constant__ CUtensorMap m3, int mode,
                      int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t base = (ptx::smem_u32(sm) + 1023u) & ~1023u;
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    ptx::mbar_init(ptx::smem_u32(&bar), 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  unsigned long long tot = 0;
  for (int it = 0; it < iters; ++it) {
    const int row0 = ((blockIdx.x * 7 + it * 13) % 200) * 40;  // different rows per CTA / iteration
    const unsigned long long t0 = clock64();
    if (threadIdx.x == 0) {
      ptx::mbar_arrive_expect_tx(ptx::smem_u32(&bar), mode == 0 ? 5120 : 40960);
      if (mode == 0) tma2(base, &m2, ptx::smem_u32(&bar), 0, row0);
      if (mode == 1)
        for (int kb = 0; kb < 8; ++kb) tma2(base + kb * 5120, &m2, ptx::smem_u32(&bar), kb * 128, row0);
      if (mode == 2) tma3(base, &m3, ptx::smem_u32(&bar), 0, row0, 0);
    }
    ptx::mbar_wait(ptx::smem_u32(&bar), it & 1);
    tot += clock64() - t0;
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = tot / iters;
}

int main() {
  const int rows = 8192, rowb = 1024;  // G: [rpad][npad / 2] bytes
  uint8_t* g;
  cudaMalloc(&g, size_t(rows) * rowb);
  cudaMemset(g, 1, size_t(rows) * rowb);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q);
  CUtensorMap m2, m3;
  {
    cuuint64_t dims[2] = {cuuint64_t(rowb), cuuint64_t(rows)};
    cuuint64_t str[1] = {cuuint64_t(rowb)};
    cuuint32_t box[2] = {128, 40}, es[2] = {1, 1};
    enc(&m2, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  {
    cuuint64_t dims[3] = {128, cuuint64_t(rows), cuuint64_t(rowb / 128)};
    cuuint64_t str[2] = {cuuint64_t(rowb), 128};
    cuuint32_t box[3] = {128, 40, 8}, es[3] = {1, 1, 1};
    CUresult r = enc(&m3, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("3d map encode: %d\n", int(r));
  }
  unsigned long long* out;
  cudaMalloc(&out, 8 * 148);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  const char* names[3] = {"one 2D box 40x128B (5 KB)", "eight 2D boxes (40 KB)", "one 3D box 128Bx40x8 (40 KB)"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int grid : {1, 148}) {
      probe<<<grid, 128, 48 * 1024>>>(m2, m3, mode, 200, out);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<unsigned long long> h(grid);
      cudaMemcpy(h.data(), out, 8 * grid, cudaMemcpyDeviceToHost);
      double s = 0;
      for (auto v : h) s += double(v);
      printf("%-32s grid %3d: %.0f cycles = %.2f us (%s)\n", names[mode], grid, s / grid, s / grid / 1965.0,
             cudaGetErrorString(e));
    }
  }
  return 0;
}
