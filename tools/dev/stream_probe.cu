// Dev probe: HBM streaming rate of the C5 J operand (n = 100000 e2m1: 100096 rows x 50048 B,
// 5 GB) into a 6-stage smem ring, one CTA per SM, as the streaming pair kernel reads it:
// (0) 2D TMA boxes of 128 rows x 128 B (SW128) from the row-major matrix, each CTA walking
//     one 128-row block along K; (1) the same bytes stored tile-contiguous ([row block][K
//     block][16 KB]) and fetched with 1D bulk copies of 16 KB; (2) like (0) with 256-row
//     boxes of 64 B (half the K bytes per row, twice the rows).
// Prints GB/s per mode. Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lcuda.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include "../../paper_2508_17655_b200/csrc/ptx.cuh"
using namespace sbg;

constexpr int STAGES = 6, TILE = 16384;

__device__ __forceinline__ void bulk1d(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void tma2(uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::
          "r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(c0), "r"(c1)
      : "memory");
}

__global__ void stream(const __grid_constant__ CUtensorMap m0, const __grid_constant__ CUtensorMap m2,
                       const uint8_t* buf, int mode, int row_blocks, int kblocks, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t base = (ptx::smem_u32(sm) + 1023u) & ~1023u;
  __shared__ uint64_t full[STAGES], empty[STAGES];
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(ptx::smem_u32(&full[s]), 1);
      ptx::mbar_init(ptx::smem_u32(&empty[s]), 1);
    }
    ptx::fence_mbar_init();
  }
  __syncthreads();
  const int kb_per = mode == 2 ? 2 * kblocks : kblocks;  // mode 2: 64-byte K blocks
  const int nrb = mode == 2 ? row_blocks / 2 : row_blocks;  // mode 2: 256-row blocks
  if (threadIdx.x == 0) {  // producer
    int st = 0;
    uint32_t ph = 0;
    for (int rb = blockIdx.x; rb < nrb; rb += gridDim.x)
      for (int kb = 0; kb < kb_per; ++kb) {
        ptx::mbar_wait(ptx::smem_u32(&empty[st]), ph ^ 1u);
        const uint32_t fb = ptx::smem_u32(&full[st]);
        ptx::mbar_arrive_expect_tx(fb, TILE);
        const uint32_t dst = base + st * TILE;
        if (mode == 0) tma2(dst, &m0, fb, kb * 128, rb * 128);
        if (mode == 1) bulk1d(dst, buf + (static_cast<size_t>(rb) * kblocks + kb) * TILE, TILE, fb);
        if (mode == 2) tma2(dst, &m2, fb, kb * 64, rb * 256);
        if (++st == STAGES) {
          st = 0;
          ph ^= 1u;
        }
      }
  } else if (threadIdx.x == 32) {  // consumer: touch one word per tile, release
    int st = 0;
    uint32_t ph = 0;
    unsigned long long acc = 0;
    for (int rb = blockIdx.x; rb < nrb; rb += gridDim.x)
      for (int kb = 0; kb < kb_per; ++kb) {
        ptx::mbar_wait(ptx::smem_u32(&full[st]), ph);
        acc += sm[(base - ptx::smem_u32(sm)) + st * TILE + (kb & 127)];
        ptx::mbar_arrive(ptx::smem_u32(&empty[st]));
        if (++st == STAGES) {
          st = 0;
          ph ^= 1u;
        }
      }
    if (acc == 0x1234567) sink[0] = acc;
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

int main() {
  const int rows = 100096, pitch = 50048, kblocks = pitch / 128;  // 391
  const int row_blocks = rows / 128;                               // 782
  const size_t bytes = static_cast<size_t>(rows) * pitch;
  uint8_t* buf;
  if (cudaMalloc(&buf, bytes) != cudaSuccess) return 1;
  cudaMemset(buf, 1, bytes);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  auto enc = encode();
  CUtensorMap m0, m2;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(pitch), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(pitch)};
  cuuint32_t box0[2] = {128, 128}, box2[2] = {64, 256}, es[2] = {1, 1};
  enc(&m0, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box0, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  enc(&m2, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dims, strides, box2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
      CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int smem = STAGES * TILE + 1024;
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const char* names[3] = {"2D TMA 128x128B row-major", "1D bulk 16KB tile-contiguous", "2D TMA 256x64B row-major"};
  for (int rep = 0; rep < 2; ++rep)
    for (int mode = 0; mode < 3; ++mode) {
      cudaEventRecord(e0);
      stream<<<sms, 64, smem>>>(m0, m2, buf, mode, row_blocks, kblocks, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const cudaError_t err = cudaGetLastError();
      printf("%-32s %8.3f ms  %7.1f GB/s %s\n", names[mode], ms, bytes / (ms * 1e-3) / 1e9,
             err == cudaSuccess ? "" : cudaGetErrorString(err));
    }
  return 0;
}
