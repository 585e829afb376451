// Dev probe: tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 (packed e2m1
// operands, unit E8M0 scales from TMEM) as an exact small-integer GEMM.
//  1. correctness: D = A B^T for random e2m1-exact integers {0,+-1,+-2,+-3,+-4,+-6},
//     M=256, N=160, K=256, operands in the K-major 128B-swizzled layout the kernels use;
//     reports which nibble of a byte holds the even K element.
//  2. exactness of long fp32 accumulation: D = 131072 then +-1 terms (C5-size sums).
//  3. throughput: back-to-back MMAs at N = 128 / 160 / 256.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2508_17655_b200/csrc/ptx.cuh"
using namespace sbg;

__host__ __device__ constexpr uint32_t idesc_mxf4(uint32_t M, uint32_t N) {
  return (1u << 7) | (1u << 10) | ((N >> 3) << 17) | (1u << 23) | ((M >> 4) << 24);
}
__device__ __forceinline__ void mma_mxf4_pair(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t sfa,
                                              uint32_t sfb, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%6], p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sfa), "r"(sfb)
      : "memory");
}

constexpr int K = 256;        // elements per row (128 bytes: one swizzle atom wide)
constexpr int ROWB = K / 2;   // bytes per row
constexpr int SF_COL = 256;   // TMEM columns [256, 264): unit scales
constexpr int NMAX = 256;

// smem byte of (row r, byte kb) in the K-major SW128 layout
__device__ __forceinline__ int sw(int r, int kb) { return (r >> 3) * 1024 + (r & 7) * 128 + (((kb >> 4) ^ (r & 7)) << 4) + (kb & 15); }

// mode 0: one K=256 product (4 MMAs); mode 1: `iters` MMAs on the same operands (accumulate)
template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    probe(const uint8_t* A, const uint8_t* B, const uint8_t* B2, int iters, int iters2, float* D, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t base = (ptx::smem_u32(sm) + 1023u) & ~1023u;
  uint8_t* s = sm + (base - ptx::smem_u32(sm));
  // A half (128 rows) at 0, B half (N/2 rows) at 16384, B2 half at 16384 + 16384
  uint64_t* bar = reinterpret_cast<uint64_t*>(s + 65536);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cr = ptx::cluster_ctarank();
  for (int i = threadIdx.x; i < 128 * ROWB; i += 128) s[sw(i / ROWB, i % ROWB)] = A[(cr * 128 + i / ROWB) * ROWB + i % ROWB];
  for (int i = threadIdx.x; i < (N / 2) * ROWB; i += 128) {
    const int r = i / ROWB, kb = i % ROWB, g = cr * (N / 2) + r;
    s[16384 + sw(r, kb)] = B[g * ROWB + kb];
    s[32768 + sw(r, kb)] = B2[g * ROWB + kb];
  }
  if (threadIdx.x == 0) { ptx::mbar_init(ptx::smem_u32(bar), 1); ptx::fence_mbar_init(); }
  if (warp == 2) { ptx::tmem_alloc_pair(ptx::smem_u32(slot), 512); ptx::tmem_relinquish_pair(); }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *slot;
  {  // unit scales: 0x7F7F7F7F in columns [SF_COL, SF_COL + 8) of every lane
    uint32_t v[8];
    for (int j = 0; j < 8; ++j) v[j] = 0x7F7F7F7Fu;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                     tmem + ((warp * 32u) << 16) + SF_COL),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync_all();
  ptx::tc_fence_after();
  if (cr == 0 && warp == 1) {
    constexpr uint32_t idesc = idesc_mxf4(256, N);
    const uint64_t ad = ptx::smem_desc_k_sw128(base), bd = ptx::smem_desc_k_sw128(base + 16384),
                   bd2 = ptx::smem_desc_k_sw128(base + 32768);
    const uint32_t sf = tmem + SF_COL;
    unsigned long long t0 = clock64();
    if (ptx::elect_one()) {
      for (int i = 0; i < iters; ++i) mma_mxf4_pair(tmem, ad + 2 * (i & 3), bd + 2 * (i & 3), idesc, sf, sf, i != 0);
      for (int i = 0; i < iters2; ++i) mma_mxf4_pair(tmem, ad + 2 * (i & 3), bd2 + 2 * (i & 3), idesc, sf, sf, 1);
      ptx::mma_commit_pair_mc(ptx::smem_u32(bar), 0x3);
    }
    __syncwarp();
    ptx::mbar_wait(ptx::smem_u32(bar), 0);
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0 && lane == 0) *cyc = t1 - t0;
  } else if (warp == 1) {
    ptx::mbar_wait(ptx::smem_u32(bar), 0);
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (blockIdx.x < 2 && D) {  // D rows of this CTA: lane = row
    for (int c = 0; c < N; c += 8) {
      uint32_t v[8];
      ptx::tmem_ld<8>(tmem + ((warp * 32u) << 16) + c, v);
      ptx::tmem_ld_wait();
      for (int j = 0; j < 8; ++j) D[(cr * 128 + warp * 32 + lane) * N + c + j] = __uint_as_float(v[j]);
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync_all();
  if (warp == 2) ptx::tmem_dealloc_pair(tmem, 512);
}

static uint8_t enc(int v) {  // e2m1 code of an e2m1-exact integer
  const int a = v < 0 ? -v : v;
  const uint8_t m = a == 0 ? 0 : a == 1 ? 2 : a == 2 ? 4 : a == 3 ? 5 : a == 4 ? 6 : 7;
  return static_cast<uint8_t>(m | (v < 0 && a ? 8 : 0));
}

template <int N>
void run() {
  const int vals[11] = {0, 1, -1, 2, -2, 3, -3, 4, -4, 6, -6};
  std::vector<int> a(256 * K), b(N * K), b2(N * K);
  srand(12345);
  for (auto& v : a) v = vals[rand() % 11];
  for (auto& v : b) v = vals[rand() % 11];
  for (auto& v : b2) v = (rand() & 1) ? 1 : -1;
  auto pack = [](const std::vector<int>& m, int rows, bool lo_first) {
    std::vector<uint8_t> p(rows * ROWB);
    for (int r = 0; r < rows; ++r)
      for (int k = 0; k < K; k += 2) {
        const uint8_t e0 = enc(m[r * K + k]), e1 = enc(m[r * K + k + 1]);
        p[r * ROWB + k / 2] = lo_first ? static_cast<uint8_t>(e0 | (e1 << 4)) : static_cast<uint8_t>(e1 | (e0 << 4));
      }
    return p;
  };
  uint8_t *dA, *dB, *dB2;
  float* dD;
  unsigned long long* dc;
  cudaMalloc(&dA, 256 * ROWB); cudaMalloc(&dB, N * ROWB); cudaMalloc(&dB2, N * ROWB);
  cudaMalloc(&dD, 256 * N * 4); cudaMalloc(&dc, 8);
  const int smem = 65536 + 1024 + 64;
  cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int lo = 1; lo >= 0; --lo) {
    auto pa = pack(a, 256, lo), pb = pack(b, N, lo), pb2 = pack(b2, N, lo);
    cudaMemcpy(dA, pa.data(), pa.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, pb.data(), pb.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB2, pb2.data(), pb2.size(), cudaMemcpyHostToDevice);
    probe<N><<<2, 128, smem>>>(dA, dB, dB2, 4, 0, dD, dc);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> D(256 * N);
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    long bad = 0;
    for (int i = 0; i < 256; ++i)
      for (int j = 0; j < N; ++j) {
        long ref = 0;
        for (int k = 0; k < K; ++k) ref += a[i * K + k] * b[j * K + k];
        if (D[i * N + j] != static_cast<float>(ref)) ++bad;
      }
    printf("N=%d nibble order %s: %ld / %d mismatches (%s) D[0]=%g\n", N, lo ? "even=low" : "even=high", bad, 256 * N,
           cudaGetErrorString(e), D[0]);
  }
  {  // long accumulation: all-ones A/B first (2048 MMAs of K=64 -> 131072), then +-1 B2 terms
    std::vector<int> ones(256 * K, 1), onesb(N * K, 1);
    auto pa = pack(ones, 256, true), pb = pack(onesb, N, true), pb2 = pack(b2, N, true);
    cudaMemcpy(dA, pa.data(), pa.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, pb.data(), pb.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB2, pb2.data(), pb2.size(), cudaMemcpyHostToDevice);
    const int it1 = 2048, it2 = 1000;
    probe<N><<<2, 128, smem>>>(dA, dB, dB2, it1, it2, dD, dc);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> D(256 * N);
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    long bad = 0;
    for (int i = 0; i < 256; ++i)
      for (int j = 0; j < N; ++j) {
        long ref = 64L * it1;
        for (int t = 0; t < it2; ++t)
          for (int k = 0; k < 64; ++k) ref += b2[j * K + (t & 3) * 64 + k];
        if (D[i * N + j] != static_cast<float>(ref)) ++bad;
      }
    printf("N=%d long accumulation (131072 then %d +-1 MMAs): %ld mismatches (%s) D[0]=%.1f\n", N, it2, bad,
           cudaGetErrorString(e), D[0]);
  }
  for (int grid : {2, 148}) {
    const int iters = 4096;
    probe<N><<<grid, 128, smem>>>(dA, dB, dB2, iters, 0, nullptr, dc);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h;
    cudaMemcpy(&h, dc, 8, cudaMemcpyDeviceToHost);
    printf("N=%d grid %d: %.1f cycles per MMA (M=256,K=64): %.0f fp4 MAC/cycle/SM (%s)\n", N, grid, double(h) / iters,
           256.0 * N * 64 / (double(h) / iters) / 2, cudaGetErrorString(e));
  }
  cudaFree(dA); cudaFree(dB); cudaFree(dB2); cudaFree(dD); cudaFree(dc);
}

int main() {
  run<48>();
  run<80>();
  run<128>();
  run<160>();
  run<256>();
  return 0;
}
