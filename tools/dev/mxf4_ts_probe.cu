// Dev probe: tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 with the A operand in
// TENSOR MEMORY (the "TS" form: [d], [a_tmem], b_desc) vs A in shared memory (SS).
//  1. correctness + layout: A row r of this CTA in TMEM lane r, K packed 8 e2m1 per 32-bit
//     column (the bytes of a packed row as little-endian words); nibble order checked;
//  2. throughput at N = 32 / 48 / 80 / 160, SS vs TS, one CTA pair and all 74 pairs.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mxf4_ts_probe mxf4_ts_probe.cu -lcuda
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
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t sf, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], %1, %2, %3, [%5], [%5], p;\n\t}" ::"r"(d),
               "l"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sf) : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t sf, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%5], [%5], p;\n\t}" ::"r"(d),
               "r"(a), "l"(b), "r"(idesc), "r"(acc), "r"(sf) : "memory");
}

constexpr int K = 256, ROWB = K / 2;
constexpr int COL_A = 256, COL_SF = 448;

__device__ __forceinline__ int sw(int r, int kb) { return (r >> 3) * 1024 + (r & 7) * 128 + (((kb >> 4) ^ (r & 7)) << 4) + (kb & 15); }

template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    probe(const uint8_t* A, const uint8_t* B, int iters, int ts, float* D, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t base = (ptx::smem_u32(sm) + 1023u) & ~1023u;
  uint8_t* s = sm + (base - ptx::smem_u32(sm));
  uint64_t* bar = reinterpret_cast<uint64_t*>(s + 65536);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cr = ptx::cluster_ctarank();
  for (int i = threadIdx.x; i < 128 * ROWB; i += 128) s[sw(i / ROWB, i % ROWB)] = A[(cr * 128 + i / ROWB) * ROWB + i % ROWB];
  for (int i = threadIdx.x; i < (N / 2) * ROWB; i += 128) {
    const int r = i / ROWB, kb = i % ROWB;
    s[16384 + sw(r, kb)] = B[(cr * (N / 2) + r) * ROWB + kb];
  }
  if (threadIdx.x == 0) { ptx::mbar_init(ptx::smem_u32(bar), 1); ptx::fence_mbar_init(); }
  if (warp == 2) { ptx::tmem_alloc_pair(ptx::smem_u32(slot), 512); ptx::tmem_relinquish_pair(); }
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *slot;
  {
    const uint32_t tl = tmem + ((warp * 32u) << 16);
    uint32_t v[8];
    for (int j = 0; j < 8; ++j) v[j] = 0x7F7F7F7Fu;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tl + COL_SF),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]) : "memory");
    // A row (this CTA's row warp*32 + lane) as 32 little-endian words -> columns [COL_A, COL_A + 32)
    const uint32_t* row = reinterpret_cast<const uint32_t*>(A + (cr * 128 + warp * 32 + lane) * ROWB);
    for (int c = 0; c < 32; c += 8) {
      uint32_t w[8];
      for (int j = 0; j < 8; ++j) w[j] = row[c + j];
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(tl + COL_A + c),
                   "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::cluster_sync_all();
  ptx::tc_fence_after();
  if (cr == 0 && warp == 1) {
    constexpr uint32_t idesc = idesc_mxf4(256, N);
    const uint64_t ad = ptx::smem_desc_k_sw128(base), bd = ptx::smem_desc_k_sw128(base + 16384);
    const uint32_t sf = tmem + COL_SF;
    unsigned long long t0 = clock64();
    if (ptx::elect_one()) {
      if (ts)
        for (int i = 0; i < iters; ++i) mma_ts(tmem, tmem + COL_A + 8 * (i & 3), bd + 2 * (i & 3), idesc, sf, i != 0);
      else
        for (int i = 0; i < iters; ++i) mma_ss(tmem, ad + 2 * (i & 3), bd + 2 * (i & 3), idesc, sf, i != 0);
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
  if (blockIdx.x < 2 && D) {
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

static uint8_t enc(int v) {
  const int a = v < 0 ? -v : v;
  const uint8_t m = a == 0 ? 0 : a == 1 ? 2 : a == 2 ? 4 : a == 3 ? 5 : a == 4 ? 6 : 7;
  return static_cast<uint8_t>(m | (v < 0 && a ? 8 : 0));
}

template <int N>
void run() {
  const int vals[11] = {0, 1, -1, 2, -2, 3, -3, 4, -4, 6, -6};
  std::vector<int> a(256 * K), b(N * K);
  srand(777);
  for (auto& v : a) v = vals[rand() % 11];
  for (auto& v : b) v = vals[rand() % 11];
  auto pack = [](const std::vector<int>& m, int rows) {
    std::vector<uint8_t> p(rows * ROWB);
    for (int r = 0; r < rows; ++r)
      for (int k = 0; k < K; k += 2) p[r * ROWB + k / 2] = static_cast<uint8_t>(enc(m[r * K + k]) | (enc(m[r * K + k + 1]) << 4));
    return p;
  };
  uint8_t *dA, *dB;
  float* dD;
  unsigned long long* dc;
  cudaMalloc(&dA, 256 * ROWB); cudaMalloc(&dB, N * ROWB); cudaMalloc(&dD, 256 * N * 4); cudaMalloc(&dc, 8);
  const int smem = 65536 + 1024 + 64;
  cudaFuncSetAttribute(probe<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  auto pa = pack(a, 256), pb = pack(b, N);
  cudaMemcpy(dA, pa.data(), pa.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, pb.data(), pb.size(), cudaMemcpyHostToDevice);
  for (int ts = 0; ts < 2; ++ts) {
    probe<N><<<2, 128, smem>>>(dA, dB, 4, ts, dD, dc);
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
    printf("N=%d %s: %ld / %d mismatches (%s)\n", N, ts ? "TS (A in TMEM)" : "SS (A in smem)", bad, 256 * N,
           cudaGetErrorString(e));
  }
  for (int ts = 0; ts < 2; ++ts)
    for (int grid : {2, 148}) {
      const int iters = 4096;
      probe<N><<<grid, 128, smem>>>(dA, dB, iters, ts, nullptr, dc);
      cudaError_t e = cudaDeviceSynchronize();
      unsigned long long h;
      cudaMemcpy(&h, dc, 8, cudaMemcpyDeviceToHost);
      printf("N=%d %s grid %d: %.1f cycles per MMA (M=256,K=64) (%s)\n", N, ts ? "TS" : "SS", grid, double(h) / iters,
             cudaGetErrorString(e));
    }
  cudaFree(dA); cudaFree(dB); cudaFree(dD); cudaFree(dc);
}

int main() {
  run<32>();
  run<48>();
  run<80>();
  run<160>();
  return 0;
}
