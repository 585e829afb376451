// Dev probe: max active 16-CTA clusters at ~208 KB smem / 640 threads, and DSMEM bulk-copy
// bandwidth/latency (each CTA pushes 8 KB to every CTA of its cluster, signalling mbarriers).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t r) { uint32_t d; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(r)); return d; }
__device__ __forceinline__ uint32_t rank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ uint32_t nrank() { uint32_t r; asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r)); return r; }
__device__ __forceinline__ void csync() { asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ bool try_wait(uint32_t bar, uint32_t ph) {
  uint32_t ok; asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p;}" : "=r"(ok) : "r"(bar), "r"(ph) : "memory"); return ok; }
extern "C" __global__ void __launch_bounds__(640, 1) probe(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* recv = sm;               // 16 x 8 KB
  uint8_t* send = sm + 16 * 8192;   // 8 KB
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 17 * 8192);
  const uint32_t r = rank(), nr = nrank();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) send[i] = uint8_t(r + i);
  __syncthreads();
  csync();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(nr * 8192u) : "memory");
    }
    csync();  // every CTA has armed its barrier for this phase
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      for (uint32_t d = 0; d < nr; ++d) {
        const uint32_t dst = mapa(smem_u32(recv + r * 8192), d), mb = mapa(smem_u32(bar), d);
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(dst), "r"(smem_u32(send)), "r"(8192), "r"(mb) : "memory");
      }
    }
    while (!try_wait(smem_u32(bar), it & 1)) {}
  }
  unsigned long long t1 = clock64();
  csync();
  if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = t1 - t0; out[1] = recv[5 * 8192 + 7]; }
}
int main() {
  const int smem = 17 * 8192 + 64 + 65536;  // + pad to ~208 KB
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 8); cfg.blockDim = dim3(640); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1; cfg.attrs = at; cfg.numAttrs = 1;
    int nclu = 0; cudaError_t e = cudaOccupancyMaxActiveClusters(&nclu, probe, &cfg);
    printf("cluster %d: max active clusters %d (%s)\n", cs, nclu, cudaGetErrorString(e));
    if (nclu < 1) continue;
    cfg.gridDim = dim3(cs * nclu);
    unsigned long long* d; cudaMalloc(&d, 16);
    const int iters = 1000;
    e = cudaLaunchKernelEx(&cfg, probe, iters, d);
    cudaDeviceSynchronize();
    unsigned long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("  launch %s: %.1f cycles per all-to-all round (%d x 8 KB pushed per CTA), check %llu\n",
           cudaGetErrorString(cudaGetLastError()), double(h[0]) / iters, cs, h[1]);
  }
  return 0;
}
