// Bulk-store (TMA, cp.async.bulk smem -> global) throughput probe: one CTA per
// SM, W warps, each with NB 4 KB staging buffers; lane 0 of each warp streams
// 4 KB bulk stores to consecutive global chunks.  Reports GB/s per
// configuration (1 GiB written per run, best of 5).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void k_store(float* dst, int W, int NB, int64_t chunks_per_warp, int hint) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* buf = sm + static_cast<size_t>(warp) * NB * 4096;
  for (int i = lane; i < NB * 1024; i += 32) reinterpret_cast<float*>(buf)[i] = 1.0f;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane != 0) return;
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * W + warp;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  for (int64_t i = 0; i < chunks_per_warp; ++i) {
    const int b = static_cast<int>(i % NB);
    if (NB == 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    else if (NB == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
    else asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
    float* g = dst + (gw * chunks_per_warp + i) * 1024;
    if (hint)
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], 4096, %2;"
                   ::"l"(g), "r"(smem_u32(buf + b * 4096)), "l"(pol) : "memory");
    else
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 4096;"
                   ::"l"(g), "r"(smem_u32(buf + b * 4096)) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int64_t total = 1ll << 30;
  float* dst;
  cudaMalloc(&dst, total * 2);
  cudaFuncSetAttribute(k_store, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  int Ws[] = {4, 8, 12, 16, 24, 32};
  int NBs[] = {1, 2, 4};
  for (int hint = 0; hint < 2; ++hint)
    for (int W : Ws)
      for (int NB : NBs) {
        if (W * NB * 4096 > 200 * 1024) continue;
        const int64_t cpw = total / 4096 / (sms * W);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
          cudaEventRecord(a);
          k_store<<<sms, 32 * W, W * NB * 4096>>>(dst, W, NB, cpw, hint);
          cudaEventRecord(b);
          cudaEventSynchronize(b);
          float ms;
          cudaEventElapsedTime(&ms, a, b);
          if (ms < best) best = ms;
        }
        const double bytes = static_cast<double>(cpw) * 4096 * sms * W;
        printf("hint %d W %2d NB %d: %7.0f GB/s (%.1f B/clk/SM at 1.9 GHz)\n", hint, W, NB,
               bytes / (best / 1e3) / 1e9, bytes / (best / 1e3) / sms / 1.9e9);
      }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
