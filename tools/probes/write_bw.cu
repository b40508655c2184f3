// Pure-write HBM bandwidth probe: 16-byte stores (default / streaming), and
// TMA-free bulk copies smem -> global (cp.async.bulk), 4 GB buffer.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void w_v4(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(1, 2, 3, 4);
}
__global__ void w_cs(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(p + i, make_uint4(1, 2, 3, 4));
}
// each block writes 16 KB chunks with cp.async.bulk from a smem buffer
__global__ void w_bulk(char* p, size_t nchunks, int chunk) {
  extern __shared__ __align__(128) char sm[];
  for (int i = threadIdx.x; i < chunk; i += blockDim.x) sm[i] = 1;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
  int inflight = 0;
  for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" :: "l"(p + c * chunk), "r"(s), "r"(chunk) : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    if (++inflight > 8) asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const size_t bytes = 4ull << 30;
  char* p;
  cudaMalloc(&p, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto run = [&](const char* name, auto launch) {
    for (int i = 0; i < 3; ++i) launch();
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-28s %7.0f GB/s  (%s)\n", name, bytes / (ms / 10) / 1e6, cudaGetErrorString(cudaGetLastError()));
  };
  for (int bpsm : {2, 4, 8}) {
    char nm[64];
    snprintf(nm, 64, "st.v4 %d blk/SM", bpsm);
    run(nm, [&] { w_v4<<<sms * bpsm, 512>>>((uint4*)p, bytes / 16); });
    snprintf(nm, 64, "st.cs.v4 %d blk/SM", bpsm);
    run(nm, [&] { w_cs<<<sms * bpsm, 512>>>((uint4*)p, bytes / 16); });
  }
  for (int chunk : {4096, 16384, 65536}) {
    cudaFuncSetAttribute(w_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
    for (int bpsm : {1, 2, 3}) {
      char nm[64];
      snprintf(nm, 64, "bulk %dB x%d/SM", chunk, bpsm);
      run(nm, [&] { w_bulk<<<sms * bpsm, 128, chunk>>>(p, bytes / chunk, chunk); });
    }
  }
  return 0;
}
