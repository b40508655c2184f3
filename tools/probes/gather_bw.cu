// Random-chunk read bandwidth probe: each warp reads whole chunks of C bytes
// at random C-aligned offsets of a large buffer (the access pattern of the
// sparse streaming column, K5s: one history-row segment per nonzero pixel).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void gather(const uint4* __restrict__ buf, const uint32_t* __restrict__ idx, int nidx,
                       int chunk16, unsigned long long* sink) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  uint32_t acc = 0;
  for (int i = warp; i < nidx; i += nwarps * 8) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = i + u * nwarps;
      v[u] = make_uint4(0, 0, 0, 0);
      if (j < nidx)
        for (int c = lane; c < chunk16; c += 32) {
          const uint4 w = __ldcs(buf + (size_t)idx[j] * chunk16 + c);
          v[u].x ^= w.x; v[u].y ^= w.y; v[u].z ^= w.z; v[u].w ^= w.w;
        }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main() {
  const size_t bytes = 16ull << 30;
  uint4* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int chunk : {64, 128, 256, 512, 1024, 4096}) {
    const size_t nchunks = bytes / chunk;
    const int nidx = (int)((size_t)(512ull << 20) / chunk);  // 512 MB read per pass
    uint32_t* h = new uint32_t[nidx];
    uint64_t s = 88172645463325252ull;
    for (int i = 0; i < nidx; ++i) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      h[i] = (uint32_t)(s % nchunks);
    }
    uint32_t* d;
    cudaMalloc(&d, nidx * 4);
    cudaMemcpy(d, h, nidx * 4, cudaMemcpyHostToDevice);
    for (int w = 0; w < 2; ++w) gather<<<148 * 8, 256>>>(buf, d, nidx, chunk / 16, sink);
    cudaEventRecord(a);
    for (int w = 0; w < 5; ++w) gather<<<148 * 8, 256>>>(buf, d, nidx, chunk / 16, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("chunk %5d B: %7.0f GB/s (%s)\n", chunk, 5.0 * nidx * chunk / (ms / 1e3) / 1e9,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
    delete[] h;
  }
  return 0;
}
