// Random-segment read bandwidth with full memory-level parallelism: a warp
// reads one C-byte segment per load instruction (C / 32 bytes per lane) at a
// random C-aligned offset, U segments in flight per lane -- the K5s access
// pattern (C = 256: one history-row segment of 256 frames per nonzero pixel)
// and its longer-segment alternatives.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int C, int U>
__global__ void gather(const uint8_t* __restrict__ buf, const uint32_t* __restrict__ idx, int nidx,
                       unsigned long long* sink) {
  constexpr int L = C / 32;  // bytes per lane: 8 / 16 / 32 / 64
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int nwarps = (gridDim.x * blockDim.x) >> 5;
  uint32_t acc = 0;
  for (int i0 = warp; i0 < nidx; i0 += nwarps * U) {
    uint4 v[U][(L + 15) / 16];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = i0 + u * nwarps;
      const uint8_t* p = buf + (size_t)(j < nidx ? idx[j] : 0) * C + lane * L;
      if (L == 8) {
        const uint2 w = __ldcs(reinterpret_cast<const uint2*>(p));
        v[u][0] = make_uint4(w.x, w.y, 0, 0);
      } else {
#pragma unroll
        for (int k = 0; k < (L + 15) / 16; ++k) v[u][k] = __ldcs(reinterpret_cast<const uint4*>(p) + k);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int k = 0; k < (L + 15) / 16; ++k) acc ^= v[u][k].x ^ v[u][k].y ^ v[u][k].z ^ v[u][k].w;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

template <int C, int U>
void run(const uint8_t* buf, size_t bytes, unsigned long long* sink, int blocks_per_sm) {
  const size_t nchunks = bytes / C;
  const int nidx = (int)((size_t)(512ull << 20) / C);
  uint32_t* h = new uint32_t[nidx];
  uint64_t s = 88172645463325252ull;
  for (int i = 0; i < nidx; ++i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    h[i] = (uint32_t)(s % nchunks);
  }
  uint32_t* d;
  cudaMalloc(&d, nidx * 4);
  cudaMemcpy(d, h, nidx * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int grid = 148 * blocks_per_sm;
  for (int w = 0; w < 2; ++w) gather<C, U><<<grid, 256>>>(buf, d, nidx, sink);
  cudaEventRecord(a);
  for (int w = 0; w < 5; ++w) gather<C, U><<<grid, 256>>>(buf, d, nidx, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("segment %5d B, %2d in flight/lane, %d blocks/SM: %7.0f GB/s (%s)\n", C, U, blocks_per_sm,
         5.0 * nidx * C / (ms / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
  delete[] h;
}

int main() {
  const size_t bytes = 8ull << 30;
  uint8_t* buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 1, bytes);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  for (int bps : {4, 8}) {
    run<256, 8>(buf, bytes, sink, bps);
    run<256, 16>(buf, bytes, sink, bps);
    run<512, 8>(buf, bytes, sink, bps);
    run<1024, 4>(buf, bytes, sink, bps);
    run<1024, 8>(buf, bytes, sink, bps);
    run<2048, 4>(buf, bytes, sink, bps);
  }
  return 0;
}
