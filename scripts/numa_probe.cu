// numa_probe.cu -- is HBM bandwidth die-local on B200?  (SM ids < 74 vs >= 74 taken as the two dies)
//
// 148 CTAs x 1024 threads are launched; only the CTAs on the chosen "die" (by %smid)
// stream, each its contiguous share of a 256 MB slice of a 2 GB buffer, with
// 16-byte loads (8 in flight per thread).  Prints GB/s for every (die, slice):
// a die-local memory layout shows up as slices one die reads much faster than the other.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o numa_probe scripts/numa_probe.cu && ./numa_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(1024, 1) rd(const uint4* __restrict__ x, size_t n16, int die, unsigned* cnt,
                                              unsigned long long* sink) {
  __shared__ unsigned slot;
  unsigned smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  const bool mine = die < 0 || (int)(smid >= 74) == die;
  if (!mine) return;
  if (threadIdx.x == 0) slot = atomicAdd(cnt, 1u);  // dense rank among participating CTAs
  __syncthreads();
  const unsigned nparts = die < 0 ? gridDim.x : 74u;
  const size_t per = (n16 + nparts - 1) / nparts;
  const size_t b = (size_t)slot * per, e = b + per < n16 ? b + per : n16;
  unsigned long long acc = 0;
  for (size_t i = b + threadIdx.x; i < e; i += 8 * 1024) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = i + u * 1024 < e ? x[i + u * 1024] : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u].x ^ v[u].w;
  }
  if (acc == 0x123456789ull) sink[0] = acc;
}

int main() {
  const size_t total = 2ull << 30, slice = 256ull << 20;
  unsigned char* x;
  unsigned *cnt;
  unsigned long long* sink;
  cudaMalloc(&x, total);
  cudaMemset(x, 1, total);
  cudaMalloc(&cnt, 4);
  cudaMalloc(&sink, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  printf("slice  die0 GB/s  die1 GB/s  both GB/s\n");
  for (size_t off = 0; off < total; off += slice) {
    float r[3];
    for (int die = -1; die <= 1; ++die) {
      float best = 1e30f;
      for (int rep = 0; rep < 4; ++rep) {
        cudaMemset(cnt, 0, 4);
        cudaEventRecord(a);
        rd<<<148, 1024>>>(reinterpret_cast<const uint4*>(x + off), slice / 16, die, cnt, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (rep && ms < best) best = ms;
      }
      r[die + 1] = slice / (best * 1e-3) / 1e9;
    }
    printf("%4zu MB  %8.1f  %8.1f  %8.1f  %s\n", off >> 20, r[1], r[2], r[0], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
