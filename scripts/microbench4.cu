// CTA dispatch spread: every CTA records globaltimer at entry
#include <cstdio>
#include <vector>
#include <algorithm>
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
template <int SMEM>
__global__ void entry_kernel(unsigned long long* out, int spin_ns) {
  __shared__ int s[SMEM / 4 > 0 ? SMEM / 4 : 1];
  unsigned long long t = gt();
  if (threadIdx.x == 0) out[blockIdx.x] = t;
  if (spin_ns) { while (gt() - t < (unsigned long long)spin_ns) {} }
  if (threadIdx.x == 0x7fffffff) s[0] = 1;
}
template <int SMEM> void run(int grid, int block, int spin) {
  unsigned long long* d; cudaMalloc(&d, 8 * grid);
  for (int r = 0; r < 3; ++r) entry_kernel<SMEM><<<grid, block>>>(d, spin);
  cudaDeviceSynchronize();
  std::vector<unsigned long long> h(grid); cudaMemcpy(h.data(), d, 8 * grid, cudaMemcpyDeviceToHost);
  std::sort(h.begin(), h.end());
  printf("grid %5d block %4d smem %6d spin %5dns: entry spread %.2f us (p50 %.2f, p90 %.2f)\n", grid, block, SMEM, spin,
         (h.back() - h.front()) / 1e3, (h[grid / 2] - h.front()) / 1e3, (h[grid * 9 / 10] - h.front()) / 1e3);
  cudaFree(d);
}
int main() {
  run<0>(148, 1024, 0); run<0>(148, 1024, 20000);
  run<0>(512, 512, 0); run<0>(512, 512, 20000);
  run<32768>(512, 512, 0); run<32768>(512, 512, 20000);
  run<0>(592, 512, 20000); run<0>(1184, 256, 20000); run<0>(296, 512, 20000);
  run<32768>(296, 512, 20000);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
