#include <cstdio>
#include "gp_common.cuh"
using namespace gp;
__device__ __forceinline__ unsigned long long gtime() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void empty_kernel() {}
__global__ void smem_kernel() { extern __shared__ int s[]; if (threadIdx.x == 0x7fffffff) s[0] = 1; }
// barrier variants
__device__ __forceinline__ void bar_nofence(uint32_t* word, uint32_t nb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t inc = blockIdx.x == 0 ? 0x80000000u - (nb - 1u) : 1u;
    const uint32_t old = atom_add_release_gpu(word, inc);
    while (((old ^ ld_acquire_gpu(word)) & 0x80000000u) == 0u) {}
  }
  __syncthreads();
}
__device__ __forceinline__ void bar_red(uint32_t* word, uint32_t nb) {
  // arrive with red (no return), poll the count: target read before arriving
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t g = ld_acquire_gpu(word);
    const uint32_t inc = blockIdx.x == 0 ? 0x80000000u - (nb - 1u) : 1u;
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" :: "l"(word), "r"(inc) : "memory");
    while (((g ^ ld_acquire_gpu(word)) & 0x80000000u) == 0u) {}
  }
  __syncthreads();
}
template <int V>
__global__ void barrier_kernel(uint32_t* word, int n, unsigned long long* out) {
  unsigned long long t0 = gtime();
  for (int i = 0; i < n; ++i) {
    if (V == 0) grid_barrier(word, gridDim.x);
    else if (V == 1) bar_nofence(word, gridDim.x);
    else bar_red(word, gridDim.x);
  }
  if (threadIdx.x == 0) out[blockIdx.x] = gtime() - t0;
}
template <class F> float tl(F f, int reps) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  f(); f(); cudaDeviceSynchronize();
  cudaEventRecord(a); for (int i = 0; i < reps; ++i) f(); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); return ms * 1000.f / reps;
}
int main() {
  uint32_t* word; unsigned long long* out; cudaMalloc(&word, 4096); cudaMemset(word, 0, 4096); cudaMalloc(&out, 8 * 4096);
  for (int blk : {128, 256, 512, 1024})
    for (int grid : {148, 296, 1184}) {
      if (grid * blk > 148 * 2048) continue;
      printf("empty %4d x %4d: %.2f us\n", grid, blk, tl([&] { empty_kernel<<<grid, blk>>>(); }, 200));
    }
  cudaFuncSetAttribute(smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  printf("empty 148 x 1024 + 160KB smem: %.2f us\n", tl([&] { smem_kernel<<<148, 1024, 160 * 1024>>>(); }, 200));
  printf("empty 148 x 512 + 160KB smem: %.2f us\n", tl([&] { smem_kernel<<<148, 512, 160 * 1024>>>(); }, 200));
  // cooperative launch overhead
  auto coop = [&](int grid, int blk) {
    cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(grid); cfg.blockDim = dim3(blk);
    cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = 1; cfg.attrs = at; cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, empty_kernel);
  };
  printf("coop empty 148x1024: %.2f us\n", tl([&] { coop(148, 1024); }, 200));
  printf("coop empty 148x256: %.2f us\n", tl([&] { coop(148, 256); }, 200));
  // graph of 20 empty launches
  {
    cudaStream_t s; cudaStreamCreate(&s); cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 20; ++i) empty_kernel<<<148, 1024, 0, s>>>();
    cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ge, g, 0);
    printf("graph 20x empty 148x1024: %.2f us per kernel\n", tl([&] { cudaGraphLaunch(ge, s); }, 50) / 20);
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < 20; ++i) empty_kernel<<<148, 256, 0, s>>>();
    cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ge, g, 0);
    printf("graph 20x empty 148x256: %.2f us per kernel\n", tl([&] { cudaGraphLaunch(ge, s); }, 50) / 20);
  }
  for (int v = 0; v < 3; ++v)
    for (int blk : {256, 1024}) {
      int n = 20;
      void* args[] = {&word, &n, &out};
      const void* fn = v == 0 ? (const void*)barrier_kernel<0> : v == 1 ? (const void*)barrier_kernel<1> : (const void*)barrier_kernel<2>;
      cudaLaunchCooperativeKernel(fn, dim3(148), dim3(blk), args, 0, 0);
      cudaDeviceSynchronize();
      unsigned long long h[148]; cudaMemcpy(h, out, 8 * 148, cudaMemcpyDeviceToHost);
      unsigned long long mx = 0; for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("barrier variant %d, 148x%d: %.3f us/barrier\n", v, blk, mx / 1e3 / n);
    }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
