// latency of a burst of independent loads at kernel start, 512 CTAs x 512 threads
#include <cstdio>
#include <vector>
#include <algorithm>
__device__ __forceinline__ unsigned long long gt() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void __launch_bounds__(512, 4) burst(const long long* idx, const float* val, long long k, int nl, unsigned long long* out) {
  unsigned long long t0 = gt();
  long long base = (k * blockIdx.x) / gridDim.x;
  long long s = 0; float f = 0;
  for (int i = 0; i < nl; ++i) { long long j = (base + threadIdx.x + i * 512) % k; s += __ldg(idx + j); f += __ldg(val + j); }
  int c = __syncthreads_count(s > 0 || f > 0);
  unsigned long long t1 = gt();
  if (threadIdx.x == 0) { out[2 * blockIdx.x] = t0; out[2 * blockIdx.x + 1] = t1 + (c == 12345); }
}
__global__ void flush(const float4* p, size_t n, float* o) { float s = 0; for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) s += p[i].x; if (s == 1.f) o[0] = s; }
int main() {
  long long k = 62914; long long* idx; float* val; cudaMalloc(&idx, 8 * k); cudaMalloc(&val, 4 * k);
  cudaMemset(idx, 0, 8 * k); cudaMemset(val, 0, 4 * k);
  float4* fb; size_t fn = (512u << 20) / 16; cudaMalloc(&fb, fn * 16); cudaMemset(fb, 0, fn * 16); float* o; cudaMalloc(&o, 64);
  unsigned long long* out; cudaMalloc(&out, 16 * 4096); std::vector<unsigned long long> h(2 * 4096);
  for (int G : {148, 512}) for (int nl : {1, 2, 8}) for (int cold = 0; cold < 2; ++cold) {
    burst<<<G, 512>>>(idx, val, k, nl, out);
    if (cold) flush<<<1184, 256>>>(fb, fn, o);
    burst<<<G, 512>>>(idx, val, k, nl, out);
    cudaDeviceSynchronize(); cudaMemcpy(h.data(), out, 16 * G, cudaMemcpyDeviceToHost);
    double mean = 0, mx = 0; for (int b = 0; b < G; ++b) { double dt = (h[2 * b + 1] - h[2 * b]) / 1e3; mean += dt / G; mx = dt > mx ? dt : mx; }
    printf("G=%d loads/thread=%d %s: mean %.2f us max %.2f us\n", G, 2 * nl, cold ? "cold(flushed)" : "warm", mean, mx);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
