// Microbenchmarks of the primitives the compress kernel is built from (development aid).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2410_12707_b200/csrc scripts/microbench.cu -o /tmp/mb
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "gp_common.cuh"

using namespace gp;

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__global__ void empty_kernel() {}

__global__ void barrier_kernel(uint32_t* word, int n, unsigned long long* out) {
  unsigned long long t0 = gtime();
  for (int i = 0; i < n; ++i) grid_barrier(word, gridDim.x);
  if (threadIdx.x == 0) out[blockIdx.x] = gtime() - t0;
}

__global__ void sync_kernel(int n, unsigned long long* out) {
  __shared__ uint32_t s[64];
  unsigned long long t0 = clock64();
  uint32_t v = threadIdx.x;
  for (int i = 0; i < n; ++i) {
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
    __syncthreads();
    v += s[(threadIdx.x >> 5) ^ 1];
  }
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0 + (v & 1);
}

__global__ void chase_kernel(const uint32_t* next, int n, unsigned long long* out) {
  uint32_t p = (n > 600) ? blockIdx.x * 97 : 0;
  unsigned long long t0 = clock64();
  for (int i = 0; i < n; ++i) p = next[p];
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0 + (p == 0xFFFFFFFF);
}

__global__ void gt_res_kernel(unsigned long long* out) {
  unsigned long long prev = gtime(), mind = ~0ull;
  for (int i = 0; i < 100000; ++i) {
    unsigned long long t = gtime();
    if (t != prev) {
      if (t - prev < mind) mind = t - prev;
      prev = t;
    }
  }
  out[0] = mind;
}

// same-address red.add contention: every CTA adds to `nbins` bins
__global__ void hot_red_kernel(uint32_t* hist, int nbins, uint32_t* word, unsigned long long* out) {
  unsigned long long t0 = gtime();
  for (int i = threadIdx.x; i < nbins; i += blockDim.x) red_add_gpu(&hist[i], 1u);
  grid_barrier(word, gridDim.x);
  if (threadIdx.x == 0) out[blockIdx.x] = gtime() - t0;
}

static float time_launches(void (*fn)(), int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  fn();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) fn();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1000.f / reps;
}

static uint32_t* g_word;
static unsigned long long* g_out;

static void launch_coop(const void* fn, void** args, int grid, int block) {
  cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(block), args, 0, 0);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaMalloc(&g_word, 4096);
  cudaMemset(g_word, 0, 4096);
  cudaMalloc(&g_out, 8 * 4096);
  std::vector<unsigned long long> h(4096);

  printf("SMs %d\n", sms);
  float t = time_launches([] { empty_kernel<<<148, 1024>>>(); }, 200);
  printf("empty kernel 148x1024 back-to-back: %.2f us/launch\n", t);

  gt_res_kernel<<<1, 1>>>(g_out);
  cudaMemcpy(h.data(), g_out, 8, cudaMemcpyDeviceToHost);
  printf("globaltimer min tick: %llu ns\n", h[0]);

  for (int n : {1, 10, 50}) {
    int nn = n;
    void* args[] = {&g_word, &nn, &g_out};
    launch_coop((const void*)barrier_kernel, args, sms, 1024);
    cudaDeviceSynchronize();
    cudaMemcpy(h.data(), g_out, 8 * sms, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0, sm = 0;
    for (int i = 0; i < sms; ++i) {
      mx = h[i] > mx ? h[i] : mx;
      sm += h[i];
    }
    printf("grid_barrier x%d (148x1024): mean %.2f us, max %.2f us -> %.3f us/barrier\n", n, sm / 1e3 / sms, mx / 1e3,
           mx / 1e3 / n);
  }
  for (int n : {10, 100}) {
    sync_kernel<<<sms, 1024>>>(n, g_out);
    cudaDeviceSynchronize();
    cudaMemcpy(h.data(), g_out, 8, cudaMemcpyDeviceToHost);
    printf("__syncthreads x%d (1024 thr): %.1f cycles each\n", n, (double)h[0] / n);
  }
  // L2 pointer chase
  {
    const int N = 1 << 20;  // 4 MB, L2 resident
    std::vector<uint32_t> nx(N);
    for (int i = 0; i < N; ++i) nx[i] = (uint32_t)((i * 2654435761ull + 12345) % N);
    uint32_t* dn;
    cudaMalloc(&dn, N * 4);
    cudaMemcpy(dn, nx.data(), N * 4, cudaMemcpyHostToDevice);
    chase_kernel<<<1, 32>>>(dn, 100, g_out);
    chase_kernel<<<1, 32>>>(dn, 1000, g_out);
    cudaDeviceSynchronize();
    cudaMemcpy(h.data(), g_out, 8, cudaMemcpyDeviceToHost);
    printf("dependent L2 load (4 MB set): %.1f cycles\n", (double)h[0] / 1000);
    const int N2 = 1 << 28;  // 1 GB, HBM
    uint32_t* dn2;
    cudaMalloc(&dn2, (size_t)N2 * 4);
    // 4096 nodes, 256 KiB apart, in a pseudo-random cycle
    for (int i = 0; i < 4096; ++i) {
      const uint32_t nxt = (uint32_t)(((i * 2654435761ull + 12345) % 4096) * 65536);
      cudaMemcpy(dn2 + (size_t)i * 65536, &nxt, 4, cudaMemcpyHostToDevice);
    }
    chase_kernel<<<1, 32>>>(dn2, 500, g_out);
    cudaDeviceSynchronize();
    cudaMemcpy(h.data(), g_out, 8, cudaMemcpyDeviceToHost);
    printf("dependent HBM load (1 GB set): %.1f cycles\n", (double)h[0] / 500);
  }
  for (int nb : {64, 300, 1000, 4000}) {
    uint32_t* hist;
    cudaMalloc(&hist, 4 * 65536);
    int nbv = nb;
    void* args[] = {&hist, &nbv, &g_word, &g_out};
    launch_coop((const void*)hot_red_kernel, args, sms, 1024);
    cudaDeviceSynchronize();
    cudaMemcpy(h.data(), g_out, 8 * sms, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("148 CTAs x red.add on %d shared bins + barrier: %.2f us\n", nb, mx / 1e3);
    cudaFree(hist);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
