// p2p_bulk_probe.cu -- can a kernel on GPU 1 stream GPU 0's memory with bulk (TMA) copies, and how fast?
//
// Reads a 256 MB buffer that lives on GPU 0 from a kernel on GPU 1 (peer access
// enabled), each CTA streaming its contiguous share through a ring of S x CHUNK
// shared-memory slots filled by cp.async.bulk (one mbarrier per slot), summing
// the words so the data is consumed.  Compared with a plain-load kernel (16-byte
// loads, U in flight per thread) and with the same kernels reading local memory.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o p2p_bulk_probe scripts/p2p_bulk_probe.cu && ./p2p_bulk_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int S, int CHUNK>
__global__ void __launch_bounds__(128) bulk_stream(const uint4* __restrict__ src, size_t n16, unsigned long long* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar[S];
  const size_t per = (n16 * 16 / gridDim.x) & ~(size_t)(CHUNK - 1);
  const unsigned char* base = reinterpret_cast<const unsigned char*>(src) + (size_t)blockIdx.x * per;
  const uint32_t nch = (uint32_t)(per / CHUNK);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (uint32_t c = 0; c < (uint32_t)S && c < nch; ++c) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[c])), "r"(CHUNK) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(sm + c * CHUNK)),
                   "l"(base + (size_t)c * CHUNK), "r"(CHUNK), "r"(smem_u32(&bar[c])) : "memory");
    }
  }
  __syncthreads();
  unsigned long long acc = 0;
  for (uint32_t c = 0; c < nch; ++c) {
    const uint32_t s = c % S;
    uint32_t ok = 0;
    do {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                   : "=r"(ok) : "r"(smem_u32(&bar[s])), "r"((c / S) & 1) : "memory");
    } while (!ok);
    const uint4* v = reinterpret_cast<const uint4*>(sm + s * CHUNK);
    for (int i = threadIdx.x; i < CHUNK / 16; i += blockDim.x) acc += v[i].x + v[i].w;
    __syncthreads();
    if (threadIdx.x == 0 && c + S < nch) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(CHUNK) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(sm + s * CHUNK)),
                   "l"(base + (size_t)(c + S) * CHUNK), "r"(CHUNK), "r"(smem_u32(&bar[s])) : "memory");
    }
  }
  if (acc == 0x1234567ull) out[0] = acc;
  if (threadIdx.x == 0) atomicAdd(out + 1, (unsigned long long)nch);
}

template <int U>
__global__ void __launch_bounds__(512) plain_stream(const uint4* __restrict__ src, size_t n16, unsigned long long* out) {
  unsigned long long acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = i + u * stride < n16 ? src[i + u * stride] : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].x + v[u].w;
  }
  if (acc == 0x1234567ull) out[0] = acc;
}

template <class F>
static float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  return best;
}

int main() {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  const size_t bytes = 256ull << 20, n16 = bytes / 16;
  uint4 *remote = nullptr, *local = nullptr;
  unsigned long long* out = nullptr;
  CK(cudaSetDevice(0));
  CK(cudaMalloc(&remote, bytes));
  CK(cudaMemset(remote, 1, bytes));
  const int rd = ndev > 1 ? 1 : 0;
  CK(cudaSetDevice(rd));
  if (rd) {
    int can = 0;
    CK(cudaDeviceCanAccessPeer(&can, 1, 0));
    printf("peer access 1->0: %d\n", can);
    CK(cudaDeviceEnablePeerAccess(0, 0));
  }
  CK(cudaMalloc(&local, bytes));
  CK(cudaMemset(local, 1, bytes));
  CK(cudaMalloc(&out, 16));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, rd));
  struct Src { const char* name; uint4* p; } srcs[2] = {{"local ", local}, {"remote", remote}};
  for (auto& s : srcs) {
    if (!rd && s.p == remote) continue;
    for (int grid : {sms, 2 * sms, 4 * sms}) {
      auto run_b = [&](auto kern, int S, int CHUNK) {
        const size_t smem = (size_t)S * CHUNK;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const float ms = timeit([&] { kern<<<grid, 128, smem>>>(s.p, n16, out); });
        const cudaError_t e = cudaGetLastError();
        printf("%s bulk  S=%d CHUNK=%5d grid=%4d: %8.1f GB/s %s\n", s.name, S, CHUNK, grid, bytes / (ms * 1e-3) / 1e9,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
      };
      run_b(bulk_stream<4, 8192>, 4, 8192);
      run_b(bulk_stream<8, 8192>, 8, 8192);
      run_b(bulk_stream<4, 16384>, 4, 16384);
      const float ms = timeit([&] { plain_stream<4><<<grid, 512>>>(s.p, n16, out); });
      printf("%s plain U=4 grid=%4d: %8.1f GB/s %s\n", s.name, grid, bytes / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
      const float ms8 = timeit([&] { plain_stream<8><<<grid, 512>>>(s.p, n16, out); });
      printf("%s plain U=8 grid=%4d: %8.1f GB/s\n", s.name, grid, bytes / (ms8 * 1e-3) / 1e9);
    }
  }
  return 0;
}
