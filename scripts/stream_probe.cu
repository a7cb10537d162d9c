// stream_probe.cu -- does a deeper per-warp TMA ring with fewer warps stream faster than the
// compress kernel's shape (1024 threads, two 2 KiB row-pair slots per warp)?
//
// Each warp streams its contiguous unit of a large fp32 buffer through a ring of SLOTS x 2 KiB
// shared-memory slots filled by bulk copies (one mbarrier per slot), tests |x| >= thr per element
// (FSETP + mask build, as the compress kernel's full steps do), and burns EXTRA dependent ALU
// instructions per step to stand in for the rest of the per-step work.  Grid = 24 CTAs (the bench's
// capped grid).  Prints GB/s per configuration.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_probe scripts/stream_probe.cu && ./stream_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok)
                 : "r"(bar), "r"(parity)
                 : "memory");
  } while (!ok);
}
__device__ __forceinline__ uint4 lds4(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}

template <int THREADS, int SLOTS, int EXTRA>
__global__ void __launch_bounds__(THREADS, 1) stream_kernel(const float* x, size_t n, float thr, unsigned* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int W = THREADS / 32;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t units = (size_t)gridDim.x * W;
  const size_t per = (n / units) & ~(size_t)511;  // whole 512-element row pairs
  const float* ux = x + ((size_t)blockIdx.x * W + w) * per;
  const uint32_t npair = (uint32_t)(per / 512);
  const uint32_t ring = smem_addr(smem) + w * SLOTS * 2048;
  const uint32_t mbar = smem_addr(smem + (size_t)W * SLOTS * 2048) + w * SLOTS * 8;
  if (lane == 0) {
    for (int s = 0; s < SLOTS; ++s) mbar_init(mbar + s * 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (uint32_t p = 0; p < (uint32_t)SLOTS && p < npair; ++p) bulk_load(ring + p * 2048, ux + (size_t)p * 512, 2048, mbar + p * 8);
  }
  __syncwarp();
  uint32_t cnt = 0, acc = lane;
  for (uint32_t p = 0; p < npair; ++p) {
    const uint32_t slot = p % SLOTS;
    mbar_wait(mbar + slot * 8, (p / SLOTS) & 1);
    uint4 v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) v[j] = lds4(ring + slot * 2048 + j * 512 + lane * 16);
    uint32_t m = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      m |= (fabsf(__uint_as_float(v[j].x)) >= thr ? 1u : 0u) << (4 * j);
      m |= (fabsf(__uint_as_float(v[j].y)) >= thr ? 2u : 0u) << (4 * j);
      m |= (fabsf(__uint_as_float(v[j].z)) >= thr ? 4u : 0u) << (4 * j);
      m |= (fabsf(__uint_as_float(v[j].w)) >= thr ? 8u : 0u) << (4 * j);
    }
    __syncwarp();
    if (lane == 0 && p + SLOTS < npair) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      bulk_load(ring + slot * 2048, ux + (size_t)(p + SLOTS) * 512, 2048, mbar + slot * 8);
    }
    cnt += __popc(__ballot_sync(0xffffffffu, m != 0));
#pragma unroll
    for (int e = 0; e < EXTRA; ++e) acc = acc * 1664525u + (m ^ (uint32_t)e);  // stand-in for per-step work
  }
  if (acc == 0x12345678u) out[1] = acc;
  if (lane == 0) atomicAdd(out, cnt);
}

template <int THREADS, int SLOTS, int EXTRA>
static void run(const float* x, size_t n, unsigned* out, int grid) {
  const size_t smem = (size_t)(THREADS / 32) * SLOTS * (2048 + 8) + 64;
  cudaFuncSetAttribute(stream_kernel<THREADS, SLOTS, EXTRA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 8; ++r) {
    cudaEventRecord(a);
    stream_kernel<THREADS, SLOTS, EXTRA><<<grid, THREADS, smem>>>(x, n, 2.58f, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (r >= 2 && ms < best) best = ms;
  }
  const cudaError_t e = cudaGetLastError();
  printf("threads %4d slots %d extra %3d smem %6zu KB: %8.1f us  %7.1f GB/s (%5.1f GB/s per SM) %s\n", THREADS, SLOTS,
         EXTRA, smem / 1024, best * 1e3, n * 4.0 / (best * 1e-3) / 1e9, n * 4.0 / (best * 1e-3) / 1e9 / grid,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  const size_t n = 64ull * 256 * 56 * 56;  // the bench's largest boundary, 205 MB fp32
  float* x;
  unsigned* out;
  cudaMalloc(&x, n * 4);
  cudaMalloc(&out, 16);
  cudaMemset(x, 0x3f, n * 4);
  for (int grid : {24, 148}) {
    printf("-- grid %d\n", grid);
    run<1024, 2, 0>(x, n, out, grid);
    run<1024, 2, 100>(x, n, out, grid);
    run<1024, 2, 200>(x, n, out, grid);
    run<512, 4, 0>(x, n, out, grid);
    run<512, 4, 100>(x, n, out, grid);
    run<512, 4, 200>(x, n, out, grid);
    run<512, 2, 0>(x, n, out, grid);
    run<512, 2, 200>(x, n, out, grid);
    run<1024, 3, 0>(x, n, out, grid);
    run<1024, 3, 200>(x, n, out, grid);
  }
  return 0;
}
