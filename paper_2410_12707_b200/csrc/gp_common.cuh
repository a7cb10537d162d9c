// gp_common.cuh — shared device helpers for the AdaTopK kernels (sm_100a).
//
// Selection total order (reference: compressor.py:91-93, np.argsort(-|x|,
// kind="stable")): +-inf > finite by |x| (denormals exact) > +-0 > NaN, every
// tie to the lower index.  It is realised as an unsigned integer key per
// element, compared as an integer, never as a float:
//     key = isnan(x) ? 0 : (bits(x) & ~sign) + 1
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace gp {

constexpr uint32_t kFull = 0xFFFFFFFFu;

// ---------------------------------------------------------------------------
// dtype traits.  `Bits` is the raw element bit pattern, `Key` the rank key.

struct TraitsF32 {
  using Elem = uint32_t;
  using Bits = uint32_t;
  using Key = uint32_t;
  static constexpr int kVec = 4;        // elements per 16-byte load
  static constexpr int kKeyBits = 31;   // significant key bits (key <= 0x7F800001)
  __device__ __forceinline__ static Key key(Bits b) {
    const uint32_t a = b & 0x7FFFFFFFu;
    return a > 0x7F800000u ? 0u : a + 1u;
  }
  __device__ __forceinline__ static float to_f32(Bits b) { return __uint_as_float(b); }
  __device__ __forceinline__ static Bits lane(const uint4& v, int e) {
    return e == 0 ? v.x : e == 1 ? v.y : e == 2 ? v.z : v.w;
  }
};

// bf16: the key of the exact fp32 upcast (bits << 16), so bf16 selection is the
// reference applied to x.float() (SURVEY.md §7 hard part 5).
struct TraitsBF16 {
  using Elem = uint16_t;
  using Bits = uint32_t;
  using Key = uint32_t;
  static constexpr int kVec = 8;
  static constexpr int kKeyBits = 31;
  __device__ __forceinline__ static Key key(Bits b) {
    const uint32_t a = b & 0x7FFFu;
    return a > 0x7F80u ? 0u : (a << 16) + 1u;
  }
  __device__ __forceinline__ static float to_f32(Bits b) { return __uint_as_float(b << 16); }
  __device__ __forceinline__ static Bits lane(const uint4& v, int e) {
    const uint32_t w = (e >> 1) == 0 ? v.x : (e >> 1) == 1 ? v.y : (e >> 1) == 2 ? v.z : v.w;
    return (e & 1) ? (w >> 16) : (w & 0xFFFFu);
  }
};

struct TraitsF64 {
  using Elem = uint64_t;
  using Bits = uint64_t;
  using Key = uint64_t;
  static constexpr int kVec = 2;
  static constexpr int kKeyBits = 63;
  __device__ __forceinline__ static Key key(Bits b) {
    const uint64_t a = b & 0x7FFFFFFFFFFFFFFFull;
    return a > 0x7FF0000000000000ull ? 0ull : a + 1ull;
  }
  __device__ __forceinline__ static float to_f32(Bits b) {
    return __double2float_rn(__longlong_as_double((long long)b));
  }
  __device__ __forceinline__ static Bits lane(const uint4& v, int e) {
    return e == 0 ? ((uint64_t)v.y << 32 | v.x) : ((uint64_t)v.w << 32 | v.z);
  }
};

// ---------------------------------------------------------------------------
// warp / memory primitives

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__device__ __forceinline__ uint4 ld_stream_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void red_add_gpu(uint32_t* p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

template <typename T>
__device__ __forceinline__ T ldcg(const T* p) { return __ldcg(p); }

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
  const uint32_t lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  return x;
}

__device__ __forceinline__ uint32_t warp_sum(uint32_t x) { return __reduce_add_sync(kFull, x); }

// Grid-wide barrier for a cooperative (co-resident) launch.  Self-resetting:
// the arrival counter returns to 0 and the generation word only increases, so
// the workspace needs no per-call reset.  Same fence pattern as
// cooperative_groups' grid.sync().
__device__ __forceinline__ void grid_barrier(uint32_t* count, uint32_t* gen, uint32_t nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t g = ld_acquire_gpu(gen);
    __threadfence();
    const uint32_t arrived = atomicAdd(count, 1u);
    if (arrived == nblocks - 1) {
      atomicExch(count, 0u);
      __threadfence();
      st_release_gpu(gen, g + 1);
    } else {
      while (ld_acquire_gpu(gen) == g) { __nanosleep(32); }
    }
    __threadfence();
  }
  __syncthreads();
}

}  // namespace gp
