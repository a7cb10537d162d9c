// gp_common.cuh — shared device helpers for the AdaTopK kernels (sm_100a).
//
// Selection total order (reference: compressor.py:91-93, np.argsort(-|x|,
// kind="stable")): +-inf > finite by |x| (denormals exact) > +-0 > NaN, every
// tie to the lower index.  It is realised as an unsigned integer key per
// element, compared as an integer, never as a float:
//     key = isnan(x) ? 0 : (bits(x) & ~sign) + 1
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace gp {

constexpr uint32_t kFull = 0xFFFFFFFFu;

// Checked build (-DGP_CHECKED, the `checked` library variant): device-side
// bounds and invariant checks that trap with the failing condition -- the
// stand-in for compute-sanitizer, which this GPU pool does not allow.  No-ops
// in the product build.
#ifdef GP_CHECKED
#define GP_CHECK(c)                                                                        \
  do {                                                                                     \
    if (!(c)) {                                                                            \
      printf("GP_CHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__,         \
             (int)blockIdx.x, (int)threadIdx.x, #c);                                       \
      __trap();                                                                            \
    }                                                                                      \
  } while (0)
#else
#define GP_CHECK(c) \
  do {              \
  } while (0)
#endif

// ---------------------------------------------------------------------------
// dtype traits.  `Bits` is the raw element bit pattern, `Key` the rank key.

struct TraitsF32 {
  using Elem = uint32_t;
  using Bits = uint32_t;
  using Key = uint32_t;
  static constexpr int kVec = 4;        // elements per 16-byte load
  static constexpr int kKeyBits = 31;   // significant key bits (key <= 0x7F800001)
  static constexpr int kExpBits = 8;
  static constexpr bool kDirectT = false;  // key bits below the fine bin vary
  static constexpr Key kInfAbs = 0x7F800000u;  // |inf| in key space; abs > kInfAbs is NaN
  __device__ __forceinline__ static Key abs_bits(Bits b) { return b & 0x7FFFFFFFu; }
  // key(b) >= lo_m1 + 1 (lo_m1 <= |inf| bits), as one |x| >= thr float compare; NaN -> false
  struct Cand {
    float thr;
    __device__ __forceinline__ bool operator()(Bits b) const { return fabsf(__uint_as_float(b)) >= thr; }
  };
  __device__ __forceinline__ static Cand make_cand(Key lo_m1) { return Cand{__uint_as_float(lo_m1)}; }
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
  static constexpr int kExpBits = 8;
  static constexpr bool kDirectT = true;  // 16-bit fine bin = the whole bf16 value
  static constexpr Key kInfAbs = 0x7F800000u;
  __device__ __forceinline__ static Key abs_bits(Bits b) { return (b & 0x7FFFu) << 16; }
  // key >= lo_m1 + 1  <=>  ceil(lo_m1 / 2^16) <= |bits16| <= |inf|  (NaN excluded)
  struct Cand {
    uint32_t t16, span16;
    __device__ __forceinline__ bool operator()(Bits b) const { return ((b & 0x7FFFu) - t16) <= span16; }
  };
  __device__ __forceinline__ static Cand make_cand(Key lo_m1) {
    const uint32_t t16 = (lo_m1 + 0xFFFFu) >> 16;
    return Cand{t16, 0x7F80u - t16};
  }
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
  static constexpr int kExpBits = 11;
  static constexpr bool kDirectT = false;
  static constexpr Key kInfAbs = 0x7FF0000000000000ull;
  __device__ __forceinline__ static Key abs_bits(Bits b) { return b & 0x7FFFFFFFFFFFFFFFull; }
  struct Cand {
    double thr;
    __device__ __forceinline__ bool operator()(Bits b) const { return fabs(__longlong_as_double((long long)b)) >= thr; }
  };
  __device__ __forceinline__ static Cand make_cand(Key lo_m1) { return Cand{__longlong_as_double((long long)lo_m1)}; }
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

__device__ __forceinline__ uint32_t sub_sat(uint32_t a, uint32_t b) { return a > b ? a - b : 0u; }

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

// ---- bulk (TMA) global->shared copies completed on an mbarrier
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
// orders this thread's (and, after a warp/CTA barrier, its peers') generic
// shared-memory accesses before later async-proxy (bulk copy) writes
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bulk_load_async(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                                uint64_t policy) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(policy)
      : "memory");
}
// ---- bulk (TMA) shared->global stores, tracked by bulk async-groups
__device__ __forceinline__ void bulk_store_async(void* dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_store_async_hint(void* dst, uint32_t src, uint32_t bytes, uint64_t policy) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst), "r"(src),
               "r"(bytes), "l"(policy)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// at most N committed groups still reading their shared-memory source
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
// every committed group complete (writes performed)
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// evict_last: lines written now and re-read after a grid barrier outlive the
// normal-priority traffic of other streams' copies (non-volatile: hoistable)
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void st_global_v2_hint(void* ptr, uint32_t a, uint32_t b, uint64_t policy) {
  asm volatile("st.global.L2::cache_hint.v2.u32 [%0], {%1, %2}, %3;" ::"l"(ptr), "r"(a), "r"(b), "l"(policy) : "memory");
}
__device__ __forceinline__ void st_global_v4_hint(void* ptr, uint4 v, uint64_t policy) {
  asm volatile("st.global.L2::cache_hint.v4.u32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(ptr), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w), "l"(policy)
               : "memory");
}
// drop a dead 128-byte line from L2 without writing it back
__device__ __forceinline__ void discard_l2_line(const void* ptr) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(ptr) : "memory");
}
// ---- per-thread async copies (cp.async / LDGSTS): 16 bytes global -> shared,
// tracked by per-thread commit groups
__device__ __forceinline__ void cp_async16_hint(uint32_t dst, const void* src, uint64_t policy) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "l"(policy)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
// at most N of this thread's committed groups still in flight
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ uint4 ld_shared_v4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x) {
  const uint32_t lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  return x;
}

__device__ __forceinline__ uint64_t warp_incl_scan64(uint64_t x) {
  const uint32_t lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  return x;
}

__device__ __forceinline__ uint32_t warp_sum(uint32_t x) { return __reduce_add_sync(kFull, x); }

__device__ __forceinline__ uint32_t atom_add_release_gpu(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// Grid-wide barrier for a cooperative (co-resident) launch, one atomic per CTA.
// CTA 0 adds 0x80000000 - (G-1), every other CTA adds 1, so the word's top bit
// flips exactly when the last CTA arrives and the low bits return to their
// previous value: self-resetting, nothing to clear between launches.
// After it, data written by other CTAs before their arrival may be read with
// plain (weak) loads: the acquire fence invalidates this SM's L1.
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

__device__ __forceinline__ void grid_barrier(uint32_t* word, uint32_t nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t inc = blockIdx.x == 0 ? 0x80000000u - (nblocks - 1u) : 1u;
    fence_acq_rel_gpu();
    const uint32_t old = atom_add_release_gpu(word, inc);
    while (((old ^ ld_acquire_gpu(word)) & 0x80000000u) == 0u) {
    }
    fence_acq_rel_gpu();
  }
  __syncthreads();
}

}  // namespace gp
