// gp_cluster.cu — AdaTopK compress of a short vector by ONE thread-block
// cluster (sm_100a).
//
// Same contract as compress_kernel (reference: pkg/src/geopipe/compressor.py:
// 79-94, `np.argsort(-np.abs(flat), kind="stable")[:k]`, kept indices in
// ascending order; the integer key of gp_common.cuh, ties to the lower index),
// for vectors that fit in the shared memory of one cluster (up to 8 CTAs x
// 192 KiB: 393,216 fp32 / 786,432 bf16 / 196,608 fp64 elements).
//
// The cooperative kernel's latency floor on short vectors is its chain of grid
// barriers through L2 (~20 us cold whatever the length or ratio).  On B200
// (scripts/cluster_probe.py, each launch after an L2 flush) this kernel takes
// 12-15 us for up to 64K fp32 elements and 16-20 us at 128K, against 20-24 us;
// warm, the cooperative grid is level from ~128K elements on, so the default
// routing sends vectors of up to 98,304 elements here.  A 16-CTA
// (non-portable) cluster costs ~10 us more than an 8-CTA one, so clusters are
// capped at 8 CTAs (GP_CL_MAX_CTAS).  Here the
// vector is read from HBM exactly once into the CTAs' shared memory and every
// later pass runs over that copy; the CTAs exchange histograms through
// distributed shared memory and synchronise with cluster barriers:
//
//   load      each CTA copies its contiguous slice (cp.async, 16 B per lane)
//   select    radix select of the k-th largest key, 11-bit digits from the top
//             (3 passes for 32-bit keys, 6 for fp64): every CTA histograms the
//             digit of its keys still matching the prefix, one cluster
//             barrier, then one warp per CTA finds the crossing over the
//             cluster (DSMEM loads: 32-bin group sums, then the bins of one
//             group; every CTA computes the same result, no second barrier)
//             -> threshold key T and the tie quota q (T-keys to keep).  Pass 1
//             also lists the keys of pass 0's bin (16 KiB of smem) and counts
//             per warp the keys above it, so the later passes read the list
//             (a CTA whose list overflows scans its slice instead)
//   count     per warp segment: keys > T and keys == T (from the list when it
//             is complete); CTA totals published, one cluster barrier, each
//             CTA sums the earlier CTAs' totals
//   write     output position of a kept element = (#keys > T before it) +
//             min(q, #keys == T before it): one packed warp scan per step
//
// No workspace is touched, so the C-ABI's zeroed-workspace contract holds.
#include <atomic>
#include <cstdlib>
#include <cooperative_groups.h>

#include "gp_kernels.cuh"

namespace gp {
namespace cg = cooperative_groups;

constexpr int kClThreads = 1024;
constexpr int kClDigitBits = 11;
constexpr int kClBins = 1 << kClDigitBits;
constexpr uint32_t kClDataBytes = 192u * 1024u;  // the resident slice of the vector
constexpr uint32_t kClListBytes = 16u * 1024u;   // pass-1 list: (slice index, bits) of the keys in the top bin
constexpr uint32_t kClSmallBytes = (2u * kClBins + 64u + 16u + 64u + 4u + 32u + 128u) * 4u;
constexpr uint32_t kClSmemBytes = kClDataBytes + kClListBytes + kClSmallBytes;
constexpr int kClMaxCtas = 16;  // DSMEM reduction width (a 16-CTA cluster only with GP_CL_MAX_CTAS=16)
#ifndef GP_CL_MAX_CTAS
#define GP_CL_MAX_CTAS 8
#endif
#ifndef GP_CL_MIN_PER_CTA
#define GP_CL_MIN_PER_CTA 8192
#endif
constexpr uint32_t kClMinPerCta = GP_CL_MIN_PER_CTA;  // elements per CTA below which the cluster shrinks
#ifndef GP_CL_AUTO_MAX
#define GP_CL_AUTO_MAX 98304
#endif
constexpr uint32_t kClAutoMax = GP_CL_AUTO_MAX;  // default routing: vectors up to this many elements

namespace {

__device__ __forceinline__ void cluster_arrive_release() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acquire() {
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <class Tr>
__device__ __forceinline__ void cl_write_out(const CompressArgs& a, void* val_out, uint32_t pos, uint32_t idx,
                                             typename Tr::Bits b) {
  using Elem = typename Tr::Elem;
  if (a.idx64) reinterpret_cast<int64_t*>(a.idx_out)[pos] = (int64_t)idx;
  else reinterpret_cast<int32_t*>(a.idx_out)[pos] = (int32_t)idx;
  if (a.val_f32) reinterpret_cast<float*>(val_out)[pos] = Tr::to_f32(b);
  else reinterpret_cast<Elem*>(val_out)[pos] = (Elem)b;
  if (a.val2_out) reinterpret_cast<Elem*>(a.val2_out)[pos] = (Elem)b;
}

template <class Tr>
__device__ __forceinline__ typename Tr::Bits cl_elem_bits(const typename Tr::Elem* p, uint32_t i) {
  return (typename Tr::Bits)p[i];
}

__device__ __forceinline__ unsigned long long cl_globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

}  // namespace

// optional per-CTA stage timestamps (development aid; a.dbg is null in production)
#define CL_STAMP(i)                                                                              \
  do {                                                                                           \
    if (a.dbg != nullptr && tid == 0 && (i) < 32) a.dbg[(size_t)c * 32 + (i)] = cl_globaltimer(); \
  } while (0)

// grid = one cluster of gridDim.x CTAs; CTA c owns elements [c*C, min(d, (c+1)*C)),
// C a multiple of 16 elements.
template <class Tr>
__global__ void __launch_bounds__(kClThreads, 1) compress_cluster_kernel(const CompressArgs a, uint32_t C) {
  using Bits = typename Tr::Bits;
  using Key = typename Tr::Key;
  using Elem = typename Tr::Elem;
  constexpr int EPS = 16 / (int)sizeof(Elem);  // elements per 16-byte vector
  constexpr int KB = Tr::kKeyBits;              // keys are < 2^KB
  constexpr int NP = (KB + kClDigitBits - 1) / kClDigitBits;

  constexpr uint32_t kListCap = kClListBytes / (4u + (uint32_t)sizeof(Bits));

  extern __shared__ __align__(16) unsigned char smem[];
  Bits* lbits = reinterpret_cast<Bits*>(smem + kClDataBytes);              // list: bits, then slice indices
  uint32_t* lidx = reinterpret_cast<uint32_t*>(smem + kClDataBytes + kListCap * sizeof(Bits));
  uint32_t* hbuf = reinterpret_cast<uint32_t*>(smem + kClDataBytes + kClListBytes);  // 2 x kClBins (pass parity)
  uint32_t* res = hbuf + 2 * kClBins + 64;                            // 16 (res[8]: list length)
  uint32_t* wcnt = res + 16;                                          // per-warp (>T, ==T) counts
  uint32_t* ccnt = wcnt + 64;                                         // this CTA's totals (read remotely)
  uint32_t* wabv = ccnt + 4;                                          // per warp: keys above pass 1's bin
  uint32_t* gbuf = wabv + 32;                                         // 2 x 64 group sums (pass parity)
  const uint32_t xs = smem_addr(smem);

  cg::cluster_group cl = cg::this_cluster();
  const uint32_t c = blockIdx.x, nc = gridDim.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t d = a.d;
  uint32_t k = a.k;
  void* val_out = a.val_out;
  if (a.k_dev != nullptr) {  // device-resident k: the same checks as compress_kernel
    const long long kk = __ldg(a.k_dev);
    if (kk < 1 || kk > (long long)a.k || kk > (long long)d) {
      if (c == 0 && tid == 0) {
        if (a.err != nullptr) atomicOr(a.err, kFlagBadK);
        if (a.header != nullptr) {
          a.header[0] = (unsigned long long)d;
          a.header[1] = ~0ull;
        }
      }
      return;  // every CTA reads the same k: none reaches a cluster barrier
    }
    k = (uint32_t)kk;
    if (a.frame_vals) val_out = reinterpret_cast<unsigned char*>(a.idx_out) + (a.idx64 ? 8ull : 4ull) * k;
  }
  CL_STAMP(0);
  if (a.header != nullptr && c == 0 && tid == 0) {
    a.header[0] = (unsigned long long)d;
    a.header[1] = (unsigned long long)k;
  }

  // ---- load: this CTA's slice into shared memory (HBM read exactly once)
  const uint32_t i0 = c * C;
  const uint32_t n = i0 < d ? min(C, d - i0) : 0u;
  const Elem* src = reinterpret_cast<const Elem*>(a.x) + i0;
  const uint32_t nbytes = n * (uint32_t)sizeof(Elem);
  uint32_t first_scalar = 0;
  if ((reinterpret_cast<uintptr_t>(src) & 15u) == 0u) {
    const uint64_t policy = l2_evict_first_policy();  // read once
    for (uint32_t o = tid * 16u; o + 16u <= nbytes; o += kClThreads * 16u)
      cp_async16_hint(xs + o, reinterpret_cast<const unsigned char*>(src) + o, policy);
    cp_async_commit();
    first_scalar = (nbytes / 16u) * 16u / (uint32_t)sizeof(Elem);
  }
  Elem* xe = reinterpret_cast<Elem*>(smem);
  for (uint32_t i = first_scalar + tid; i < n; i += kClThreads) xe[i] = src[i];
  for (uint32_t i = tid; i < 2u * kClBins; i += kClThreads) hbuf[i] = 0u;
  if (tid == 0) res[8] = 0u;
  cp_async_wait<0>();
  __syncthreads();
  CL_STAMP(1);

  const uint32_t nfull = n / EPS;                // complete 16-byte vectors
  const uint32_t nv = (n + EPS - 1) / EPS;       // vectors, the last one possibly partial
  const uint32_t nlast = n - (nv ? nv - 1 : 0u) * EPS;
  // warp segments (contiguous vectors, index order) of pass 1, the count and the write
  const uint32_t S = (nv + 31u) / 32u;
  const uint32_t v0 = min(nv, w * S), v1 = min(nv, v0 + S);
  bool list_ok = false;  // pass 1's list holds every key of its bin (this CTA)

  // ---- radix select: T = the k-th largest key over the cluster, q = T-keys to keep
  Key P = 0;
  uint32_t kr = k;
#pragma unroll 1
  for (int p = 0; p < NP; ++p) {
    const int hi = KB - p * kClDigitBits;
    const int lo = hi > kClDigitBits ? hi - kClDigitBits : 0;
    const int width = hi - lo;
    const uint32_t mask = (1u << width) - 1u;
    uint32_t* h = hbuf + (p & 1) * kClBins;
    if (p >= 2) {  // every CTA's reads of this buffer (pass p-2) ended before the last cluster barrier
      for (uint32_t i = tid; i < (uint32_t)kClBins; i += kClThreads) h[i] = 0u;
      __syncthreads();
    }
    auto add = [&](Bits b) {
      const Key kk = Tr::key(b);
      if ((kk >> hi) == P) atomicAdd(&h[(uint32_t)(kk >> lo) & mask], 1u);
    };
    if (p == 1) {
      // pass 1, over the warp segments: the keys of pass 0's bin are also
      // listed (their number is small unless the bin is crowded), and each
      // warp counts its keys above the bin (all > T); later passes and the
      // count then read the list instead of the slice
      uint32_t abv = 0;
      // the bin is [lo_in, hi_in) in key space; when both edges are finite
      // non-zero keys each test is one |x| >= threshold compare (Tr::Cand, NaN
      // false), else the integer key is computed (warp-uniform choice)
      const Key lo_in = P << hi, hi_in = (P + 1) << hi;
      const bool fast = lo_in >= 1 && hi_in - 1 <= Tr::kInfAbs;
      const typename Tr::Cand c_lo = Tr::make_cand(fast ? lo_in - 1 : (Key)0);
      const typename Tr::Cand c_hi = Tr::make_cand(fast ? hi_in - 1 : (Key)0);
      for (uint32_t v = v0 + lane; v < v1; v += 32u) {
        const uint4 q4 = ld_shared_v4(xs + v * 16u);
        const uint32_t ne = v + 1u == nv ? nlast : (uint32_t)EPS;
        uint32_t m = 0;  // keys of the bin: rare, handled below without per-element branches
        if (fast) {
#pragma unroll
          for (int e = 0; e < EPS; ++e) {
            const Bits b = Tr::lane(q4, e);
            const bool valid = (uint32_t)e < ne, above = c_hi(b);
            m |= (uint32_t)(valid && !above && c_lo(b)) << e;
            abv += (uint32_t)(valid && above);
          }
        } else {
#pragma unroll
          for (int e = 0; e < EPS; ++e) {
            const Key top = Tr::key(Tr::lane(q4, e)) >> hi;
            const bool valid = (uint32_t)e < ne;
            m |= (uint32_t)(valid && top == P) << e;
            abv += (uint32_t)(valid && top > P);
          }
        }
        while (m) {  // one list slot per key (a per-warp reservation measured 2x slower)
          const int e = __ffs(m) - 1;
          m &= m - 1;
          const Bits b = Tr::lane(q4, e);
          atomicAdd(&h[(uint32_t)(Tr::key(b) >> lo) & mask], 1u);
          const uint32_t j = atomicAdd(&res[8], 1u);
          if (j < kListCap) {
            lbits[j] = b;
            lidx[j] = v * (uint32_t)EPS + (uint32_t)e;
          }
        }
      }
      abv = warp_sum(abv);
      if (lane == 0) wabv[w] = abv;
    } else if (p >= 2 && list_ok) {
      const uint32_t nl = res[8];
      for (uint32_t j = tid; j < nl; j += kClThreads) add(lbits[j]);
    } else if (p == 0) {  // every key matches the empty prefix: no test, no branch
      for (uint32_t v = tid; v < nfull; v += kClThreads) {
        const uint4 q4 = ld_shared_v4(xs + v * 16u);
#pragma unroll
        for (int e = 0; e < EPS; ++e) atomicAdd(&h[(uint32_t)(Tr::key(Tr::lane(q4, e)) >> lo) & mask], 1u);
      }
      if (tid < n - nfull * EPS) add(cl_elem_bits<Tr>(xe, nfull * EPS + tid));
    } else {
      for (uint32_t v = tid; v < nfull; v += kClThreads) {
        const uint4 q4 = ld_shared_v4(xs + v * 16u);
#pragma unroll
        for (int e = 0; e < EPS; ++e) add(Tr::lane(q4, e));
      }
      if (tid < n - nfull * EPS) add(cl_elem_bits<Tr>(xe, nfull * EPS + tid));
    }
    // group sums (32 bins each) for the two-level cluster reduction below
    const uint32_t NB = 1u << width, NG = NB / 32u;  // NB >= 256: 8..64 groups
    uint32_t* gs = gbuf + (p & 1) * 64u;
    __syncthreads();
    for (uint32_t g = w; g < NG; g += 32u) {
      const uint32_t t = warp_sum(h[g * 32u + lane]);
      if (lane == 0) gs[g] = t;
    }
    CL_STAMP(2 + 3 * p);
    cl.sync();
    CL_STAMP(3 + 3 * p);
    if (p == 1) list_ok = res[8] <= kListCap;  // final: the cluster barrier ordered every append
    // warp 0 finds the crossing: the group over the cluster's group sums (DSMEM,
    // lane l owns groups NG-1-2l, NG-2-2l), then the bin inside that group (lane l
    // owns bin 31-l of it); every CTA computes the same result, no second barrier
    if (w == 0) {
      uint32_t g0 = 0, g1 = 0;  // groups a = NG-1-2l (higher), b = a-1
      const bool own = 2u * lane < NG;
      if (own) {
        uint2 v[kClMaxCtas];
        const uint32_t gb = NG - 2u - 2u * lane;
#pragma unroll
        for (int r = 0; r < kClMaxCtas; ++r)
          v[r] = (uint32_t)r < nc ? *reinterpret_cast<const uint2*>(cl.map_shared_rank(gs + gb, r)) : make_uint2(0u, 0u);
#pragma unroll
        for (int r = 0; r < kClMaxCtas; ++r) {
          g1 += v[r].x;
          g0 += v[r].y;
        }
      }
      const uint32_t incl = warp_incl_scan(g0 + g1);
      const uint32_t ex = incl - (g0 + g1);
      uint32_t hit = 0, gabove = 0, grp = 0;
      if (own) {
        if (ex < kr && kr <= ex + g0) {
          hit = 1u;
          grp = NG - 1u - 2u * lane;
          gabove = ex;
        } else if (ex + g0 < kr && kr <= ex + g0 + g1) {
          hit = 1u;
          grp = NG - 2u - 2u * lane;
          gabove = ex + g0;
        }
      }
      const uint32_t hb = __ballot_sync(kFull, hit != 0u);
      GP_CHECK(__popc(hb) == 1);
      const int src = __ffs(hb) - 1;
      grp = __shfl_sync(kFull, grp, src);
      gabove = __shfl_sync(kFull, gabove, src);
      const uint32_t bin = grp * 32u + 31u - lane;
      uint32_t hv[kClMaxCtas];
#pragma unroll
      for (int r = 0; r < kClMaxCtas; ++r) hv[r] = (uint32_t)r < nc ? *cl.map_shared_rank(h + bin, r) : 0u;
      uint32_t hs = 0;
#pragma unroll
      for (int r = 0; r < kClMaxCtas; ++r) hs += hv[r];
      const uint32_t bi = warp_incl_scan(hs);
      const uint32_t bex = gabove + bi - hs;
      if (bex < kr && kr <= bex + hs) {
        res[0] = bin;
        res[1] = bex;
      }
    }
    __syncthreads();
    P = (P << width) | (Key)res[0];
    kr -= res[1];
    CL_STAMP(4 + 3 * p);
    GP_CHECK(kr >= 1u);
  }
  const Key T = P;
  const uint32_t q = kr;  // keys equal to T that are kept: the q lowest-indexed ones

  // ---- count: per warp segment (contiguous vectors, index order) keys > T and == T
  if (list_ok) {
    // keys > T: those above pass 1's bin (counted there) and the listed ones
    // above T; keys == T are all listed
    if (tid < 32) {
      wcnt[tid] = wabv[tid];
      wcnt[32 + tid] = 0u;
    }
    __syncthreads();
    const uint32_t nl = res[8];
    for (uint32_t j = tid; j < nl; j += kClThreads) {
      const Key kk = Tr::key(lbits[j]);
      const uint32_t ws = (lidx[j] / (uint32_t)EPS) / S;  // the warp segment holding the entry
      if (kk > T) atomicAdd(&wcnt[ws], 1u);
      else if (kk == T) atomicAdd(&wcnt[32 + ws], 1u);
    }
    __syncthreads();
    if (w == 0) {
      const uint32_t g = wcnt[lane], e = wcnt[32 + lane];
      const uint32_t gi = warp_incl_scan(g), ei = warp_incl_scan(e);
      wcnt[lane] = gi - g;
      wcnt[32 + lane] = ei - e;
      if (lane == 31) {
        ccnt[0] = gi;
        ccnt[1] = ei;
      }
    }
  } else {
    uint32_t gt = 0, eq = 0;
    for (uint32_t v = v0 + lane; v < v1; v += 32u) {
      const uint4 q4 = ld_shared_v4(xs + v * 16u);
      const uint32_t ne = v + 1u == nv ? nlast : (uint32_t)EPS;
#pragma unroll
      for (int e = 0; e < EPS; ++e) {
        const Key kk = Tr::key(Tr::lane(q4, e));
        if ((uint32_t)e < ne) {
          gt += kk > T;
          eq += kk == T;
        }
      }
    }
    gt = warp_sum(gt);
    eq = warp_sum(eq);
    if (lane == 0) {
      wcnt[w] = gt;
      wcnt[32 + w] = eq;
    }
    __syncthreads();
    if (w == 0) {
      const uint32_t g = wcnt[lane], e = wcnt[32 + lane];
      const uint32_t gi = warp_incl_scan(g), ei = warp_incl_scan(e);
      wcnt[lane] = gi - g;
      wcnt[32 + lane] = ei - e;
      if (lane == 31) {
        ccnt[0] = gi;
        ccnt[1] = ei;
      }
    }
  }
  CL_STAMP(20);
  cl.sync();
  CL_STAMP(21);
  if (w == 0) {  // the earlier CTAs' totals
    uint32_t g = 0, e = 0;
    if (lane < c) {
      const uint32_t* rc = cl.map_shared_rank(ccnt, lane);
      g = rc[0];
      e = rc[1];
    }
    g = warp_sum(g);
    e = warp_sum(e);
    if (lane == 0) {
      res[4] = g;
      res[5] = e;
    }
  }
  cluster_arrive_release();  // this CTA's remote reads are done; it waits before exiting
  __syncthreads();
  CL_STAMP(23);

  // ---- write: kept (index, value) pairs in index order; two 32-vector steps
  // per iteration, so their load -> scan -> store chains overlap
  uint32_t gtb = res[4] + wcnt[w], eqb = res[5] + wcnt[32 + w];
  // key > T as one |x| >= threshold compare and key == T as abs-bits == T - 1
  // when T is a finite non-zero key (warp-uniform), else the integer key
  const bool fastw = T >= 1 && T <= Tr::kInfAbs;
  const typename Tr::Cand c_gt = Tr::make_cand(fastw ? T : (Key)0);
  const Key tm1 = T - 1;
  auto masks = [&](uint32_t v, uint4& q4, uint32_t& gm, uint32_t& em) {
    gm = 0u;
    em = 0u;
    q4 = make_uint4(0u, 0u, 0u, 0u);
    if (v < v1) {
      q4 = ld_shared_v4(xs + v * 16u);
      const uint32_t ne = v + 1u == nv ? nlast : (uint32_t)EPS;
      if (fastw) {
#pragma unroll
        for (int e = 0; e < EPS; ++e) {
          const Bits b = Tr::lane(q4, e);
          const bool valid = (uint32_t)e < ne;
          gm |= (uint32_t)(valid && c_gt(b)) << e;
          em |= (uint32_t)(valid && Tr::abs_bits(b) == tm1) << e;
        }
      } else {
#pragma unroll
        for (int e = 0; e < EPS; ++e) {
          const Key kk = Tr::key(Tr::lane(q4, e));
          const bool valid = (uint32_t)e < ne;
          gm |= (uint32_t)(valid && kk > T) << e;
          em |= (uint32_t)(valid && kk == T) << e;
        }
      }
    }
  };
  auto emit = [&](uint32_t v, const uint4& q4, uint32_t gm, uint32_t em, uint32_t g, uint32_t e2) {
    const uint32_t base = i0 + v * (uint32_t)EPS;
    uint32_t all = gm | em;  // in index order; a tie is kept while its rank is below q
    while (all) {
      const int e = __ffs(all) - 1;
      all &= all - 1;
      if ((gm >> e) & 1u) {
        const uint32_t pos = g + min(q, e2);
        GP_CHECK(pos < k);
        cl_write_out<Tr>(a, val_out, pos, base + e, Tr::lane(q4, e));
        ++g;
      } else {
        if (e2 < q) {
          GP_CHECK(g + e2 < k);
          cl_write_out<Tr>(a, val_out, g + e2, base + e, Tr::lane(q4, e));
        }
        ++e2;
      }
    }
  };
  for (uint32_t vb = v0; vb < v1; vb += 64u) {
    const uint32_t va = vb + lane, vc = vb + 32u + lane;
    uint4 qa, qc;
    uint32_t ga, ea, gc, ec;
    masks(va, qa, ga, ea);
    masks(vc, qc, gc, ec);
    if (!__any_sync(kFull, (ga | ea | gc | ec) != 0u)) continue;  // nothing kept or tied in either step
    const uint32_t pa = (uint32_t)__popc(ga) | ((uint32_t)__popc(ea) << 16);
    const uint32_t pc = (uint32_t)__popc(gc) | ((uint32_t)__popc(ec) << 16);
    const uint32_t ia = warp_incl_scan(pa), ic = warp_incl_scan(pc);
    const uint32_t ta = __shfl_sync(kFull, ia, 31), tc = __shfl_sync(kFull, ic, 31);
    if (ga | ea) emit(va, qa, ga, ea, gtb + ((ia - pa) & 0xFFFFu), eqb + ((ia - pa) >> 16));
    gtb += ta & 0xFFFFu;
    eqb += ta >> 16;
    if (gc | ec) emit(vc, qc, gc, ec, gtb + ((ic - pc) & 0xFFFFu), eqb + ((ic - pc) >> 16));
    gtb += tc & 0xFFFFu;
    eqb += tc >> 16;
  }
  CL_STAMP(22);
  cluster_wait_acquire();  // no CTA leaves while another may still read its counts
}

// ---------------------------------------------------------------------------
// host side

static uint32_t env_u32(const char* name, uint32_t dflt) {  // development knobs
  const char* s = std::getenv(name);
  return (s != nullptr && s[0] >= '0' && s[0] <= '9') ? (uint32_t)std::strtoul(s, nullptr, 10) : dflt;
}

template <class Tr>
static int launch_cluster_t(const CompressArgs& a, const DeviceInfo& dev, cudaStream_t stream) {
  // per device: largest launchable cluster (GP_CL_MAX_CTAS, halved until one fits; 0 = none), found once
  static std::atomic<int> max_nc[kMaxDevices];
  if (dev.ordinal < 0 || dev.ordinal >= kMaxDevices) return -1;
  int mnc = max_nc[dev.ordinal].load(std::memory_order_acquire);
  if (mnc == 0) {
    mnc = -1;
    if (cudaFuncSetAttribute(compress_cluster_kernel<Tr>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kClSmemBytes) == cudaSuccess &&
        cudaFuncSetAttribute(compress_cluster_kernel<Tr>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) ==
            cudaSuccess) {
      const int want = (int)std::min<uint32_t>(kClMaxCtas, std::max<uint32_t>(1u, env_u32("GP_CL_MAX_CTAS", GP_CL_MAX_CTAS)));
      for (int nc = want; nc >= 1 && mnc < 0; nc /= 2) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(nc);
        cfg.blockDim = dim3(kClThreads);
        cfg.dynamicSmemBytes = kClSmemBytes;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = nc;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, compress_cluster_kernel<Tr>, &cfg) == cudaSuccess &&
            nclusters >= 1)
          mnc = nc;
      }
    }
    (void)cudaGetLastError();  // a refused probe leaves no sticky state
    max_nc[dev.ordinal].store(mnc, std::memory_order_release);
  }
  if (mnc < 0) return -1;
  uint32_t ncap = (uint32_t)mnc;
  if (dev.max_ctas > 0) ncap = std::min(ncap, (uint32_t)dev.max_ctas);
  constexpr uint32_t kCap = kClDataBytes / sizeof(typename Tr::Elem);  // elements per CTA
  if ((uint64_t)a.d > (uint64_t)ncap * kCap) return -1;
  static const uint32_t min_per_cta = std::max<uint32_t>(1u, env_u32("GP_CL_MIN_PER_CTA", kClMinPerCta));
  static const uint32_t short_rule = env_u32("GP_CL_NC_RULE", 1u);
  uint64_t want = std::max<uint64_t>(1, (a.d + min_per_cta - 1) / min_per_cta);
  // short vectors: up to 4 CTAs of >= 2048 elements (B200: 8K-32K elements
  // 1.5-2.5 us faster on 4 CTAs than on 1-2 of 8192)
  if (short_rule) want = std::max<uint64_t>(want, std::min<uint64_t>(4, (a.d + 2047) / 2048));
  uint32_t nc = (uint32_t)std::min<uint64_t>(ncap, want);
  nc = std::max<uint32_t>(nc, (uint32_t)((a.d + kCap - 1) / kCap));
  const uint32_t C = (uint32_t)((((uint64_t)a.d + nc - 1) / nc + 15) & ~15ull);

  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nc);
  cfg.blockDim = dim3(kClThreads);
  cfg.dynamicSmemBytes = kClSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = nc;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, compress_cluster_kernel<Tr>, a, C) == cudaSuccess ? 0 : 5;
}

// 0: off, 1: vectors of at most kClAutoMax elements (default), 2: every vector
// that fits the cluster (tests, A/B)
static std::atomic<int> g_cluster_path{-1};  // -1: not yet read from the environment

int cluster_path_mode() {
  int v = g_cluster_path.load(std::memory_order_acquire);
  if (v < 0) {  // GP_CLUSTER_PATH=0/1/2 (development aid), GP_NO_CLUSTER=1 = 0
    int env = (int)env_u32("GP_CLUSTER_PATH", 1u);
    const char* s = std::getenv("GP_NO_CLUSTER");
    if (s != nullptr && s[0] == '1') env = 0;
    if (env > 2) env = 1;
    g_cluster_path.compare_exchange_strong(v, env, std::memory_order_acq_rel);
    v = g_cluster_path.load(std::memory_order_acquire);
  }
  return v;
}

int set_cluster_path(int mode) {
  const int prev = cluster_path_mode();
  g_cluster_path.store(mode < 0 ? 0 : (mode > 2 ? 2 : mode), std::memory_order_release);
  return prev;
}

// -1: not applicable (too long, no cluster launchable, or the path switched
// off); otherwise the launch status
int launch_compress_cluster(int dtype, const CompressArgs& a, const DeviceInfo& dev, cudaStream_t stream) {
  const int mode = cluster_path_mode();
  if (mode == 0) return -1;
  // auto: only where it beats the cooperative grid (B200 A/B, scripts/cluster_probe.py:
  // 16K fp32 elements 14 us vs 22-24 us cold, 64K 14-15 vs 21-22 cold and 13-14 vs
  // 15-16 warm; at 128K 16-20 vs 20-22 cold but 15-18 vs 15-17 warm)
  static const uint32_t auto_max = env_u32("GP_CL_AUTO_MAX", kClAutoMax);
  if (mode == 1 && a.d > auto_max) return -1;
  switch (dtype) {
    case 0: return launch_cluster_t<TraitsF32>(a, dev, stream);
    case 1: return launch_cluster_t<TraitsBF16>(a, dev, stream);
    case 2: return launch_cluster_t<TraitsF64>(a, dev, stream);
    default: return -1;
  }
}

}  // namespace gp
