// gp_compress.cu — AdaTopK compress on sm_100a.
//
// Replaces topk_compress (reference: pkg/src/geopipe/compressor.py:79-94):
//     order = np.argsort(-np.abs(flat), kind="stable"); kept = np.sort(order[:k])
//     values = flat[kept]
// i.e. the k largest |x| (NaN lowest, ties to the lower index), emitted in
// ascending index order.  No sort is performed; the kernel is a radix *select*
// followed by an index-ordered stream compaction, bit-exact with the reference.
//
// One persistent cooperative launch, 1024 threads x one CTA per SM (or fewer
// CTAs, gp_topk_compress_*_ctas, so independent compresses share the GPU).  The
// vector is split into G*32 contiguous "units", one per warp, in index order,
// so that a warp-ordered compaction of every unit concatenated in unit order
// is globally index ordered.  A unit streams through a per-warp shared-memory
// ring of two 2 KiB row-pair slots; each lane fills (cp.async) and tests the
// two 16-byte pieces of every row it owns.
//
//   stage 0  each CTA takes a low watermark lo0 from a sample of its warps'
//            first rows (4 keys per lane, no extra traffic): the key whose
//            expected population is ~k plus a 4-sigma margin.
//   stage 1  the single full read of x: every element with |x| >= lo0 (one
//            FSETP) is a candidate; candidates go to the warp's index-ordered
//            list (shared memory, spilling to the workspace) and into an fb-bit
//            "fine" histogram (smem window starting at the watermark, flushed by
//            red.add into the global histogram, GP_HIST_COPIES replicas).  Sparse steps place
//            candidates with ballots; dense steps with one packed warp scan.
//            -- grid barrier B1 --
//   stage 2  every CTA sums the replicas from the top and finds the fine bin
//            B1 holding the k-th largest key.  If some CTA's watermark sat
//            above B1, only those CTAs re-stream with a lowered watermark
//            (one extra barrier; B1 can only move up).  Keys above B1 are kept
//            ("sure"); keys inside B1 are final candidates (FC).  Fast path
//            (<= 64K FC keys): each CTA publishes [sure, |FC|, FC keys].
//            -- grid barrier B2 --
//   stage 3  one round trip reads every CTA's first 32 words; the exact
//            threshold key T and the tie quota come from a radix select over
//            the unordered FC keys (bf16: T is B1); a CTA's output offset needs
//            only the earlier CTAs' counts and its own FC keys' tie prefix;
//            each warp then writes its kept (index, value) pairs.
//   slow path (too many FC keys, or a CTA overflowing its region) resolves
//            the low bits with global per-level histograms + barriers, then
//            one more barrier for the tie prefix.
//
// fb (fine-histogram bits) grows with d so |B1| stays small: 16 bits below 2^21
// elements, one more per doubling, at most 20 (GP_FB_SHIFT 5; against 7 on a
// B200 A/B: 26 MB compresses at r = 10 -8%, the bench +0.7%).
// All histogram state is left zeroed for the next call and the grid barrier
// is self-resetting, so the workspace needs to be zeroed only once.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <type_traits>

#include "gp_kernels.cuh"

#ifndef GP_LIST_KB
#define GP_LIST_KB 40
#endif

namespace gp {

constexpr int kMaxGridSpec = 160;      // largest grid: the one-round-trip FC gather stages G*32 keys in smem
constexpr uint32_t kRing = 4;          // 1 KiB rows in flight per warp (two 2-row bulk copies into smem)
constexpr uint32_t kFcCapBig = 65536;  // final candidates the fast path accepts in total
#ifndef GP_DEFER_REST
#define GP_DEFER_REST 1
#endif
#ifndef GP_GROUP_COPY
#define GP_GROUP_COPY 0
#endif
#ifndef GP_SKIP_EMPTY
#define GP_SKIP_EMPTY 0
#endif
#ifndef GP_WM_REFINE
#define GP_WM_REFINE 1
#endif
constexpr int kWmFineBins = 4096;      // watermark refinement: fine sample bins (in the window's smem)
#ifndef GP_REFINE_MIN_ROWS
#define GP_REFINE_MIN_ROWS 32
#endif
constexpr size_t kRefineMinUnitBytes = (size_t)GP_REFINE_MIN_ROWS * 1024;  // refine for units of >= this many rows
#ifndef GP_LIST_EVICT_LAST
#define GP_LIST_EVICT_LAST 0
#endif
#ifndef GP_LIST_DISCARD
#define GP_LIST_DISCARD 1
#endif
#ifndef GP_LDGSTS
#define GP_LDGSTS 1  // ring filled by per-lane cp.async (1) or by one bulk (TMA) copy per row pair (0)
#endif
#ifndef GP_ISSUE_FULL
#define GP_ISSUE_FULL 1  // full row pairs refilled without per-piece bounds
#endif
#ifndef GP_PREFETCH_ROWS
#define GP_PREFETCH_ROWS 8
#endif
constexpr uint32_t kPrefetchRows = GP_PREFETCH_ROWS;  // further rows prefetched to L2 at kernel start

// ---------------------------------------------------------------------------
// list entries: (global index, raw bits) — 8 B for 16/32-bit, 16 B for 64-bit

template <class Tr>
struct Entry {
  static constexpr uint32_t kBytes = sizeof(typename Tr::Bits) == 4 ? 8 : 16;
  // per-CTA shared-memory candidate lists (a larger list starves L1, where
  // the few register spills of the stream loop live)
  static constexpr uint32_t kListBytes = GP_LIST_KB * 1024;
  static constexpr uint32_t kSmemCap = kListBytes / (32 * kBytes);  // entries per warp in smem

  __device__ __forceinline__ static void put(unsigned char* base, uint32_t pos, uint32_t idx, typename Tr::Bits b) {
    if constexpr (kBytes == 8) {
      reinterpret_cast<uint2*>(base)[pos] = make_uint2(idx, (uint32_t)b);
    } else {
      reinterpret_cast<uint4*>(base)[pos] = make_uint4(idx, 0u, (uint32_t)b, (uint32_t)((uint64_t)b >> 32));
    }
  }
  // a spilled (global) entry: L2 evict_last (GP_LIST_EVICT_LAST), so the list
  // survives other streams' normal-priority traffic until the walk
  __device__ __forceinline__ static void put_glob(unsigned char* base, uint32_t pos, uint32_t idx,
                                                  typename Tr::Bits b) {
#if GP_LIST_EVICT_LAST
    if constexpr (kBytes == 8) {
      st_global_v2_hint(reinterpret_cast<uint2*>(base) + pos, idx, (uint32_t)b, l2_evict_last_policy());
    } else {
      st_global_v4_hint(reinterpret_cast<uint4*>(base) + pos,
                        make_uint4(idx, 0u, (uint32_t)b, (uint32_t)((uint64_t)b >> 32)), l2_evict_last_policy());
    }
#else
    put(base, pos, idx, b);
#endif
  }
  // plain loads: global entries were written by this warp, and grid barriers
  // (acquire fences) separate any cross-SM producer
  __device__ __forceinline__ static void get(const unsigned char* base, uint32_t pos, uint32_t& idx,
                                             typename Tr::Bits& b) {
    if constexpr (kBytes == 8) {
      const uint2 e = reinterpret_cast<const uint2*>(base)[pos];
      idx = e.x;
      b = e.y;
    } else {
      const uint4 e = reinterpret_cast<const uint4*>(base)[pos];
      idx = e.x;
      b = (typename Tr::Bits)(((uint64_t)e.w << 32) | e.z);
    }
  }
};

// A warp's candidate list: the first kSmemCap entries in shared memory, the
// rest in the unit's workspace region (same positions).
template <class Tr>
struct WarpList {
  unsigned char* smem;
  unsigned char* glob;
  __device__ __forceinline__ void put(uint32_t j, uint32_t idx, typename Tr::Bits b) const {
    if (j < Entry<Tr>::kSmemCap) Entry<Tr>::put(smem, j, idx, b);
    else Entry<Tr>::put_glob(glob, j, idx, b);
  }
  // after the last pass over an L-entry list: its spilled lines are dead, drop
  // them from L2 instead of writing them back (GP_LIST_DISCARD)
  __device__ __forceinline__ void discard(uint32_t L) const {
#if GP_LIST_DISCARD
    constexpr uint32_t kB = Entry<Tr>::kBytes;
    static_assert(Entry<Tr>::kSmemCap * kB % 128 == 0, "the global part starts on a line");
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t ln = Entry<Tr>::kSmemCap * kB / 128 + lane; ln < (L * kB + 127) / 128; ln += 32)
      discard_l2_line(glob + (size_t)ln * 128);
#endif
  }
  __device__ __forceinline__ void get(uint32_t j, uint32_t& idx, typename Tr::Bits& b) const {
    Entry<Tr>::get(j < Entry<Tr>::kSmemCap ? smem : glob, j, idx, b);
  }
};

// Visit entries [j0, L) of a warp's list in index order, 32 per step, with
// the loads of kScanDepth steps in flight (spilled entries live in L2/HBM: one
// round trip per step would serialise the pass).  body(valid, idx, bits) runs
// warp-wide.
// development aid: GP_EXIT_AT=n ends the kernel after phase n (timing by differences)
#ifndef GP_EXIT_AT
#define GP_EXIT_AT 99
#endif
#define EXIT_AT(n) \
  do {             \
    if (GP_EXIT_AT == (n)) return; \
  } while (0)

#ifndef GP_SCAN_DEPTH
#define GP_SCAN_DEPTH 4
#endif
constexpr int kScanDepth = GP_SCAN_DEPTH;
template <class Tr, class F>
__device__ __forceinline__ void list_scan(const WarpList<Tr>& list, uint32_t L, F&& body, uint32_t j0 = 0) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t base = j0; base < L; base += kScanDepth * 32u) {
    uint32_t idx[kScanDepth];
    typename Tr::Bits b[kScanDepth];
#pragma unroll
    for (int q = 0; q < kScanDepth; ++q) {
      const uint32_t j = base + q * 32u + lane;
      idx[q] = 0;
      b[q] = 0;
      if (j < L) list.get(j, idx[q], b[q]);
    }
#pragma unroll
    for (int q = 0; q < kScanDepth; ++q)
      if (base + q * 32u < L) body(base + q * 32u + lane < L, idx[q], b[q]);
  }
}

// Same, two consecutive entries per lane (one 16-byte load for 8-byte
// entries): 64 entries per step, lane l holding entries 2l and 2l+1, so index
// order is (lane, e) and positions come from two ballots, no scan.
// body(v0, idx0, bits0, v1, idx1, bits1) runs warp-wide.
template <class Tr, class F>
__device__ __forceinline__ void list_scan2(const WarpList<Tr>& list, uint32_t L, F&& body) {
  const uint32_t lane = threadIdx.x & 31;
  constexpr uint32_t kCap = Entry<Tr>::kSmemCap;
  static_assert(kCap % 2 == 0, "entry pairs never straddle smem/global");
  for (uint32_t base = 0; base < L; base += kScanDepth * 64u) {
    uint32_t idx[kScanDepth][2];
    typename Tr::Bits b[kScanDepth][2];
#pragma unroll
    for (int q = 0; q < kScanDepth; ++q) {
      const uint32_t j = base + q * 64u + 2u * lane;
      idx[q][0] = idx[q][1] = 0;
      b[q][0] = b[q][1] = 0;
      if (j < L) {
        const unsigned char* src = j < kCap ? list.smem : list.glob;
        if constexpr (Entry<Tr>::kBytes == 8) {
          const uint4 e = *reinterpret_cast<const uint4*>(src + (size_t)j * 8);
          idx[q][0] = e.x;
          b[q][0] = e.y;
          idx[q][1] = e.z;
          b[q][1] = e.w;
        } else {
          Entry<Tr>::get(src, j, idx[q][0], b[q][0]);
          Entry<Tr>::get(src, j + 1, idx[q][1], b[q][1]);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < kScanDepth; ++q) {
      const uint32_t j = base + q * 64u + 2u * lane;
      if (base + q * 64u < L) body(j < L, idx[q][0], b[q][0], j + 1 < L, idx[q][1], b[q][1]);
    }
  }
}

template <class Tr>
__device__ __forceinline__ typename Tr::Bits load_bits(const void* x, uint32_t i) {
  return (typename Tr::Bits)__ldg(reinterpret_cast<const typename Tr::Elem*>(x) + i);
}

// ---------------------------------------------------------------------------
// one element's raw bits from shared memory

template <class Tr>
__device__ __forceinline__ typename Tr::Bits ld_shared_elem(uint32_t addr) {
  if constexpr (sizeof(typename Tr::Elem) == 4) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
  } else if constexpr (sizeof(typename Tr::Elem) == 2) {
    uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
    return (typename Tr::Bits)v;
  } else {
    uint64_t v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(addr));
    return v;
  }
}

// ---------------------------------------------------------------------------
// scans / crossing searches

// 1024-thread exclusive scan, two barriers; sh32 holds 64 words.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* sh32, uint32_t* total) {
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t x = warp_incl_scan(v);
  if (lane == 31) sh32[w] = x;
  __syncthreads();
  if (w == 0) sh32[32 + lane] = warp_incl_scan(sh32[lane]);
  __syncthreads();
  *total = sh32[63];
  return (w ? sh32[32 + w - 1] : 0u) + x - v;
}

// One warp: scanning smem bins downward from `top` to 0, 256 per step, find b
// with above(b) < target <= above(b) + h(b).  Results are warp-uniform.
__device__ __forceinline__ bool warp_cross_desc(const uint32_t* hist, int top, uint32_t target, uint32_t* bin,
                                                uint32_t* above) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t base = 0;
  for (int t0 = top; t0 >= 0; t0 -= 256) {
    uint32_t v[8], s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int b = t0 - 8 * (int)lane - i;
      v[i] = b >= 0 ? hist[b] : 0u;
      s += v[i];
    }
    const uint32_t incl = warp_incl_scan(s);
    uint32_t run = base + incl - s;
    const bool mine = run < target && run + s >= target;
    const uint32_t who = __ballot_sync(kFull, mine);
    if (who) {
      uint32_t rb = 0, ra = 0;
      if (mine) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (run < target && run + v[i] >= target) {
            rb = (uint32_t)(t0 - 8 * (int)lane - i);
            ra = run;
          }
          run += v[i];
        }
      }
      const int src = __ffs(who) - 1;
      *bin = __shfl_sync(kFull, rb, src);
      *above = __shfl_sync(kFull, ra, src);
      return true;
    }
    base += __shfl_sync(kFull, incl, 31);
  }
  return false;
}

// ---------------------------------------------------------------------------
// output

template <class Tr>
__device__ __forceinline__ void write_out(const CompressArgs& a, void* val_out, uint32_t pos, uint32_t idx,
                                          typename Tr::Bits b) {
  using Elem = typename Tr::Elem;
  if (a.idx64) reinterpret_cast<int64_t*>(a.idx_out)[pos] = (int64_t)idx;
  else reinterpret_cast<int32_t*>(a.idx_out)[pos] = (int32_t)idx;
  if (a.val_f32) reinterpret_cast<float*>(val_out)[pos] = Tr::to_f32(b);
  else reinterpret_cast<Elem*>(val_out)[pos] = (Elem)b;
  if (a.val2_out) reinterpret_cast<Elem*>(a.val2_out)[pos] = (Elem)b;
}

// ---------------------------------------------------------------------------
// optional stage timestamps (development aid; a.dbg is null in production)

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define STAMP(i)                                                        \
  do {                                                                  \
    if (a.dbg != nullptr && tid == 0) {                                 \
      a.dbg[(size_t)c * 32 + (i)] = globaltimer_ns();                   \
      a.dbg[(size_t)c * 32 + 16 + (i)] = (unsigned long long)clock64(); \
    }                                                                   \
  } while (0)

// ---------------------------------------------------------------------------
// shared-memory layout (bytes)

template <class Tr>
struct Smem {
  static constexpr size_t coarse = 0;                                   // kCoarseBins u32
  static constexpr size_t win = coarse + kCoarseBins * 4;               // kWinBins u32
  static constexpr size_t low = win + kWinBins * 4;                     // kLowBins u32
  static constexpr size_t lvl = low + kLowBins * 4;                     // 256 u32
  static constexpr size_t s32 = lvl + 256 * 4;                          // 64 u32
  static constexpr size_t res = s32 + 64 * 4;                           // 32 u32
  static constexpr size_t warp = res + 32 * 4;                          // 4 x 32 u32
  static constexpr size_t fcoff = warp + 4 * 32 * 4;                    // kMaxGrid+4 u32
  static constexpr size_t mbar = (fcoff + (kMaxGrid + 4) * 4 + 7) & ~size_t(7);  // 32 x kRing mbarriers
  static constexpr size_t ring = (mbar + 32 * kRing * 8 + 127) & ~size_t(127);   // 32 x kRing x 1 KiB rows
  // the final-candidate arrays are used only after the stream: they alias the ring
  static constexpr size_t fcpre = ring;                                           // kFcCap+4 u32
  static constexpr size_t fckey = (fcpre + (kFcCap + 4) * 4 + 15) & ~size_t(15);  // kFcCap keys
  static_assert(fckey + kFcCap * sizeof(typename Tr::Key) <= ring + 32 * kRing * 1024, "FC arrays fit the ring");
  static constexpr size_t list = ring + 32 * kRing * 1024;                        // Entry::kListBytes
  static constexpr size_t total = list + Entry<Tr>::kListBytes;
  static_assert(total <= 227 * 1024, "shared memory");
};

// ---------------------------------------------------------------------------
// the kernel

template <class Tr, bool kRefine>
__global__ void __launch_bounds__(kCompressThreads, 1) compress_kernel(const CompressArgs a) {
  using Bits = typename Tr::Bits;
  using Key = typename Tr::Key;
  using Elem = typename Tr::Elem;
  using SL = Smem<Tr>;
  constexpr int CS = Tr::kKeyBits - 12;        // coarse bin = key >> CS (12 bits)
  constexpr int EPL = 32 / (int)sizeof(Elem);  // elements per lane chunk (8 f32, 16 bf16, 4 f64)
  constexpr int EPS = 16 / (int)sizeof(Elem);  // elements per 16-byte piece
  constexpr uint32_t kEntryBytes = Entry<Tr>::kBytes;
  const int FB = a.fb;                         // fine-histogram bits
  const int FS = Tr::kKeyBits - FB;            // fine bin = key >> FS
  const uint32_t nfine = 1u << FB;

  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* sh_coarse = reinterpret_cast<uint32_t*>(smem + SL::coarse);
  uint32_t* sh_win = reinterpret_cast<uint32_t*>(smem + SL::win);
  uint32_t* sh_low = reinterpret_cast<uint32_t*>(smem + SL::low);
  uint32_t* sh_lvl = reinterpret_cast<uint32_t*>(smem + SL::lvl);
  uint32_t* sh32 = reinterpret_cast<uint32_t*>(smem + SL::s32);
  uint32_t* sh_res = reinterpret_cast<uint32_t*>(smem + SL::res);
  uint32_t* w_a = reinterpret_cast<uint32_t*>(smem + SL::warp);
  uint32_t* w_b = w_a + 32;
  uint32_t* w_aoff = w_b + 32;
  uint32_t* w_boff = w_aoff + 32;
  uint32_t* sh_fcoff = reinterpret_cast<uint32_t*>(smem + SL::fcoff);
  uint32_t* sh_fcpre = reinterpret_cast<uint32_t*>(smem + SL::fcpre);
  Key* sh_fckey = reinterpret_cast<Key*>(smem + SL::fckey);

  const uint32_t G = gridDim.x, c = blockIdx.x, tid = threadIdx.x;
  // warp index broadcast from lane 0: ptxas then keeps the unit, ring and
  // row addresses derived from it in uniform registers (A/B with the cp.async
  // ring: +0.5% bench, +2% GPT-2 batch; with the bulk-copy ring it had cost 5%)
  const uint32_t lane = tid & 31, w = __shfl_sync(kFull, tid >> 5, 0);
  const uint32_t d = a.d;
  uint32_t k = a.k;
  void* val_out = a.val_out;
  if (a.k_dev != nullptr) {
    // device-resident k (an on-device AdaTopK plan): every CTA reads the same
    // value, so an invalid k ends every CTA here (no grid barrier is reached)
    const long long kk = __ldg(a.k_dev);
    if (kk < 1 || kk > (long long)a.k || kk > (long long)d) {
      if (c == 0 && tid == 0) {
        if (a.err != nullptr) atomicOr(a.err, kFlagBadK);
        if (a.header != nullptr) {
          a.header[0] = (unsigned long long)d;
          a.header[1] = ~0ull;  // an invalid frame: the receiver flags it
        }
      }
      return;
    }
    k = (uint32_t)kk;
    if (a.frame_vals) val_out = reinterpret_cast<unsigned char*>(a.idx_out) + (a.idx64 ? 8ull : 4ull) * k;
    if (k == d) {  // ratio <= 1: every element kept, in index order (the pass-through)
      if (a.header != nullptr && c == 0 && tid == 0) {
        a.header[0] = (unsigned long long)d;
        a.header[1] = (unsigned long long)k;
      }
      for (uint32_t i = c * blockDim.x + tid; i < d; i += gridDim.x * blockDim.x)
        write_out<Tr>(a, val_out, i, i, load_bits<Tr>(a.x, i));
      return;
    }
  }
  const uint32_t unit = c * 32u + w;
  const uint32_t u0 = (uint32_t)min((uint64_t)unit * a.W, (uint64_t)d);
  const uint32_t u1 = (uint32_t)min((uint64_t)u0 + a.W, (uint64_t)d);
  const uint32_t n = u1 - u0;
  const Elem* x = reinterpret_cast<const Elem*>(a.x);
  const WarpList<Tr> list{smem + SL::list + (size_t)w * Entry<Tr>::kSmemCap * kEntryBytes,
                          reinterpret_cast<unsigned char*>(a.lists) + (size_t)unit * a.W * kEntryBytes};
  uint32_t* ctrl = a.ctrl;
  uint32_t* bar = &ctrl[kCtrlBar];
  // this CTA's histogram replica (kHistCopies replicas cut same-address atomic contention)
  uint32_t* hist = a.hist1 + (size_t)(c & (kHistCopies - 1)) * kFineBinsMax;

  STAMP(0);
  if (a.header != nullptr && c == 0 && tid == 0) {
    a.header[0] = (unsigned long long)d;
    a.header[1] = (unsigned long long)k;
  }

  // ---- the unit's rows (1 KiB each) stream through a per-warp ring of two
  // 2 KiB slots, each holding a row pair filled by one bulk (TMA) copy that
  // completes on the slot's mbarrier; row pair 0 (the watermark's sample) is
  // requested before anything else, the rest once it has arrived
  const uint32_t nch = a.aligned ? n / EPL : 0u;  // full 32-byte chunks in the unit
  const uint32_t nrow = (nch + 31) / 32;
  const uint32_t npair = (nrow + 1) / 2;
  const uint32_t* xw = reinterpret_cast<const uint32_t*>(x + u0);
  constexpr uint32_t kPairs = kRing / 2;            // row-pair slots per warp
  const uint32_t ring = smem_addr(smem + SL::ring) + w * (kRing * 1024u);
  const uint32_t mbar = smem_addr(smem + SL::mbar) + w * (kRing * 8u);
  const uint64_t policy = l2_evict_first_policy();  // x is read once: keep L2 for the lists
  uint32_t seq = 0;                                 // row pairs this warp has issued into the ring
#if GP_LDGSTS
  static_assert(!GP_GROUP_COPY, "cp.async ring: one row pair per commit group");
  // every lane: the four 16-byte pieces of row pair p it reads itself (piece
  // j*32 + lane of the pair), one commit group per call; rings are only ever
  // read by the lane that filled the piece, so a per-thread wait is the only
  // synchronisation (A/B on B200: a bulk copy per warp and row pair streams at
  // ~25-40 GB/s per SM, per-lane cp.async at up to 150, scripts/layout_probe.cu)
  auto issue = [&](uint32_t p, uint32_t q) {
    const uint32_t slot = q % kPairs;
    const uint32_t nb = min(64u, nch - p * 64u) * 32u;  // valid bytes of the pair
    const unsigned char* src = reinterpret_cast<const unsigned char*>(xw + (size_t)p * 512u);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const uint32_t o = (uint32_t)j * 512u + lane * 16u;
      if (o < nb) cp_async16_hint(ring + slot * 2048u + o, src + o, policy);
    }
    cp_async_commit();
  };
  // the same for a pair with all 64 chunks (the stream loop's case): one
  // source pointer, immediate offsets, no per-piece bounds
  auto issue_full = [&](uint32_t p, uint32_t q) {
    const uint32_t d0 = ring + (q % kPairs) * 2048u + lane * 16u;
    const unsigned char* s0 = reinterpret_cast<const unsigned char*>(xw + (size_t)p * 512u) + lane * 16u;
#pragma unroll
    for (int j = 0; j < 4; ++j) cp_async16_hint(d0 + (uint32_t)j * 512u, s0 + j * 512, policy);
    cp_async_commit();
  };
#else
  auto issue = [&](uint32_t p, uint32_t q) {        // lane 0: row pair p as ring sequence number q
    const uint32_t slot = q % kPairs;
    bulk_load_async(ring + slot * 2048u, xw + (size_t)p * 512u, min(64u, nch - p * 64u) * 32u, mbar + slot * 8u,
                    policy);
  };
#endif
#if GP_GROUP_COPY
  // group mode: both ring slots (contiguous in smem) refilled by ONE 4 KiB
  // copy of two consecutive row pairs, completing on slot 0's mbarrier
  auto issue_group = [&](uint32_t g) {
    bulk_load_async(ring, xw + (size_t)g * 1024u, min(128u, nch - g * 128u) * 32u, mbar, policy);
  };
#endif
  // the rest of the warp's opening requests: the other ring pairs and, for a
  // short unit, its remaining rows sent to L2 (no second HBM round trip)
  auto issue_rest = [&]() {
#if GP_LDGSTS
    for (uint32_t p = 1; p < kPairs; ++p) {  // every lane; one group per slot, empty past the unit
      if (p < npair) issue(p, p);
      else cp_async_commit();
    }
    if (lane == 0 && nrow > kRing && nrow <= kRing + kPrefetchRows)
      prefetch_l2_bulk(xw + (size_t)kRing * 256u, (nch - kRing * 32u) * 32u);
#else
    if (!GP_GROUP_COPY)
      for (uint32_t p = 1; p < min(npair, kPairs); ++p) issue(p, p);
    if (nrow > kRing && nrow <= kRing + kPrefetchRows)
      prefetch_l2_bulk(xw + (size_t)kRing * 256u, (nch - kRing * 32u) * 32u);
#endif
  };
#if GP_LDGSTS
  if (npair > 0) issue(0, 0);
  if (!GP_DEFER_REST) issue_rest();
  if (false) {
#else
  if (lane == 0) {
#endif
    for (uint32_t s = 0; s < kPairs; ++s) mbar_init(mbar + s * 8u, 1u);
    fence_mbar_init();
#if GP_GROUP_COPY
    if (npair > 0) issue_group(0);
#else
    if (npair > 0) issue(0, 0);
#endif
    if (!GP_DEFER_REST) issue_rest();
  }
  __syncwarp();

  // ---- stage 0: low watermark from a sample of this CTA's row 0s (no extra
  // traffic): 4 elements per lane, one warp finds the crossing from the top
  // Watermark refinement (below) for large units only (>= GP_REFINE_MIN_ROWS
  // rows per warp: the bench's capped grids, GPT-2 tensors in flight): its
  // ~2 us of prologue outweigh the candidates it saves on smaller units (A/B
  // on B200: 21-row units +1-3 us, 43-row neutral, 87-row and longer -4..-9%).
  constexpr bool refine = GP_WM_REFINE && kRefine;  // the launcher picks the instantiation by unit size
  for (uint32_t i = tid; i < kCoarseBins; i += kCompressThreads) sh_coarse[i] = 0u;
  if (refine)  // the refinement's fine sample bins (the window, free until the stream)
    for (uint32_t i = tid; i < kWmFineBins; i += kCompressThreads) sh_win[i] = 0u;
  if (tid < 32) sh_res[tid] = 0u;
  __syncthreads();
  if (nrow > 0) {
#if GP_LDGSTS
    if (GP_DEFER_REST) cp_async_wait<0>();  // row pair 0 (the only group so far)
    else cp_async_wait<kPairs - 1>();
    // deferred: the watermark needs only row pair 0 of every warp, so the
    // rest of the unit is requested once this warp's pair 0 is in (it then
    // streams in under the watermark's barriers instead of ahead of row 0s)
    if (GP_DEFER_REST) issue_rest();
#else
    mbar_wait(mbar, 0u);  // row pair 0
    // deferred: the watermark needs only row pair 0 of every warp, so the
    // rest of the unit is requested once this warp's pair 0 is in (it then
    // streams in under the watermark's barriers instead of ahead of row 0s)
    if (GP_DEFER_REST && lane == 0) issue_rest();
#endif
    uint32_t ns = 0, mb = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint32_t piece = h * 32u + lane;  // 16-byte piece of row 0
      if (piece < 2u * nch) {
        const uint4 v = ld_shared_v4(ring + piece * 16u);
#pragma unroll
        for (int e = 0; e < EPS; e += EPS / 2) {
          const uint32_t bin = (uint32_t)(Tr::key(Tr::lane(v, e)) >> CS);
          atomicAdd(&sh_coarse[bin], 1u);
          mb = max(mb, bin + 1u);
          ++ns;
        }
      }
    }
    ns = warp_sum(ns);
    mb = __reduce_max_sync(kFull, mb);
    if (lane == 0 && ns) {
      atomicAdd(&sh_res[19], ns);
      atomicMax(&sh_res[16], mb);
    }
  }
  __syncthreads();
  if (w == 0 && sh_res[16]) {
    const uint32_t S = sh_res[19];
    const double mu = (double)S * (double)k / (double)d;
    const double rs = ceil(mu + 4.0 * sqrt(mu) + 8.0);
    if (rs < (double)S) {
      uint32_t bin = 0, above = 0;
      if (warp_cross_desc(sh_coarse, (int)sh_res[16] - 1, (uint32_t)rs, &bin, &above) && lane == 0)
        sh_res[17] = bin + 1u;
    }
  }
  __syncthreads();
  Key lo0 = sh_res[17] ? (Key)(sh_res[17] - 1) << CS : (Key)0;
  // refinement: the coarse watermark above sits on a 12-bit bin edge from 4
  // keys per lane, so its margin and its rounding let through up to ~5x k
  // candidates (r = 1000).  Every key of row pair 0 (16 per lane for fp32) at
  // or above it goes into 4096 sample bins 8 key bits finer, and the
  // watermark moves up to the fine bin where the expected population of the
  // larger sample, plus the same 4-sigma+8 margin, is reached.  It only ever
  // rises, and a watermark above the threshold is still caught by the rescan.
  if (refine && sh_res[17] != 0u) {
    constexpr int RS = CS - 8;
    const Key la = lo0;
    if (nrow > 0) {
      uint32_t ns = 0, na = 0;
      const uint32_t npc = 2u * min(nch, 64u);  // 16-byte pieces of row pair 0
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t piece = q * 32u + lane;
        if (piece < npc) {
          const uint4 v = ld_shared_v4(ring + piece * 16u);
#pragma unroll
          for (int e = 0; e < EPS; ++e) {
            const Key kk = Tr::key(Tr::lane(v, e));
            if (kk >= la) {
              const Key off = (kk - la) >> RS;
              atomicAdd(&sh_win[off < (Key)(kWmFineBins - 1) ? (uint32_t)off : (uint32_t)(kWmFineBins - 1)], 1u);
              ++na;
            }
          }
          ns += EPS;
        }
      }
      ns = warp_sum(ns);
      na = warp_sum(na);
      if (lane == 0 && ns) {
        atomicAdd(&sh_res[23], ns);
        atomicAdd(&sh_res[22], na);
      }
    }
    __syncthreads();
    const double mu2 = (double)sh_res[23] * (double)k / (double)d;
    const double rs2 = ceil(mu2 + 4.0 * sqrt(mu2) + 8.0);
    if (rs2 <= (double)sh_res[22]) {  // CTA-uniform
      static_assert(kWmFineBins == 4 * kCompressThreads, "one block scan over the fine sample bins");
      uint32_t v[4], sum = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {  // thread order = descending bins
        v[b] = sh_win[kWmFineBins - 1 - 4 * tid - b];
        sum += v[b];
      }
      uint32_t tot;
      uint32_t run = block_excl_scan(sum, sh32, &tot);  // sample keys in higher bins
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        if ((double)run < rs2 && (double)(run + v[b]) >= rs2) sh_res[21] = kWmFineBins - 4 * tid - b;  // bin + 1
        run += v[b];
      }
      __syncthreads();
      // down to a fine-histogram bin edge: a CTA must count every key of its
      // lowest histogram bin, or the threshold bin's population is short
      if (sh_res[21] != 0u) lo0 = ((la + ((Key)(sh_res[21] - 1u) << RS)) >> FS) << FS;
    }
  }
  const uint32_t cmax = sh_res[16] ? sh_res[16] - 1 : (uint32_t)(kCoarseBins - 1);  // highest sampled coarse bin
  // top of the smem histogram window: two exponents above the sample maximum
  const uint32_t top = min(nfine, ((cmax + 1u) << (FB - 12)) + (2u << (FB - Tr::kExpBits)));

  STAMP(1);
  if (GP_EXIT_AT == 1) {  // drain the ring first: no bulk copy may outlive the CTA
#if GP_LDGSTS
    cp_async_wait<0>();
#else
    for (uint32_t p = 0; p < (GP_GROUP_COPY ? min(npair, 1u) : min(npair, kPairs)); ++p) mbar_wait(mbar + p * 8u, 0u);
#endif
    return;
  }
  uint32_t L = 0;                              // this warp's candidate count
  uint32_t my_lobin = (uint32_t)(lo0 >> FS);   // lowest fine bin this CTA histograms

  // ---- stage 1 (and the rare rescan): stream the unit, keep keys >= lo and
  // histogram those whose fine bin is below add_below
  auto stream_unit = [&](Key lo, uint32_t add_below, bool preloaded) {
    const uint32_t lob = (uint32_t)(lo >> FS);
    // smem window: candidates are densest right above the watermark, so the
    // window starts there (at 20 fine bits it spans only two octaves); with no
    // watermark (every element a candidate) it ends at the top of the sample
    // range.  Bins outside it take global atomics.
    uint32_t wb = lob > 0u ? lob : (top > (uint32_t)kWinBins ? top - kWinBins : 0u);
    wb = min(wb, nfine - kWinBins);
    const uint32_t lowlim = min((uint32_t)kLowBins, wb);
    for (uint32_t i = tid; i < kWinBins; i += kCompressThreads) sh_win[i] = 0u;
    if (tid < kLowBins) sh_low[tid] = 0u;
    if (tid == 0) {
      sh_res[18] = 0u;
      sh_res[20] = 0u;
    }
    __syncthreads();
    L = 0;
    uint32_t mymax = 0;
    const Key lo_m1 = lo ? lo - 1 : (Key)0;
    // histogram one candidate (run warp-cooperatively over freshly appended entries)
    auto count = [&](Bits b) {
      const uint32_t fb = (uint32_t)(Tr::key(b) >> FS);
      if (fb < add_below) {
        const uint32_t off = fb - wb;
        if (off < (uint32_t)kWinBins) atomicAdd(&sh_win[off], 1u);
        else if (fb < lowlim) atomicAdd(&sh_low[fb], 1u);
        else atomicAdd(&hist[fb], 1u);
        mymax = max(mymax, fb + 1u);
      }
    };
    // Candidate test in the value domain: one |x| >= thr compare per element
    // (FSETP/DSETP with the abs modifier; NaN compares false, its key is 0).
    const typename Tr::Cand test = Tr::make_cand(lo_m1);
    const bool all = lo == 0;  // every element is a candidate, NaN included
    // the warp histograms the entries it just appended, one per lane
    // Entries that spilled to global memory are histogrammed after the loop
    // (reading them back here would put an L2 round trip on every row pair).
    constexpr uint32_t kCap = Entry<Tr>::kSmemCap;
    auto count_new = [&](uint32_t from) {
      __syncwarp();
      const uint32_t end = min(L, kCap);
      for (uint32_t j = from + lane; j < end; j += 32u) {
        uint32_t idx;
        Bits b;
        list.get(j, idx, b);
        count(b);
      }
    };
    // one 1 KiB row from ring slot `so`: lane holds 16-byte pieces h*32+lane
    // (h = 0, 1), i.e. elements [h*32*EPS + lane*EPS, +EPS) of the row
    // Rows r and r+1 (ring slots so0, so1) in one step: the four 512-byte
    // sub-rows j = 2*row + h are tested together and placed with one packed
    // scan, so a warp's per-row dependent chain (scan, append, histogram) is
    // paid once per two rows.  Lane holds 16-byte piece h*32+lane of each row,
    // i.e. elements [h*32*EPS + lane*EPS, +EPS).
    // FULL (both rows complete: no per-piece bounds) and ALL (every element a
    // candidate) are compile-time in the hot loop: a full step is four
    // back-to-back 16-byte smem loads, then one compare and one predicated OR
    // per element, with no branch.
    auto process2 = [&](uint32_t r, uint32_t so0, uint32_t so1, auto full_c, auto all_c) {
      constexpr bool FULL = decltype(full_c)::value;
      constexpr bool ALL = decltype(all_c)::value;
      uint32_t m[4];
      if constexpr (FULL) {
        uint4 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = ld_shared_v4((j < 2 ? so0 : so1) + ((j & 1) * 32u + lane) * 16u);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint32_t mm = 0;
#pragma unroll
          for (int e = 0; e < EPS; ++e) mm |= (ALL || test(Tr::lane(v[j], e))) ? (1u << e) : 0u;
          m[j] = mm;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t rr = r + (j >> 1);
          const uint32_t piece = (j & 1) * 32u + lane;
          uint32_t mm = 0;
          if (rr < nrow && piece < 2u * min(32u, nch - rr * 32u)) {
            const uint4 v = ld_shared_v4((j < 2 ? so0 : so1) + piece * 16u);
#pragma unroll
            for (int e = 0; e < EPS; ++e) mm |= (ALL || test(Tr::lane(v, e))) ? (1u << e) : 0u;
          }
          m[j] = mm;
        }
      }
#if GP_SKIP_EMPTY
      // no candidate anywhere in the step (about a quarter of the steps at
      // r = 1000 with the refined watermark): done after one vote
      if (!__any_sync(kFull, (m[0] | m[1] | m[2] | m[3]) != 0u)) return;
#endif
      // per-sub-row counts packed into one scan: 8-bit fields when a sub-row
      // holds at most 32*EPS <= 128 candidates (f32, f64), else 16-bit fields
      constexpr int kField = EPS * 32 < 256 ? 8 : 16;
      using Packed = typename std::conditional<kField == 8, uint32_t, uint64_t>::type;
      // sparse step (the common case above r ~ 50): no lane holds two
      // candidates in one sub-row, so ballots give every position directly and
      // each candidate is histogrammed where it is appended
      const uint32_t two = (m[0] & (m[0] - 1)) | (m[1] & (m[1] - 1)) | (m[2] & (m[2] - 1)) | (m[3] & (m[3] - 1));
      if (!__any_sync(kFull, two)) {
        const uint32_t lt = lanemask_lt();
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t bj = __ballot_sync(kFull, m[j] != 0u);
#if GP_SKIP_EMPTY
          if (bj == 0u) continue;  // warp-uniform: no candidate in this sub-row
#endif
          if (m[j]) {
            const uint32_t e = __ffs(m[j]) - 1;
            const uint32_t piece = (j & 1) * 32u + lane;
            const Bits bv = ld_shared_elem<Tr>((j < 2 ? so0 : so1) + piece * 16u + e * (uint32_t)sizeof(Elem));
            list.put(L + __popc(bj & lt), u0 + (r + (j >> 1)) * (32u * EPL) + piece * EPS + e, bv);
            if (L + __popc(bj & lt) < kCap) count(bv);  // spilled entries are counted after the loop
          }
          L += __popc(bj);
        }
        return;
      }
      if (__any_sync(kFull, (m[0] | m[1] | m[2] | m[3]) != 0u)) {
        // (built only here: the sparse steps above never need the counts)
        const Packed packed = (Packed)__popc(m[0]) | ((Packed)__popc(m[1]) << kField) |
                              ((Packed)__popc(m[2]) << (2 * kField)) | ((Packed)__popc(m[3]) << (3 * kField));
        Packed incl;
        if constexpr (kField == 8) incl = warp_incl_scan(packed);
        else incl = warp_incl_scan64(packed);
        const Packed excl = incl - packed, tot = __shfl_sync(kFull, incl, 31);
        constexpr uint32_t kMask = (1u << kField) - 1u;
        const uint32_t from = L;
        uint32_t pos[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          pos[j] = L + ((uint32_t)(excl >> (kField * j)) & kMask);
        }
        {  // every earlier sub-row's total precedes sub-row j
          uint32_t run = 0;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            pos[j] += run;
            run += (uint32_t)(tot >> (kField * j)) & kMask;
          }
          L += run;
        }
        // append (divergent): each candidate is one LDS from its ring slot;
        // once a warp's list is past its smem part (dense steps), entries go
        // straight to global memory without a per-entry placement test
        auto append = [&](auto glob_only) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint32_t mm = m[j];
            const uint32_t piece = (j & 1) * 32u + lane;
            const uint32_t base = u0 + (r + (j >> 1)) * (32u * EPL) + piece * EPS;
            const uint32_t src = (j < 2 ? so0 : so1) + piece * 16u;
            while (mm) {
              const uint32_t e = __ffs(mm) - 1;
              mm &= mm - 1;
              const Bits bv = ld_shared_elem<Tr>(src + e * (uint32_t)sizeof(Elem));
              if constexpr (decltype(glob_only)::value) Entry<Tr>::put_glob(list.glob, pos[j]++, base + e, bv);
              else list.put(pos[j]++, base + e, bv);
            }
          }
        };
        if (from >= kCap) append(std::true_type{});
        else append(std::false_type{});
        count_new(from);
      }
    };
    static_assert(kRing == 4, "two row-pair slots");
#if GP_GROUP_COPY
    const uint32_t q0 = seq;  // groups of two row pairs issued so far (mbarrier phases of slot 0)
    const uint32_t ngroups = (npair + 1) / 2;
    if (!preloaded && lane == 0 && npair > 0) {
      fence_proxy_async_smem();
      issue_group(0);
    }
    auto run_pairs = [&](auto all_c) {
      const uint32_t nfull = nch / 64u;
      for (uint32_t p = 0; p < npair; ++p) {
        const uint32_t g = p >> 1, slot = p & 1u;
        if (slot == 0) mbar_wait(mbar, (q0 + g) & 1u);
        if (p < nfull) process2(2u * p, ring + slot * 2048u, ring + slot * 2048u + 1024u, std::true_type{}, all_c);
        else process2(2u * p, ring + slot * 2048u, ring + slot * 2048u + 1024u, std::false_type{}, all_c);
        if (slot == 1 || p + 1 == npair) {
          __syncwarp();
          if (lane == 0 && g + 1 < ngroups) {  // both slots consumed: refill them with the next group
            fence_proxy_async_smem();
            issue_group(g + 1);
          }
        }
      }
    };
    if (all) run_pairs(std::true_type{});
    else run_pairs(std::false_type{});
    seq = q0 + ngroups;
#else
    const uint32_t q0 = seq;
#if GP_LDGSTS
    if (!preloaded) {  // every lane: kPairs groups, empty past the unit
      for (uint32_t p = 0; p < kPairs; ++p) {
        if (p < npair) issue(p, q0 + p);
        else cp_async_commit();
      }
    }
#else
    if (!preloaded && lane == 0) {
      fence_proxy_async_smem();
      for (uint32_t p = 0; p < min(npair, kPairs); ++p) issue(p, q0 + p);
    }
#endif
    auto run_pairs = [&](auto all_c) {
      const uint32_t nfull = nch / 64u;  // row pairs with both rows complete
      for (uint32_t p = 0; p < npair; ++p) {
        const uint32_t q = q0 + p, slot = q % kPairs;
#if GP_LDGSTS
        cp_async_wait<kPairs - 1>();  // exactly kPairs - 1 groups were committed after this pair's
#else
        mbar_wait(mbar + slot * 8u, (q / kPairs) & 1u);
#endif
        if (p < nfull) process2(2u * p, ring + slot * 2048u, ring + slot * 2048u + 1024u, std::true_type{}, all_c);
        else process2(2u * p, ring + slot * 2048u, ring + slot * 2048u + 1024u, std::false_type{}, all_c);
        __syncwarp();
#if GP_LDGSTS
        // refill the slot just consumed (every lane); an empty group past the
        // unit keeps the wait count exact
        if (GP_ISSUE_FULL && p + kPairs < nfull) issue_full(p + kPairs, q + kPairs);
        else if (p + kPairs < npair) issue(p + kPairs, q + kPairs);
        else cp_async_commit();
#else
        if (lane == 0 && p + kPairs < npair) {  // refill the slot just consumed
          fence_proxy_async_smem();
          issue(p + kPairs, q + kPairs);
        }
#endif
      }
    };
    if (all) run_pairs(std::true_type{});
    else run_pairs(std::false_type{});
    seq = q0 + npair;
#endif
    const Key span = lo ? Tr::kInfAbs - lo_m1 : ~(Key)0;
    for (uint32_t i0 = nch * EPL; i0 < n; i0 += 32u) {  // scalar tail / unaligned input
      const uint32_t i = i0 + lane;
      Bits b = 0;
      bool f = false;
      if (i < n) {
        b = load_bits<Tr>(x, u0 + i);
        f = (Key)(Tr::abs_bits(b) - lo_m1) <= span;
      }
      const uint32_t mk = __ballot_sync(kFull, f);
      const uint32_t from = L;
      if (f) list.put(L + __popc(mk & lanemask_lt()), u0 + i, b);
      L += __popc(mk);
      count_new(from);
    }
    list_scan<Tr>(list, L, [&](bool valid, uint32_t, Bits b) { if (valid) count(b); }, kCap);  // spilled tail
    mymax = __reduce_max_sync(kFull, mymax);
    if (lane == 0) {
      if (mymax) atomicMax(&sh_res[18], mymax);
      if (L) atomicAdd(&sh_res[20], L);
    }
    __syncthreads();
    for (uint32_t i = tid; i < kWinBins; i += kCompressThreads) {
      const uint32_t v = sh_win[i];
      if (v) red_add_gpu(&hist[wb + i], v);
    }
    if (tid < lowlim && sh_low[tid]) red_add_gpu(&hist[tid], sh_low[tid]);
    if (tid == 0) {
      if (sh_res[18]) atomicMax(&ctrl[kCtrlMaxBin], sh_res[18]);
      if (sh_res[20]) red_add_gpu(&ctrl[kCtrlCands], sh_res[20]);
    }
  };

  // ---- stage 2 helper: sum the replicas from the top, 4096 bins per step,
  // and find the fine bin holding the k-th largest key
  uint32_t B1 = 0, G1 = 0, M = 0;
  uint32_t pop_lo = 0, pop_hi = 0;  // every populated bin of every replica lies in [pop_lo, pop_hi)
  auto find_b1 = [&](uint32_t mb, uint32_t minlo_c) -> bool {
    const int lowest = (int)(0xFFFFFFFFu - minlo_c);  // no bin below any watermark is populated
    pop_lo = (uint32_t)lowest;
    pop_hi = mb;
    if (tid == 0) sh_res[0] = 0u;
    uint32_t base = 0;
    for (int t0 = (int)mb - 1; t0 >= lowest; t0 -= 4 * kCompressThreads) {
      uint32_t v[4], s = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {  // thread order = descending bins
        const int bin = t0 - 4 * (int)tid - b;
        v[b] = 0;
        if (bin >= lowest) {
#pragma unroll
          for (int r = 0; r < kHistCopies; ++r) v[b] += a.hist1[(size_t)r * kFineBinsMax + bin];
        }
        s += v[b];
      }
      uint32_t tot;
      uint32_t run = base + block_excl_scan(s, sh32, &tot);  // keys in higher bins
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        if (run < k && run + v[b] >= k) {
          sh_res[0] = 1u;
          sh_res[1] = (uint32_t)(t0 - 4 * (int)tid - b);
          sh_res[2] = run;
          sh_res[3] = v[b];
        }
        run += v[b];
      }
      __syncthreads();
      if (sh_res[0]) break;
      base += tot;
    }
    B1 = sh_res[1];
    G1 = sh_res[2];
    M = sh_res[3];
    return sh_res[0] != 0u;
  };

  // first pass, and at most one partial rescan: a CTA whose watermark sat
  // above B1 (or all of them, if too few candidates overall) re-streams its
  // chunk with the watermark lowered to B1's edge, adding just the newly
  // covered bins; B1 can only move up, so one rescan suffices.
  {
    Key lo = lo0;
    uint32_t add_below = 0xFFFFFFFFu;
    for (int pass = 0;; ++pass) {
      if (pass == 0 || my_lobin > (uint32_t)(lo >> FS)) {
        stream_unit(lo, add_below, pass == 0);
        if (pass == 1) my_lobin = (uint32_t)(lo >> FS);
        if (tid == 0) {
          atomicMax(&ctrl[kCtrlMaxLoBin], my_lobin + 1u);
          atomicMax(&ctrl[kCtrlMinLoBin], 0xFFFFFFFFu - my_lobin);  // min, stored complemented
        }
      }
      if (pass == 0) STAMP(2);
      EXIT_AT(2);
      grid_barrier(bar, G);  // ---- B1 (and the rescan barrier)
      if (pass == 0) STAMP(3);
      EXIT_AT(3);
      // every control word in one round trip (four independent loads), not
      // one dependent L2 trip per decision
      const uint32_t c_mb = ctrl[kCtrlMaxBin], c_maxlo = ctrl[kCtrlMaxLoBin], c_cands = ctrl[kCtrlCands],
                     c_minlo = ctrl[kCtrlMinLoBin];
      const bool found = (pass == 1 || c_cands >= k) && find_b1(c_mb, c_minlo);
      if (pass == 1 || (found && c_maxlo - 1u <= B1)) break;
      lo = (Key)(found ? B1 : 0u) << FS;
      add_below = my_lobin;
    }
  }
  STAMP(4);
  EXIT_AT(4);

  // bf16: the bits below the fine bin are constant, so B1 already is the key
  // (except bin 0, which holds both NaN, key 0, and +-0, key 1)
  const bool kDirectT = Tr::kDirectT && B1 != 0;

  // fast path: every CTA's final candidates fit its window (bf16: they are
  // all equal to T, so only their per-CTA counts are exchanged and any number
  // fits).  Up to kFcCapBig in total they usually do; a CTA that overflows is
  // seen by every CTA after B2 and all of them take the slow path.
  bool fast = kDirectT || M + 2 <= kFcCapBig;
  if (fast) {
    // ================= fast path =================
    // Each CTA's FC region: [0] sure count, [1] FC count, [2..] FC keys in
    // index order, so one coalesced read of 32 words per CTA after B2 returns
    // every count and (usually) every key.
    Key* fcreg = reinterpret_cast<Key*>(a.fcreg) + (size_t)c * kFcCap;
    // One pass over the list: per-warp sure / FC counts, with the FC keys
    // staged in the (still unused) FC smem, kStageW per warp.
    constexpr uint32_t kStageW = kFcCap / 32;
    Key* stagew = sh_fckey + w * kStageW;
    {
      uint32_t ca = 0, cb = 0;
      const uint32_t lt = lanemask_lt();
      list_scan2<Tr>(list, L, [&](bool v0, uint32_t, Bits b0, bool v1, uint32_t, Bits b1) {
        const Key k0 = Tr::key(b0), k1 = Tr::key(b1);
        const uint32_t f0 = (uint32_t)(k0 >> FS), f1 = (uint32_t)(k1 >> FS);
        const bool fc0 = v0 && f0 == B1, fc1 = v1 && f1 == B1;
        const uint32_t m0 = __ballot_sync(kFull, fc0), m1 = __ballot_sync(kFull, fc1);
        ca += __popc(__ballot_sync(kFull, v0 && f0 > B1)) + __popc(__ballot_sync(kFull, v1 && f1 > B1));
        if (!kDirectT && (m0 | m1)) {
          const uint32_t p0 = cb + __popc(m0 & lt) + __popc(m1 & lt);
          if (fc0 && p0 < kStageW) stagew[p0] = k0;
          if (fc1 && p0 + fc0 < kStageW) stagew[p0 + fc0] = k1;
        }
        cb += __popc(m0) + __popc(m1);
      });
      if (lane == 0) {
        w_a[w] = ca;
        w_b[w] = cb;
      }
    }
    __syncthreads();
    if (w == 0) {
      const uint32_t va = w_a[lane], vb = w_b[lane];
      const uint32_t ia = warp_incl_scan(va), ib = warp_incl_scan(vb);
      w_aoff[lane] = ia - va;
      w_boff[lane] = ib - vb;
      if (lane == 31) {
        sh_res[8] = ia;
        sh_res[9] = ib;
      }
    }
    __syncthreads();
    if (!kDirectT) {  // publish the staged keys at the warp's place in the CTA's index order
      const uint32_t cb = w_b[w];
      Key* dst = fcreg + 2 + w_boff[w];
      const uint32_t room = sub_sat(kFcCap - 2, w_boff[w]);  // never past the CTA's region
      for (uint32_t i = lane; i < min(min(cb, kStageW), room); i += 32u) dst[i] = stagew[i];
      if (cb > kStageW && room > kStageW) {  // rare: this warp alone holds more than its staging share
        uint32_t r = 0;
        for (uint32_t base = 0; base < L; base += 32u) {
          const uint32_t j = base + lane;
          bool isfc = false;
          Key kk = 0;
          if (j < L) {
            uint32_t idx;
            Bits b;
            list.get(j, idx, b);
            kk = Tr::key(b);
            isfc = (uint32_t)(kk >> FS) == B1;
          }
          const uint32_t fm = __ballot_sync(kFull, isfc);
          const uint32_t p = r + __popc(fm & lanemask_lt());
          if (isfc && p >= kStageW && p < room) dst[p] = kk;
          r += __popc(fm);
        }
      }
    }
    if (tid == 0) {
      fcreg[0] = (Key)sh_res[8];
      fcreg[1] = (Key)sh_res[9];
    }
    // the rest of the 32-word window every CTA reads after B2 is written too
    // (zeros past the keys): an unwritten sector of it would be read from DRAM
    // on the critical path after an L2 flush, instead of from L2
    if (!kDirectT && tid >= 2 && tid < 32 && tid - 2 >= sh_res[9]) fcreg[tid] = (Key)0;
    if (tid < 256) {
      sh_lvl[tid] = 0u;  // radix digit histograms of stage 3 (two levels, alternating)
      sh_low[tid] = 0u;
    }
    if (tid < 2) sh_res[24 + tid] = 0u;
    STAMP(5);
    EXIT_AT(5);
    grid_barrier(bar, G);  // ---- B2
    STAMP(6);
    EXIT_AT(6);

    // ---- stage 3: one round trip for every CTA's window [sure count, FC
    // count, first kSpec-2 FC keys]; warp w handles CTAs w, w+32, ... with
    // lane j holding word j, so per-CTA sums are warp reductions.
    constexpr uint32_t kSpec = 32;
    static_assert(kSpec == 32, "one CTA window per warp");
    constexpr int R = (kMaxGridSpec + 31) / 32;
    Key* stage = reinterpret_cast<Key*>(smem + SL::coarse);  // coarse + window smem, free after stage 1
    static_assert(kMaxGridSpec * kSpec * sizeof(Key) <= (kCoarseBins + kWinBins) * 4, "staging fits");
    const Key* fcall = reinterpret_cast<const Key*>(a.fcreg);
    // the first radix level needs no prefix test (every FC key is in bin B1):
    // its digit histogram is built straight from the gathered registers
    const int nb0 = FS < 8 ? FS : 8;
    const int lob0 = FS - nb0;
    bool extra = false;  // some CTA holds more than kSpec-2 FC keys
    {
      Key v[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint32_t c2 = w + 32u * r;
        if (c2 < G) v[r] = fcall[(size_t)c2 * kFcCap + lane];
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint32_t c2 = w + 32u * r;
        if (c2 < G) {
          stage[c2 * kSpec + lane] = v[r];
          const uint32_t cnt = (uint32_t)__shfl_sync(kFull, v[r], 1);
          if (!kDirectT && lane >= 2 && lane - 2 < cnt)
            atomicAdd(&sh_lvl[(uint32_t)(v[r] >> lob0) & ((1u << nb0) - 1u)], 1u);
          extra |= cnt > kSpec - 2;
        }
      }
    }
    extra = __syncthreads_or(extra);
    STAMP(9);
    // Keys beyond the first kSpec-2 of a CTA (many FC keys, e.g. r = 10 on a
    // large tensor) are fetched once, in one round trip, into sh_fckey
    // (flattened; sh_fcoff[c2] = offset of CTA c2's extras, sh_fcoff[G] = total).
    bool xg = false;  // the extras exceed smem: read them from the CTA regions
    if (!kDirectT && extra) {
      if (w == 0) {
        const uint32_t per = (G + 31) / 32;
        uint32_t sx = 0, mx = 0;
        for (uint32_t i = 0; i < per; ++i) {
          const uint32_t c2 = lane * per + i;
          if (c2 < G) {
            sx += sub_sat((uint32_t)stage[c2 * kSpec + 1], kSpec - 2);
            mx = max(mx, (uint32_t)stage[c2 * kSpec + 1]);
          }
        }
        const uint32_t incl = warp_incl_scan(sx);
        mx = __reduce_max_sync(kFull, mx);
        uint32_t run = incl - sx;
        for (uint32_t i = 0; i < per; ++i) {
          const uint32_t c2 = lane * per + i;
          if (c2 < G) {
            sh_fcoff[c2] = run;
            run += sub_sat((uint32_t)stage[c2 * kSpec + 1], kSpec - 2);
          }
        }
        if (lane == 31) {
          sh_fcoff[G] = incl;
          sh_res[26] = mx > (uint32_t)kFcCap - 2;  // some CTA's keys overflowed its region
        }
      }
      __syncthreads();
      const uint32_t nx = sh_fcoff[G];
      if (sh_res[26]) {
        fast = false;  // the same decision in every CTA
      } else if (nx <= (uint32_t)kFcCap) {
        constexpr int PER = kFcCap / kCompressThreads;
        Key v[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) {
          const uint32_t p = tid + i * kCompressThreads;
          if (p < nx) {
            uint32_t lo = 0, hi = G;  // sh_fcoff[lo] <= p < sh_fcoff[hi]
            while (hi - lo > 1u) {
              const uint32_t mid = (lo + hi) >> 1;
              if (sh_fcoff[mid] <= p) lo = mid;
              else hi = mid;
            }
            v[i] = fcall[(size_t)lo * kFcCap + kSpec + (p - sh_fcoff[lo])];
          }
        }
#pragma unroll
        for (int i = 0; i < PER; ++i) {
          const uint32_t p = tid + i * kCompressThreads;
          if (p < nx) {
            sh_fckey[p] = v[i];
            atomicAdd(&sh_lvl[(uint32_t)(v[i] >> lob0) & ((1u << nb0) - 1u)], 1u);
          }
        }
        __syncthreads();
      } else {  // very many final candidates (r ~ 10 on >= 2^26 elements): extras stay in global memory
        xg = true;
        for (uint32_t r = 0; r < (G + 31) / 32; ++r) {
          const uint32_t c2 = w + 32u * r;
          if (c2 < G) {
            const uint32_t cnt = (uint32_t)stage[c2 * kSpec + 1];
            for (uint32_t j = kSpec - 2 + lane; j < cnt; j += 32u) {
              const Key kk = fcall[(size_t)c2 * kFcCap + 2 + j];
              atomicAdd(&sh_lvl[(uint32_t)(kk >> lob0) & ((1u << nb0) - 1u)], 1u);
            }
          }
        }
        __syncthreads();
      }
    }
    if (fast) {
    // every FC key of every CTA (staged window, then the CTA's extras);
    // fn(key) runs on this warp's lanes
    auto for_fc_keys = [&](uint32_t c2, auto&& fn) {
      const uint32_t cnt = (uint32_t)stage[c2 * kSpec + 1];
      if (lane >= 2 && lane - 2 < cnt) fn(stage[c2 * kSpec + lane]);
      for (uint32_t j = lane; j + (kSpec - 2) < cnt; j += 32u)
        fn(xg ? fcall[(size_t)c2 * kFcCap + kSpec + j] : sh_fckey[sh_fcoff[c2] + j]);
    };
    uint32_t need = k - G1;
    Key T = (Key)B1 << FS;
    if (kDirectT) {
      T |= 1;  // every FC key equals T; the tie quota is the whole need
    } else {
      // radix select over the low FS bits of the (unordered) final candidates
      for (int hib = FS, li = 0; hib > 0; ++li) {
        const int nb = hib < 8 ? hib : 8;
        const int lob = hib - nb;
        uint32_t* H = (li & 1) ? sh_low : sh_lvl;
        if (li > 0) {  // level 0 was counted during the gather
          for (int r = 0; r < R; ++r) {
            const uint32_t c2 = w + 32u * r;
            if (c2 < G)
              for_fc_keys(c2, [&](Key kk) {
                if ((kk >> hib) == (T >> hib)) atomicAdd(&H[(uint32_t)(kk >> lob) & ((1u << nb) - 1u)], 1u);
              });
          }
          __syncthreads();
        }
        if (w == 0) {
          uint32_t dig = 0, above = 0;
          warp_cross_desc(H, (1 << nb) - 1, need, &dig, &above);
          if (lane == 0) {
            sh_res[12] = dig;
            sh_res[13] = above;
          }
        }
        __syncthreads();
        T |= (Key)sh_res[12] << lob;
        need -= sh_res[13];
        hib = lob;
        if (tid < 256) H[tid] = 0u;  // reused two levels on, after at least one more barrier
      }
    }
    const uint32_t need_eq = need;  // number of key == T final candidates kept
    STAMP(7);
    EXIT_AT(7);
    // CTAs before this one: sure + (key > T) counts, and (key == T) counts;
    // this CTA's own FC keys (index order): per-position (gt, eq) prefix
    {
      uint32_t acc_a = 0, acc_e = 0;
      for (int r = 0; r < R; ++r) {
        const uint32_t c2 = w + 32u * r;
        if (c2 >= G || c2 > c) break;
        const uint32_t cnt = (uint32_t)stage[c2 * kSpec + 1];
        if (c2 < c) {
          uint32_t gt = 0, eq = 0;
          if (kDirectT) {
            eq = lane == 0 ? cnt : 0u;
          } else {
            for_fc_keys(c2, [&](Key kk) {
              gt += kk > T;
              eq += kk == T;
            });
          }
          acc_a += (lane == 0 ? (uint32_t)stage[c2 * kSpec] : 0u) + gt;
          acc_e += eq;
        } else if (!kDirectT) {  // own CTA: sh_fcpre[i] = (gt << 16) | eq over own keys before i
          uint32_t run = 0;
          for (uint32_t j0 = 0; j0 < cnt; j0 += 32u) {
            const uint32_t i = j0 + lane;
            Key kk = T;
            if (i < cnt && !kDirectT)
              kk = i < kSpec - 2 ? stage[c2 * kSpec + 2 + i]
                   : (xg ? fcall[(size_t)c2 * kFcCap + 2 + i] : sh_fckey[sh_fcoff[c2] + i - (kSpec - 2)]);
            const bool valid = i < cnt;
            const uint32_t v = valid ? ((kk > T ? 0x10000u : 0u) | (kk == T ? 1u : 0u)) : 0u;
            const uint32_t incl = warp_incl_scan(v);
            if (valid) sh_fcpre[i] = run + incl - v;
            run += __shfl_sync(kFull, incl, 31);
          }
          if (lane == 0) sh_fcpre[cnt] = run;
        }
      }
      acc_a = warp_sum(acc_a);
      acc_e = warp_sum(acc_e);
      if (lane == 0) {
        if (acc_a) atomicAdd(&sh_res[24], acc_a);
        if (acc_e) atomicAdd(&sh_res[25], acc_e);
      }
    }
    __syncthreads();
    STAMP(10);
    const uint32_t eq_before = sh_res[25];  // key == T final candidates in earlier CTAs
    const uint32_t kept_eq0 = min(eq_before, need_eq);
    // kept own final candidates before own FC position p
    auto fcsel = [&](uint32_t p) {
      if (kDirectT) return min(eq_before + p, need_eq) - kept_eq0;  // every own FC key == T
      const uint32_t v = sh_fcpre[p];
      return (v >> 16) + min(eq_before + (v & 0xFFFFu), need_eq) - kept_eq0;
    };
    uint32_t o = sh_res[24] + kept_eq0 + w_aoff[w] + fcsel(w_boff[w]);
    uint32_t jfc = w_boff[w];
    const uint32_t lt = lanemask_lt();
    auto walk = [&](auto frame_out) {
      list_scan2<Tr>(list, L, [&](bool v0, uint32_t i0, Bits b0, bool v1, uint32_t i1, Bits b1) {
        const Key k0 = Tr::key(b0), k1 = Tr::key(b1);
        const uint32_t f0 = (uint32_t)(k0 >> FS), f1 = (uint32_t)(k1 >> FS);
        const bool fc0 = v0 && f0 == B1, fc1 = v1 && f1 == B1;
        const uint32_t m0 = __ballot_sync(kFull, fc0), m1 = __ballot_sync(kFull, fc1);
        bool s0 = v0 && f0 > B1, s1 = v1 && f1 > B1;
        if (m0 | m1) {  // final candidates: T and the tie quota decide
          const uint32_t p0 = jfc + __popc(m0 & lt) + __popc(m1 & lt);
          if (kDirectT) {
            if (fc0) s0 = eq_before + p0 < need_eq;
            if (fc1) s1 = eq_before + p0 + fc0 < need_eq;
          } else {
            if (fc0) s0 = k0 > T || (k0 == T && eq_before + (sh_fcpre[p0] & 0xFFFFu) < need_eq);
            if (fc1) s1 = k1 > T || (k1 == T && eq_before + (sh_fcpre[p0 + fc0] & 0xFFFFu) < need_eq);
          }
          jfc += __popc(m0) + __popc(m1);
        }
        const uint32_t q0 = __ballot_sync(kFull, s0), q1 = __ballot_sync(kFull, s1);
        const uint32_t p = o + __popc(q0 & lt) + __popc(q1 & lt);
        if constexpr (decltype(frame_out)::value) {  // reference frame: i64 indices, f32 values
          if (s0) {
            reinterpret_cast<int64_t*>(a.idx_out)[p] = (int64_t)i0;
            reinterpret_cast<float*>(val_out)[p] = Tr::to_f32(b0);
          }
          if (s1) {
            reinterpret_cast<int64_t*>(a.idx_out)[p + s0] = (int64_t)i1;
            reinterpret_cast<float*>(val_out)[p + s0] = Tr::to_f32(b1);
          }
        } else {
          if (s0) write_out<Tr>(a, val_out, p, i0, b0);
          if (s1) write_out<Tr>(a, val_out, p + s0, i1, b1);
        }
        o += __popc(q0) + __popc(q1);
      });
    };
    if (a.idx64 && a.val_f32 && a.val2_out == nullptr) walk(std::true_type{});
    else walk(std::false_type{});
    list.discard(L);
    }  // fast (no CTA overflowed)
  }
  if (!fast) {
    // ================= slow path: many keys share the fine bin B1 =================
    uint32_t need = k - G1;
    Key T = (Key)B1 << FS;
    int lvl = 0;
    if (kDirectT) {
      T |= 1;
    } else {
      for (int hib = FS; hib > 0; ++lvl) {
        const int nb = hib < 8 ? hib : 8;
        const int lob = hib - nb;
        if (tid < 256) sh_lvl[tid] = 0u;
        __syncthreads();
        list_scan<Tr>(list, L, [&](bool valid, uint32_t, Bits b) {
          const Key kk = Tr::key(b);
          if (valid && (kk >> hib) == (T >> hib)) atomicAdd(&sh_lvl[(uint32_t)(kk >> lob) & ((1u << nb) - 1u)], 1u);
        });
        __syncthreads();
        if (tid < 256 && sh_lvl[tid]) red_add_gpu(&a.hist_lvl[lvl * 256 + tid], sh_lvl[tid]);
        grid_barrier(bar, G);
        if (tid < 256) sh_lvl[tid] = a.hist_lvl[lvl * 256 + tid];
        __syncthreads();
        if (w == 0) {
          uint32_t dig = 0, above = 0;
          warp_cross_desc(sh_lvl, (1 << nb) - 1, need, &dig, &above);
          if (lane == 0) {
            sh_res[12] = dig;
            sh_res[13] = above;
          }
        }
        __syncthreads();
        T |= (Key)sh_res[12] << lob;
        need -= sh_res[13];
        hib = lob;
      }
    }
    const uint32_t need_eq = need;
    {
      uint32_t gt = 0, eq = 0;
      list_scan<Tr>(list, L, [&](bool valid, uint32_t, Bits b) {
        const Key kk = Tr::key(b);
        gt += valid && kk > T;
        eq += valid && kk == T;
      });
      gt = warp_sum(gt);
      eq = warp_sum(eq);
      if (lane == 0) {
        w_a[w] = gt;
        w_b[w] = eq;
      }
    }
    __syncthreads();
    if (w == 0) {
      const uint32_t va = w_a[lane], vb = w_b[lane];
      const uint32_t ia = warp_incl_scan(va), ib = warp_incl_scan(vb);
      w_aoff[lane] = ia - va;
      w_boff[lane] = ib - vb;
      if (lane == 31) {
        a.cta_a[c] = ia;
        a.cta_b[c] = ib;
      }
    }
    grid_barrier(bar, G);
    {
      const uint32_t va = tid < G ? a.cta_a[tid] : 0u;
      const uint32_t vb = tid < G ? a.cta_b[tid] : 0u;
      uint32_t ta, tb;
      const uint32_t ea = block_excl_scan(va, sh32, &ta);
      const uint32_t eb = block_excl_scan(vb, sh32, &tb);
      if (tid == c) {
        sh_res[10] = ea;
        sh_res[11] = eb;
      }
    }
    __syncthreads();
    const uint32_t gt_c = sh_res[10], eq_c = sh_res[11];
    const uint32_t eqw = eq_c + w_boff[w];
    uint32_t o = gt_c + min(eq_c, need_eq) + w_aoff[w] + (min(eqw, need_eq) - min(eq_c, need_eq));
    uint32_t er = eqw;
    list_scan<Tr>(list, L, [&](bool valid, uint32_t idx, Bits b) {
      const Key kk = Tr::key(b);
      const bool iseq = valid && kk == T;
      const uint32_t em = __ballot_sync(kFull, iseq);
      const bool sel = valid && (kk > T || (iseq && er + __popc(em & lanemask_lt()) < need_eq));
      const uint32_t sm = __ballot_sync(kFull, sel);
      if (sel) write_out<Tr>(a, val_out, o + __popc(sm & lanemask_lt()), idx, b);
      o += __popc(sm);
      er += __popc(em);
    });
    list.discard(L);
    if (c == 0) {
      for (uint32_t i = tid; i < (uint32_t)(lvl * 256); i += kCompressThreads) a.hist_lvl[i] = 0u;
    }
  }
  STAMP(8);
  EXIT_AT(8);

  // ---- leave the workspace clean: the populated range of every replica,
  // [pop_lo, pop_hi), is zeroed in 1/G slices (one CTA per slice, not one per
  // contributor); all histogram / control reads happened before the last grid
  // barrier.
  {
    const uint32_t span = pop_hi > pop_lo ? pop_hi - pop_lo : 0u;
    for (uint32_t i = c * kCompressThreads + tid; i < span * kHistCopies; i += G * kCompressThreads)
      a.hist1[(size_t)(i / span) * kFineBinsMax + pop_lo + i % span] = 0u;
  }
  if (c == 0 && tid == 0) {
    ctrl[kCtrlMaxBin] = 0u;
    ctrl[kCtrlMaxLoBin] = 0u;
    ctrl[kCtrlMinLoBin] = 0u;
    ctrl[kCtrlCands] = 0u;
  }
}

// k == d: every element is kept, in index order.
template <class Tr>
__global__ void __launch_bounds__(256) keep_all_kernel(const CompressArgs a) {
  if (a.header != nullptr && blockIdx.x == 0 && threadIdx.x == 0) {
    a.header[0] = (unsigned long long)a.d;
    a.header[1] = (unsigned long long)a.k;
  }
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < a.d; i += gridDim.x * blockDim.x)
    write_out<Tr>(a, a.val_out, i, i, load_bits<Tr>(a.x, i));
}

// ---------------------------------------------------------------------------
// host side

// Fine-histogram resolution: 16 bits up to 2^23 elements, +1 bit per doubling
// (max 20), so the population of the threshold bin stays roughly constant.
#ifndef GP_FB_SHIFT
#define GP_FB_SHIFT 5
#endif
static int fine_bits_for(bool direct_t, uint64_t d) {
  if (direct_t) return 16;
  int fb = 16;
  while (fb < kFineBitsMax && (d >> (fb + GP_FB_SHIFT)) != 0) ++fb;
  return fb;
}
template <class Tr>
static int fine_bits(uint64_t d) {
  return fine_bits_for(Tr::kDirectT, d);
}

// Largest cooperative grid a length-d compress can launch on any device
// (launch_compress_t: G <= kMaxGridSpec and G <= ceil(d / kMinPerCta)).
static uint32_t grid_bound(uint64_t d) {
  return (uint32_t)std::min<uint64_t>(kMaxGridSpec, std::max<uint64_t>(1, (d + kMinPerCta - 1) / kMinPerCta));
}

template <class Tr>
static int launch_compress_t(CompressArgs a, const DeviceInfo& dev, cudaStream_t stream) {
  if (a.k == a.d && a.k_dev == nullptr) {
    const uint32_t blocks = (uint32_t)std::min<uint64_t>(((uint64_t)a.d + 255) / 256, (uint64_t)dev.num_sms * 8);
    keep_all_kernel<Tr><<<blocks, 256, 0, stream>>>(a);
    return cudaGetLastError() == cudaSuccess ? 0 : 5;
  }
  // per-device: the kernels' smem attribute set once and their occupancy (0 =
  // not yet known); concurrent first calls do the same idempotent setup
  static std::atomic<int> blocks_per_sm[kMaxDevices];
  const size_t smem = Smem<Tr>::total;
  if (dev.ordinal < 0 || dev.ordinal >= kMaxDevices) return 5;
  int nb = blocks_per_sm[dev.ordinal].load(std::memory_order_acquire);
  if (!nb) {
    if (cudaFuncSetAttribute(compress_kernel<Tr, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess ||
        cudaFuncSetAttribute(compress_kernel<Tr, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
      return 5;
    int nb2 = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, compress_kernel<Tr, false>, kCompressThreads, smem) !=
            cudaSuccess ||
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb2, compress_kernel<Tr, true>, kCompressThreads, smem) !=
            cudaSuccess)
      return 5;
    nb = std::min(nb, nb2);
    if (nb < 1) return 5;
    blocks_per_sm[dev.ordinal].store(nb, std::memory_order_release);
  }
  uint32_t gmax = (uint32_t)std::min(dev.num_sms * nb, kMaxGridSpec);
  if (dev.max_ctas > 0) gmax = std::min(gmax, (uint32_t)dev.max_ctas);
  const uint32_t G =
      (uint32_t)std::min<uint64_t>(gmax, std::max<uint64_t>(1, ((uint64_t)a.d + kMinPerCta - 1) / kMinPerCta));
  const uint64_t per_unit = ((uint64_t)a.d + (uint64_t)G * 32 - 1) / ((uint64_t)G * 32);
  a.W = (uint32_t)((per_unit + 15) & ~15ull);  // 32-byte aligned unit starts for every dtype
  a.fb = fine_bits<Tr>(a.d);

  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(kCompressThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  // watermark refinement for units of >= GP_REFINE_MIN_ROWS rows (see the kernel)
  const bool refine = (size_t)a.W * sizeof(typename Tr::Elem) >= kRefineMinUnitBytes;
  const cudaError_t e = refine ? cudaLaunchKernelEx(&cfg, compress_kernel<Tr, true>, a)
                               : cudaLaunchKernelEx(&cfg, compress_kernel<Tr, false>, a);
  return e == cudaSuccess ? 0 : 5;
}

int launch_compress(int dtype, CompressArgs a, const DeviceInfo& dev, cudaStream_t stream) {
  // vectors that fit one cluster's shared memory: gp_cluster.cu (no grid barriers)
  if (!(a.k == a.d && a.k_dev == nullptr)) {
    const int rc = launch_compress_cluster(dtype, a, dev, stream);
    if (rc >= 0) return rc;
  }
  switch (dtype) {
    case 0: return launch_compress_t<TraitsF32>(a, dev, stream);
    case 1: return launch_compress_t<TraitsBF16>(a, dev, stream);
    case 2: return launch_compress_t<TraitsF64>(a, dev, stream);
    default: return 6;
  }
}

// Workspace layout.  The state that must stay zeroed between calls (control
// words, level histograms, the fine histogram) sits at the front at offsets
// that depend only on ws_bytes: the fine histogram is sized for the largest
// vector any call could fit in ws_bytes (lists take >= 8 B per element, so
// d <= ws_bytes / 8).  Every call on a buffer therefore sees the same state
// region, whatever its d and dtype, and the per-call regions behind it (per-CTA
// counters and final-candidate regions sized by the grid d can get, candidate
// lists sized by d) never overlap it.
static size_t state_bytes(size_t ws_bytes) {
  auto up = [](size_t v) { return (v + 255) & ~(size_t)255; };
  const size_t nfine = (size_t)1 << fine_bits_for(false, ws_bytes / 8);
  return up(256) + up((size_t)8 * 256 * 4) + up(((size_t)(kHistCopies - 1) * kFineBinsMax + nfine) * 4);
}

size_t workspace_state_bytes(size_t ws_bytes) { return state_bytes(ws_bytes); }

size_t compress_workspace_layout(uint64_t d, int dtype, size_t ws_bytes, WsLayout* out) {
  const size_t entry = dtype == 2 ? 16 : 8;
  const size_t key = dtype == 2 ? 8 : 4;
  const size_t gmax = grid_bound(d);
  auto up = [](size_t v) { return (v + 255) & ~(size_t)255; };
  WsLayout l;
  size_t off = 0;
  l.ctrl = off;
  off = up(off + 256);
  l.hist_lvl = off;
  off = up(off + (size_t)8 * 256 * 4);
  l.hist1 = off;  // replica r at r * kFineBinsMax; capacity for any d that fits ws_bytes
  off = state_bytes(ws_bytes);
  l.cta_a = off;
  off = up(off + gmax * 4);
  l.cta_b = off;
  off = up(off + gmax * 4);
  l.fcreg = off;
  off = up(off + gmax * kFcCap * key);
  l.lists = off;
  off = up(off + ((size_t)d + gmax * 32 * 16) * entry);
  l.total = off;
  if (out) *out = l;
  return off;
}

// Smallest buffer whose layout fits a length-d compress: the fine histogram
// grows with the buffer, so iterate to the fixed point (a few steps at most).
size_t compress_workspace_bytes(uint64_t d, int dtype) {
  size_t ws = compress_workspace_layout(d, dtype, 0, nullptr);
  for (int i = 0; i < 8; ++i) {
    const size_t need = compress_workspace_layout(d, dtype, ws, nullptr);
    if (need <= ws) break;
    ws = need;
  }
  return ws;
}

}  // namespace gp
