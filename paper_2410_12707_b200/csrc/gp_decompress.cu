// gp_decompress.cu — AdaTopK decompress on sm_100a.
//
// Replaces topk_decompress (reference: pkg/src/geopipe/compressor.py:97-103):
//     if k and (indices.min() < 0 or indices.max() >= d): raise IndexOutOfRange
//     out = np.zeros(d, values.dtype); out[indices] = values
//
// Fast path (indices strictly increasing, as topk_compress emits them): four
// 512-thread CTAs per SM, each owning one contiguous output range.  One round
// of 512 probes around the interpolation guess k*o0/d brackets the range's
// first entry (a 32-ary warp search when the probes miss); then the range is
// produced as 16 KiB tiles built in shared memory (zeros, or for mode 1 --
// residual add, not in the reference -- the current contents), the tile's
// entries are streamed in coalesced batches and scattered into smem, and each
// full tile is written to HBM once by a bulk (TMA) shared->global store issued
// by one thread (three tile buffers rotate, so none is refilled before its
// store has read it).  No output line is touched twice: a zero-then-scatter in
// global memory re-reads every line a value lands in once the output exceeds
// L2.  Sparse payloads that fit in L2 take a fill+scatter kernel instead.  The
// same launch validates the index array: each CTA checks a 1/grid share of the
// k-1 adjacent pairs (strictly increasing) and CTA 0 checks idx[0] >= 0 and
// idx[k-1] < d; violations are reported in an asynchronous device flag
// (GP_FLAG_*).
//
// General path (unsorted / repeated indices) reproduces numpy's
// last-write-wins `out[indices] = values` with an atomicMax "winner" pass.
#include <algorithm>
#include <atomic>
#include <type_traits>

#include "gp_kernels.cuh"

namespace gp {

#ifndef GP_DEC_TILE_KB
#define GP_DEC_TILE_KB 16
#endif
#ifndef GP_DEC_BLOCKS_PER_SM
#define GP_DEC_BLOCKS_PER_SM 4
#endif
constexpr int kDecThreads = 512;
#ifndef GP_DEC_PROBES
#define GP_DEC_PROBES 128  // 512 before: -7 MB of probe reads per 205 MB r = 10 decompress, +1% (A/B)
#endif
// threads probing for a CTA's first entry: the probe window spans +-3 sigma of
// a uniform spread around the interpolation guess; its stride must stay below
// a batch (kDecThreads) so that the first batch brackets the entry
constexpr int kProbes = GP_DEC_PROBES;
static_assert(kProbes <= kDecThreads && kProbes % 32 == 0, "probes are whole warps of the CTA");
constexpr int kDecBlocksPerSm = GP_DEC_BLOCKS_PER_SM;
constexpr int kTileBytes = GP_DEC_TILE_KB * 1024;   // smem output tile
#ifndef GP_DEC_EVICT_FIRST
#define GP_DEC_EVICT_FIRST 1
#endif
#ifndef GP_DEC_TMA
#define GP_DEC_TMA 1
#endif
// full tiles leave shared memory by one bulk (TMA) store: three buffers, so a
// buffer is refilled only after its store has read it (no extra barrier)
constexpr int kTileBufs = GP_DEC_TMA ? 3 : 2;
constexpr int64_t kMinChunk = 8192;
#ifndef GP_SPARSE_DENSITY_INV
#define GP_SPARSE_DENSITY_INV 20
#endif
constexpr int64_t kSparseDensityInv = GP_SPARSE_DENSITY_INV;  // fill+scatter when k/d <= 1/this
constexpr int64_t kSparseMaxBytes = 64ll << 20;  // ... and the output fits well inside L2 (126 MB)

// ---- value conversions (exact for f32<->f64 widening and bf16<->f32 of bf16 values)
__device__ __forceinline__ float bf16_to_f32(uint16_t b) { return __uint_as_float((uint32_t)b << 16); }
__device__ __forceinline__ uint16_t f32_to_bf16_rn(float f) {
  uint32_t u = __float_as_uint(f);
  if ((u & 0x7FFFFFFFu) > 0x7F800000u) return (uint16_t)((u >> 16) | 0x40u);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

template <class T> struct Val;
template <> struct Val<float> {
  __device__ static double to_d(float v) { return (double)v; }
  __device__ static float to_f(float v) { return v; }
};
template <> struct Val<uint16_t> {
  __device__ static double to_d(uint16_t v) { return (double)bf16_to_f32(v); }
  __device__ static float to_f(uint16_t v) { return bf16_to_f32(v); }
};
template <> struct Val<double> {
  __device__ static double to_d(double v) { return v; }
  __device__ static float to_f(double v) { return __double2float_rn(v); }
};

template <class O, class V>
__device__ __forceinline__ O cvt(V v) {
  if constexpr (std::is_same<O, V>::value) return v;
  else if constexpr (std::is_same<O, double>::value) return Val<V>::to_d(v);
  else if constexpr (std::is_same<O, float>::value) return Val<V>::to_f(v);
  else return f32_to_bf16_rn(Val<V>::to_f(v));
}

template <class O>
__device__ __forceinline__ O add_vals(O a, O b) {
  if constexpr (std::is_same<O, uint16_t>::value) return f32_to_bf16_rn(bf16_to_f32(a) + bf16_to_f32(b));
  else return a + b;
}

// first j in [0, n) with idx[j] >= target (n if none), computed by one warp.
// The first round probes 32 positions around `guess` (k*target/d, exact for
// uniformly spread indices) with a stride of ~sqrt(n)/8, so for top-k payloads
// the bracket is usually found in one round trip and finished in a second.
template <class IT>
__device__ __forceinline__ int64_t warp_lower_bound(const IT* __restrict__ idx, int64_t n, int64_t target,
                                                    int64_t guess) {
  const uint32_t lane = threadIdx.x & 31;
  int64_t lo = 0, hi = n;
  if (n > 32) {
    const int64_t stride = max((int64_t)1, (int64_t)(sqrtf((float)n) * 0.125f));
    int64_t p = guess + ((int64_t)lane - 16) * stride;
    p = p < 0 ? 0 : (p >= n ? n - 1 : p);
    const bool pred = (int64_t)__ldg(idx + p) < target;
    const int cnt = __popc(__ballot_sync(kFull, pred));
    const int64_t below = __shfl_sync(kFull, p, cnt > 0 ? cnt - 1 : 0);
    const int64_t above = __shfl_sync(kFull, p, cnt < 32 ? cnt : 31);
    if (cnt > 0) lo = below + 1;
    if (cnt < 32) hi = above;
    if (lo > hi) lo = hi;  // only for unsorted input; the pair check flags it
  }
  while (hi - lo > 32) {
    const int64_t span = hi - lo;
    const int64_t p = lo + (span * (lane + 1)) / 33;
    const bool pred = (int64_t)__ldg(idx + p) < target;
    const int cnt = __popc(__ballot_sync(kFull, pred));
    const int64_t nlo = cnt > 0 ? lo + (span * cnt) / 33 + 1 : lo;
    const int64_t nhi = cnt < 32 ? lo + (span * (cnt + 1)) / 33 : hi;
    lo = nlo;
    hi = nhi;
  }
  const int64_t p = lo + lane;
  const bool pred = p < hi && (int64_t)__ldg(idx + p) < target;
  return lo + __popc(__ballot_sync(kFull, pred));
}

// The rest of a CTA's share of the adjacent-pair checks (idx[j] < idx[j+1]
// for j in [j0, pe), stride kDecThreads), four independent load pairs in
// flight per thread: at r = 10 a share is ~17 pairs per thread and a plain loop
// is a serial chain of round trips at the end of the kernel.
template <class IT>
__device__ __forceinline__ bool pair_check_rest(const IT* __restrict__ idx, int64_t j0, int64_t pe) {
  constexpr int U = 4;
  bool bad = false;
  for (int64_t j = j0; j < pe; j += U * kDecThreads) {
    IT a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t jj = j + (int64_t)u * kDecThreads;
      a[u] = 0;
      b[u] = 1;
      if (jj < pe) {
        a[u] = __ldg(idx + jj);
        b[u] = __ldg(idx + jj + 1);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) bad |= !((int64_t)a[u] < (int64_t)b[u]);
  }
  return bad;
}

template <class IT, class VT, class OT>
__global__ void __launch_bounds__(kDecThreads, kDecBlocksPerSm) decompress_kernel(
    const IT* __restrict__ idx, const VT* __restrict__ vals, int64_t k, int64_t d, int64_t chunk,
    OT* __restrict__ out, int mode_bits, uint32_t* err, unsigned long long* dbg, const unsigned long long* hdr,
    int dev_k) {
  constexpr int kTileElems = kTileBytes / (int)sizeof(OT);
  const int mode = mode_bits & 1;                // 1: residual add
  const bool trusted = (mode_bits & 2) != 0;     // indices from gp_topk_compress: no sortedness scan
  if (hdr != nullptr) {  // the frame's {d, k} header against what the receiver expects
    const unsigned long long hd = __ldg(hdr), hk = __ldg(hdr + 1);
    const bool ok = hd == (unsigned long long)d &&
                    (dev_k ? hk >= 1ull && hk <= (unsigned long long)k : hk == (unsigned long long)k);
    if (!ok) {
      if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(err, kFlagHeader);
      k = 0;  // nothing is scattered: zeros (mode 0) or the untouched residual (mode 1)
    } else if (dev_k) {
      k = (int64_t)hk;
      vals = reinterpret_cast<const VT*>(idx + k);  // reference frame: the values follow the k indices
    }
  }

  constexpr int kVecs = kTileBytes / 16;
#define DSTAMP(i)                                                \
  do {                                                           \
    if (dbg != nullptr && threadIdx.x == 0) {                    \
      unsigned long long t_;                                     \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));     \
      dbg[(size_t)blockIdx.x * 8 + (i)] = t_;                    \
    }                                                            \
  } while (0)
  DSTAMP(0);
  extern __shared__ __align__(128) unsigned char dec_smem[];  // kTileBufs tiles
  OT(*tiles)[kTileElems] = reinterpret_cast<OT(*)[kTileElems]>(dec_smem);
  __shared__ int64_t sh_lo;
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  const int64_t o0 = min((int64_t)blockIdx.x * chunk, d);
  const int64_t o1 = min(o0 + chunk, d);
  bool bad = false;
  // This CTA's 1/grid share of the k-1 adjacent-pair checks (covers every
  // pair whatever the input); the first pair per thread is loaded now and
  // compared at the end, so its latency overlaps the rest.
  const int64_t P = (k > 1 && !trusted) ? k - 1 : 0;  // adjacent pairs this launch checks
  const int64_t pb = (P * (int64_t)blockIdx.x) / gridDim.x;
  const int64_t pe = (P * ((int64_t)blockIdx.x + 1)) / gridDim.x;
  int64_t pa = 0, pz = 1;
  if (pb + tid < pe) {
    pa = (int64_t)__ldg(idx + pb + tid);
    pz = (int64_t)__ldg(idx + pb + tid + 1);
  }
  int64_t first = 0, last = 0;
  if (blockIdx.x == 0 && tid == 0 && k > 0) {
    first = (int64_t)__ldg(idx);
    last = (int64_t)__ldg(idx + k - 1);
  }
  // Entries are consumed in index order through a register window of one
  // entry per thread (batch of kDecThreads) with the next batch prefetched.
  // The first batch is loaded around the interpolation guess k*o0/d, so for
  // well-spread indices the start of this CTA's entries is found inside it
  // (a block count) with no separate search round trip.
  int64_t ci = 0, ni = 0;
  VT cv = VT(0), nv = VT(0);
  auto fetch = [&](int64_t b, int64_t& i, VT& v) {
    const int64_t j = b + tid;
    if (j >= 0 && j < k) {
      i = (int64_t)__ldg(idx + j);
      v = __ldg(vals + j);
      return true;
    }
    return false;
  };
  // Round trip 1: all threads probe the index array around the interpolation
  // guess k*o0/d with a stride covering +-3 sigma of a uniform spread, which
  // brackets lower_bound(o0) to within one stride (< one batch).  Round trip
  // 2 loads the batch starting at the bracket.  Clustered indices that the
  // probe window misses fall back to a 32-ary search.
  const int64_t guess = d ? (int64_t)((double)k * (double)o0 / (double)d) : 0;  // a guess; rounding is harmless
  const int64_t stride = max((int64_t)1, (int64_t)(3.0f * sqrtf((float)k) / kProbes) + 1);
  auto probe_pos = [&](int64_t t) {
    const int64_t p = guess + (t - kProbes / 2) * stride;
    return p < 0 ? (int64_t)0 : (p >= k ? k - 1 : p);
  };
  int64_t base = 0;
  if (k > 0) {
    const int64_t pv = tid < (uint32_t)kProbes ? (int64_t)__ldg(idx + probe_pos(tid)) : 0;
    // consume the early loads here (not at the end, where the compiler would
    // otherwise sink them into an extra serialized round trip)
    if (!(pa < pz)) bad = true;
    if (blockIdx.x == 0 && tid == 0 && (first < 0 || last >= d)) atomicOr(err, kFlagOutOfRange);
    const int below = __syncthreads_count(tid < (uint32_t)kProbes && pv < o0);
    const int64_t p_first = probe_pos(0), p_last = probe_pos(kProbes - 1);
    if ((below == 0 && p_first > 0) || (below == kProbes && p_last < k - 1)) {
      if (tid < 32) {  // probe window missed (clustered indices)
        const int64_t r = warp_lower_bound(idx, k, o0, guess);
        if (lane == 0) sh_lo = r;
      }
      __syncthreads();
      base = sh_lo;
    } else {
      base = below == 0 ? 0 : probe_pos(below - 1) + 1;  // lower_bound(o0) in [base, base + stride]
    }
  }
  const bool have = fetch(base, ci, cv);
  bool nhave = fetch(base + kDecThreads, ni, nv);
  bool pend = have && ci >= o0;  // entries below o0 belong to earlier CTAs
  DSTAMP(1);
  const bool vec_ok = ((uintptr_t)out % 16) == 0;
  int par = 0;
  DSTAMP(2);
  // Output tiles are built in shared memory (zeros or, mode 1, the current
  // contents), the tile's entries are scattered into smem, and the tile is
  // written once with 128-bit stores: every output line reaches HBM once.
  for (int64_t t0 = o0; t0 < o1; t0 += kTileElems, par = par + 1 == kTileBufs ? 0 : par + 1) {
    OT* tile = tiles[par];
    const int n = (int)min((int64_t)kTileElems, o1 - t0);
    const bool full = vec_ok && n == kTileElems;
    uint4* tv = reinterpret_cast<uint4*>(tile);
    if (mode == 0) {
      for (int i = tid; i < kVecs; i += kDecThreads) tv[i] = make_uint4(0u, 0u, 0u, 0u);
    } else if (full) {
      const uint4* ov = reinterpret_cast<const uint4*>(out + t0);
      for (int i = tid; i < kVecs; i += kDecThreads) tv[i] = ov[i];
    } else {
      for (int i = tid; i < n; i += kDecThreads) tile[i] = out[t0 + i];
    }
    __syncthreads();
    const int64_t t1 = t0 + n;
    for (;;) {
      if (pend && ci < t1) {
        if (ci >= t0) {
          const OT v = cvt<OT>(cv);
          tile[ci - t0] = mode == 0 ? v : add_vals<OT>(tile[ci - t0], v);
        } else {
          bad = true;  // below the tile: only possible for unsorted input
        }
        pend = false;
      }
      // barrier + "is the whole batch consumed?" (sorted input consumes prefixes)
      if (__syncthreads_count(pend) != 0 || base + kDecThreads >= k) break;
      base += kDecThreads;
      ci = ni;
      cv = nv;
      pend = nhave;
      nhave = fetch(base + kDecThreads, ni, nv);
    }
    if (full) {
      if (GP_DEC_TMA) {
        // the tile is complete (the loop left after a barrier): one thread
        // hands it to the bulk-copy engine; waiting until at most this group
        // is still reading keeps every buffer's refill, two tiles on, behind
        // a barrier that follows the wait
        if (tid == 0) {
          fence_proxy_async_smem();
          if (GP_DEC_EVICT_FIRST)  // output lines leave L2 first: the frame stays for the pair checks
            bulk_store_async_hint(out + t0, smem_addr(tile), (uint32_t)kTileBytes, l2_evict_first_policy());
          else
            bulk_store_async(out + t0, smem_addr(tile), (uint32_t)kTileBytes);
          bulk_commit();
          bulk_wait_read<1>();
        }
      } else {
        uint4* ov = reinterpret_cast<uint4*>(out + t0);
        for (int i = tid; i < kVecs; i += kDecThreads) ov[i] = tv[i];
      }
    } else {
      for (int i = tid; i < n; i += kDecThreads) out[t0 + i] = tile[i];
    }
  }
  if (GP_DEC_TMA && tid == 0) bulk_wait_all();  // the stores must finish before the CTA's smem goes away
  DSTAMP(3);
  if (pair_check_rest(idx, pb + tid + kDecThreads, pe)) bad = true;
  if (__syncthreads_or(bad) && tid == 0) atomicOr(err, kFlagUnsorted);
  DSTAMP(4);
#undef DSTAMP
}

// Sparse fast path (mode 0, k/d <= 1/20, output <= 64 MB): each CTA zero-fills
// its output range with 128-bit stores straight away, overlapping the round
// trips that locate its entries, then scatters those entries (after a CTA
// barrier, so each value lands after the zero written to its address by a
// sibling thread).  The output fits in L2, so the scattered sectors merge there
// and HBM still sees every output line once; no smem staging, no per-tile
// barriers.  (For larger outputs the fill evicts lines before the scatter and
// the tiled kernel wins.)  Validation is the same as the tiled kernel's.
template <class IT, class VT, class OT>
__global__ void __launch_bounds__(kDecThreads, kDecBlocksPerSm) decompress_sparse_kernel(
    const IT* __restrict__ idx, const VT* __restrict__ vals, int64_t k, int64_t d, int64_t chunk,
    OT* __restrict__ out, uint32_t* err, const unsigned long long* hdr, int dev_k, bool trusted) {
  if (hdr != nullptr) {  // the frame's {d, k} header against what the receiver expects
    const unsigned long long hd = __ldg(hdr), hk = __ldg(hdr + 1);
    const bool ok = hd == (unsigned long long)d &&
                    (dev_k ? hk >= 1ull && hk <= (unsigned long long)k : hk == (unsigned long long)k);
    if (!ok) {
      if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(err, kFlagHeader);
      k = 0;  // nothing is scattered: zeros (mode 0) or the untouched residual (mode 1)
    } else if (dev_k) {
      k = (int64_t)hk;
      vals = reinterpret_cast<const VT*>(idx + k);  // reference frame: the values follow the k indices
    }
  }
  const uint32_t tid = threadIdx.x;
  const int64_t o0 = min((int64_t)blockIdx.x * chunk, d);
  const int64_t o1 = min(o0 + chunk, d);
  bool bad = false;
  const int64_t P = (k > 1 && !trusted) ? k - 1 : 0;  // adjacent pairs this launch checks
  const int64_t pb = (P * (int64_t)blockIdx.x) / gridDim.x;
  const int64_t pe = (P * ((int64_t)blockIdx.x + 1)) / gridDim.x;
  int64_t pa = 0, pz = 1;
  if (pb + tid < pe) {
    pa = (int64_t)__ldg(idx + pb + tid);
    pz = (int64_t)__ldg(idx + pb + tid + 1);
  }
  int64_t first = 0, last = 0;
  if (blockIdx.x == 0 && tid == 0 && k > 0) {
    first = (int64_t)__ldg(idx);
    last = (int64_t)__ldg(idx + k - 1);
  }
  const int64_t guess = d ? (int64_t)((double)k * (double)o0 / (double)d) : 0;
  const int64_t stride = max((int64_t)1, (int64_t)(3.0f * sqrtf((float)k) / kProbes) + 1);
  auto probe_pos = [&](int64_t t) {
    const int64_t p = guess + (t - kProbes / 2) * stride;
    return p < 0 ? (int64_t)0 : (p >= k ? k - 1 : p);
  };
  int64_t pv = 0;
  if (k > 0 && tid < (uint32_t)kProbes) pv = (int64_t)__ldg(idx + probe_pos(tid));
  // zero fill of the whole range while the probes are in flight
  if (((uintptr_t)(out + o0) % 16) == 0) {
    constexpr int V = 16 / (int)sizeof(OT);
    const int64_t nvec = (o1 - o0) / V;
    uint4* ov = reinterpret_cast<uint4*>(out + o0);
    for (int64_t i = tid; i < nvec; i += kDecThreads) ov[i] = make_uint4(0u, 0u, 0u, 0u);
    for (int64_t i = o0 + nvec * V + tid; i < o1; i += kDecThreads) out[i] = OT(0);
  } else {
    for (int64_t i = o0 + tid; i < o1; i += kDecThreads) out[i] = OT(0);
  }
  if (k == 0) return;
  if (!(pa < pz)) bad = true;
  if (blockIdx.x == 0 && tid == 0 && (first < 0 || last >= d)) atomicOr(err, kFlagOutOfRange);
  __shared__ int64_t sh_lo;
  const int below = __syncthreads_count(tid < (uint32_t)kProbes && pv < o0);  // also orders the fill before the scatter
  int64_t base;
  const int64_t p_first = probe_pos(0), p_last = probe_pos(kProbes - 1);
  if ((below == 0 && p_first > 0) || (below == kProbes && p_last < k - 1)) {
    if (tid < 32) {  // probe window missed (clustered indices)
      const int64_t r = warp_lower_bound(idx, k, o0, guess);
      if ((tid & 31) == 0) sh_lo = r;
    }
    __syncthreads();
    base = sh_lo;
  } else {
    base = below == 0 ? 0 : probe_pos(below - 1) + 1;  // lower_bound(o0) in [base, base + stride]
  }
  for (;; base += kDecThreads) {
    const int64_t j = base + tid;
    bool past = j >= k;
    if (!past) {
      const int64_t i = (int64_t)__ldg(idx + j);
      if (i >= o1) past = true;
      else if (i >= o0) out[i] = cvt<OT>(__ldg(vals + j));  // base may trail lower_bound(o0) by < stride
    }
    if (__syncthreads_or(past)) break;
  }
  if (pair_check_rest(idx, pb + tid + kDecThreads, pe)) bad = true;
  if (__syncthreads_or(bad) && tid == 0) atomicOr(err, kFlagUnsorted);
}

// ---- general path
template <class OT>
__global__ void zero_kernel(OT* out, int64_t d) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < d; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = OT(0);
}

template <class IT>
__global__ void winner_kernel(const IT* idx, int64_t k, int64_t d, int32_t* win, uint32_t* err) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < k; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = (int64_t)idx[j];
    if (i < 0 || i >= d) atomicOr(err, kFlagOutOfRange);
    else atomicMax(&win[i], (int32_t)j);
  }
}

template <class IT, class VT, class OT>
__global__ void scatter_kernel(const IT* idx, const VT* vals, int64_t k, int64_t d, const int32_t* win, OT* out) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < k; j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = (int64_t)idx[j];
    if (i >= 0 && i < d && win[i] == (int32_t)j) out[i] = cvt<OT>(vals[j]);
  }
}

// ---- dispatch
template <class IT, class VT, class OT>
static int run_fast(const DecompressArgs& a, const DeviceInfo& dev, cudaStream_t s) {
  if (a.d <= 0) return 0;
  const int64_t blocks = std::min<int64_t>((int64_t)dev.num_sms * kDecBlocksPerSm, (a.d + kMinChunk - 1) / kMinChunk);
  int64_t chunk = (a.d + blocks - 1) / blocks;
  const int64_t tile_elems = kTileBytes / (int64_t)sizeof(OT);
  chunk = (chunk + tile_elems - 1) / tile_elems * tile_elems;  // whole, 16-byte aligned tiles
  const int64_t grid = (a.d + chunk - 1) / chunk;
  // 4 CTAs x 32 KiB per SM needs the max-shared carveout (set once per device; idempotent)
  static std::atomic<bool> carveout_set[kMaxDevices];
  if (dev.ordinal < 0 || dev.ordinal >= kMaxDevices) return 5;
  if (!carveout_set[dev.ordinal].load(std::memory_order_acquire)) {
    if (cudaFuncSetAttribute(decompress_kernel<IT, VT, OT>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared) != cudaSuccess ||
        cudaFuncSetAttribute(decompress_kernel<IT, VT, OT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kTileBufs * kTileBytes) != cudaSuccess)
      return 5;
    carveout_set[dev.ordinal].store(true, std::memory_order_release);
  }
  if ((a.mode & 1) == 0 && a.k * kSparseDensityInv <= a.d && a.d * (int64_t)sizeof(OT) <= kSparseMaxBytes) {
    decompress_sparse_kernel<IT, VT, OT><<<(unsigned)grid, kDecThreads, 0, s>>>(
        (const IT*)a.idx, (const VT*)a.vals, a.k, a.d, chunk, (OT*)a.out, a.err, a.hdr, a.dev_k, (a.mode & 2) != 0);
  } else {
    decompress_kernel<IT, VT, OT><<<(unsigned)grid, kDecThreads, kTileBufs * kTileBytes, s>>>(
        (const IT*)a.idx, (const VT*)a.vals, a.k, a.d, chunk, (OT*)a.out, a.mode, a.err, a.dbg, a.hdr, a.dev_k);
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}

template <class IT, class VT, class OT>
static int run_general(const DecompressArgs& a, void* scratch, const DeviceInfo& dev, cudaStream_t s) {
  const unsigned blocks = (unsigned)dev.num_sms * 8;
  zero_kernel<OT><<<blocks, 256, 0, s>>>((OT*)a.out, a.d);
  if (cudaMemsetAsync(scratch, 0xFF, (size_t)a.d * 4, s) != cudaSuccess) return 5;
  winner_kernel<IT><<<blocks, 256, 0, s>>>((const IT*)a.idx, a.k, a.d, (int32_t*)scratch, a.err);
  scatter_kernel<IT, VT, OT><<<blocks, 256, 0, s>>>((const IT*)a.idx, (const VT*)a.vals, a.k, a.d,
                                                    (const int32_t*)scratch, (OT*)a.out);
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}

template <class IT, class VT>
static int pick_out(const DecompressArgs& a, void* scratch, const DeviceInfo& dev, cudaStream_t s, bool general) {
  switch (a.out_dtype) {
    case 0: return general ? run_general<IT, VT, float>(a, scratch, dev, s) : run_fast<IT, VT, float>(a, dev, s);
    case 1: return general ? run_general<IT, VT, uint16_t>(a, scratch, dev, s) : run_fast<IT, VT, uint16_t>(a, dev, s);
    case 2: return general ? run_general<IT, VT, double>(a, scratch, dev, s) : run_fast<IT, VT, double>(a, dev, s);
    default: return 6;
  }
}

template <class IT>
static int pick_val(const DecompressArgs& a, void* scratch, const DeviceInfo& dev, cudaStream_t s, bool general) {
  switch (a.val_dtype) {
    case 0: return pick_out<IT, float>(a, scratch, dev, s, general);
    case 1: return pick_out<IT, uint16_t>(a, scratch, dev, s, general);
    case 2: return pick_out<IT, double>(a, scratch, dev, s, general);
    default: return 6;
  }
}

int launch_decompress(const DecompressArgs& a, const DeviceInfo& dev, cudaStream_t s) {
  return a.idx64 ? pick_val<int64_t>(a, nullptr, dev, s, false) : pick_val<int32_t>(a, nullptr, dev, s, false);
}

int launch_decompress_unsorted(const DecompressArgs& a, void* scratch, const DeviceInfo& dev, cudaStream_t s) {
  return a.idx64 ? pick_val<int64_t>(a, scratch, dev, s, true) : pick_val<int32_t>(a, scratch, dev, s, true);
}

}  // namespace gp

namespace gp {
// development aid: resident CTAs per SM of the fast decompress kernel (f32, i64 indices)
int debug_decompress_occupancy() {
  int nb = -1;
  cudaFuncSetAttribute(decompress_kernel<int64_t, float, float>, cudaFuncAttributePreferredSharedMemoryCarveout,
                       cudaSharedmemCarveoutMaxShared);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, decompress_kernel<int64_t, float, float>, kDecThreads,
                                                kTileBufs * kTileBytes);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, decompress_kernel<int64_t, float, float>);
  return nb * 1000000 + fa.numRegs * 1000 + (int)(fa.sharedSizeBytes / 1024);
}
}  // namespace gp
