// gp_compress.cu — AdaTopK compress on sm_100a.
//
// Replaces topk_compress (reference: pkg/src/geopipe/compressor.py:79-94):
//     order = np.argsort(-np.abs(flat), kind="stable"); kept = np.sort(order[:k])
//     values = flat[kept]
// i.e. the k largest |x| (NaN lowest, ties to the lower index), emitted in
// ascending index order.  No sort is performed; the kernel is a radix *select*
// followed by an index-ordered stream compaction, bit-exact with the reference.
//
// One persistent cooperative launch, 1024 threads x one CTA per SM.  The
// vector is split into G*32 contiguous "units", one per warp, in index order,
// so that a warp-ordered compaction of every unit concatenated in unit order
// is globally index ordered.
//
//   stage 0  every CTA draws the same stratified 2048-element sample, builds a
//            12-bit coarse histogram of its keys and picks a low watermark
//            lo0 whose expected population is ~k plus a 4-sigma margin;
//            meanwhile each warp issues a bulk L2 prefetch of its unit.
//   stage 1  the single full read of x: every element with key >= lo0 is a
//            candidate; candidates go into the warp's index-ordered list and a
//            16-bit "fine" histogram (smem window, flushed to L2 by red.add).
//            -- grid barrier B1 --
//   stage 2  every CTA scans the global fine histogram from the top and finds
//            the fine bin B1 holding the k-th largest key.  Keys above B1 are
//            certainly kept ("sure"); keys inside B1 are "final candidates".
//            Fast path (|B1| <= kFcCap): every CTA publishes its final
//            candidates, in index order, to its own region.  -- barrier B2 --
//   stage 3  every CTA loads the whole (small, index-ordered) final-candidate
//            list, resolves the exact threshold key T and the tie quota by an
//            in-smem radix select over the remaining low bits, derives its own
//            output offset, and each warp writes its kept (index, value) pairs.
//   slow path (|B1| > kFcCap) resolves the low bits with global per-level
//            histograms + barriers, then one more barrier for the tie prefix.
//   retry    if the sample overestimated lo0 (fewer than k candidates), stage 1
//            is redone with lo0 = 0.
//
// All histogram state is left zeroed for the next call; the grid barrier is
// self-resetting, so the workspace needs to be zeroed only once.
#include <algorithm>

#include "gp_kernels.cuh"

namespace gp {

// ---------------------------------------------------------------------------
// list entries: (global index, raw bits) — 8 B for 16/32-bit, 16 B for 64-bit

template <class Tr>
__device__ __forceinline__ void store_entry(void* base, uint32_t pos, uint32_t idx, typename Tr::Bits b) {
  if constexpr (sizeof(typename Tr::Bits) == 4) {
    reinterpret_cast<uint2*>(base)[pos] = make_uint2(idx, (uint32_t)b);
  } else {
    reinterpret_cast<uint4*>(base)[pos] = make_uint4(idx, 0u, (uint32_t)b, (uint32_t)((uint64_t)b >> 32));
  }
}

template <class Tr>
__device__ __forceinline__ void load_entry(const void* base, uint32_t pos, uint32_t& idx, typename Tr::Bits& b) {
  if constexpr (sizeof(typename Tr::Bits) == 4) {
    const uint2 e = __ldcg(reinterpret_cast<const uint2*>(base) + pos);
    idx = e.x;
    b = e.y;
  } else {
    const uint4 e = __ldcg(reinterpret_cast<const uint4*>(base) + pos);
    idx = e.x;
    b = (typename Tr::Bits)(((uint64_t)e.w << 32) | e.z);
  }
}

template <class Tr>
__device__ __forceinline__ typename Tr::Bits load_bits(const void* x, uint32_t i) {
  return (typename Tr::Bits)__ldg(reinterpret_cast<const typename Tr::Elem*>(x) + i);
}

// ---------------------------------------------------------------------------
// 1024-thread block scan / crossing search

__device__ __forceinline__ uint32_t block_incl_scan(uint32_t v, uint32_t* sh32, uint32_t* total) {
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t x = warp_incl_scan(v);
  if (lane == 31) sh32[w] = x;
  __syncthreads();
  if (w == 0) sh32[lane] = warp_incl_scan(sh32[lane]);
  __syncthreads();
  const uint32_t pre = w ? sh32[w - 1] : 0u;
  *total = sh32[31];
  __syncthreads();
  return x + pre;
}

// Thread t holds bins [4t, 4t+4) of a 4096-bin window (ascending).  Counting
// from the top, with `base` keys already above the window, find the bin b with
//     base + above(b) < target <= base + above(b) + h(b).
// Returns true (in every thread) when found; outputs are block-uniform.
__device__ __forceinline__ bool block_cross4(const uint32_t v[4], uint32_t base, uint32_t target,
                                             uint32_t* sh32, uint32_t* sh_res, uint32_t* bin,
                                             uint32_t* above, uint32_t* cnt, uint32_t* total) {
  if (threadIdx.x == 0) sh_res[0] = 0u;
  const uint32_t ts = v[0] + v[1] + v[2] + v[3];
  uint32_t tot;
  const uint32_t incl = block_incl_scan(ts, sh32, &tot);  // syncs order the reset above
  uint32_t run = base + (tot - incl);
#pragma unroll
  for (int b = 3; b >= 0; --b) {
    if (run < target && run + v[b] >= target) {
      sh_res[0] = 1u;
      sh_res[1] = 4u * threadIdx.x + (uint32_t)b;
      sh_res[2] = run;
      sh_res[3] = v[b];
    }
    run += v[b];
  }
  __syncthreads();
  const bool found = sh_res[0] != 0u;
  *bin = sh_res[1];
  *above = sh_res[2];
  *cnt = sh_res[3];
  *total = tot;
  __syncthreads();
  return found;
}

__device__ __forceinline__ uint32_t hash32(uint32_t s) {
  s ^= s >> 16;
  s *= 0x7feb352dU;
  s ^= s >> 15;
  s *= 0x846ca68bU;
  s ^= s >> 16;
  return s;
}

// ---------------------------------------------------------------------------
// output

template <class Tr>
__device__ __forceinline__ void write_out(const CompressArgs& a, uint32_t pos, uint32_t idx, typename Tr::Bits b) {
  using Elem = typename Tr::Elem;
  if (a.idx64) reinterpret_cast<int64_t*>(a.idx_out)[pos] = (int64_t)idx;
  else reinterpret_cast<int32_t*>(a.idx_out)[pos] = (int32_t)idx;
  if (a.val_f32) reinterpret_cast<float*>(a.val_out)[pos] = Tr::to_f32(b);
  else reinterpret_cast<Elem*>(a.val_out)[pos] = (Elem)b;
  if (a.val2_out) reinterpret_cast<Elem*>(a.val2_out)[pos] = (Elem)b;
}

// ---------------------------------------------------------------------------
// the kernel

template <class Tr>
__global__ void __launch_bounds__(kCompressThreads, 1) compress_kernel(const CompressArgs a) {
  using Bits = typename Tr::Bits;
  using Key = typename Tr::Key;
  using Elem = typename Tr::Elem;
  constexpr int FS = Tr::kKeyBits - 16;  // fine bin  = key >> FS  (16 bits)
  constexpr int CS = Tr::kKeyBits - 12;  // coarse bin = key >> CS (12 bits)
  constexpr int VEC = Tr::kVec;
  constexpr int U = 4;                   // 16-byte loads in flight per lane
  constexpr size_t kEntryBytes = sizeof(Bits) == 4 ? 8 : 16;

  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* sh_coarse = reinterpret_cast<uint32_t*>(smem);  // kCoarseBins
  uint32_t* sh_win = sh_coarse + kCoarseBins;                // kWinBins
  uint32_t* sh_low = sh_win + kWinBins;                      // kLowBins
  uint32_t* sh_lvl = sh_low + kLowBins;                      // 256
  uint32_t* sh32 = sh_lvl + 256;                             // 32
  uint32_t* sh_res = sh32 + 32;                              // 32
  uint32_t* w_len = sh_res + 32;                             // 32
  uint32_t* w_a = w_len + 32;
  uint32_t* w_b = w_a + 32;
  uint32_t* w_aoff = w_b + 32;
  uint32_t* w_boff = w_aoff + 32;
  uint32_t* sh_fcoff = w_boff + 32;                          // kMaxGrid + 4
  uint32_t* sh_fcpre = sh_fcoff + kMaxGrid + 4;              // kFcCap + 4
  Key* sh_fckey = reinterpret_cast<Key*>(sh_fcpre + kFcCap + 4);  // kFcCap

  const uint32_t G = gridDim.x, c = blockIdx.x, tid = threadIdx.x;
  const uint32_t lane = tid & 31, w = tid >> 5;
  const uint32_t d = a.d, k = a.k;
  const uint32_t unit = c * 32u + w;
  const uint32_t u0 = (uint32_t)min((uint64_t)unit * a.W, (uint64_t)d);
  const uint32_t u1 = (uint32_t)min((uint64_t)u0 + a.W, (uint64_t)d);
  const uint32_t n = u1 - u0;
  const Elem* x = reinterpret_cast<const Elem*>(a.x);
  unsigned char* my_list = reinterpret_cast<unsigned char*>(a.lists) + (size_t)unit * a.W * kEntryBytes;
  uint32_t* ctrl = a.ctrl;

  if (a.header != nullptr && c == 0 && tid == 0) {
    a.header[0] = (unsigned long long)d;
    a.header[1] = (unsigned long long)k;
  }

  // ---- stage 0: L2 prefetch of this warp's unit, sample-based low watermark
  if (lane == 0 && n > 0 && a.aligned) {
    const uint32_t bytes = (uint32_t)min((uint64_t)n * sizeof(Elem), (uint64_t)a.prefetch_bytes) & ~15u;
    if (bytes >= 16) prefetch_l2_bulk(x + u0, bytes);
  }
  for (uint32_t i = tid; i < kCoarseBins; i += kCompressThreads) sh_coarse[i] = 0u;
  if (tid == 0) sh_res[16] = 0u;
  __syncthreads();
  const uint32_t S = d < (uint32_t)kSamples ? d : (uint32_t)kSamples;
  {
    const uint32_t stride = d / S;
    for (uint32_t s = tid; s < S; s += kCompressThreads) {
      const uint32_t pos = (S == d) ? s : s * stride + hash32(s) % stride;
      const Key kk = Tr::key(load_bits<Tr>(x, pos));
      atomicAdd(&sh_coarse[(uint32_t)(kk >> CS)], 1u);
    }
  }
  __syncthreads();
  Key lo0 = 0;
  uint32_t cmax;  // highest non-empty coarse bin of the sample
  {
    uint32_t v[4], m = 0;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      v[b] = sh_coarse[4 * tid + b];
      if (v[b]) m = 4 * tid + b + 1;
    }
    m = __reduce_max_sync(kFull, m);
    if (lane == 0 && m) atomicMax(&sh_res[16], m);
    const double mu = (double)S * (double)k / (double)d;
    const double rs = ceil(mu + 4.0 * sqrt(mu) + 4.0);
    const bool want = rs < (double)S;
    uint32_t bin, above, cnt, tot;
    const bool found = block_cross4(v, 0u, want ? (uint32_t)rs : 0xFFFFFFFFu, sh32, sh_res, &bin, &above, &cnt, &tot);
    if (want && found) lo0 = (Key)bin << CS;
    cmax = sh_res[16] ? sh_res[16] - 1 : 0u;
  }
  const uint32_t top = min((uint32_t)kFineBins, ((cmax + 1u) << 4) + 512u);

  uint32_t L = 0;              // this warp's candidate count
  uint32_t B1 = 0, G1 = 0, M = 0, lobin = 0, maxb = 0;
  for (int attempt = 0;; ++attempt) {
    if (attempt == 1) lo0 = 0;
    lobin = (uint32_t)(lo0 >> FS);
    uint32_t wb = top > (uint32_t)kWinBins ? top - kWinBins : 0u;
    wb = max(wb, lobin);
    wb = min(wb, (uint32_t)(kFineBins - kWinBins));
    const uint32_t lowlim = min((uint32_t)kLowBins, wb);

    for (uint32_t i = tid; i < kWinBins; i += kCompressThreads) sh_win[i] = 0u;
    if (tid < kLowBins) sh_low[tid] = 0u;
    if (tid == 0) sh_res[17] = 0u;
    __syncthreads();

    // ---- stage 1: the one full pass over x
    L = 0;
    uint32_t mymax = 0;  // 1 + highest fine bin among my candidates
    auto hist_add = [&](uint32_t fb) {
      const uint32_t off = fb - wb;
      if (off < (uint32_t)kWinBins) atomicAdd(&sh_win[off], 1u);
      else if (fb < lowlim) atomicAdd(&sh_low[fb], 1u);
      else atomicAdd(&a.hist1[fb], 1u);
      mymax = max(mymax, fb + 1u);
    };
    const uint32_t nv = a.aligned ? n / VEC : 0u;
    const uint4* xv = reinterpret_cast<const uint4*>(x + u0);
    for (uint32_t v0 = 0; v0 < nv; v0 += 32u * U) {
      uint4 r[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const uint32_t vi = v0 + q * 32u + lane;
        r[q] = vi < nv ? ld_stream_v4(xv + vi) : make_uint4(0u, 0u, 0u, 0u);
      }
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const uint32_t vi = v0 + q * 32u + lane;
        uint32_t flags = 0;
        if (vi < nv) {
#pragma unroll
          for (int e = 0; e < VEC; ++e)
            if (Tr::key(Tr::lane(r[q], e)) >= lo0) flags |= 1u << e;
        }
        if (__any_sync(kFull, flags)) {
          const uint32_t cnt = __popc(flags);
          const uint32_t incl = warp_incl_scan(cnt);
          uint32_t pos = L + incl - cnt;
#pragma unroll
          for (int e = 0; e < VEC; ++e) {
            if ((flags >> e) & 1u) {
              const Bits b = Tr::lane(r[q], e);
              hist_add((uint32_t)(Tr::key(b) >> FS));
              store_entry<Tr>(my_list, pos++, u0 + vi * VEC + e, b);
            }
          }
          L += __shfl_sync(kFull, incl, 31);
        }
      }
    }
    for (uint32_t i0 = nv * VEC; i0 < n; i0 += 32u) {  // scalar tail / unaligned input
      const uint32_t i = i0 + lane;
      Bits b = 0;
      bool f = false;
      if (i < n) {
        b = load_bits<Tr>(x, u0 + i);
        f = Tr::key(b) >= lo0;
      }
      const uint32_t m = __ballot_sync(kFull, f);
      if (f) {
        hist_add((uint32_t)(Tr::key(b) >> FS));
        store_entry<Tr>(my_list, L + __popc(m & lanemask_lt()), u0 + i, b);
      }
      L += __popc(m);
    }
    mymax = __reduce_max_sync(kFull, mymax);
    if (lane == 0 && mymax) atomicMax(&sh_res[17], mymax);
    __syncthreads();
    for (uint32_t i = tid; i < kWinBins; i += kCompressThreads) {
      const uint32_t v = sh_win[i];
      if (v) red_add_gpu(&a.hist1[wb + i], v);
    }
    if (tid < lowlim && sh_low[tid]) red_add_gpu(&a.hist1[tid], sh_low[tid]);
    if (tid == 0 && sh_res[17]) atomicMax(&ctrl[kCtrlMaxBin], sh_res[17]);
    grid_barrier(&ctrl[kCtrlBarCount], &ctrl[kCtrlBarGen], G);  // ---- B1

    // ---- stage 2: locate the fine bin B1 that holds the k-th largest key
    maxb = __ldcg(&ctrl[kCtrlMaxBin]);
    bool found = false;
    {
      uint32_t base = 0;
      int hi = (int)maxb - 1;
      while (!found && hi >= (int)lobin) {
        const int cb = hi - 4095;
        uint32_t v[4];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int bin = cb + 4 * (int)tid + b;
          v[b] = (bin >= (int)lobin && bin <= hi) ? __ldcg(&a.hist1[bin]) : 0u;
        }
        uint32_t bin, above, cnt, tot;
        found = block_cross4(v, base, k, sh32, sh_res, &bin, &above, &cnt, &tot);
        if (found) {
          B1 = (uint32_t)(cb + (int)bin);
          G1 = above;
          M = cnt;
        }
        base += tot;
        hi = cb - 1;
      }
    }
    if (found) break;
    // lo0 overestimated: clear and redo stage 1 with every element a candidate
    grid_barrier(&ctrl[kCtrlBarCount], &ctrl[kCtrlBarGen], G);
    {
      const uint32_t span = maxb > lobin ? maxb - lobin : 0u;
      const uint32_t z0 = lobin + (uint32_t)(((uint64_t)span * c) / G);
      const uint32_t z1 = lobin + (uint32_t)(((uint64_t)span * (c + 1)) / G);
      for (uint32_t i = z0 + tid; i < z1; i += kCompressThreads) a.hist1[i] = 0u;
      if (c == 0 && tid == 0) ctrl[kCtrlMaxBin] = 0u;
    }
    grid_barrier(&ctrl[kCtrlBarCount], &ctrl[kCtrlBarGen], G);
  }

  // per-warp split of my candidates: sure (fine bin > B1) / final (== B1)
  {
    uint32_t ca = 0, cb = 0;
    for (uint32_t j = lane; j < L; j += 32u) {
      uint32_t idx;
      Bits b;
      load_entry<Tr>(my_list, j, idx, b);
      const uint32_t fb = (uint32_t)(Tr::key(b) >> FS);
      ca += fb > B1;
      cb += fb == B1;
    }
    ca = warp_sum(ca);
    cb = warp_sum(cb);
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

  if (M <= (uint32_t)kFcCap) {
    // ================= fast path =================
    Key* fcreg = reinterpret_cast<Key*>(a.fcreg) + (size_t)c * kFcCap;
    {
      uint32_t j0 = w_boff[w];
      for (uint32_t base = 0; base < L; base += 32u) {
        const uint32_t j = base + lane;
        bool isfc = false;
        Key kk = 0;
        if (j < L) {
          uint32_t idx;
          Bits b;
          load_entry<Tr>(my_list, j, idx, b);
          kk = Tr::key(b);
          isfc = (uint32_t)(kk >> FS) == B1;
        }
        const uint32_t m = __ballot_sync(kFull, isfc);
        if (isfc) fcreg[j0 + __popc(m & lanemask_lt())] = kk;
        j0 += __popc(m);
      }
    }
    if (tid == 0) {
      a.cta_a[c] = sh_res[8];
      a.cta_b[c] = sh_res[9];
    }
    grid_barrier(&ctrl[kCtrlBarCount], &ctrl[kCtrlBarGen], G);  // ---- B2

    // ---- stage 3: exact threshold inside B1, offsets, output
    {
      const uint32_t va = tid < G ? __ldcg(&a.cta_a[tid]) : 0u;
      const uint32_t vb = tid < G ? __ldcg(&a.cta_b[tid]) : 0u;
      uint32_t ta, tb;
      const uint32_t ia = block_incl_scan(va, sh32, &ta);
      const uint32_t ib = block_incl_scan(vb, sh32, &tb);
      if (tid < G) sh_fcoff[tid] = ib - vb;
      if (tid == 0) sh_fcoff[G] = tb;
      if (tid == c) sh_res[10] = ia - va;
    }
    __syncthreads();
    const uint32_t Mt = sh_fcoff[G];
    const uint32_t sure_off = sh_res[10];
    for (uint32_t p = tid; p < Mt; p += kCompressThreads) {
      uint32_t lo = 0, hi = G - 1;
      while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (sh_fcoff[mid] <= p) lo = mid;
        else hi = mid - 1;
      }
      sh_fckey[p] = __ldcg(reinterpret_cast<const Key*>(a.fcreg) + (size_t)lo * kFcCap + (p - sh_fcoff[lo]));
    }
    __syncthreads();
    // in-smem radix select over the low FS bits of the final candidates
    uint32_t need = k - G1;
    Key T = (Key)B1 << FS;
    for (int hib = FS; hib > 0;) {
      const int nb = hib < 8 ? hib : 8;
      const int lob = hib - nb;
      if (tid < 256) sh_lvl[tid] = 0u;
      __syncthreads();
      for (uint32_t p = tid; p < Mt; p += kCompressThreads) {
        const Key kk = sh_fckey[p];
        if ((kk >> hib) == (T >> hib)) atomicAdd(&sh_lvl[(uint32_t)(kk >> lob) & ((1u << nb) - 1u)], 1u);
      }
      __syncthreads();
      uint32_t v[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) v[b] = (4 * tid + b < 256u) ? sh_lvl[4 * tid + b] : 0u;
      uint32_t dig, above, cnt, tot;
      block_cross4(v, 0u, need, sh32, sh_res, &dig, &above, &cnt, &tot);
      T |= (Key)dig << lob;
      need -= above;
      hib = lob;
    }
    const uint32_t need_eq = need;  // number of key == T final candidates kept
    {
      uint32_t pk[4], s = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const uint32_t p = 4 * tid + b;
        uint32_t v = 0;
        if (p < Mt) {
          const Key kk = sh_fckey[p];
          v = (kk > T ? 0x10000u : 0u) | (kk == T ? 1u : 0u);
        }
        pk[b] = v;
        s += v;
      }
      uint32_t tot;
      uint32_t run = block_incl_scan(s, sh32, &tot) - s;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        sh_fcpre[4 * tid + b] = run;
        run += pk[b];
      }
      if (tid == 0) sh_fcpre[kFcCap] = tot;
    }
    __syncthreads();
    auto fcsel = [&](uint32_t p) {
      const uint32_t v = sh_fcpre[p];
      return (v >> 16) + min(v & 0xFFFFu, need_eq);
    };
    const uint32_t fc_c = sh_fcoff[c];
    const uint32_t fcw = fc_c + w_boff[w];
    uint32_t o = sure_off + fcsel(fc_c) + w_aoff[w] + (fcsel(fcw) - fcsel(fc_c));
    uint32_t jfc = fcw;
    for (uint32_t base = 0; base < L; base += 32u) {
      const uint32_t j = base + lane;
      uint32_t idx = 0;
      Bits b = 0;
      Key kk = 0;
      uint32_t fb = 0;
      const bool valid = j < L;
      if (valid) {
        load_entry<Tr>(my_list, j, idx, b);
        kk = Tr::key(b);
        fb = (uint32_t)(kk >> FS);
      }
      const bool isfc = valid && fb == B1;
      const uint32_t fm = __ballot_sync(kFull, isfc);
      const uint32_t p = jfc + __popc(fm & lanemask_lt());
      const bool sel = valid && (fb > B1 || (isfc && (kk > T || (kk == T && (sh_fcpre[p] & 0xFFFFu) < need_eq))));
      const uint32_t sm = __ballot_sync(kFull, sel);
      if (sel) write_out<Tr>(a, o + __popc(sm & lanemask_lt()), idx, b);
      o += __popc(sm);
      jfc += __popc(fm);
    }
  } else {
    // ================= slow path: many keys share the fine bin B1 =================
    uint32_t need = k - G1;
    Key T = (Key)B1 << FS;
    int lvl = 0;
    for (int hib = FS; hib > 0; ++lvl) {
      const int nb = hib < 8 ? hib : 8;
      const int lob = hib - nb;
      if (tid < 256) sh_lvl[tid] = 0u;
      __syncthreads();
      for (uint32_t j = lane; j < L; j += 32u) {
        uint32_t idx;
        Bits b;
        load_entry<Tr>(my_list, j, idx, b);
        const Key kk = Tr::key(b);
        if ((kk >> hib) == (T >> hib)) atomicAdd(&sh_lvl[(uint32_t)(kk >> lob) & ((1u << nb) - 1u)], 1u);
      }
      __syncthreads();
      if (tid < 256 && sh_lvl[tid]) red_add_gpu(&a.hist_lvl[lvl * 256 + tid], sh_lvl[tid]);
      grid_barrier(&ctrl[kCtrlBarCount], &ctrl[kCtrlBarGen], G);
      uint32_t v[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) v[b] = (4 * tid + b < 256u) ? __ldcg(&a.hist_lvl[lvl * 256 + 4 * tid + b]) : 0u;
      uint32_t dig, above, cnt, tot;
      block_cross4(v, 0u, need, sh32, sh_res, &dig, &above, &cnt, &tot);
      T |= (Key)dig << lob;
      need -= above;
      hib = lob;
    }
    const uint32_t need_eq = need;
    {
      uint32_t gt = 0, eq = 0;
      for (uint32_t j = lane; j < L; j += 32u) {
        uint32_t idx;
        Bits b;
        load_entry<Tr>(my_list, j, idx, b);
        const Key kk = Tr::key(b);
        gt += kk > T;
        eq += kk == T;
      }
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
    grid_barrier(&ctrl[kCtrlBarCount], &ctrl[kCtrlBarGen], G);
    {
      const uint32_t va = tid < G ? __ldcg(&a.cta_a[tid]) : 0u;
      const uint32_t vb = tid < G ? __ldcg(&a.cta_b[tid]) : 0u;
      uint32_t ta, tb;
      const uint32_t ia = block_incl_scan(va, sh32, &ta);
      const uint32_t ib = block_incl_scan(vb, sh32, &tb);
      if (tid == c) {
        sh_res[10] = ia - va;
        sh_res[11] = ib - vb;
      }
    }
    __syncthreads();
    const uint32_t gt_c = sh_res[10], eq_c = sh_res[11];
    const uint32_t eqw = eq_c + w_boff[w];
    uint32_t o = gt_c + min(eq_c, need_eq) + w_aoff[w] + (min(eqw, need_eq) - min(eq_c, need_eq));
    uint32_t er = eqw;
    for (uint32_t base = 0; base < L; base += 32u) {
      const uint32_t j = base + lane;
      uint32_t idx = 0;
      Bits b = 0;
      Key kk = 0;
      const bool valid = j < L;
      if (valid) {
        load_entry<Tr>(my_list, j, idx, b);
        kk = Tr::key(b);
      }
      const bool iseq = valid && kk == T;
      const uint32_t em = __ballot_sync(kFull, iseq);
      const bool sel = valid && (kk > T || (iseq && er + __popc(em & lanemask_lt()) < need_eq));
      const uint32_t sm = __ballot_sync(kFull, sel);
      if (sel) write_out<Tr>(a, o + __popc(sm & lanemask_lt()), idx, b);
      o += __popc(sm);
      er += __popc(em);
    }
    if (c == 0) {
      for (uint32_t i = tid; i < (uint32_t)(lvl * 256); i += kCompressThreads) a.hist_lvl[i] = 0u;
    }
  }

  // ---- leave the workspace clean: every histogram bin that can be non-zero
  // lies in [lobin, maxb); all reads of hist1 / maxbin happened before the
  // last barrier.
  {
    const uint32_t span = maxb > lobin ? maxb - lobin : 0u;
    const uint32_t z0 = lobin + (uint32_t)(((uint64_t)span * c) / G);
    const uint32_t z1 = lobin + (uint32_t)(((uint64_t)span * (c + 1)) / G);
    for (uint32_t i = z0 + tid; i < z1; i += kCompressThreads) a.hist1[i] = 0u;
    if (c == 0 && tid == 0) ctrl[kCtrlMaxBin] = 0u;
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
    write_out<Tr>(a, i, i, load_bits<Tr>(a.x, i));
}

// ---------------------------------------------------------------------------
// host side

template <class Tr>
static size_t compress_smem_bytes() {
  return (size_t)(kCoarseBins + kWinBins + kLowBins + 256 + 32 * 8 + kMaxGrid + 4 + kFcCap + 4) * 4 +
         (size_t)kFcCap * sizeof(typename Tr::Key);
}

template <class Tr>
static int launch_compress_t(CompressArgs a, const DeviceInfo& dev, cudaStream_t stream) {
  if (a.k == a.d) {
    const uint32_t blocks = (uint32_t)std::min<uint64_t>(((uint64_t)a.d + 255) / 256, (uint64_t)dev.num_sms * 8);
    keep_all_kernel<Tr><<<blocks, 256, 0, stream>>>(a);
    return cudaGetLastError() == cudaSuccess ? 0 : 5;
  }
  static int configured[64] = {0};
  static int max_blocks_per_sm[64] = {0};
  const size_t smem = compress_smem_bytes<Tr>();
  if (!configured[dev.ordinal]) {
    if (cudaFuncSetAttribute(compress_kernel<Tr>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return 5;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, compress_kernel<Tr>, kCompressThreads, smem) != cudaSuccess ||
        nb < 1)
      return 5;
    max_blocks_per_sm[dev.ordinal] = nb;
    configured[dev.ordinal] = 1;
  }
  const uint32_t gmax = (uint32_t)std::min(dev.num_sms * max_blocks_per_sm[dev.ordinal], kMaxGrid);
  uint32_t G = (uint32_t)std::min<uint64_t>(gmax, std::max<uint64_t>(1, ((uint64_t)a.d + kMinPerCta - 1) / kMinPerCta));
  const uint64_t per_unit = ((uint64_t)a.d + (uint64_t)G * 32 - 1) / ((uint64_t)G * 32);
  a.W = (uint32_t)((per_unit + 7) & ~7ull);
  const uint64_t total_bytes = (uint64_t)a.d * sizeof(typename Tr::Elem);
  const uint64_t budget = 64ull << 20;  // keep the prefetched prefix within L2
  a.prefetch_bytes = (uint32_t)std::min<uint64_t>(
      total_bytes <= budget ? (uint64_t)a.W * sizeof(typename Tr::Elem) : budget / ((uint64_t)G * 32), 1u << 30);

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
  return cudaLaunchKernelEx(&cfg, compress_kernel<Tr>, a) == cudaSuccess ? 0 : 5;
}

int launch_compress(int dtype, CompressArgs a, const DeviceInfo& dev, cudaStream_t stream) {
  switch (dtype) {
    case 0: return launch_compress_t<TraitsF32>(a, dev, stream);
    case 1: return launch_compress_t<TraitsBF16>(a, dev, stream);
    case 2: return launch_compress_t<TraitsF64>(a, dev, stream);
    default: return 6;
  }
}

size_t compress_workspace_layout(uint64_t d, int dtype, int gmax, WsLayout* out) {
  const size_t entry = dtype == 2 ? 16 : 8;
  const size_t key = dtype == 2 ? 8 : 4;
  auto up = [](size_t v) { return (v + 255) & ~(size_t)255; };
  WsLayout l;
  size_t off = 0;
  l.ctrl = off;
  off = up(off + 256);
  l.hist1 = off;
  off = up(off + (size_t)kFineBins * 4);
  l.hist_lvl = off;
  off = up(off + (size_t)8 * 256 * 4);
  l.cta_a = off;
  off = up(off + (size_t)kMaxGrid * 4);
  l.cta_b = off;
  off = up(off + (size_t)kMaxGrid * 4);
  l.fcreg = off;
  off = up(off + (size_t)gmax * kFcCap * key);
  l.lists = off;
  off = up(off + ((size_t)d + (size_t)gmax * 32 * 8) * entry);
  l.total = off;
  if (out) *out = l;
  return off;
}

}  // namespace gp
