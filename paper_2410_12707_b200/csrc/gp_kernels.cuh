// gp_kernels.cuh — internal interfaces between the C-ABI layer and the kernels.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "gp_common.cuh"

namespace gp {

constexpr int kCompressThreads = 1024;  // 32 warps; block scans assume exactly this
constexpr int kMaxGrid = 1024;          // max CTAs of the cooperative compress grid
#ifndef GP_MIN_PER_CTA
#define GP_MIN_PER_CTA 16384
#endif
constexpr int kMinPerCta = GP_MIN_PER_CTA;  // elements per CTA below which the grid shrinks
constexpr int kCoarseBins = 1 << 12;    // sample histogram (key >> (bits-12))
constexpr int kFineBitsMax = 20;        // fine candidate histogram: 16..20 bits (grows with d)
constexpr int kFineBinsMax = 1 << kFineBitsMax;
constexpr int kWinBins = 8192;          // smem window of the fine histogram
constexpr int kLowBins = 256;           // smem low window (zeros, NaN, denormals)
constexpr int kFcCap = 8192;            // final-candidate capacity of the fast path

// control words at the head of the workspace
#ifndef GP_HIST_COPIES
#define GP_HIST_COPIES 1
#endif
constexpr int kHistCopies = GP_HIST_COPIES;  // replicas of the fine histogram (CTA c uses c % copies)
constexpr int kCtrlBar = 0;             // grid-barrier word (top bit flips per barrier)
constexpr int kCtrlMaxBin = 2;          // 1 + highest fine bin with a candidate
constexpr int kCtrlMaxLoBin = 3;        // 1 + highest per-CTA watermark bin
constexpr int kCtrlCands = 4;           // total candidates of stage 1
constexpr int kCtrlMinLoBin = 5;        // ~(lowest per-CTA watermark bin), via atomicMax

// asynchronous device error flags (include/adatopk.h GP_FLAG_*)
constexpr uint32_t kFlagOutOfRange = 1u;
constexpr uint32_t kFlagUnsorted = 2u;
constexpr uint32_t kFlagHeader = 4u;
constexpr uint32_t kFlagBadK = 8u;

struct CompressArgs {
  const void* x;
  uint32_t d;
  uint32_t k;
  void* idx_out;
  int idx64;
  void* val_out;
  int val_f32;
  void* val2_out;
  unsigned long long* header;
  uint32_t* ctrl;
  uint32_t* hist1;
  uint32_t* hist_lvl;
  uint32_t* cta_a;
  uint32_t* cta_b;
  void* fcreg;
  void* lists;
  uint32_t W;               // elements per warp unit (multiple of 8), set by the launcher
  int aligned;              // x is 32-byte aligned (256-bit row loads)
  int fb;                   // fine-histogram bits, set by the launcher
  unsigned long long* dbg;  // optional per-CTA stage timestamps (32 words per CTA)
  // device-resident k (adaptive plans without a host round trip): when set,
  // k = *k_dev, bounded by the capacity a.k; with frame_vals the values start
  // right after the k indices (reference frame layout), so val_out is derived
  const long long* k_dev;
  int frame_vals;
  uint32_t* err;            // GP_FLAG_BAD_K when *k_dev is outside [1, min(k_cap, d)]
};

struct WsLayout {
  size_t ctrl, hist1, hist_lvl, cta_a, cta_b, fcreg, lists, total;
};

constexpr int kMaxDevices = 64;  // per-device launch configuration caches

struct DeviceInfo {
  int ordinal;
  int num_sms;
  int max_ctas = 0;  // compress grid cap (0: one CTA per SM); lets independent compresses share the GPU
};

int launch_compress(int dtype, CompressArgs a, const DeviceInfo& dev, cudaStream_t stream);
// one-cluster compress of a short vector (gp_cluster.cu); -1 when not applicable
int launch_compress_cluster(int dtype, const CompressArgs& a, const DeviceInfo& dev, cudaStream_t stream);
int cluster_path_mode();
int set_cluster_path(int mode);  // returns the previous mode
size_t compress_workspace_layout(uint64_t d, int dtype, size_t ws_bytes, WsLayout* out);
size_t compress_workspace_bytes(uint64_t d, int dtype);
size_t workspace_state_bytes(size_t ws_bytes);

struct DecompressArgs {
  const void* idx;
  int idx64;
  const void* vals;
  int val_dtype;
  int64_t k;
  int64_t d;
  void* out;
  int out_dtype;
  int mode;
  uint32_t* err;
  unsigned long long* dbg;  // optional per-CTA stage timestamps (8 words per CTA)
  // frame header {d, k} to validate (nullable): GP_FLAG_HEADER on a mismatch.
  // dev_k: k is read from the header (bounded by the capacity a.k) and the
  // values start right after the k indices.
  const unsigned long long* hdr;
  int dev_k;
};

int launch_decompress(const DecompressArgs& a, const DeviceInfo& dev, cudaStream_t stream);
int launch_decompress_unsorted(const DecompressArgs& a, void* scratch, const DeviceInfo& dev, cudaStream_t stream);

int launch_adatopk_plan(const double* R, int n, double base_ratio, const int64_t* d_per_link, double* r_out,
                        int64_t* k_out, int32_t* status, cudaStream_t stream);

}  // namespace gp
