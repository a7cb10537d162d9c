// gp_kernels.cuh — internal interfaces between the C-ABI layer and the kernels.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "gp_common.cuh"

namespace gp {

constexpr int kCompressThreads = 1024;  // 32 warps; block scans assume exactly this
constexpr int kMaxGrid = 1024;          // max CTAs of the cooperative compress grid
constexpr int kMinPerCta = 16384;       // elements per CTA below which the grid shrinks
constexpr int kCoarseBins = 1 << 12;    // sample histogram (key >> (bits-12))
constexpr int kFineBins = 1 << 16;      // global candidate histogram (key >> (bits-16))
constexpr int kWinBins = 8192;          // smem window of the fine histogram
constexpr int kLowBins = 256;           // smem low window (zeros, NaN, denormals)
constexpr int kFcCap = 4096;            // final-candidate capacity of the fast path
constexpr int kSamples = 2048;          // sample size of the watermark estimate

// control words at the head of the workspace
constexpr int kCtrlBarCount = 0;
constexpr int kCtrlBarGen = 1;
constexpr int kCtrlMaxBin = 2;

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
  uint32_t prefetch_bytes;  // per-unit L2 prefetch length, set by the launcher
  int aligned;              // x is 16-byte aligned
};

struct WsLayout {
  size_t ctrl, hist1, hist_lvl, cta_a, cta_b, fcreg, lists, total;
};

struct DeviceInfo {
  int ordinal;
  int num_sms;
};

int launch_compress(int dtype, CompressArgs a, const DeviceInfo& dev, cudaStream_t stream);
size_t compress_workspace_layout(uint64_t d, int dtype, int gmax, WsLayout* out);

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
};

int launch_decompress(const DecompressArgs& a, const DeviceInfo& dev, cudaStream_t stream);
int launch_decompress_unsorted(const DecompressArgs& a, void* scratch, const DeviceInfo& dev, cudaStream_t stream);

int launch_adatopk_plan(const double* R, int n, double base_ratio, const int64_t* d_per_link, double* r_out,
                        int64_t* k_out, int32_t* status, cudaStream_t stream);

}  // namespace gp
