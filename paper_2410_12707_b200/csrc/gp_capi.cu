// gp_capi.cu — the extern "C" boundary (include/adatopk.h) and the on-device
// AdaTopK bookkeeping kernel.
//
// Reference interfaces replaced (pkg/src/geopipe/compressor.py):
//   select_k        :73-76    -> gp_select_k
//   wire_bytes      :106-108  -> gp_wire_bytes
//   topk_compress   :79-94    -> gp_topk_compress / gp_topk_compress_frame
//   topk_decompress :97-103   -> gp_topk_decompress / _frame / _unsorted
//   adatopk_plan    :111-129  -> gp_adatopk_plan (device) / gp_adatopk_plan_host
//   SparsePayload.to_bytes :39-44 -> the *_frame variants write/read that layout
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>

#include "../../include/adatopk.h"
#include "gp_kernels.cuh"

namespace {

int device_info(gp::DeviceInfo* info) {
  // per-device SM count, cached; concurrent first calls from several host
  // threads store the same value (atomics: no data race)
  static std::atomic<int> cached_sms[gp::kMaxDevices];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= gp::kMaxDevices) return GP_ERR_CUDA;
  int sms = cached_sms[dev].load(std::memory_order_acquire);
  if (!sms) {
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms < 1)
      return GP_ERR_CUDA;
    cached_sms[dev].store(sms, std::memory_order_release);
  }
  info->ordinal = dev;
  info->num_sms = sms;
  return GP_OK;
}

unsigned long long* g_debug_stamps = nullptr;  // development aid, see gp_debug_stamps
unsigned long long* g_debug_dec = nullptr;     // development aid, see gp_debug_dec_stamps

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Python: `max(1, math.floor(d / ratio))` with `ratio < 1 -> InvalidRatio`.
int select_k_impl(int64_t d, double ratio, int64_t* k_out) {
  if (ratio < 1.0) return GP_ERR_INVALID_RATIO;
  if (std::isnan(ratio)) return GP_ERR_INVALID_ARGUMENT;  // math.floor(nan) raises ValueError
  const double q = (double)d / ratio;
  const double f = std::floor(q);
  int64_t k = (int64_t)f;
  if (k < 1) k = 1;
  *k_out = k;
  return GP_OK;
}

// Eq. 6 (compressor.py:118-125), operation order preserved:
//   r_max = max(R); r_i = max(1.0, 3.0 * base_ratio * R_i / r_max)
__host__ __device__ inline int plan_impl(const double* R, int n, double base, const int64_t* dl, double* r_out,
                                         int64_t* k_out) {
  if (base < 1.0) return GP_ERR_INVALID_RATIO;
  double r_max = 0.0;  // max(values, default=0.0): first element, then strictly-greater updates
  for (int i = 0; i < n; ++i)
    if (i == 0 || R[i] > r_max) r_max = R[i];
  if (r_max <= 0.0) return GP_ERR_NO_COMMUNICATION;
  for (int i = 0; i < n; ++i) {
    double t = 3.0 * base;
    t = t * R[i];
    t = t / r_max;
    const double r = (t > 1.0) ? t : 1.0;  // max(1.0, t)
    if (r_out) r_out[i] = r;
    if (k_out && dl) {
      double f = floor((double)dl[i] / r);
      int64_t k = (int64_t)f;
      k_out[i] = k < 1 ? 1 : k;
    }
  }
  return GP_OK;
}

__global__ void plan_kernel(const double* R, int n, double base, const int64_t* dl, double* r_out, int64_t* k_out,
                            int32_t* status) {
  if (blockIdx.x == 0 && threadIdx.x == 0) *status = plan_impl(R, n, base, dl, r_out, k_out);
}

}  // namespace

namespace gp {
int debug_decompress_occupancy();
int launch_adatopk_plan(const double* R, int n, double base, const int64_t* dl, double* r_out, int64_t* k_out,
                        int32_t* status, cudaStream_t s) {
  plan_kernel<<<1, 32, 0, s>>>(R, n, base, dl, r_out, k_out, status);
  return cudaGetLastError() == cudaSuccess ? GP_OK : GP_ERR_CUDA;
}
}  // namespace gp

extern "C" {

const char* gp_version(void) { return "adatopk-b200 0.1.0 sm_100a"; }

int gp_set_cluster_path(int mode) { return gp::set_cluster_path(mode); }

// Development aid (not part of the public header): when non-NULL, every
// compress launch writes per-CTA stage timestamps (globaltimer ns, clock64)
// into this device buffer of G*32 u64.
void gp_debug_stamps(void* dev_buf) { g_debug_stamps = static_cast<unsigned long long*>(dev_buf); }
void gp_debug_dec_stamps(void* dev_buf) { g_debug_dec = static_cast<unsigned long long*>(dev_buf); }
int gp_debug_dec_occupancy(void) { return gp::debug_decompress_occupancy(); }

int gp_select_k(int64_t d, double ratio, int64_t* k_out) {
  if (!k_out) return GP_ERR_INVALID_ARGUMENT;
  return select_k_impl(d, ratio, k_out);
}

int gp_wire_bytes(int64_t d, double ratio, int64_t* bytes_out) {
  if (!bytes_out) return GP_ERR_INVALID_ARGUMENT;
  int64_t k = 0;
  const int st = select_k_impl(d, ratio, &k);
  if (st) return st;
  *bytes_out = k * 12;
  return GP_OK;
}

size_t gp_topk_workspace_bytes(int64_t d, int dtype) {
  if (d < 0) d = 0;
  return gp::compress_workspace_bytes((uint64_t)d, dtype);
}

int gp_workspace_init(void* ws, size_t ws_bytes, void* stream) {
  if (!ws) return GP_ERR_INVALID_ARGUMENT;
  // the state region (its extent depends only on ws_bytes); once: every call
  // leaves it zeroed again
  size_t n = gp::workspace_state_bytes(ws_bytes);
  if (n > ws_bytes) n = ws_bytes;
  return cudaMemsetAsync(ws, 0, n, as_stream(stream)) == cudaSuccess ? GP_OK : GP_ERR_CUDA;
}

static int compress_impl(const void* x, int dtype, int64_t d, int64_t k, void* idx_out, int idx_bytes,
                         void* val_out, int val_dtype, void* val2_out, void* header_out, void* ws, size_t ws_bytes,
                         void* stream, int max_ctas, const int64_t* k_dev = nullptr, uint32_t* err = nullptr) {
  if (d <= 0) return GP_ERR_EMPTY_VECTOR;
  if (!x || !idx_out || (!val_out && !k_dev) || !ws) return GP_ERR_INVALID_ARGUMENT;
  if (dtype < 0 || dtype > 2) return GP_ERR_INVALID_ARGUMENT;
  if (d >= (int64_t)1 << 31 || k < 1 || k > d) return GP_ERR_INVALID_ARGUMENT;
  if (idx_bytes != 4 && idx_bytes != 8) return GP_ERR_INVALID_ARGUMENT;
  if (val_dtype != GP_DTYPE_F32 && val_dtype != dtype) return GP_ERR_INVALID_ARGUMENT;
  gp::WsLayout l;
  const size_t need = gp::compress_workspace_layout((uint64_t)d, dtype, ws_bytes, &l);
  if (ws_bytes < need) return GP_ERR_INVALID_ARGUMENT;
  gp::DeviceInfo dev;
  if (device_info(&dev)) return GP_ERR_CUDA;
  dev.max_ctas = max_ctas;
  unsigned char* base = static_cast<unsigned char*>(ws);
  gp::CompressArgs a = {};
  a.x = x;
  a.d = (uint32_t)d;
  a.k = (uint32_t)k;
  a.idx_out = idx_out;
  a.idx64 = idx_bytes == 8;
  a.val_out = val_out;
  a.val_f32 = val_dtype == GP_DTYPE_F32;
  a.val2_out = val2_out;
  a.header = static_cast<unsigned long long*>(header_out);
  a.ctrl = reinterpret_cast<uint32_t*>(base + l.ctrl);
  a.hist1 = reinterpret_cast<uint32_t*>(base + l.hist1);
  a.hist_lvl = reinterpret_cast<uint32_t*>(base + l.hist_lvl);
  a.cta_a = reinterpret_cast<uint32_t*>(base + l.cta_a);
  a.cta_b = reinterpret_cast<uint32_t*>(base + l.cta_b);
  a.fcreg = base + l.fcreg;
  a.lists = base + l.lists;
  a.aligned = ((uintptr_t)x % 32) == 0;
  a.dbg = g_debug_stamps;
  a.k_dev = reinterpret_cast<const long long*>(k_dev);
  a.frame_vals = k_dev != nullptr && val_out == nullptr;
  a.err = err;
  return gp::launch_compress(dtype, a, dev, as_stream(stream));
}

int gp_topk_compress(const void* x, int dtype, int64_t d, int64_t k, void* idx_out, int idx_bytes, void* val_out,
                     int val_dtype, void* val2_out, void* header_out, void* ws, size_t ws_bytes, void* stream) {
  return compress_impl(x, dtype, d, k, idx_out, idx_bytes, val_out, val_dtype, val2_out, header_out, ws, ws_bytes,
                       stream, 0);
}

int gp_topk_compress_ctas(const void* x, int dtype, int64_t d, int64_t k, void* idx_out, int idx_bytes, void* val_out,
                          int val_dtype, void* val2_out, void* header_out, void* ws, size_t ws_bytes, void* stream,
                          int max_ctas) {
  if (max_ctas < 0) return GP_ERR_INVALID_ARGUMENT;
  return compress_impl(x, dtype, d, k, idx_out, idx_bytes, val_out, val_dtype, val2_out, header_out, ws, ws_bytes,
                       stream, max_ctas);
}

int gp_topk_compress_frame_ctas(const void* x, int dtype, int64_t d, int64_t k, void* frame_out, void* ws,
                                size_t ws_bytes, void* stream, int max_ctas) {
  if (!frame_out || ((uintptr_t)frame_out % 8) != 0 || max_ctas < 0) return GP_ERR_INVALID_ARGUMENT;
  unsigned char* f = static_cast<unsigned char*>(frame_out);
  return compress_impl(x, dtype, d, k, f + GP_FRAME_HEADER_BYTES, 8, f + GP_FRAME_HEADER_BYTES + 8 * k,
                       GP_DTYPE_F32, nullptr, f, ws, ws_bytes, stream, max_ctas);
}

int gp_topk_compress_frame_dk(const void* x, int dtype, int64_t d, const int64_t* k_dev, int64_t k_cap,
                              void* frame_out, uint32_t* d_err_flag, void* ws, size_t ws_bytes, void* stream,
                              int max_ctas) {
  if (!frame_out || !k_dev || ((uintptr_t)frame_out % 8) != 0 || max_ctas < 0) return GP_ERR_INVALID_ARGUMENT;
  if (k_cap < 1 || k_cap > d) return GP_ERR_INVALID_ARGUMENT;
  unsigned char* f = static_cast<unsigned char*>(frame_out);
  // k_cap sizes the launch-independent checks; the kernel reads k and places the values after the k indices
  return compress_impl(x, dtype, d, k_cap, f + GP_FRAME_HEADER_BYTES, 8, nullptr, GP_DTYPE_F32, nullptr, f, ws,
                       ws_bytes, stream, max_ctas, k_dev, d_err_flag);
}

int gp_topk_compress_frame(const void* x, int dtype, int64_t d, int64_t k, void* frame_out, void* ws,
                           size_t ws_bytes, void* stream) {
  return gp_topk_compress_frame_ctas(x, dtype, d, k, frame_out, ws, ws_bytes, stream, 0);
}

static int decompress_common(const void* idx, int idx_bytes, const void* vals, int val_dtype, int64_t k, int64_t d,
                             void* out, int out_dtype, int mode, uint32_t* d_err_flag, void* stream,
                             void* scratch, const void* hdr = nullptr, int dev_k = 0) {
  if (k < 0 || d < 0) return GP_ERR_INVALID_ARGUMENT;
  if (idx_bytes != 4 && idx_bytes != 8) return GP_ERR_INVALID_ARGUMENT;
  if (val_dtype < 0 || val_dtype > 2 || out_dtype < 0 || out_dtype > 2) return GP_ERR_INVALID_ARGUMENT;
  if (mode < 0 || mode > 3) return GP_ERR_INVALID_ARGUMENT;  // GP_DECOMPRESS_RESIDUAL | GP_DECOMPRESS_TRUSTED
  if (!d_err_flag || (k > 0 && (!idx || (!vals && !dev_k))) || (d > 0 && !out)) return GP_ERR_INVALID_ARGUMENT;
  if (d == 0 && k > 0) return GP_ERR_INDEX_OUT_OF_RANGE;  // every index is >= d
  gp::DeviceInfo dev;
  if (device_info(&dev)) return GP_ERR_CUDA;
  gp::DecompressArgs a = {idx, idx_bytes == 8, vals, val_dtype, k, d, out, out_dtype, mode, d_err_flag, g_debug_dec,
                          static_cast<const unsigned long long*>(hdr), dev_k};
  if (scratch) return gp::launch_decompress_unsorted(a, scratch, dev, as_stream(stream));
  return gp::launch_decompress(a, dev, as_stream(stream));
}

int gp_topk_decompress(const void* idx, int idx_bytes, const void* vals, int val_dtype, int64_t k, int64_t d,
                       void* out, int out_dtype, int mode, uint32_t* d_err_flag, void* stream) {
  return decompress_common(idx, idx_bytes, vals, val_dtype, k, d, out, out_dtype, mode, d_err_flag, stream, nullptr);
}

int gp_topk_decompress_frame(const void* frame, int64_t k, int64_t d, void* out, int out_dtype, int mode,
                             uint32_t* d_err_flag, void* stream) {
  if (!frame || ((uintptr_t)frame % 8) != 0) return GP_ERR_INVALID_ARGUMENT;
  const unsigned char* f = static_cast<const unsigned char*>(frame);
  // the frame's own {d, k} header is checked against (d, k) in the same launch (GP_FLAG_HEADER)
  return decompress_common(f + GP_FRAME_HEADER_BYTES, 8, f + GP_FRAME_HEADER_BYTES + 8 * k, GP_DTYPE_F32, k, d, out,
                           out_dtype, mode, d_err_flag, stream, nullptr, f, 0);
}

int gp_topk_decompress_frame_dk(const void* frame, int64_t d, int64_t k_cap, void* out, int out_dtype, int mode,
                                uint32_t* d_err_flag, void* stream) {
  if (!frame || ((uintptr_t)frame % 8) != 0 || k_cap < 1) return GP_ERR_INVALID_ARGUMENT;
  const unsigned char* f = static_cast<const unsigned char*>(frame);
  return decompress_common(f + GP_FRAME_HEADER_BYTES, 8, nullptr, GP_DTYPE_F32, k_cap, d, out, out_dtype, mode,
                           d_err_flag, stream, nullptr, f, 1);
}

// ---- OpData envelope (opdag.py:67-86) ahead of a stage-boundary message
namespace {
struct Envelope {
  long long f[GP_ENVELOPE_WORDS];
};

__global__ void envelope_write_kernel(long long* env, Envelope e) {
  if (threadIdx.x < GP_ENVELOPE_WORDS) env[threadIdx.x] = e.f[threadIdx.x];
}

__global__ void envelope_check_kernel(const long long* env, Envelope e, unsigned long long mask, uint32_t* err) {
  const int i = threadIdx.x;
  const bool bad = i < GP_ENVELOPE_WORDS && ((mask >> i) & 1ull) && env[i] != e.f[i];
  if (__any_sync(0xFFFFFFFFu, bad) && i == 0) atomicOr(err, GP_FLAG_ENVELOPE);
}
}  // namespace

int gp_envelope_write(void* env_dev, const int64_t* fields, void* stream) {
  if (!env_dev || !fields || ((uintptr_t)env_dev % 8) != 0) return GP_ERR_INVALID_ARGUMENT;
  Envelope e;
  for (int i = 0; i < GP_ENVELOPE_WORDS; ++i) e.f[i] = fields[i];
  envelope_write_kernel<<<1, 32, 0, as_stream(stream)>>>(static_cast<long long*>(env_dev), e);
  return cudaGetLastError() == cudaSuccess ? GP_OK : GP_ERR_CUDA;
}

int gp_envelope_check(const void* env_dev, const int64_t* expected, uint64_t mask, uint32_t* d_err_flag,
                      void* stream) {
  if (!env_dev || !expected || !d_err_flag || ((uintptr_t)env_dev % 8) != 0) return GP_ERR_INVALID_ARGUMENT;
  Envelope e;
  for (int i = 0; i < GP_ENVELOPE_WORDS; ++i) e.f[i] = expected[i];
  envelope_check_kernel<<<1, 32, 0, as_stream(stream)>>>(static_cast<const long long*>(env_dev), e,
                                                          (unsigned long long)mask, d_err_flag);
  return cudaGetLastError() == cudaSuccess ? GP_OK : GP_ERR_CUDA;
}

// ---- standalone frame pack / unpack (SparsePayload.to_bytes / from_bytes, compressor.py:39-53)
namespace {
__device__ __forceinline__ float val_as_f32(const void* v, int dt, int64_t j) {
  if (dt == GP_DTYPE_F32) return static_cast<const float*>(v)[j];
  if (dt == GP_DTYPE_BF16) return __uint_as_float((uint32_t)static_cast<const uint16_t*>(v)[j] << 16);
  return __double2float_rn(static_cast<const double*>(v)[j]);
}

__global__ void pack_frame_kernel(const void* idx, int idx64, const void* vals, int val_dtype, int64_t k, int64_t d,
                                  unsigned char* frame) {
  unsigned long long* h = reinterpret_cast<unsigned long long*>(frame);
  int64_t* fi = reinterpret_cast<int64_t*>(frame + GP_FRAME_HEADER_BYTES);
  float* fv = reinterpret_cast<float*>(frame + GP_FRAME_HEADER_BYTES + 8 * k);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    h[0] = (unsigned long long)d;
    h[1] = (unsigned long long)k;
  }
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < k; j += (int64_t)gridDim.x * blockDim.x) {
    fi[j] = idx64 ? static_cast<const int64_t*>(idx)[j] : (int64_t) static_cast<const int32_t*>(idx)[j];
    fv[j] = val_as_f32(vals, val_dtype, j);
  }
}

// k comes from the frame header (device memory); frames with k > k_cap or a
// header other than {d_expect, .} (d_expect >= 0) raise GP_FLAG_HEADER and
// unpack nothing.  hdr_out (nullable) receives the header as read.
__global__ void unpack_frame_kernel(const unsigned char* frame, int64_t k_cap, int64_t d_expect, int64_t* idx_out,
                                    void* vals_out, int val_dtype, int64_t* hdr_out, uint32_t* err) {
  const unsigned long long hd = reinterpret_cast<const unsigned long long*>(frame)[0];
  const unsigned long long hk = reinterpret_cast<const unsigned long long*>(frame)[1];
  const bool ok = hk <= (unsigned long long)k_cap && (d_expect < 0 || hd == (unsigned long long)d_expect);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (hdr_out) {
      hdr_out[0] = (int64_t)hd;
      hdr_out[1] = (int64_t)hk;
    }
    if (!ok && err) atomicOr(err, GP_FLAG_HEADER);
  }
  if (!ok) return;
  const int64_t k = (int64_t)hk;
  const int64_t* fi = reinterpret_cast<const int64_t*>(frame + GP_FRAME_HEADER_BYTES);
  const float* fv = reinterpret_cast<const float*>(frame + GP_FRAME_HEADER_BYTES + 8 * k);
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < k; j += (int64_t)gridDim.x * blockDim.x) {
    idx_out[j] = fi[j];
    const float v = fv[j];
    if (val_dtype == GP_DTYPE_F64) static_cast<double*>(vals_out)[j] = (double)v;
    else if (val_dtype == GP_DTYPE_F32) static_cast<float*>(vals_out)[j] = v;
    else static_cast<uint16_t*>(vals_out)[j] = (uint16_t)(__float_as_uint(v) >> 16);  // exact for bf16-valued frames
  }
}

unsigned frame_grid(int64_t k) {
  const int64_t b = (k + 255) / 256;
  return (unsigned)(b < 1 ? 1 : (b > 1184 ? 1184 : b));
}
}  // namespace

int gp_pack_frame(const void* idx, int idx_bytes, const void* vals, int val_dtype, int64_t k, int64_t d,
                  void* frame_out, void* stream) {
  if (!frame_out || ((uintptr_t)frame_out % 8) != 0 || k < 0 || d < 0) return GP_ERR_INVALID_ARGUMENT;
  if ((idx_bytes != 4 && idx_bytes != 8) || val_dtype < 0 || val_dtype > 2) return GP_ERR_INVALID_ARGUMENT;
  if (k > 0 && (!idx || !vals)) return GP_ERR_INVALID_ARGUMENT;
  pack_frame_kernel<<<frame_grid(k), 256, 0, as_stream(stream)>>>(idx, idx_bytes == 8, vals, val_dtype, k, d,
                                                                  static_cast<unsigned char*>(frame_out));
  return cudaGetLastError() == cudaSuccess ? GP_OK : GP_ERR_CUDA;
}

int gp_unpack_frame(const void* frame, int64_t k_cap, int64_t d_expect, int64_t* idx_out, void* vals_out,
                    int val_dtype, int64_t* hdr_out, uint32_t* d_err_flag, void* stream) {
  if (!frame || ((uintptr_t)frame % 8) != 0 || k_cap < 0 || val_dtype < 0 || val_dtype > 2) return GP_ERR_INVALID_ARGUMENT;
  if (k_cap > 0 && (!idx_out || !vals_out)) return GP_ERR_INVALID_ARGUMENT;
  unpack_frame_kernel<<<frame_grid(k_cap), 256, 0, as_stream(stream)>>>(
      static_cast<const unsigned char*>(frame), k_cap, d_expect, idx_out, vals_out, val_dtype, hdr_out, d_err_flag);
  return cudaGetLastError() == cudaSuccess ? GP_OK : GP_ERR_CUDA;
}

int gp_topk_decompress_unsorted(const void* idx, int idx_bytes, const void* vals, int val_dtype, int64_t k,
                                int64_t d, void* out, int out_dtype, void* scratch, uint32_t* d_err_flag,
                                void* stream) {
  if (!scratch) return GP_ERR_INVALID_ARGUMENT;
  if (d >= (int64_t)1 << 31 || k >= (int64_t)1 << 31) return GP_ERR_INVALID_ARGUMENT;
  return decompress_common(idx, idx_bytes, vals, val_dtype, k, d, out, out_dtype, 0, d_err_flag, stream, scratch);
}

int gp_adatopk_plan(const double* R, int n, double base_ratio, const int64_t* d_per_link, double* r_out,
                    int64_t* k_out, int32_t* d_status, void* stream) {
  if (!R || !d_status || n < 0) return GP_ERR_INVALID_ARGUMENT;
  return gp::launch_adatopk_plan(R, n, base_ratio, d_per_link, r_out, k_out, d_status, as_stream(stream));
}

int gp_adatopk_plan_host(const double* R, int n, double base_ratio, const int64_t* d_per_link, double* r_out,
                         int64_t* k_out) {
  if ((!R && n > 0) || n < 0) return GP_ERR_INVALID_ARGUMENT;
  return plan_impl(R, n, base_ratio, d_per_link, r_out, k_out);
}

// ---- peer-memory transport (executor.py:248-297 inbox delivery, on NVLink)
static_assert(sizeof(cudaIpcMemHandle_t) == GP_IPC_HANDLE_BYTES, "IPC handle size");
static_assert(sizeof(cudaIpcEventHandle_t) == GP_IPC_HANDLE_BYTES, "IPC event handle size");
static int cuda_status(cudaError_t e) { return e == cudaSuccess ? GP_OK : GP_ERR_CUDA; }

int gp_peer_alloc(size_t bytes, void** ptr_out) {
  if (!ptr_out || bytes == 0) return GP_ERR_INVALID_ARGUMENT;
  return cuda_status(cudaMalloc(ptr_out, bytes));
}
int gp_peer_free(void* ptr) { return cuda_status(cudaFree(ptr)); }
int gp_ipc_mem_handle(void* ptr, void* handle_out) {
  if (!ptr || !handle_out) return GP_ERR_INVALID_ARGUMENT;
  return cuda_status(cudaIpcGetMemHandle(static_cast<cudaIpcMemHandle_t*>(handle_out), ptr));
}
int gp_ipc_open_mem(const void* handle, void** ptr_out) {
  if (!handle || !ptr_out) return GP_ERR_INVALID_ARGUMENT;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  return cuda_status(cudaIpcOpenMemHandle(ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
}
int gp_ipc_close_mem(void* ptr) { return cuda_status(cudaIpcCloseMemHandle(ptr)); }
int gp_ipc_event_create(void** event_out, void* handle_out) {
  if (!event_out || !handle_out) return GP_ERR_INVALID_ARGUMENT;
  cudaEvent_t ev;
  if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming | cudaEventInterprocess) != cudaSuccess) return GP_ERR_CUDA;
  *event_out = ev;
  return cuda_status(cudaIpcGetEventHandle(static_cast<cudaIpcEventHandle_t*>(handle_out), ev));
}
int gp_ipc_open_event(const void* handle, void** event_out) {
  if (!handle || !event_out) return GP_ERR_INVALID_ARGUMENT;
  cudaIpcEventHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  cudaEvent_t ev;
  if (cudaIpcOpenEventHandle(&ev, h) != cudaSuccess) return GP_ERR_CUDA;
  *event_out = ev;
  return GP_OK;
}
int gp_event_destroy(void* event) { return cuda_status(cudaEventDestroy(static_cast<cudaEvent_t>(event))); }
int gp_event_record(void* event, void* stream) {
  return cuda_status(cudaEventRecord(static_cast<cudaEvent_t>(event), as_stream(stream)));
}
int gp_stream_wait_event(void* stream, void* event) {
  return cuda_status(cudaStreamWaitEvent(as_stream(stream), static_cast<cudaEvent_t>(event), 0));
}
// the same inside a CUDA-graph capture as real (external) event record / wait
// nodes: another process's stream or graph can then wait on a record made by
// a graph replay here, and a graph can wait on another process's record
static bool capturing(cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  return cudaStreamIsCapturing(s, &st) == cudaSuccess && st == cudaStreamCaptureStatusActive;
}
int gp_event_record_external(void* event, void* stream) {
  const cudaStream_t s = as_stream(stream);
  if (!capturing(s)) return cuda_status(cudaEventRecord(static_cast<cudaEvent_t>(event), s));
  return cuda_status(cudaEventRecordWithFlags(static_cast<cudaEvent_t>(event), s, cudaEventRecordExternal));
}
int gp_stream_wait_event_external(void* stream, void* event) {
  const cudaStream_t s = as_stream(stream);
  return cuda_status(cudaStreamWaitEvent(s, static_cast<cudaEvent_t>(event), capturing(s) ? cudaEventWaitExternal : 0));
}
int gp_copy_async(void* dst, const void* src, size_t bytes, void* stream) {
  if ((!dst || !src) && bytes) return GP_ERR_INVALID_ARGUMENT;
  return cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, as_stream(stream)));
}

}  // extern "C"
