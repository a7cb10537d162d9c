/*
 * adatopk.h — C-ABI of the B200-native AdaTopK compressor (sm_100a).
 *
 * This is the drop-in boundary for the hot path named in BASELINE.json
 * `north_star`: the Top-K compressor of FusionLLM's reference
 * (`geopipe.compressor`, /root/reference/pkg/src/geopipe/compressor.py) and the
 * per-link adaptive ratio bookkeeping (Eq. 6).  Every entry point below cites
 * the reference function it replaces.  Plain pointers and sizes only: device
 * pointers for tensors, `void* stream` is a `cudaStream_t` (NULL = legacy
 * default stream).  All GPU calls are stream-ordered, never synchronise, and
 * never allocate; the caller owns every buffer.
 *
 * Status codes map 1:1 onto the reference exception classes
 * (/root/reference/pkg/src/geopipe/errors.py:46-59).
 */
#ifndef ADATOPK_H_
#define ADATOPK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define GP_OK                       0
#define GP_ERR_INVALID_RATIO        1  /* errors.py:46  InvalidRatio      */
#define GP_ERR_EMPTY_VECTOR         2  /* errors.py:50  EmptyVector       */
#define GP_ERR_INDEX_OUT_OF_RANGE   3  /* errors.py:54  IndexOutOfRange   */
#define GP_ERR_NO_COMMUNICATION     4  /* errors.py:58  NoCommunication   */
#define GP_ERR_CUDA                 5  /* CUDA launch / runtime error      */
#define GP_ERR_INVALID_ARGUMENT     6  /* bad dtype, size, alignment, ... */

/* ---- element types ----------------------------------------------------- */
#define GP_DTYPE_F32   0   /* float32  (reference fp32 path)               */
#define GP_DTYPE_BF16  1   /* bfloat16 (selection == reference on x.float()) */
#define GP_DTYPE_F64   2   /* float64  (reference executor's dtype)        */

/* ---- asynchronous device error flags (decompress) ---------------------- */
#define GP_FLAG_OUT_OF_RANGE  1u   /* some index < 0 or >= d  (compressor.py:99-100) */
#define GP_FLAG_UNSORTED      2u   /* indices not strictly increasing (fast path invalid) */
#define GP_FLAG_HEADER        4u   /* frame header {d,k} disagrees with the receiver's (d, k / k_cap) */
#define GP_FLAG_BAD_K         8u   /* device-resident k outside [1, min(k_cap, d)] (compress) */
#define GP_FLAG_ENVELOPE     16u   /* a message's OpData envelope differs from what the receiver expects */

/* Wire frame of the reference (compressor.py:39-44): little-endian
 * {d:u64, k:u64} header, k x i64 indices, k x f32 values. */
#define GP_FRAME_HEADER_BYTES 16
static inline size_t gp_frame_bytes(int64_t k) { return (size_t)GP_FRAME_HEADER_BYTES + (size_t)k * 12u; }

/* Library version string. */
const char* gp_version(void);

/* k = max(1, floor(d / ratio)); GP_ERR_INVALID_RATIO if ratio < 1.
 * Replaces select_k, compressor.py:73-76 (IEEE double divide, same order). */
int gp_select_k(int64_t d, double ratio, int64_t* k_out);

/* Bytes on the wire for a compressed length-d vector = 12 * k.
 * Replaces wire_bytes, compressor.py:106-108. */
int gp_wire_bytes(int64_t d, double ratio, int64_t* bytes_out);

/* Scratch needed by gp_topk_compress for a length-d vector of `dtype`
 * (sized by d: about 8 B per element for the candidate lists plus per-CTA
 * regions).  A buffer serves every call whose own requirement fits in it.  Its
 * state region (extent a function of the buffer size only) must be zeroed once
 * with gp_workspace_init and is left zeroed by every call; one workspace per
 * concurrent stream. */
size_t gp_topk_workspace_bytes(int64_t d, int dtype);
int gp_workspace_init(void* ws, size_t ws_bytes, void* stream);

/* Top-K by |x| with lower-index tie break; NaN ranks below every number.
 * Writes k indices (strictly increasing; int64 if idx_bytes == 8 else int32)
 * and k values (val_dtype: GP_DTYPE_F32 or the input dtype).  val2_out, if
 * non-NULL, receives the values again in the input dtype (lets the caller get
 * both the f32 wire values and the dtype-preserving SparsePayload.values in one
 * pass).  header_out, if non-NULL, receives the {d, k} frame header.
 * Replaces topk_compress, compressor.py:79-94 (np.argsort(-|x|, stable), take
 * k, sort kept, gather).  d must be < 2^31. */
int gp_topk_compress(const void* x, int dtype, int64_t d, int64_t k,
                     void* idx_out, int idx_bytes,
                     void* val_out, int val_dtype,
                     void* val2_out,
                     void* header_out,
                     void* ws, size_t ws_bytes, void* stream);

/* Same, writing the reference wire frame (16 + 12k bytes) directly. */
int gp_topk_compress_frame(const void* x, int dtype, int64_t d, int64_t k,
                           void* frame_out, void* ws, size_t ws_bytes, void* stream);

/* Short vectors can be compressed by a single thread-block cluster -- one HBM
 * read into the CTAs' shared memory, DSMEM histograms, cluster barriers --
 * instead of the cooperative grid (identical results).  mode 1 (default): the
 * cluster kernel for vectors of at most 98,304 elements, where it is the
 * faster one on B200 (1.4-1.9x cold at 1K-64K elements); 2: for every vector that fits one
 * 8-CTA cluster (up to 393,216 fp32 / 786,432 bf16 / 196,608 fp64 elements,
 * within max_ctas);
 * 0: never (also when the environment sets GP_NO_CLUSTER=1).  Returns the
 * previous mode.  Process-wide; for A/B measurements and tests. */
int gp_set_cluster_path(int mode);

/* decompress `mode` bits */
#define GP_DECOMPRESS_RESIDUAL 1   /* add into `out` instead of zero-filling (extension) */
#define GP_DECOMPRESS_TRUSTED  2   /* indices written by gp_topk_compress* and unmodified: strictly
                                      increasing by construction, so the O(k) sortedness scan is skipped
                                      (the O(1) range check and the frame header check remain) */

/* Dense length-d output: values at their indices, zero (mode 0) or added to
 * the existing contents (mode 1, residual extension) elsewhere.  Fast path,
 * requires strictly increasing indices; violations and out-of-range indices are
 * reported asynchronously in *d_err_flag (GP_FLAG_*; the caller zeroes it).
 * Replaces topk_decompress, compressor.py:97-103. */
int gp_topk_decompress(const void* idx, int idx_bytes,
                       const void* vals, int val_dtype, int64_t k, int64_t d,
                       void* out, int out_dtype, int mode,
                       uint32_t* d_err_flag, void* stream);

/* gp_topk_compress with the cooperative grid capped at `max_ctas` CTAs (see
 * gp_topk_compress_frame_ctas). */
int gp_topk_compress_ctas(const void* x, int dtype, int64_t d, int64_t k,
                          void* idx_out, int idx_bytes, void* val_out, int val_dtype,
                          void* val2_out, void* header_out, void* ws, size_t ws_bytes,
                          void* stream, int max_ctas);

/* Same, with the cooperative grid capped at `max_ctas` CTAs (0 = one per SM):
 * independent compresses on different streams (each with its own workspace)
 * then share the GPU, one's barrier-bound tail overlapping another's HBM
 * stream. */
int gp_topk_compress_frame_ctas(const void* x, int dtype, int64_t d, int64_t k,
                                void* frame_out, void* ws, size_t ws_bytes,
                                void* stream, int max_ctas);

/* Decompress straight from a reference wire frame on the device.  The frame's
 * {d, k} header is checked against (d, k) in the same launch: a mismatch
 * raises GP_FLAG_HEADER and nothing is scattered. */
int gp_topk_decompress_frame(const void* frame, int64_t k, int64_t d,
                             void* out, int out_dtype, int mode,
                             uint32_t* d_err_flag, void* stream);

/* ---- device-resident k (north_star item 4: adaptive bookkeeping kept on the
 * device).  k is read from device memory at kernel start -- e.g. the k_out of
 * gp_adatopk_plan -- so re-planning k never round-trips through the host.
 * Frames are sized for a host-known capacity k_cap (16 + 12*k_cap bytes; the
 * frame written is 16 + 12*k, values right after the k indices as in the
 * reference layout).  *k_dev outside [1, min(k_cap, d)] writes nothing but an
 * invalid header {d, ~0} and raises GP_FLAG_BAD_K; k == d keeps every element
 * (ratio <= 1, the executor's pass-through, executor.py:210-212).
 * Replaces topk_compress + to_bytes (compressor.py:79-94, :39-44) with k from
 * select_k/adatopk_plan evaluated on the device (compressor.py:73-76,111-129). */
int gp_topk_compress_frame_dk(const void* x, int dtype, int64_t d, const int64_t* k_dev, int64_t k_cap,
                              void* frame_out, uint32_t* d_err_flag, void* ws, size_t ws_bytes,
                              void* stream, int max_ctas);

/* Decompress a frame whose k is read from its own header (1 <= k <= k_cap and
 * header d == d, else GP_FLAG_HEADER and nothing is scattered).  The receive
 * buffer is sized for k_cap; no size handshake precedes the payload.
 * Replaces topk_decompress(SparsePayload.from_bytes(raw)), compressor.py:46-53,97-103. */
int gp_topk_decompress_frame_dk(const void* frame, int64_t d, int64_t k_cap, void* out, int out_dtype, int mode,
                                uint32_t* d_err_flag, void* stream);

/* Standalone on-device frame pack: {d, k} header, k indices widened to i64,
 * k values rounded to f32 (IEEE round-to-nearest; exact for f32 / bf16).
 * Replaces SparsePayload.to_bytes, compressor.py:39-44. */
int gp_pack_frame(const void* idx, int idx_bytes, const void* vals, int val_dtype, int64_t k, int64_t d,
                  void* frame_out, void* stream);

/* Standalone on-device frame unpack: k from the frame's header (must be
 * <= k_cap; d_expect >= 0 also checks the header's d), i64 indices and the
 * values converted to val_dtype (GP_DTYPE_F64 = the reference's from_bytes,
 * which returns float64 values).  hdr_out (nullable, device) receives {d, k}.
 * A bad header raises GP_FLAG_HEADER and unpacks nothing.
 * Replaces SparsePayload.from_bytes, compressor.py:46-53. */
int gp_unpack_frame(const void* frame, int64_t k_cap, int64_t d_expect, int64_t* idx_out, void* vals_out,
                    int val_dtype, int64_t* hdr_out, uint32_t* d_err_flag, void* stream);

/* ---- OpData envelope.  The reference wraps every cross-device payload in an
 * OpData (opdag.py:67-86: producer, consumers, iteration, micro-batch,
 * compress_cfg {algo, shape}) and routes it by those fields
 * (executor.py:248-297).  Here a 128-byte envelope of GP_ENVELOPE_WORDS int64
 * travels ahead of each stage-boundary message in the same buffer; the
 * fields are the caller's (the Python transport uses: magic, iteration,
 * micro-batch, source stage, destination stage, kind, compressed flag,
 * payload bytes, ndim, shape[4]).  Both calls are stream-ordered kernels with
 * the fields passed by value (no host copy); a mismatch in any field selected
 * by `mask` raises GP_FLAG_ENVELOPE. */
#define GP_ENVELOPE_WORDS 16
#define GP_ENVELOPE_BYTES (GP_ENVELOPE_WORDS * 8)
int gp_envelope_write(void* env_dev, const int64_t* fields, void* stream);
int gp_envelope_check(const void* env_dev, const int64_t* expected, uint64_t mask, uint32_t* d_err_flag,
                      void* stream);

/* General scatter for arbitrary (unsorted, possibly repeated) indices with
 * numpy's last-write-wins semantics for `out[indices] = values`.  `scratch`
 * holds d int32.  Mode 0 only. */
int gp_topk_decompress_unsorted(const void* idx, int idx_bytes,
                                const void* vals, int val_dtype, int64_t k, int64_t d,
                                void* out, int out_dtype, void* scratch,
                                uint32_t* d_err_flag, void* stream);

/* On-device AdaTopK bookkeeping (Eq. 6): r_i = max(1, 3*r*R_i/max R) in IEEE
 * double, same operation order as compressor.py:111-129, then
 * k_i = max(1, floor(d_i / r_i)) (compressor.py:73-76).  R, d_per_link, r_out,
 * k_out are device arrays of n entries; *d_status receives GP_OK,
 * GP_ERR_INVALID_RATIO or GP_ERR_NO_COMMUNICATION. */
int gp_adatopk_plan(const double* R, int n, double base_ratio,
                    const int64_t* d_per_link, double* r_out, int64_t* k_out,
                    int32_t* d_status, void* stream);

/* Host twin of gp_adatopk_plan (same arithmetic), returns the status. */
int gp_adatopk_plan_host(const double* R, int n, double base_ratio,
                         const int64_t* d_per_link, double* r_out, int64_t* k_out);

/* ---- Stage-boundary transport over peer memory (NVLink / NVSwitch).
 * Replaces the reference's in-process inbox delivery of compressed payloads
 * (executor.py:248-297, `dest.inbox[key] = _maybe_decompress(...)`): a sender
 * GPU copies its frames straight into the receiving GPU's buffer with the copy
 * engines (no SMs, so transfers overlap the next compress) and signals an
 * interprocess event the receiver's stream waits on.  Buffers and events are
 * shared between processes as opaque 64-byte IPC handles. */
#define GP_IPC_HANDLE_BYTES 64

/* Device buffer that can be exported with gp_ipc_mem_handle. */
int gp_peer_alloc(size_t bytes, void** ptr_out);
int gp_peer_free(void* ptr);
/* Export / import a gp_peer_alloc buffer (peer access enabled lazily). */
int gp_ipc_mem_handle(void* ptr, void* handle_out);
int gp_ipc_open_mem(const void* handle, void** ptr_out);
int gp_ipc_close_mem(void* ptr);
/* Interprocess event (timing disabled) and its import. */
int gp_ipc_event_create(void** event_out, void* handle_out);
int gp_ipc_open_event(const void* handle, void** event_out);
int gp_event_destroy(void* event);
int gp_event_record(void* event, void* stream);
int gp_stream_wait_event(void* stream, void* event);
/* As above, but inside a CUDA-graph capture they become external event record
 * / wait nodes, so a replayed graph can signal, or wait for, another process's
 * stream (per-frame hand-off of the peer transport). */
int gp_event_record_external(void* event, void* stream);
int gp_stream_wait_event_external(void* stream, void* event);
/* Device-to-device (local or peer) async copy on `stream`. */
int gp_copy_async(void* dst, const void* src, size_t bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* ADATOPK_H_ */
