/*
 * mgrc_gpu.h — C-ABI of the B200 (sm_100a) compress / decompress path.
 *
 * Drop-in boundary for the reference's container API
 * (/root/reference/proj/include/mgrc/container.hpp:66-83) and the CLI
 * multiblock driver (tools/mgrc.cpp:363-542).  Plain pointers and sizes only;
 * no CUDA or torch types.  Every entry point returns 0 on success or the
 * reference's errc ordinal + 1 (error.hpp:11-31; MGRC_E_*), with the message
 * available from mgrc_gpu_last_error() on the calling thread.  Buffers may be
 * host or device (CUDA) pointers: residency is detected per call.
 *
 * There is no CPU fallback: without a usable CUDA device every compute entry
 * point fails with MGRC_E_CUDA.  Header-only entry points (inspect, describe,
 * plan_chunks) run on the host.
 */
#ifndef MGRC_GPU_H
#define MGRC_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MGRC_GPU_API __attribute__((visibility("default")))

/* status codes: errc ordinal + 1 (error.hpp:11-31) */
enum {
  MGRC_OK = 0,
  MGRC_E_INVALID_SHAPE = 1,
  MGRC_E_TOO_MANY_DIMS = 2,
  MGRC_E_LEVEL_OUT_OF_RANGE = 3,
  MGRC_E_SHAPE_MISMATCH = 4,
  MGRC_E_NON_FINITE_INPUT = 5,
  MGRC_E_DEGENERATE_DATA = 6,
  MGRC_E_OVERFLOW = 7,
  MGRC_E_UNKNOWN_CODEC = 8,
  MGRC_E_CORRUPT_STREAM = 9,
  MGRC_E_BAD_MAGIC = 10,
  MGRC_E_UNSUPPORTED_VERSION = 11,
  MGRC_E_CHECKSUM_MISMATCH = 12,
  MGRC_E_TOLERANCE_UNREACHABLE = 13,
  MGRC_E_PLANE_COUNT_OUT_OF_RANGE = 14,
  MGRC_E_UNSATISFIABLE_TOLERANCE = 15,
  MGRC_E_INVALID_STATE = 16,
  MGRC_E_PREFIX_VIOLATION = 17,
  MGRC_E_BUDGET_TOO_SMALL = 18,
  MGRC_E_IO_ERROR = 19,
  MGRC_E_CUDA = 100,            /* CUDA runtime failure / no device */
  MGRC_E_INVALID_ARGUMENT = 101 /* null pointer, buffer too small */
};

enum { MGRC_DTYPE_F32 = 0, MGRC_DTYPE_F64 = 1 };             /* container.hpp:18 */
enum { MGRC_NORM_INF = 0, MGRC_NORM_S = 1 };                 /* error_control.hpp:15 */
enum { MGRC_MODE_ABS = 0, MGRC_MODE_REL = 1 };               /* error_control.hpp:16 */
enum { MGRC_CODEC_RAW = 0, MGRC_CODEC_VARINT = 1, MGRC_CODEC_HUFFMAN = 2 }; /* codec.hpp:14 */

/* ContainerInfo (container.hpp:37-51); coordinates are not returned here. */
typedef struct {
  uint16_t version;
  uint8_t constant_field, coords_present, dtype, ndims, nlevels, codec_id;
  uint64_t shape[4];
  uint8_t mode, norm;
  double smoothness, tol;
  double bin_widths[65];
  uint64_t payload_len;
  uint32_t checksum;
  uint64_t header_size;
  uint8_t l2_projection; /* header flag 0x04: the L2-corrected decomposition (not readable by the reference) */
} mgrc_container_info;

/* Replaces mgrc::compress(span<const float|double>, TensorGrid, ErrorSpec,
 * Codec, exec) — container.hpp:69-74.  `coords` is NULL (index coordinates,
 * make_grid(shape), grid.cpp:56) or ndims pointers to per-axis coordinates
 * (make_grid(shape, coords), grid.cpp:70).  *out is a host buffer owned by
 * the caller (release with mgrc_gpu_free). */
MGRC_GPU_API int mgrc_gpu_compress(const void* data, int dtype, int ndims, const uint64_t* shape,
                                   const double* const* coords, double tol, int norm, double smoothness, int mode,
                                   int codec, uint8_t** out, uint64_t* out_len);

/* Same, writing the container into a caller buffer (host or device).  With
 * dst == NULL only *out_len is produced (the container stays staged). */
MGRC_GPU_API int mgrc_gpu_compress_to(const void* data, int dtype, int ndims, const uint64_t* shape,
                                      const double* const* coords, double tol, int norm, double smoothness, int mode,
                                      int codec, void* dst, uint64_t dst_capacity, uint64_t* out_len);

/* The same two on the decomposition with MGARD's L2-projection correction
 * (mgrc_gpu_forward_transform_l2): the reference's quantiser, accept loop and
 * lossless stage on the corrected coefficients, the a-posteriori error taken
 * through the corrected recomposition.  The container carries header flag
 * 0x04 (the reference rejects it as unknown, container.cpp:143); the
 * decompress entry points below read it. */
MGRC_GPU_API int mgrc_gpu_compress_l2(const void* data, int dtype, int ndims, const uint64_t* shape,
                                      const double* const* coords, double tol, int norm, double smoothness, int mode,
                                      int codec, uint8_t** out, uint64_t* out_len);
MGRC_GPU_API int mgrc_gpu_compress_l2_to(const void* data, int dtype, int ndims, const uint64_t* shape,
                                         const double* const* coords, double tol, int norm, double smoothness,
                                         int mode, int codec, void* dst, uint64_t dst_capacity, uint64_t* out_len);

/* Replaces mgrc::decompress(span<const uint8_t>, exec) — container.hpp:76-77.
 * *out is a host buffer of prod(shape) floats (dtype f32) or doubles. */
MGRC_GPU_API int mgrc_gpu_decompress(const uint8_t* in, uint64_t len, void** out, int* dtype, int* ndims,
                                     uint64_t* shape);

/* Same, into a caller buffer (host or device) of dst_capacity bytes. */
MGRC_GPU_API int mgrc_gpu_decompress_into(const uint8_t* in, uint64_t len, void* dst, uint64_t dst_capacity,
                                          int* dtype, int* ndims, uint64_t* shape);

/* Replaces mgrc::inspect / mgrc::describe — container.hpp:79-83 (host only). */
MGRC_GPU_API int mgrc_gpu_inspect(const uint8_t* in, uint64_t len, mgrc_container_info* info);
MGRC_GPU_API int mgrc_gpu_describe(const uint8_t* in, uint64_t len, char** text);

/* Replaces mgrc::plan_chunks (chunking.hpp:38-44).  ranges[(b*ndims + a)*2 +
 * {0,1}] = [begin, end) of block b on axis a, row-major block order. */
MGRC_GPU_API int mgrc_gpu_plan_chunks(int ndims, const uint64_t* shape, int dtype, uint64_t budget,
                                      uint64_t* nblocks, uint64_t* ranges, uint64_t cap_blocks);

/* The CLI's multiblock compress (tools/mgrc.cpp:363-484) on one GPU: global
 * REL normalisation, per-block ABS compress with the block's coordinate
 * slice, and the u32 count | u64 offsets | containers framing. */
MGRC_GPU_API int mgrc_gpu_compress_chunked(const void* data, int dtype, int ndims, const uint64_t* shape,
                                           const double* const* coords, double tol, int norm, double smoothness,
                                           int mode, int codec, uint64_t chunk_mem, uint8_t** out,
                                           uint64_t* out_len);

/* The CLI's multiblock decompress (tools/mgrc.cpp:490-542): offset
 * validation, placement from the blocks' coordinate slices, decode. */
MGRC_GPU_API int mgrc_gpu_decompress_chunked(const uint8_t* in, uint64_t len, void** out, int* dtype, int* ndims,
                                             uint64_t* shape);

/* The same two on `ngpus` GPUs of one process: one host thread
 * per rank, rank g on device g % device_count, slab b on rank floor(b*G/B)
 * (contiguous rows and stream ranges); the per-block compressed sizes are
 * all-gathered with NCCL (ncclCommInitAll + ncclAllGather, loaded at run
 * time) when the ranks sit on distinct devices.  Host inputs (a device input
 * is compressed on its own device); the output stream is byte-identical for
 * every ngpus. */
MGRC_GPU_API int mgrc_gpu_compress_chunked_multi(const void* data, int dtype, int ndims, const uint64_t* shape,
                                                 const double* const* coords, double tol, int norm, double smoothness,
                                                 int mode, int codec, uint64_t chunk_mem, int ngpus, uint8_t** out,
                                                 uint64_t* out_len);
MGRC_GPU_API int mgrc_gpu_decompress_chunked_multi(const uint8_t* in, uint64_t len, int ngpus, void** out, int* dtype,
                                                   int* ndims, uint64_t* shape);

/* ---- the decomposition and the quantiser as entry points of their own ----
 * f64 arrays, row-major over the grid (shape, coords as in mgrc_gpu_compress);
 * host or device pointers.  Bit-identical to the reference library. */

/* GridHierarchy::nlevels of make_grid(shape[, coords]) (grid.cpp:100-153). */
MGRC_GPU_API int mgrc_gpu_nlevels(int ndims, const uint64_t* shape, const double* const* coords, int* nlevels);
/* initial_bin_widths (error_control.cpp:42-60): widths[0..nlevels]. */
MGRC_GPU_API int mgrc_gpu_initial_bin_widths(double tau_abs, int norm, double smoothness, int ndims, int nlevels,
                                             double* widths);
/* Replaces forward_transform (transform.hpp:24-26, transform.cpp:163-178):
 * c = multilevel coefficients of u.  NonFiniteInput on NaN/Inf. */
MGRC_GPU_API int mgrc_gpu_forward_transform(const double* u, int ndims, const uint64_t* shape,
                                            const double* const* coords, double* c);
/* Replaces inverse_transform (transform.hpp:28-30, transform.cpp:180-191). */
MGRC_GPU_API int mgrc_gpu_inverse_transform(const double* c, int ndims, const uint64_t* shape,
                                            const double* const* coords, double* u);
/* The decomposition / recomposition with MGARD's L2-projection correction
 * (opt-in; the reference is interpolation-only): after the
 * level-l coefficients are formed the coarse values receive
 * z = M_{l-1}^{-1} R M_l c (mass-matrix multiply, restriction, tridiagonal
 * solve, axis by axis), so each coarse level is the L2 projection of the
 * finer one.  Same arguments as mgrc_gpu_forward/inverse_transform. */
MGRC_GPU_API int mgrc_gpu_forward_transform_l2(const double* u, int ndims, const uint64_t* shape,
                                               const double* const* coords, double* c);
MGRC_GPU_API int mgrc_gpu_inverse_transform_l2(const double* c, int ndims, const uint64_t* shape,
                                               const double* const* coords, double* u);
/* Replaces quantize (quantize.hpp:32-36, quantize.cpp:72-132): q = rne(c/delta_tag)
 * and (if residuals != NULL) r = c - q*delta_tag; nwidths must be nlevels+1
 * (ShapeMismatch), widths > 0 (InvalidState); Overflow when |c/delta| >= 2^63;
 * *outliers (nullable) = count of |q| > 2^31-1. */
MGRC_GPU_API int mgrc_gpu_quantize(const double* c, int ndims, const uint64_t* shape, const double* const* coords,
                                   const double* widths, int nwidths, int64_t* q, double* residuals,
                                   uint64_t* outliers);
/* Replaces dequantize (quantize.hpp:38-40, quantize.cpp:134-158): c = (double)q*delta_tag. */
MGRC_GPU_API int mgrc_gpu_dequantize(const int64_t* q, int ndims, const uint64_t* shape, const double* const* coords,
                                     const double* widths, int nwidths, double* c);

/* ---- MDR refactor / recompose (refactor.hpp:81-117) ----------------------
 * refactor: multilevel coefficients per level in node scan order, B-bit
 * fixed point against the level exponent, split into B bit planes (plane 0
 * interleaves the sign with the top magnitude bit), each (level, plane)
 * segment canonical-Huffman coded with its CRC-32 — byte-identical to the
 * reference's segments.  request: the reference's greedy planner.
 * reconstruct: applies segments in per-level prefix order to a
 * device-resident state and synthesises the field (inverse transform). */
typedef struct {
  int ndims;
  uint64_t shape[4];
  int nlevels;
  uint32_t planes;
  int32_t level_exponents[65]; /* INT32_MIN: the level is empty (all coefficients 0) */
  uint64_t level_counts[65];
  double value_min, value_max, value_rms;
} mgrc_mdr_manifest;
typedef struct {
  uint64_t bytes, raw_bits;
  uint32_t crc32;
} mgrc_mdr_segment;

/* refactor (refactor.cpp:144-218): f64 input (host or device); *store is an
 * opaque handle (mgrc_gpu_mdr_store_free). */
MGRC_GPU_API int mgrc_gpu_mdr_refactor(const double* u, int ndims, const uint64_t* shape,
                                       const double* const* coords, uint32_t planes, void** store);
/* The store's manifest and its (nlevels+1)*planes segment table (level-major; segs nullable). */
MGRC_GPU_API int mgrc_gpu_mdr_store_manifest(const void* store, mgrc_mdr_manifest* m, mgrc_mdr_segment* segs);
/* A segment payload (owned by the store). */
MGRC_GPU_API int mgrc_gpu_mdr_store_segment(const void* store, uint32_t level, uint32_t plane, const uint8_t** data,
                                            uint64_t* len);
MGRC_GPU_API void mgrc_gpu_mdr_store_free(void* store);
/* request (refactor.cpp:226-272) from a state with fetched[l] planes (NULL: none). */
MGRC_GPU_API int mgrc_gpu_mdr_request(const mgrc_mdr_manifest* m, const mgrc_mdr_segment* segs, double tol_abs,
                                      int norm, double smoothness, const uint32_t* fetched, uint32_t* levels,
                                      uint32_t* planes, uint64_t cap, uint64_t* n, uint64_t* total_bytes,
                                      double* predicted, int* satisfiable);
/* A retrieval session (make_initial_state, refactor.cpp:210-221) on the current device. */
MGRC_GPU_API int mgrc_gpu_mdr_session_new(const mgrc_mdr_manifest* m, const mgrc_mdr_segment* segs,
                                          const double* const* coords, void** session);
/* reconstruct (refactor.cpp:274-357): applies the n segments (their payloads in
 * request order; checksum and per-level prefix order enforced) and writes the
 * refined field to out (host or device, prod(shape) doubles). */
MGRC_GPU_API int mgrc_gpu_mdr_reconstruct(void* session, const uint32_t* levels, const uint32_t* planes, uint64_t n,
                                          const uint8_t* const* payloads, const uint64_t* lens, int norm,
                                          double smoothness, double* out, double* accrued, uint32_t* fetched_out);
MGRC_GPU_API void mgrc_gpu_mdr_session_free(void* session);

/* Non-finite flag, min and max of an array (host or device) — the per-rank
 * statistics of the multi-GPU driver's global REL normalisation. */
MGRC_GPU_API int mgrc_gpu_field_stats(const void* data, int dtype, uint64_t n, double* min, double* max,
                                      int* nonfinite);

/* s0 + sum of v_i*v_i, added serially in index order with one rounding per
 * addition (exactly the CLI's scan_stats accumulation, tools/mgrc.cpp:227),
 * reproduced bit for bit on the device; host or device array.  Ranks holding
 * consecutive row ranges chain it (s0 = the previous rank's result) so the
 * multi-GPU S-REL tolerance equals the single-scan one. */
MGRC_GPU_API int mgrc_gpu_serial_sumsq(const void* data, int dtype, uint64_t n, double s0, double* out);

/* Page-locked host buffers for fast host<->device staging (the CLI's raw-file
 * reads land in one; any host pointer is accepted by the calls above). */
MGRC_GPU_API int mgrc_gpu_host_alloc(uint64_t bytes, void** p);
MGRC_GPU_API void mgrc_gpu_host_free(void* p);

MGRC_GPU_API const char* mgrc_gpu_last_error(void);
MGRC_GPU_API void mgrc_gpu_free(void* p);
MGRC_GPU_API int mgrc_gpu_set_device(int device);
/* Stream used by subsequent calls on this thread (a cudaStream_t; NULL = own stream). */
MGRC_GPU_API int mgrc_gpu_set_stream(void* stream);
/* Per-phase CUDA-event timing of the last call on this thread. */
MGRC_GPU_API int mgrc_gpu_set_profiling(int on);
MGRC_GPU_API int mgrc_gpu_profile_count(void);
MGRC_GPU_API int mgrc_gpu_profile_entry(int i, const char** name, double* ms, double* bytes);
MGRC_GPU_API const char* mgrc_gpu_version(void);
/* Accept decision of the calling thread's last compress (container.cpp:93-123):
 * the absolute tolerance tau, the achieved error the decision compared with
 * tau*(1-1e-9) (error_control.cpp:62-101; for S(s!=0) the reference's
 * level-weighted estimator), the shrink passes run, and how it was decided:
 * 0 none (constant field), 1 a-priori bound (L+1)*max|r| (reported in
 * *achieved), 2 the exact a-posteriori value, 3 the same after the S(s!=0)
 * estimator's fixed-order sum could not certify the decision and the
 * reference's serial per-level sums were reproduced exactly. */
MGRC_GPU_API int mgrc_gpu_last_compress_stats(double* tau_abs, double* achieved, int* passes, int* decided_by);
/* Kernels launched by the calling thread through this library so far. */
MGRC_GPU_API uint64_t mgrc_gpu_launch_count(void);

#ifdef __cplusplus
}
#endif

#endif /* MGRC_GPU_H */
