// Device pipeline: compress / decompress of one container on one GPU.
#pragma once

#include <cuda_runtime.h>

#include <climits>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "host.hpp"

namespace mgrc_gpu {

struct PhaseTime {
  std::string name;
  double ms;
  double bytes;  // algorithmic bytes moved by the phase (0 when not a kernel of interest)
};

// A compressed container split into a host part (container header, plus the
// Huffman table header for codec 2) and a device part (the coded stream).
struct ContainerParts {
  std::vector<uint8_t> head;   // host bytes
  const uint8_t* dev = nullptr;  // device bytes (owned by the context workspace)
  uint64_t dev_len = 0;
  std::vector<uint8_t> host_tail;  // tail bytes kept on the host (constant field payload)
  uint64_t total() const { return head.size() + dev_len + host_tail.size(); }
};

struct DecodedInfo {
  DType dtype;
  int ndims;
  uint64_t shape[kMaxDims];
};

class Context;

// Per-thread, per-device context (streams + grow-only workspace); calls are
// reentrant across threads because no state is shared between contexts.
Context& context_for_current_device();
void context_set_stream(Context& c, cudaStream_t s);
cudaStream_t context_stream(Context& c);
void context_set_profiling(Context& c, bool on);
const std::vector<PhaseTime>& context_profile(Context& c);

// data: host or device pointer (auto-detected), N elements of dtype.
ContainerParts compress(Context& ctx, const void* data, DType dtype, const Grid& grid, const ErrorSpec& spec,
                        Codec codec);

// The same on the L²-corrected decomposition (header flag 0x04; transform.cu).
ContainerParts compress_l2(Context& ctx, const void* data, DType dtype, const Grid& grid, const ErrorSpec& spec,
                           Codec codec);

// Parses and validates; decodes into `out` (host or device, capacity checked).
DecodedInfo decompress_into(Context& ctx, const uint8_t* in, uint64_t len, void* out, uint64_t out_capacity_bytes);
ContainerInfo inspect_any(Context& ctx, const uint8_t* in, uint64_t len);

bool is_device_pointer(const void* p);

// Accept decision of the last compress on this thread (container.cpp:93-123):
// τ_abs, the achieved error the decision used (the reference's exact value, or
// for decided_by == 1 the a-priori bound (L+1)·max|r| that already passes),
// the number of shrink passes, and how it was decided (0 = constant field /
// not run, 1 = bound, 2 = exact a-posteriori value).
struct CompressStats {
  double tau_abs, achieved;
  int passes, decided_by;
};
const CompressStats& last_compress_stats();

// Number of kernels this thread has launched through the library.
unsigned long long launch_count();

// Input statistics used by the multi-GPU driver for global REL normalisation.
struct FieldStats {
  double min, max;
  bool nonfinite;
};
FieldStats field_stats(Context& ctx, const void* data, DType dtype, uint64_t n);

// Whole-array statistics of the CLI's scan_stats (tools/mgrc.cpp:197-233):
// min, max, non-finite flag and Σv² summed serially in index order, bit-exact
// (host arrays are streamed through a bounded device staging buffer).
struct GlobalStats {
  double min, max, sumsq;
  bool nonfinite;
};
GlobalStats global_stats(Context& ctx, const void* data, DType dtype, uint64_t n, bool want_sumsq);

// s0 + Σ p_i in index order with one rounding per addition (p_i = v_i² when
// `square`), reproduced exactly on the device (serial_sum.cuh).  Terms ≥ 0.
double exact_serial_sum(Context& ctx, const void* v, DType dtype, uint64_t n, bool square, double s0);
// s0 + Σ v_i² serially in index order over a host or device array (the
// continuation of the CLI's scan_stats sum, tools/mgrc.cpp:227).
double serial_sumsq(Context& ctx, const void* data, DType dtype, uint64_t n, double s0);


// ---- MDR refactor / request / reconstruct (refactor.hpp:81-117) ----------
// Per-(level, bitplane) precision segments of the multilevel coefficients,
// each canonical-Huffman coded with its CRC; the greedy planner on the host;
// progressive reconstruction on the device.
constexpr int kMdrEmptyExponent = INT32_MIN;  // empty_level_exponent (error_control.hpp:40)
struct MdrSegment {
  uint64_t bytes = 0, raw_bits = 0;
  uint32_t crc = 0;
};
struct MdrManifest {  // StoreManifest (refactor.hpp:33-45); dtype is always f64
  Grid grid;
  int nlevels = 0;
  uint32_t planes = 32;
  std::vector<int> exps;
  std::vector<uint64_t> counts;
  double vmin = 0, vmax = 0, vrms = 0;
  std::vector<std::vector<MdrSegment>> seg;  // [level][plane]
};
struct MdrStore {
  MdrManifest m;
  std::vector<std::vector<std::vector<uint8_t>>> payload;  // [level][plane]
};
struct MdrRequest {
  std::vector<std::pair<uint32_t, uint32_t>> segs;  // (level, plane) in fetch order
  uint64_t bytes = 0;
  double predicted = 0;
  bool satisfiable = true;
};
MdrStore mdr_refactor(Context& ctx, const double* u, const Grid& grid, uint32_t planes);
double mdr_estimator(const MdrManifest& m, const std::vector<uint32_t>& fetched, Norm norm, double s);
MdrRequest mdr_request(const MdrManifest& m, double tol_abs, Norm norm, double s, std::vector<uint32_t> fetched);
class MdrSession;  // device-resident RetrievalState (refactor.hpp:56-62)
MdrSession* mdr_session_new(const MdrManifest& m);
void mdr_session_free(MdrSession* s);
const std::vector<uint32_t>& mdr_session_fetched(const MdrSession* s);
// Applies the segments (payloads given in request order), then writes the
// refined field (host or device pointer); returns the accrued estimator.
double mdr_reconstruct(Context& ctx, MdrSession& ss, const std::vector<std::pair<uint32_t, uint32_t>>& segs,
                       const std::vector<const uint8_t*>& payloads, const std::vector<uint64_t>& lens, Norm norm,
                       double s, double* out);

}  // namespace mgrc_gpu
