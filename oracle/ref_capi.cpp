// TEST INFRASTRUCTURE ONLY — not part of the product.
//
// extern "C" shim over the *unmodified* reference library.  oracle/Makefile
// compiles this file together with /root/reference/proj/src/*.cpp (read in
// place, never copied) into oracle/_ref/libmgrc_ref.so.  It exports the same
// oc_* API as the C restatement (oracle/mgrc_oracle.c) so the parity tests
// can pin the restatement against the real reference, and bench.py's
// reference arm can time the reference's own CPU path.
//
// The only restated logic here is the CLI multiblock driver
// (oc_compress_chunked, tools/mgrc.cpp:363-484): the CLI itself cannot be
// built in this image (CLI11.hpp absent, tools/mgrc.cpp:16).

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <span>
#include <string>
#include <vector>

#include "mgrc/bytes.hpp"
#include "mgrc/chunking.hpp"
#include "mgrc/codec.hpp"
#include "mgrc/container.hpp"
#include "mgrc/error.hpp"
#include "mgrc/error_control.hpp"
#include "mgrc/exec.hpp"
#include "mgrc/grid.hpp"
#include "mgrc/quantize.hpp"
#include "mgrc/refactor.hpp"
#include "mgrc/transform.hpp"
#include "support/test_support.hpp"

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

thread_local std::string g_err;

template <class Fn>
int guard(Fn fn) {
  try {
    fn();
    return 0;
  } catch (const mgrc::error& e) {
    g_err = e.what();
    return static_cast<int>(e.code()) + 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 100;
  }
}

mgrc::TensorGrid grid_of(int ndims, const uint64_t* shape, const double* coords) {
  std::vector<std::size_t> s(shape, shape + ndims);
  if (!coords) return mgrc::make_grid(s);
  std::vector<std::vector<double>> c(ndims);
  std::size_t off = 0;
  for (int a = 0; a < ndims; ++a) {
    c[a].assign(coords + off, coords + off + shape[a]);
    off += shape[a];
  }
  return mgrc::make_grid(s, c);
}

uint64_t count_of(int ndims, const uint64_t* shape) {
  uint64_t n = 1;
  for (int a = 0; a < ndims; ++a) n *= shape[a];
  return n;
}

mgrc::ErrorSpec spec_of(double tol, int norm, double s, int mode) {
  mgrc::ErrorSpec sp;
  sp.tol = tol;
  sp.norm = static_cast<mgrc::Norm>(norm);
  sp.smoothness = s;
  sp.mode = static_cast<mgrc::Mode>(mode);
  return sp;
}

template <class T>
T* dup(const std::vector<T>& v) {
  T* p = static_cast<T*>(std::malloc(v.size() * sizeof(T) + 1));
  if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(T));
  return p;
}

struct oc_info {
  uint16_t version;
  uint8_t constant_field, coords_present, dtype, ndims, nlevels, codec_id;
  uint64_t shape[4];
  uint8_t mode, norm;
  double smoothness, tol;
  double bin_widths[65];
  uint64_t payload_len;
  uint32_t checksum;
  uint64_t header_size;
};

}  // namespace

extern "C" {

const char* oc_last_error(void) { return g_err.c_str(); }
void oc_free(void* p) { std::free(p); }
int oc_set_threads(int n) {
  mgrc::set_worker_count(n);
  return mgrc::worker_count();
}
const char* oc_impl(void) { return "reference"; }

int oc_compress(const void* data, int dtype, int ndims, const uint64_t* shape, const double* coords, double tol, int norm,
                double s, int mode, int codec, uint8_t** out, uint64_t* out_len) {
  return guard([&] {
    const auto g = grid_of(ndims, shape, coords);
    const auto sp = spec_of(tol, norm, s, mode);
    const uint64_t n = count_of(ndims, shape);
    mgrc::CompressedContainer c =
        dtype == 0 ? mgrc::compress(std::span<const float>(static_cast<const float*>(data), n), g, sp,
                                    static_cast<mgrc::Codec>(codec))
                   : mgrc::compress(std::span<const double>(static_cast<const double*>(data), n), g, sp,
                                    static_cast<mgrc::Codec>(codec));
    *out = dup(c.bytes);
    *out_len = c.bytes.size();
  });
}

int oc_decompress(const uint8_t* in, uint64_t len, void** out, int* dtype, int* ndims, uint64_t* shape) {
  return guard([&] {
    auto a = mgrc::decompress(std::span<const uint8_t>(in, len));
    *dtype = static_cast<int>(a.dtype);
    *ndims = static_cast<int>(a.shape.size());
    for (std::size_t i = 0; i < a.shape.size(); ++i) shape[i] = a.shape[i];
    if (a.dtype == mgrc::DType::f32) *out = dup(std::get<std::vector<float>>(a.values));
    else *out = dup(std::get<std::vector<double>>(a.values));
  });
}

int oc_inspect(const uint8_t* in, uint64_t len, oc_info* info) {
  return guard([&] {
    const auto ci = mgrc::inspect(std::span<const uint8_t>(in, len));
    std::memset(info, 0, sizeof *info);
    info->version = ci.version;
    info->constant_field = ci.constant_field;
    info->coords_present = ci.coords_present;
    info->dtype = static_cast<uint8_t>(ci.dtype);
    info->ndims = static_cast<uint8_t>(ci.shape.size());
    info->nlevels = ci.nlevels;
    info->codec_id = ci.codec_id;
    for (std::size_t a = 0; a < ci.shape.size(); ++a) info->shape[a] = ci.shape[a];
    info->mode = static_cast<uint8_t>(ci.spec.mode);
    info->norm = static_cast<uint8_t>(ci.spec.norm);
    info->smoothness = ci.spec.smoothness;
    info->tol = ci.spec.tol;
    for (std::size_t l = 0; l < ci.bin_widths.size() && l < 65; ++l) info->bin_widths[l] = ci.bin_widths[l];
    info->payload_len = ci.payload_len;
    info->checksum = ci.checksum;
    info->header_size = ci.header_size;
  });
}

int oc_describe(const uint8_t* in, uint64_t len, char** text) {
  return guard([&] {
    const std::string s = mgrc::describe(mgrc::inspect(std::span<const uint8_t>(in, len)));
    *text = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(*text, s.c_str(), s.size() + 1);
  });
}

int oc_hierarchy(int ndims, const uint64_t* shape, const double* coords, int* nlevels, uint8_t* axis_level,
                 uint64_t* node_counts, uint64_t* level_sizes, int cap_levels) {
  return guard([&] {
    const auto h = mgrc::build_hierarchy(grid_of(ndims, shape, coords));
    *nlevels = static_cast<int>(h.nlevels);
    uint64_t off = 0;
    for (int a = 0; a < ndims; ++a) {
      if (axis_level) std::memcpy(axis_level + off, h.axis_level[a].data(), shape[a]);
      off += shape[a];
    }
    for (std::size_t l = 0; l <= h.nlevels && static_cast<int>(l) < cap_levels; ++l) {
      if (node_counts) node_counts[l] = h.level_node_counts[l];
      if (level_sizes)
        for (int a = 0; a < ndims; ++a) level_sizes[l * ndims + a] = h.level_shapes[l][a];
    }
  });
}

int oc_level_set(int ndims, const uint64_t* shape, int level, int axis, uint64_t* out, uint64_t* n) {
  return guard([&] {
    const auto h = mgrc::build_hierarchy(grid_of(ndims, shape, nullptr));
    if (level < 0 || static_cast<std::size_t>(level) > h.nlevels)
      mgrc::raise(mgrc::errc::level_out_of_range, "level");
    const auto& s = h.level_index_sets[level][axis];
    *n = s.size();
    if (out)
      for (std::size_t i = 0; i < s.size(); ++i) out[i] = s[i];
  });
}

int oc_forward(int ndims, const uint64_t* shape, const double* coords, const double* u, double* c) {
  return guard([&] {
    const auto h = mgrc::build_hierarchy(grid_of(ndims, shape, coords));
    const uint64_t n = count_of(ndims, shape);
    const auto mc = mgrc::forward_transform(std::span<const double>(u, n), h);
    std::memcpy(c, mc.values.data(), n * 8);
  });
}

int oc_inverse(int ndims, const uint64_t* shape, const double* coords, const double* c, double* u) {
  return guard([&] {
    const auto h = mgrc::build_hierarchy(grid_of(ndims, shape, coords));
    const uint64_t n = count_of(ndims, shape);
    mgrc::MultilevelCoefficients mc{std::vector<double>(c, c + n), &h};
    const auto v = mgrc::inverse_transform(mc);
    std::memcpy(u, v.data(), n * 8);
  });
}

int oc_quantize(int ndims, const uint64_t* shape, const double* coords, const double* c, const double* widths, int64_t* q,
                double* res, uint64_t* outliers) {
  return guard([&] {
    const auto h = mgrc::build_hierarchy(grid_of(ndims, shape, coords));
    const uint64_t n = count_of(ndims, shape);
    mgrc::MultilevelCoefficients mc{std::vector<double>(c, c + n), &h};
    mgrc::LevelBudget b;
    b.bin_widths.assign(widths, widths + h.nlevels + 1);
    const auto qr = mgrc::quantize(mc, b);
    std::memcpy(q, qr.q.qvalues.data(), n * 8);
    std::memcpy(res, qr.residuals.values.data(), n * 8);
    if (outliers) *outliers = qr.q.outlier_count;
  });
}

int oc_dequantize(int ndims, const uint64_t* shape, const double* coords, const int64_t* q, const double* widths, double* c) {
  return guard([&] {
    const auto h = mgrc::build_hierarchy(grid_of(ndims, shape, coords));
    const uint64_t n = count_of(ndims, shape);
    mgrc::QuantizedCoefficients qc;
    qc.qvalues.assign(q, q + n);
    qc.budget.bin_widths.assign(widths, widths + h.nlevels + 1);
    const auto mc = mgrc::dequantize(qc, h);
    std::memcpy(c, mc.values.data(), n * 8);
  });
}

double oc_round_half_even(double x) { return mgrc::round_half_even(x); }

int oc_absolute_tolerance(const double* u, uint64_t n, double tol, int norm, double s, int mode, double* out) {
  return guard([&] { *out = mgrc::absolute_tolerance(spec_of(tol, norm, s, mode), std::span<const double>(u, n)); });
}

int oc_bin_widths(double tau, int norm, double s, int ndims, int nlevels, double* out) {
  return guard([&] {
    // initial_bin_widths reads only nlevels and ndims from the hierarchy.
    mgrc::GridHierarchy h;
    h.grid.shape.assign(ndims, 2);
    h.nlevels = nlevels;
    const auto b = mgrc::initial_bin_widths(tau, spec_of(1.0, norm, s, 0), h);
    for (std::size_t l = 0; l < b.bin_widths.size(); ++l) out[l] = b.bin_widths[l];
  });
}

int oc_achieved_error(int ndims, const uint64_t* shape, const double* coords, const double* res, int norm, double s,
                      double* out) {
  return guard([&] {
    const auto h = mgrc::build_hierarchy(grid_of(ndims, shape, coords));
    const uint64_t n = count_of(ndims, shape);
    mgrc::MultilevelCoefficients mc{std::vector<double>(res, res + n), &h};
    *out = mgrc::achieved_error(mc, spec_of(1.0, norm, s, 0), h).value;
  });
}

double oc_sum_squares(const double* v, uint64_t n) {
  return mgrc::kernels::sum_squares(std::span<const double>(v, n), mgrc::exec::parallel);
}

uint32_t oc_crc32(const uint8_t* data, uint64_t n) { return mgrc::crc32(std::span<const uint8_t>(data, n)); }

int oc_huffman_pack(const uint8_t* in, uint64_t n, uint8_t** out, uint64_t* out_len) {
  return guard([&] {
    const auto v = mgrc::huffman_pack_bytes(std::span<const uint8_t>(in, n));
    *out = dup(v);
    *out_len = v.size();
  });
}

int oc_huffman_unpack(const uint8_t* in, uint64_t n, uint64_t count, uint8_t* out) {
  return guard([&] {
    const auto v = mgrc::huffman_unpack_bytes(std::span<const uint8_t>(in, n), count);
    std::memcpy(out, v.data(), v.size());
  });
}

int oc_lossless_encode(const int64_t* v, uint64_t n, int codec, uint8_t** out, uint64_t* out_len) {
  return guard([&] {
    const auto b = mgrc::lossless_encode(std::span<const int64_t>(v, n), static_cast<mgrc::Codec>(codec));
    *out = dup(b.payload);
    *out_len = b.payload.size();
  });
}

int oc_lossless_decode(const uint8_t* p, uint64_t len, uint64_t count, int codec, int64_t* out) {
  return guard([&] {
    mgrc::LosslessBlock b;
    b.codec_id = static_cast<uint8_t>(codec);
    b.payload.assign(p, p + len);
    b.original_count = count;
    const auto v = mgrc::lossless_decode(b);
    std::memcpy(out, v.data(), v.size() * 8);
  });
}

int oc_plan_chunks(int ndims, const uint64_t* shape, int dtype, uint64_t budget, uint64_t* nblocks, uint64_t* out,
                   uint64_t cap_blocks) {
  return guard([&] {
    std::vector<std::size_t> s(shape, shape + ndims);
    const auto plan = mgrc::plan_chunks(s, static_cast<mgrc::DType>(dtype), budget);
    *nblocks = plan.block_count();
    if (out && plan.block_count() <= cap_blocks)
      for (std::size_t b = 0; b < plan.block_count(); ++b) {
        const auto r = plan.block(b);
        for (int a = 0; a < ndims; ++a) {
          out[(b * ndims + a) * 2] = r[a].begin;
          out[(b * ndims + a) * 2 + 1] = r[a].end;
        }
      }
  });
}

// Restatement of tools/mgrc.cpp:363-484 on an in-memory array: REL is
// normalised by the CLI's serial whole-file scan (:197-233), blocks are
// compressed with exec::serial under an OpenMP dynamic loop (:432-473), and
// the multiblock file is written as u32 count | u64 offsets | containers
// (:258-275).
int oc_compress_chunked(const void* data, int dtype, int ndims, const uint64_t* shape, const double* coords, double tol,
                        int norm, double s, int mode, int codec, uint64_t chunk_mem, uint8_t** out, uint64_t* out_len) {
  return guard([&] {
    std::vector<std::size_t> sh(shape, shape + ndims);
    const auto dt = static_cast<mgrc::DType>(dtype);
    const uint64_t count = count_of(ndims, shape);
    const auto spec = spec_of(tol, norm, s, mode);
    const auto plan = mgrc::plan_chunks(sh, dt, chunk_mem > 0 ? chunk_mem : UINT64_MAX);
    const std::size_t nb = plan.block_count();
    auto value = [&](uint64_t i) {
      return dtype == 0 ? static_cast<double>(static_cast<const float*>(data)[i]) : static_cast<const double*>(data)[i];
    };
    std::vector<std::vector<double>> user_coords;
    if (coords) {
      user_coords.resize(ndims);
      std::size_t off = 0;
      for (int a = 0; a < ndims; ++a) {
        user_coords[a].assign(coords + off, coords + off + shape[a]);
        off += shape[a];
      }
    }
    std::vector<std::vector<uint8_t>> blocks(nb);
    const std::size_t unit = mgrc::dtype_size(dt);
    if (nb == 1) {
      const auto g = user_coords.empty() ? mgrc::make_grid(sh) : mgrc::make_grid(sh, user_coords);
      blocks[0] = dtype == 0 ? mgrc::compress(std::span<const float>(static_cast<const float*>(data), count), g, spec,
                                              static_cast<mgrc::Codec>(codec))
                                   .bytes
                             : mgrc::compress(std::span<const double>(static_cast<const double*>(data), count), g,
                                              spec, static_cast<mgrc::Codec>(codec))
                                   .bytes;
    } else {
      mgrc::ErrorSpec bspec = spec;
      bspec.mode = mgrc::Mode::abs;
      if (spec.mode == mgrc::Mode::rel) {
        double mn = 0, mx = 0, sumsq = 0;
        for (uint64_t i = 0; i < count; ++i) {
          const double v = value(i);
          if (!std::isfinite(v)) mgrc::raise(mgrc::errc::non_finite_input, "input contains NaN or Inf");
          if (i == 0 || v < mn) mn = v;
          if (i == 0 || v > mx) mx = v;
          sumsq += v * v;
        }
        const double nrm = spec.norm == mgrc::Norm::inf ? mx - mn : std::sqrt(sumsq / static_cast<double>(count));
        if (nrm == 0.0) mgrc::raise(mgrc::errc::degenerate_data, "relative bound on a constant file");
        bspec.tol = spec.tol * nrm;
      }
      std::vector<std::vector<double>> cs = user_coords;
      if (cs.empty()) {
        cs.resize(ndims);
        for (int a = 0; a < ndims; ++a) {
          cs[a].resize(shape[a]);
          for (uint64_t i = 0; i < shape[a]; ++i) cs[a][i] = static_cast<double>(i);
        }
      }
      std::vector<std::size_t> stride(ndims, 1);
      for (int a = ndims - 1; a-- > 0;) stride[a] = stride[a + 1] * shape[a + 1];
      std::exception_ptr failure;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic) num_threads(mgrc::worker_count())
#endif
      for (std::ptrdiff_t bi = 0; bi < static_cast<std::ptrdiff_t>(nb); ++bi) {
        try {
          const auto b = static_cast<std::size_t>(bi);
          const auto ranges = plan.block(b);
          std::vector<std::size_t> bshape(ndims);
          std::vector<std::vector<double>> bc(ndims);
          std::size_t bn = 1;
          for (int a = 0; a < ndims; ++a) {
            bshape[a] = ranges[a].length();
            bn *= bshape[a];
            bc[a].assign(cs[a].begin() + ranges[a].begin, cs[a].begin() + ranges[a].end);
          }
          std::vector<uint8_t> bd(bn * unit);
          std::vector<std::size_t> idx(ndims, 0);
          for (std::size_t f = 0; f < bn; ++f) {
            std::size_t src = 0;
            for (int a = 0; a < ndims; ++a) src += (ranges[a].begin + idx[a]) * stride[a];
            std::memcpy(bd.data() + f * unit, static_cast<const uint8_t*>(data) + src * unit, unit);
            for (int a = ndims; a-- > 0;) {
              if (++idx[a] < bshape[a]) break;
              idx[a] = 0;
            }
          }
          const auto g = mgrc::make_grid(bshape, bc);
          blocks[b] = dtype == 0 ? mgrc::compress(std::span<const float>(reinterpret_cast<const float*>(bd.data()), bn),
                                                  g, bspec, static_cast<mgrc::Codec>(codec), mgrc::exec::serial)
                                       .bytes
                                 : mgrc::compress(std::span<const double>(reinterpret_cast<const double*>(bd.data()), bn),
                                                  g, bspec, static_cast<mgrc::Codec>(codec), mgrc::exec::serial)
                                       .bytes;
        } catch (...) {
#ifdef _OPENMP
#pragma omp critical
#endif
          if (!failure) failure = std::current_exception();
        }
      }
      if (failure) std::rethrow_exception(failure);
    }
    std::vector<uint8_t> file;
    mgrc::put_u32(file, static_cast<uint32_t>(nb));
    uint64_t off = 4 + 8 * nb;
    for (const auto& b : blocks) {
      mgrc::put_u64(file, off);
      off += b.size();
    }
    for (const auto& b : blocks) file.insert(file.end(), b.begin(), b.end());
    *out = dup(file);
    *out_len = file.size();
  });
}


// ---- MDR refactor / request / reconstruct (refactor.hpp:81-117) -----------
// The reference's own functions; a store and a retrieval session are opaque
// handles (test infrastructure for the GPU refactor's parity).

struct OcSession {
  mgrc::StoreManifest manifest;
  const mgrc::RefactoredStore* store;
  mgrc::RetrievalState state;
};

void* oc_mdr_refactor(const double* u, int ndims, const uint64_t* shape, const double* coords, uint32_t planes) {
  void* out = nullptr;
  if (guard([&] {
        const auto g = grid_of(ndims, shape, coords);
        auto* st = new mgrc::RefactoredStore(
            mgrc::refactor(std::span<const double>(u, count_of(ndims, shape)), g, planes));
        out = st;
      }) != 0)
    return nullptr;
  return out;
}

int oc_mdr_manifest_json(void* store, char** out) {
  return guard([&] {
    const std::string j = mgrc::manifest_to_json(static_cast<mgrc::RefactoredStore*>(store)->manifest);
    *out = static_cast<char*>(std::malloc(j.size() + 1));
    std::memcpy(*out, j.c_str(), j.size() + 1);
  });
}

int oc_mdr_segment(void* store, uint32_t l, uint32_t p, uint8_t** out, uint64_t* n) {
  return guard([&] {
    const auto& seg = static_cast<mgrc::RefactoredStore*>(store)->segments.at(l).at(p);
    *out = dup(seg);
    *n = seg.size();
  });
}

void oc_mdr_free(void* store) { delete static_cast<mgrc::RefactoredStore*>(store); }

int oc_mdr_request(const char* manifest_json, double tol_abs, int norm, double s, const uint32_t* fetched,
                   uint32_t* levels, uint32_t* planes, uint64_t cap, uint64_t* nseg, uint64_t* bytes,
                   double* predicted, int* satisfiable) {
  return guard([&] {
    const mgrc::StoreManifest m = mgrc::manifest_from_json(manifest_json);
    mgrc::RetrievalState st = mgrc::make_initial_state(m);
    for (std::size_t l = 0; l < st.planes_fetched.size(); ++l) st.planes_fetched[l] = fetched ? fetched[l] : 0;
    const mgrc::SegmentRequest r = mgrc::request(m, tol_abs, static_cast<mgrc::Norm>(norm), s, st);
    *nseg = r.segments.size();
    for (std::size_t i = 0; i < r.segments.size() && i < cap; ++i) {
      levels[i] = r.segments[i].level;
      planes[i] = r.segments[i].plane;
    }
    *bytes = r.total_bytes;
    *predicted = r.predicted.value;
    *satisfiable = r.satisfiable ? 1 : 0;
  });
}

void* oc_mdr_session(const char* manifest_json, void* store) {
  void* out = nullptr;
  if (guard([&] {
        auto* ss = new OcSession;
        ss->manifest = mgrc::manifest_from_json(manifest_json);
        ss->store = static_cast<mgrc::RefactoredStore*>(store);
        ss->state = mgrc::make_initial_state(ss->manifest);
        out = ss;
      }) != 0)
    return nullptr;
  return out;
}

int oc_mdr_reconstruct(void* sess, const uint32_t* levels, const uint32_t* planes, uint64_t nseg, int norm, double s,
                       double* out, double* accrued) {
  return guard([&] {
    auto* ss = static_cast<OcSession*>(sess);
    mgrc::SegmentRequest req;
    for (uint64_t i = 0; i < nseg; ++i) req.segments.push_back({levels[i], planes[i]});
    req.predicted.norm = static_cast<mgrc::Norm>(norm);
    req.predicted.smoothness = s;
    const auto* store = ss->store;
    const mgrc::SegmentSource src = [store](std::uint32_t l, std::uint32_t p) { return store->segments.at(l).at(p); };
    const std::vector<double> v = mgrc::reconstruct(ss->manifest, src, req, ss->state);
    std::memcpy(out, v.data(), v.size() * sizeof(double));
    *accrued = ss->state.accrued.value;
  });
}

void oc_mdr_session_free(void* sess) { delete static_cast<OcSession*>(sess); }

void oc_multisine(int ndims, const uint64_t* shape, double* out) {
  std::vector<std::size_t> s(shape, shape + ndims);
  const auto u = mgrc::test::multisine(s);
  std::memcpy(out, u.data(), u.size() * 8);
}

void oc_mt19937_64(uint64_t seed, uint64_t n, uint64_t* out) {
  mgrc::test::Rng r(seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = r.bits();
}

void oc_random_field(uint64_t n, uint64_t seed, double lo, double hi, double* out) {
  mgrc::test::Rng r(seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = r.uniform(lo, hi);
}

void oc_multisine_noisy(int ndims, const uint64_t* shape, uint64_t seed, double noise, double* out) {
  std::vector<std::size_t> s(shape, shape + ndims);
  mgrc::test::Rng r(seed);
  const auto u = mgrc::test::multisine_noisy(s, r, noise);
  std::memcpy(out, u.data(), u.size() * 8);
}

}  // extern "C"
