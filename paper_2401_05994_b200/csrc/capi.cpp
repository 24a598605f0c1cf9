// extern "C" boundary (include/mgrc_gpu.h).  Exceptions never cross it: every
// entry point maps mgrc_gpu::Error to its errc ordinal + 1 and keeps the
// message in a thread-local slot, mirroring mgrc::error (error.hpp:34-47).
#include <cuda_runtime.h>

#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/mgrc_gpu.h"
#include "host.hpp"
#include "pipeline.hpp"
#include "transform.hpp"

using namespace mgrc_gpu;

namespace {

thread_local std::string g_last_error;

template <class Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    g_last_error.clear();
    return MGRC_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return static_cast<int>(e.code());
  } catch (const std::bad_alloc&) {
    g_last_error = "out of host memory";
    return MGRC_E_CUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return MGRC_E_CUDA;
  }
}

void require(bool ok, const char* what) {
  if (!ok) raise(Errc::invalid_argument, what);
}

DType to_dtype(int d) {
  if (d != 0 && d != 1) raise(Errc::invalid_argument, "dtype must be 0 (f32) or 1 (f64)");
  return static_cast<DType>(d);
}

ErrorSpec to_spec(double tol, int norm, double s, int mode) {
  if (norm != 0 && norm != 1) raise(Errc::invalid_argument, "norm must be 0 (inf) or 1 (s)");
  if (mode != 0 && mode != 1) raise(Errc::invalid_argument, "mode must be 0 (abs) or 1 (rel)");
  ErrorSpec sp;
  sp.tol = tol;
  sp.norm = static_cast<Norm>(norm);
  sp.smoothness = s;
  sp.mode = static_cast<Mode>(mode);
  return sp;
}

Codec to_codec(int c) {
  if (c < 0 || c > 2) raise(Errc::unknown_codec, "codec " + std::to_string(c));
  return static_cast<Codec>(c);
}

void ensure_device() {
  int n = 0;
  const cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    raise(Errc::cuda, "no CUDA device available (the sm_100a path has no CPU fallback)");
  }
}

// Writes a container (host head + device body + host tail) to dst (host or device).
void emit_parts(Context& ctx, const ContainerParts& parts, uint8_t* dst, bool dst_dev) {
  cudaStream_t s = context_stream(ctx);
  const uint64_t h = parts.head.size();
  if (dst_dev) {
    if (h && cudaMemcpyAsync(dst, parts.head.data(), h, cudaMemcpyHostToDevice, s) != cudaSuccess)
      raise(Errc::cuda, "header copy failed");
    if (parts.dev_len &&
        cudaMemcpyAsync(dst + h, parts.dev, parts.dev_len, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      raise(Errc::cuda, "payload copy failed");
    if (!parts.host_tail.empty() &&
        cudaMemcpyAsync(dst + h + parts.dev_len, parts.host_tail.data(), parts.host_tail.size(),
                        cudaMemcpyHostToDevice, s) != cudaSuccess)
      raise(Errc::cuda, "tail copy failed");
  } else {
    std::memcpy(dst, parts.head.data(), h);
    if (parts.dev_len &&
        cudaMemcpyAsync(dst + h, parts.dev, parts.dev_len, cudaMemcpyDeviceToHost, s) != cudaSuccess)
      raise(Errc::cuda, "payload copy failed");
    if (!parts.host_tail.empty()) std::memcpy(dst + h + parts.dev_len, parts.host_tail.data(), parts.host_tail.size());
  }
  if (cudaStreamSynchronize(s) != cudaSuccess) raise(Errc::cuda, "stream synchronize failed");
}

Grid grid_from(int ndims, const uint64_t* shape, const double* const* coords) {
  require(shape != nullptr, "shape is null");
  if (ndims > kMaxDims) raise(Errc::too_many_dims, "grid has " + std::to_string(ndims) + " axes, max is 4");
  return make_grid(ndims, shape, coords);
}

void fill_info(const ContainerInfo& ci, mgrc_container_info* info) {
  std::memset(info, 0, sizeof *info);
  info->version = ci.version;
  info->constant_field = ci.constant_field;
  info->l2_projection = ci.l2_projection;
  info->coords_present = ci.coords_present;
  info->dtype = static_cast<uint8_t>(ci.dtype);
  info->ndims = static_cast<uint8_t>(ci.ndims);
  info->nlevels = static_cast<uint8_t>(ci.nlevels);
  info->codec_id = ci.codec_id;
  for (int a = 0; a < ci.ndims; ++a) info->shape[a] = ci.shape[a];
  info->mode = static_cast<uint8_t>(ci.spec.mode);
  info->norm = static_cast<uint8_t>(ci.spec.norm);
  info->smoothness = ci.spec.smoothness;
  info->tol = ci.spec.tol;
  for (size_t l = 0; l < ci.bin_widths.size() && l < 65; ++l) info->bin_widths[l] = ci.bin_widths[l];
  info->payload_len = ci.payload_len;
  info->checksum = ci.checksum;
  info->header_size = ci.header_size;
}

// ---- multiblock framing (tools/mgrc.cpp:258-293) ----------------------------

std::vector<std::pair<uint64_t, uint64_t>> split_multiblock(const uint8_t* f, uint64_t n) {
  auto rd = [&](uint64_t at, int bytes) {
    if (at + bytes > n) raise(Errc::corrupt_stream, "truncated stream");
    uint64_t v = 0;
    for (int i = bytes - 1; i >= 0; --i) v = (v << 8) | f[at + i];
    return v;
  };
  const uint64_t count = rd(0, 4);
  if (count == 0) raise(Errc::corrupt_stream, "no blocks");
  const uint64_t hdr = 4 + 8 * count;
  std::vector<uint64_t> off(count);
  for (uint64_t i = 0; i < count; ++i) off[i] = rd(4 + 8 * i, 8);
  std::vector<std::pair<uint64_t, uint64_t>> out(count);
  for (uint64_t i = 0; i < count; ++i) {
    const uint64_t b = off[i], e = i + 1 < count ? off[i + 1] : n;
    if (b < hdr || e > n || b > e) raise(Errc::corrupt_stream, "bad block offsets");
    out[i] = {b, e - b};
  }
  return out;
}


// Owned device allocation (RAII).
struct DeviceArray {
  void* p = nullptr;
  size_t n = 0;
  void alloc(size_t bytes) {
    if (bytes <= n) return;
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
      cudaGetLastError();
      raise(Errc::cuda, "cudaMalloc of " + std::to_string(bytes) + " bytes failed");
    }
    n = bytes;
  }
  ~DeviceArray() {
    if (p) cudaFree(p);
  }
};

// Block `rng` of a device array of `shape`: a pointer into it when the block
// is contiguous (only leading axes split), else a device gather of the box
// (cudaMemcpy3D over the last three axes, looped over the first).
const void* copy_box(cudaStream_t st, const void* data, size_t unit, int d, const uint64_t* shape,
                     const std::vector<Range>& rng, DeviceArray& tmp) {
  uint64_t stride[kMaxDims];
  stride[d - 1] = 1;
  for (int a = d - 1; a > 0; --a) stride[a - 1] = stride[a] * shape[a];
  int first_partial = -1;
  for (int a = 0; a < d; ++a)
    if (rng[a].length() != shape[a]) {
      first_partial = a;
      break;
    }
  bool contiguous = true;
  for (int a = first_partial + 1; first_partial >= 0 && a < d; ++a)
    if (rng[a].length() != shape[a]) contiguous = false;
  uint64_t origin = 0, bcount = 1;
  for (int a = 0; a < d; ++a) {
    origin += rng[a].begin * stride[a];
    bcount *= rng[a].length();
  }
  const uint8_t* base = static_cast<const uint8_t*>(data);
  if (contiguous) return base + origin * unit;
  tmp.alloc(bcount * unit);
  // view as [outer][n2][n1][n0] with the last three axes copied by cudaMemcpy3D
  const int k = d >= 3 ? d - 3 : 0;  // axes [0, k) are looped
  uint64_t ext[3] = {1, 1, 1}, full[3] = {1, 1, 1}, beg[3] = {0, 0, 0};
  for (int a = k, j = 3 - (d - k); a < d; ++a, ++j) {
    ext[j] = rng[a].length();
    full[j] = shape[a];
    beg[j] = rng[a].begin;
  }
  uint64_t nouter = 1;
  for (int a = 0; a < k; ++a) nouter *= rng[a].length();
  uint8_t* dst = static_cast<uint8_t*>(tmp.p);
  std::vector<uint64_t> pos(std::max(k, 1), 0);
  for (uint64_t o = 0; o < nouter; ++o) {
    uint64_t src_off = 0;
    for (int a = 0; a < k; ++a) src_off += (rng[a].begin + pos[a]) * stride[a];
    cudaMemcpy3DParms p{};
    p.srcPtr = make_cudaPitchedPtr(const_cast<uint8_t*>(base + src_off * unit), full[2] * unit, full[2], full[1]);
    p.srcPos = make_cudaPos(beg[2] * unit, beg[1], beg[0]);
    p.dstPtr = make_cudaPitchedPtr(dst + o * ext[0] * ext[1] * ext[2] * unit, ext[2] * unit, ext[2], ext[1]);
    p.dstPos = make_cudaPos(0, 0, 0);
    p.extent = make_cudaExtent(ext[2] * unit, ext[1], ext[0]);
    p.kind = cudaMemcpyDeviceToDevice;
    if (cudaMemcpy3DAsync(&p, st) != cudaSuccess) raise(Errc::cuda, "block gather failed");
    for (int a = k - 1; a >= 0; --a) {
      if (++pos[a] < rng[a].length()) break;
      pos[a] = 0;
    }
  }
  return tmp.p;
}

// Block `rng` of a HOST array: a pointer into it when the block is contiguous,
// else the box gathered row by row into `tmp` (write_block's inverse).
const void* host_box(const void* data, size_t unit, int d, const uint64_t* shape, const std::vector<Range>& rng,
                     std::vector<uint8_t>& tmp) {
  uint64_t stride[kMaxDims];
  stride[d - 1] = 1;
  for (int a = d - 1; a > 0; --a) stride[a - 1] = stride[a] * shape[a];
  int first_partial = -1;
  for (int a = 0; a < d; ++a)
    if (rng[a].length() != shape[a]) {
      first_partial = a;
      break;
    }
  bool contiguous = true;
  for (int a = first_partial + 1; first_partial >= 0 && a < d; ++a)
    if (rng[a].length() != shape[a]) contiguous = false;
  uint64_t origin = 0, bcount = 1;
  for (int a = 0; a < d; ++a) {
    origin += rng[a].begin * stride[a];
    bcount *= rng[a].length();
  }
  const uint8_t* base = static_cast<const uint8_t*>(data);
  if (contiguous) return base + origin * unit;
  tmp.resize(bcount * unit);
  const uint64_t run = rng[d - 1].length();
  std::vector<uint64_t> pos(d, 0);
  for (uint64_t row = 0; row < bcount / run; ++row) {
    uint64_t off = rng[d - 1].begin;
    for (int a = 0; a + 1 < d; ++a) off += (rng[a].begin + pos[a]) * stride[a];
    std::memcpy(tmp.data() + row * run * unit, base + off * unit, run * unit);
    for (int a = d - 2; a >= 0; --a) {
      if (++pos[a] < rng[a].length()) break;
      pos[a] = 0;
    }
  }
  return tmp.data();
}


// ---- single-process multi-GPU chunked driver ---------------------------------
//
// One host thread per rank, rank g on device g % device_count (each thread has
// its own per-device context: stream + workspace), slab b on rank floor(b*G/B)
// (contiguous rows and stream ranges, as the torch.distributed driver).  The
// blocks are independent containers; the only collective is the
// all-gather of the per-block compressed sizes, done with NCCL (loaded at run
// time: the process may already hold torch's copy) when the ranks sit on
// distinct devices, on the host when a device carries several ranks.

struct Nccl {
  using comm_t = void*;
  int (*init_all)(comm_t*, int, const int*) = nullptr;
  int (*all_gather)(const void*, void*, size_t, int, comm_t, cudaStream_t) = nullptr;
  int (*group_start)() = nullptr;
  int (*group_end)() = nullptr;
  int (*destroy)(comm_t) = nullptr;
  bool ok = false;
};

const Nccl& nccl() {
  static const Nccl n = [] {
    Nccl r;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return r;
    r.init_all = reinterpret_cast<decltype(r.init_all)>(dlsym(h, "ncclCommInitAll"));
    r.all_gather = reinterpret_cast<decltype(r.all_gather)>(dlsym(h, "ncclAllGather"));
    r.group_start = reinterpret_cast<decltype(r.group_start)>(dlsym(h, "ncclGroupStart"));
    r.group_end = reinterpret_cast<decltype(r.group_end)>(dlsym(h, "ncclGroupEnd"));
    r.destroy = reinterpret_cast<decltype(r.destroy)>(dlsym(h, "ncclCommDestroy"));
    r.ok = r.init_all && r.all_gather && r.group_start && r.group_end && r.destroy;
    return r;
  }();
  return n;
}
constexpr int kNcclUint64 = 5;  // ncclUint64 (nccl.h)

uint64_t owner_of(uint64_t b, uint64_t nb, int G) { return (b * static_cast<uint64_t>(G)) / nb; }

// Runs fn(rank) on G host threads, rank g on device g % ndev; rethrows the first failure.
template <class Fn>
void on_ranks(int G, Fn fn) {
  if (G == 1) {  // the calling thread, its context and stream
    fn(0);
    return;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) raise(Errc::cuda, "no CUDA device");
  std::vector<std::thread> th;
  std::exception_ptr failure;
  std::mutex mu;
  for (int g = 0; g < G; ++g)
    th.emplace_back([&, g] {
      try {
        if (cudaSetDevice(g % ndev) != cudaSuccess) raise(Errc::cuda, "cudaSetDevice failed");
        fn(g);
      } catch (...) {
        std::lock_guard<std::mutex> lk(mu);
        if (!failure) failure = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  if (failure) std::rethrow_exception(failure);
}

// All-gather of the per-rank size vectors (every rank contributes nb entries,
// zeros outside its blocks) -> the summed sizes of every block.
std::vector<uint64_t> gather_sizes(int G, const std::vector<std::vector<uint64_t>>& local, uint64_t nb) {
  std::vector<uint64_t> sizes(nb, 0);
  int ndev = 0;
  cudaGetDeviceCount(&ndev);
  const Nccl& n = nccl();
  if (G > 1 && G <= ndev && n.ok) {
    std::vector<Nccl::comm_t> comms(G, nullptr);
    std::vector<int> devs(G);
    for (int g = 0; g < G; ++g) devs[g] = g;
    if (n.init_all(comms.data(), G, devs.data()) != 0) raise(Errc::cuda, "ncclCommInitAll failed");
    std::vector<uint64_t*> send(G, nullptr), recv(G, nullptr);
    std::vector<cudaStream_t> st(G, nullptr);
    for (int g = 0; g < G; ++g) {
      cudaSetDevice(g);
      cudaStreamCreate(&st[g]);
      cudaMalloc(&send[g], nb * 8);
      cudaMalloc(&recv[g], nb * 8 * G);
      cudaMemcpy(send[g], local[g].data(), nb * 8, cudaMemcpyHostToDevice);
    }
    n.group_start();
    for (int g = 0; g < G; ++g) n.all_gather(send[g], recv[g], nb, kNcclUint64, comms[g], st[g]);
    n.group_end();
    std::vector<uint64_t> all(nb * G);
    cudaSetDevice(0);
    cudaStreamSynchronize(st[0]);
    cudaMemcpy(all.data(), recv[0], nb * 8 * G, cudaMemcpyDeviceToHost);
    for (int g = 0; g < G; ++g) {
      cudaSetDevice(g);
      cudaStreamSynchronize(st[g]);
      cudaFree(send[g]);
      cudaFree(recv[g]);
      cudaStreamDestroy(st[g]);
      n.destroy(comms[g]);
    }
    cudaSetDevice(0);
    for (int g = 0; g < G; ++g)
      for (uint64_t b = 0; b < nb; ++b) sizes[b] += all[g * nb + b];
  } else {  // ranks sharing a device (or no NCCL): the vectors are already on the host
    for (int g = 0; g < G; ++g)
      for (uint64_t b = 0; b < nb; ++b) sizes[b] += local[g][b];
  }
  return sizes;
}

MdrManifest manifest_from(const mgrc_mdr_manifest* m, const mgrc_mdr_segment* segs, const double* const* coords) {
  require(m != nullptr && segs != nullptr, "null argument");
  MdrManifest r;
  r.grid = grid_from(m->ndims, m->shape, coords);
  r.nlevels = m->nlevels;
  r.planes = m->planes;
  if (m->nlevels < 0 || m->nlevels > 64) raise(Errc::corrupt_stream, "manifest level count out of range");
  for (int l = 0; l <= m->nlevels; ++l) {
    r.exps.push_back(m->level_exponents[l]);
    r.counts.push_back(m->level_counts[l]);
    std::vector<MdrSegment> row(m->planes);
    for (uint32_t p = 0; p < m->planes; ++p) {
      const mgrc_mdr_segment& sg = segs[static_cast<size_t>(l) * m->planes + p];
      row[p].bytes = sg.bytes;
      row[p].raw_bits = sg.raw_bits;
      row[p].crc = sg.crc32;
    }
    r.seg.push_back(row);
  }
  r.vmin = m->value_min;
  r.vmax = m->value_max;
  r.vrms = m->value_rms;
  return r;
}

// Multiblock compress (tools/mgrc.cpp:363-484) on `ngpus` ranks: global REL
// normalisation, per-block ABS compress with the block's coordinate slice,
// the u32 count | u64 offsets | containers framing.  Blocks split only along
// leading axes are contiguous sub-arrays and are compressed in place (device
// inputs) or uploaded one block at a time (host inputs, read_block :91-145);
// other blocks are gathered first.
void compress_chunked_impl(const void* data, int dtype, int ndims, const uint64_t* shape,
                                  const double* const* coords, double tol, int norm, double smoothness, int mode,
                                  int codec, uint64_t chunk_mem, int ngpus, uint8_t** out, uint64_t* out_len) {
  require(data != nullptr && out != nullptr && out_len != nullptr, "null argument");
  const Grid whole = grid_from(ndims, shape, coords);
  const DType dt = to_dtype(dtype);
  const ErrorSpec spec = to_spec(tol, norm, smoothness, mode);
  const Codec cd = to_codec(codec);
  const ChunkPlan plan = plan_chunks(ndims, shape, dt, chunk_mem > 0 ? chunk_mem : UINT64_MAX);
  const uint64_t nb = plan.block_count();
  ensure_device();
  const bool on_dev = is_device_pointer(data);
  // ranks: at most one per block; a device-resident input stays on its device
  const int G = on_dev ? 1 : static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(ngpus > 0 ? ngpus : 1, nb)));
  int dev0 = 0;
  cudaGetDevice(&dev0);
  const size_t unit = dtype_size(dt);
  std::vector<std::vector<uint8_t>> blocks(nb);
  ErrorSpec bspec = spec;
  if (nb > 1) {
    bspec.mode = Mode::abs;
    if (spec.mode == Mode::rel) {  // global normalisation (tools/mgrc.cpp:405-418, scan_stats :197-233)
      const uint64_t count = whole.count();
      GlobalStats gs{0.0, 0.0, 0.0, false};
      if (spec.norm == Norm::s || G == 1) {
        // Σu² in file order, exactly (serial_sum.cuh) — one rank streams the whole array
        gs = global_stats(context_for_current_device(), data, dt, count, spec.norm == Norm::s);
      } else {  // min / max are order-free: each rank scans its own rows
        std::vector<GlobalStats> part(G);
        on_ranks(G, [&](int g) {
          uint64_t lo = UINT64_MAX, hi = 0;
          for (uint64_t b = 0; b < nb; ++b)
            if (static_cast<int>(owner_of(b, nb, G)) == g) {
              const auto r = plan.block(b);
              lo = std::min<uint64_t>(lo, r[0].begin);
              hi = std::max<uint64_t>(hi, r[0].end);
            }
          const uint64_t row = count / shape[0];
          part[g] = global_stats(context_for_current_device(), static_cast<const uint8_t*>(data) + lo * row * unit,
                                 dt, (hi - lo) * row, false);
        });
        gs = part[0];
        for (int g = 1; g < G; ++g) {
          gs.nonfinite = gs.nonfinite || part[g].nonfinite;
          gs.min = std::min(gs.min, part[g].min);
          gs.max = std::max(gs.max, part[g].max);
        }
      }
      if (gs.nonfinite) raise(Errc::non_finite_input, "input contains NaN or Inf");
      const double nrm = spec.norm == Norm::s ? std::sqrt(gs.sumsq / static_cast<double>(count)) : gs.max - gs.min;
      if (nrm == 0.0) raise(Errc::degenerate_data, "relative bound on a constant file");
      bspec.tol = spec.tol * nrm;
    }
  }
  std::vector<std::vector<uint64_t>> local(G, std::vector<uint64_t>(nb, 0));
  on_ranks(G, [&](int g) {
    Context& ctx = context_for_current_device();
    cudaStream_t st = context_stream(ctx);
    DeviceArray gather;
    std::vector<uint8_t> hostbox;
    for (uint64_t b = 0; b < nb; ++b) {
      if (static_cast<int>(owner_of(b, nb, G)) != g) continue;
      if (nb == 1) {  // single block: the user's grid and spec (mgrc.cpp:389-404)
        const ContainerParts parts = compress(ctx, data, dt, whole, spec, cd);
        blocks[0].resize(parts.total());
        emit_parts(ctx, parts, blocks[0].data(), false);
      } else {
        const auto rng = plan.block(b);
        uint64_t bshape[kMaxDims];
        std::vector<double> bc[kMaxDims];
        const double* cptr[kMaxDims];
        for (int a = 0; a < ndims; ++a) {
          bshape[a] = rng[a].length();
          bc[a].assign(whole.coords[a].begin() + rng[a].begin, whole.coords[a].begin() + rng[a].end);
          cptr[a] = bc[a].data();
        }
        const void* bdata = on_dev ? copy_box(st, data, unit, ndims, shape, rng, gather)
                                   : host_box(data, unit, ndims, shape, rng, hostbox);
        const Grid bg = make_grid(ndims, bshape, cptr);
        const ContainerParts parts = compress(ctx, bdata, dt, bg, bspec, cd);
        blocks[b].resize(parts.total());
        emit_parts(ctx, parts, blocks[b].data(), false);
      }
      local[g][b] = blocks[b].size();
    }
  });
  const std::vector<uint64_t> sizes = gather_sizes(G, local, nb);
  cudaSetDevice(dev0);
  uint64_t total = 4 + 8 * nb;
  for (const uint64_t z : sizes) total += z;
  uint8_t* buf = static_cast<uint8_t*>(std::malloc(total));
  if (!buf) throw std::bad_alloc();
  uint64_t at = 0;
  auto put = [&](uint64_t v, int bytes) {
    for (int i = 0; i < bytes; ++i) buf[at++] = static_cast<uint8_t>(v >> (8 * i));
  };
  put(nb, 4);
  uint64_t off = 4 + 8 * nb;
  std::vector<uint64_t> offs(nb);
  for (uint64_t b = 0; b < nb; ++b) {
    offs[b] = off;
    put(off, 8);
    off += sizes[b];
  }
  for (uint64_t b = 0; b < nb; ++b) std::memcpy(buf + offs[b], blocks[b].data(), blocks[b].size());
  *out = buf;
  *out_len = total;
}

// Multiblock decompress (tools/mgrc.cpp:490-542) on `ngpus` ranks: offset
// validation, placement from the blocks' coordinate slices, decode; a block
// that is a contiguous slab of the output is decoded straight into place.
void decompress_chunked_impl(const uint8_t* in, uint64_t len, int ngpus, void** out, int* dtype, int* ndims,
                                    uint64_t* shape) {
  require(in != nullptr && out != nullptr, "null argument");
  ensure_device();
  const auto blocks = split_multiblock(in, len);
  std::vector<ContainerInfo> infos;
  for (const auto& b : blocks) infos.push_back(parse_header(in + b.first, b.second));
  const DType dt = infos[0].dtype;
  for (const auto& i : infos)
    if (i.dtype != dt) raise(Errc::corrupt_stream, "blocks disagree on dtype");
  const int d = infos[0].ndims;
  uint64_t gshape[kMaxDims] = {0, 0, 0, 0};
  std::vector<std::vector<Range>> place(blocks.size());
  if (blocks.size() == 1) {
    for (int a = 0; a < d; ++a) {
      gshape[a] = infos[0].shape[a];
      place[0].push_back({0, gshape[a]});
    }
  } else {  // derive_placement (tools/mgrc.cpp:302-347)
    for (int a = 0; a < d; ++a) {
      std::vector<std::pair<double, uint64_t>> ranges;
      for (const auto& info : infos) {
        if (!info.coords_present || info.ndims != d)
          raise(Errc::corrupt_stream, "multi-block container lacks placement coordinates");
        const double start = info.coords[a][0];
        const uint64_t l = info.shape[a];
        bool found = false;
        for (auto& r : ranges)
          if (r.first == start) {
            if (r.second != l) raise(Errc::corrupt_stream, "inconsistent block grid");
            found = true;
          }
        if (!found) ranges.push_back({start, l});
      }
      std::sort(ranges.begin(), ranges.end());
      uint64_t at = 0;
      std::vector<std::pair<double, Range>> placed;
      for (const auto& r : ranges) {
        placed.push_back({r.first, {at, at + r.second}});
        at += r.second;
      }
      gshape[a] = at;
      for (size_t i = 0; i < infos.size(); ++i)
        for (const auto& pr : placed)
          if (pr.first == infos[i].coords[a][0]) {
            place[i].push_back(pr.second);
            break;
          }
      for (const auto& br : place)
        if (static_cast<int>(br.size()) != a + 1) raise(Errc::corrupt_stream, "block placement failed");
    }
  }
  uint64_t count = 1;
  for (int a = 0; a < d; ++a) count *= gshape[a];
  const size_t unit = dtype_size(dt);
  uint8_t* buf = static_cast<uint8_t*>(std::malloc(count * unit + 1));
  if (!buf) throw std::bad_alloc();
  const uint64_t nb = blocks.size();
  const int G = static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(ngpus > 0 ? ngpus : 1, nb)));
  int dev0 = 0;
  cudaGetDevice(&dev0);
  try {
    uint64_t stride[kMaxDims];
    stride[d - 1] = 1;
    for (int a = d - 1; a > 0; --a) stride[a - 1] = stride[a] * gshape[a];
    on_ranks(G, [&](int g) {
        Context& ctx = context_for_current_device();
      std::vector<uint8_t> tmp;
      for (uint64_t b = 0; b < nb; ++b) {
        if (static_cast<int>(owner_of(b, nb, G)) != g) continue;
        const auto& r = place[b];
        uint64_t bcount = 1, origin = 0;
        int first_partial = -1;
        for (int a = 0; a < d; ++a) {
          bcount *= r[a].length();
          origin += r[a].begin * stride[a];
          if (first_partial < 0 && r[a].length() != gshape[a]) first_partial = a;
        }
        bool contiguous = true;  // only leading axes split: the block is one run of the output
        for (int a = first_partial + 1; first_partial >= 0 && a < d; ++a)
          if (r[a].length() != gshape[a]) contiguous = false;
        if (contiguous) {
          decompress_into(ctx, in + blocks[b].first, blocks[b].second, buf + origin * unit, bcount * unit);
          continue;
        }
        tmp.resize(bcount * unit);
        decompress_into(ctx, in + blocks[b].first, blocks[b].second, tmp.data(), tmp.size());
        const uint64_t run = r[d - 1].length();
        std::vector<uint64_t> pos(d, 0);
        for (uint64_t row = 0; row < bcount / run; ++row) {  // write_block (tools/mgrc.cpp:148-190)
          uint64_t off = r[d - 1].begin;
          for (int a = 0; a + 1 < d; ++a) off += (r[a].begin + pos[a]) * stride[a];
          std::memcpy(buf + off * unit, tmp.data() + row * run * unit, run * unit);
          for (int a = d - 2; a >= 0; --a) {
            if (++pos[a] < r[a].length()) break;
            pos[a] = 0;
          }
        }
      }
    });
    cudaSetDevice(dev0);
  } catch (...) {
    cudaSetDevice(dev0);
    std::free(buf);
    throw;
  }
  *out = buf;
  if (dtype) *dtype = static_cast<int>(dt);
  if (ndims) *ndims = d;
  if (shape)
    for (int a = 0; a < d; ++a) shape[a] = gshape[a];
}

}  // namespace

extern "C" {

const char* mgrc_gpu_version(void) { return "mgrc_gpu 0.1 (sm_100a)"; }
const char* mgrc_gpu_last_error(void) { return g_last_error.c_str(); }
void mgrc_gpu_free(void* p) { std::free(p); }
uint64_t mgrc_gpu_launch_count(void) { return launch_count(); }

int mgrc_gpu_last_compress_stats(double* tau_abs, double* achieved, int* passes, int* decided_by) {
  const CompressStats& c = last_compress_stats();
  if (tau_abs) *tau_abs = c.tau_abs;
  if (achieved) *achieved = c.achieved;
  if (passes) *passes = c.passes;
  if (decided_by) *decided_by = c.decided_by;
  return MGRC_OK;
}

int mgrc_gpu_host_alloc(uint64_t bytes, void** p) {
  return guarded([&] {
    require(p != nullptr, "null output pointer");
    ensure_device();
    *p = nullptr;
    if (cudaHostAlloc(p, bytes ? bytes : 1, cudaHostAllocDefault) != cudaSuccess) {
      cudaGetLastError();
      raise(Errc::cuda, "cudaHostAlloc of " + std::to_string(bytes) + " bytes failed");
    }
  });
}

void mgrc_gpu_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int mgrc_gpu_set_device(int device) {
  return guarded([&] {
    ensure_device();
    if (cudaSetDevice(device) != cudaSuccess) raise(Errc::cuda, "cudaSetDevice failed");
  });
}

int mgrc_gpu_set_stream(void* stream) {
  return guarded([&] {
    ensure_device();
    Context& c = context_for_current_device();
    if (stream) {
      context_set_stream(c, static_cast<cudaStream_t>(stream));
    } else {
      cudaStream_t s;
      if (cudaStreamCreateWithFlags(&s, cudaStreamDefault) != cudaSuccess) raise(Errc::cuda, "stream create");
      context_set_stream(c, s);
    }
  });
}

int mgrc_gpu_set_profiling(int on) {
  return guarded([&] {
    ensure_device();
    context_set_profiling(context_for_current_device(), on != 0);
  });
}

int mgrc_gpu_profile_count(void) {
  int n = 0;
  guarded([&] { n = static_cast<int>(context_profile(context_for_current_device()).size()); });
  return n;
}

int mgrc_gpu_profile_entry(int i, const char** name, double* ms, double* bytes) {
  return guarded([&] {
    const auto& p = context_profile(context_for_current_device());
    require(i >= 0 && i < static_cast<int>(p.size()), "profile index out of range");
    *name = p[i].name.c_str();
    *ms = p[i].ms;
    *bytes = p[i].bytes;
  });
}

static int compress_to_impl(bool l2, const void* data, int dtype, int ndims, const uint64_t* shape, const double* const* coords,
                         double tol, int norm, double smoothness, int mode, int codec, void* dst,
                         uint64_t dst_capacity, uint64_t* out_len) {
  return guarded([&] {
    require(data != nullptr && out_len != nullptr, "null argument");
    const Grid g = grid_from(ndims, shape, coords);
    const ErrorSpec sp = to_spec(tol, norm, smoothness, mode);
    const Codec cd = to_codec(codec);
    const DType dt = to_dtype(dtype);
    ensure_device();
    Context& ctx = context_for_current_device();
    const ContainerParts parts = l2 ? compress_l2(ctx, data, dt, g, sp, cd) : compress(ctx, data, dt, g, sp, cd);
    *out_len = parts.total();
    if (!dst) return;
    if (dst_capacity < parts.total()) raise(Errc::invalid_argument, "destination buffer too small");
    emit_parts(ctx, parts, static_cast<uint8_t*>(dst), is_device_pointer(dst));
  });
}

static int compress_impl(bool l2, const void* data, int dtype, int ndims, const uint64_t* shape, const double* const* coords,
                      double tol, int norm, double smoothness, int mode, int codec, uint8_t** out,
                      uint64_t* out_len) {
  return guarded([&] {
    require(data != nullptr && out != nullptr && out_len != nullptr, "null argument");
    const Grid g = grid_from(ndims, shape, coords);
    const ErrorSpec sp = to_spec(tol, norm, smoothness, mode);
    const Codec cd = to_codec(codec);
    const DType dt = to_dtype(dtype);
    ensure_device();
    Context& ctx = context_for_current_device();
    const ContainerParts parts = l2 ? compress_l2(ctx, data, dt, g, sp, cd) : compress(ctx, data, dt, g, sp, cd);
    uint8_t* buf = static_cast<uint8_t*>(std::malloc(parts.total() + 1));
    if (!buf) throw std::bad_alloc();
    try {
      emit_parts(ctx, parts, buf, false);
    } catch (...) {
      std::free(buf);
      throw;
    }
    *out = buf;
    *out_len = parts.total();
  });
}

int mgrc_gpu_compress_to(const void* data, int dtype, int ndims, const uint64_t* shape, const double* const* coords,
                         double tol, int norm, double smoothness, int mode, int codec, void* dst,
                         uint64_t dst_capacity, uint64_t* out_len) {
  return compress_to_impl(false, data, dtype, ndims, shape, coords, tol, norm, smoothness, mode, codec, dst,
                          dst_capacity, out_len);
}

int mgrc_gpu_compress_l2_to(const void* data, int dtype, int ndims, const uint64_t* shape, const double* const* coords,
                            double tol, int norm, double smoothness, int mode, int codec, void* dst,
                            uint64_t dst_capacity, uint64_t* out_len) {
  return compress_to_impl(true, data, dtype, ndims, shape, coords, tol, norm, smoothness, mode, codec, dst,
                          dst_capacity, out_len);
}

int mgrc_gpu_compress(const void* data, int dtype, int ndims, const uint64_t* shape, const double* const* coords,
                      double tol, int norm, double smoothness, int mode, int codec, uint8_t** out,
                      uint64_t* out_len) {
  return compress_impl(false, data, dtype, ndims, shape, coords, tol, norm, smoothness, mode, codec, out, out_len);
}

int mgrc_gpu_compress_l2(const void* data, int dtype, int ndims, const uint64_t* shape, const double* const* coords,
                         double tol, int norm, double smoothness, int mode, int codec, uint8_t** out,
                         uint64_t* out_len) {
  return compress_impl(true, data, dtype, ndims, shape, coords, tol, norm, smoothness, mode, codec, out, out_len);
}

int mgrc_gpu_decompress_into(const uint8_t* in, uint64_t len, void* dst, uint64_t dst_capacity, int* dtype,
                             int* ndims, uint64_t* shape) {
  return guarded([&] {
    require(in != nullptr && dst != nullptr, "null argument");
    ensure_device();
    Context& ctx = context_for_current_device();
    const DecodedInfo di = decompress_into(ctx, in, len, dst, dst_capacity);
    if (dtype) *dtype = static_cast<int>(di.dtype);
    if (ndims) *ndims = di.ndims;
    if (shape)
      for (int a = 0; a < di.ndims; ++a) shape[a] = di.shape[a];
  });
}

int mgrc_gpu_decompress(const uint8_t* in, uint64_t len, void** out, int* dtype, int* ndims, uint64_t* shape) {
  return guarded([&] {
    require(in != nullptr && out != nullptr, "null argument");
    ensure_device();
    Context& ctx = context_for_current_device();
    const ContainerInfo info = inspect_any(ctx, in, len);
    uint64_t n = 1;
    for (int a = 0; a < info.ndims; ++a) n *= info.shape[a];
    const uint64_t bytes = n * dtype_size(info.dtype);
    void* buf = std::malloc(bytes + 1);
    if (!buf) throw std::bad_alloc();
    try {
      const DecodedInfo di = decompress_into(ctx, in, len, buf, bytes);
      if (dtype) *dtype = static_cast<int>(di.dtype);
      if (ndims) *ndims = di.ndims;
      if (shape)
        for (int a = 0; a < di.ndims; ++a) shape[a] = di.shape[a];
    } catch (...) {
      std::free(buf);
      throw;
    }
    *out = buf;
  });
}

int mgrc_gpu_inspect(const uint8_t* in, uint64_t len, mgrc_container_info* info) {
  return guarded([&] {
    require(in != nullptr && info != nullptr, "null argument");
    fill_info(parse_header(in, len), info);
  });
}

int mgrc_gpu_describe(const uint8_t* in, uint64_t len, char** text) {
  return guarded([&] {
    require(in != nullptr && text != nullptr, "null argument");
    const std::string s = describe(parse_header(in, len));
    char* t = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(t, s.c_str(), s.size() + 1);
    *text = t;
  });
}

int mgrc_gpu_plan_chunks(int ndims, const uint64_t* shape, int dtype, uint64_t budget, uint64_t* nblocks,
                         uint64_t* ranges, uint64_t cap_blocks) {
  return guarded([&] {
    require(shape != nullptr && nblocks != nullptr, "null argument");
    const ChunkPlan plan = plan_chunks(ndims, shape, to_dtype(dtype), budget);
    *nblocks = plan.block_count();
    if (ranges && plan.block_count() <= cap_blocks)
      for (uint64_t b = 0; b < plan.block_count(); ++b) {
        const auto r = plan.block(b);
        for (int a = 0; a < ndims; ++a) {
          ranges[(b * ndims + a) * 2] = r[a].begin;
          ranges[(b * ndims + a) * 2 + 1] = r[a].end;
        }
      }
  });
}

int mgrc_gpu_serial_sumsq(const void* data, int dtype, uint64_t n, double s0, double* out) {
  return guarded([&] {
    require(data != nullptr && out != nullptr, "null argument");
    ensure_device();
    *out = serial_sumsq(context_for_current_device(), data, to_dtype(dtype), n, s0);
  });
}

int mgrc_gpu_field_stats(const void* data, int dtype, uint64_t n, double* mn, double* mx, int* nonfinite) {
  return guarded([&] {
    require(data != nullptr && n > 0, "null argument");
    ensure_device();
    const FieldStats st = field_stats(context_for_current_device(), data, to_dtype(dtype), n);
    if (mn) *mn = st.min;
    if (mx) *mx = st.max;
    if (nonfinite) *nonfinite = st.nonfinite;
  });
}

// ---- decomposition / quantiser entry points (transform.hpp:24-30, quantize.hpp:32-42) ----

int mgrc_gpu_nlevels(int ndims, const uint64_t* shape, const double* const* coords, int* nlevels) {
  return guarded([&] {
    require(nlevels != nullptr, "null argument");
    *nlevels = build_hierarchy(grid_from(ndims, shape, coords)).L;
  });
}

int mgrc_gpu_initial_bin_widths(double tau_abs, int norm, double smoothness, int ndims, int nlevels, double* widths) {
  return guarded([&] {
    require(widths != nullptr && nlevels >= 0 && nlevels < 64, "bad argument");
    const auto w = initial_bin_widths(tau_abs, to_spec(tau_abs, norm, smoothness, 0), ndims, nlevels);
    for (int l = 0; l <= nlevels; ++l) widths[l] = w[l];
  });
}

int mgrc_gpu_forward_transform(const double* u, int ndims, const uint64_t* shape, const double* const* coords,
                               double* c) {
  return guarded([&] {
    require(u != nullptr && c != nullptr, "null argument");
    const Grid g = grid_from(ndims, shape, coords);
    ensure_device();
    forward_transform(context_for_current_device(), u, c, g);
  });
}

int mgrc_gpu_inverse_transform(const double* c, int ndims, const uint64_t* shape, const double* const* coords,
                               double* u) {
  return guarded([&] {
    require(u != nullptr && c != nullptr, "null argument");
    const Grid g = grid_from(ndims, shape, coords);
    ensure_device();
    inverse_transform(context_for_current_device(), c, u, g);
  });
}

int mgrc_gpu_forward_transform_l2(const double* u, int ndims, const uint64_t* shape, const double* const* coords,
                                  double* c) {
  return guarded([&] {
    require(u != nullptr && c != nullptr, "null argument");
    const Grid g = grid_from(ndims, shape, coords);
    ensure_device();
    forward_transform_l2(context_for_current_device(), u, c, g);
  });
}

int mgrc_gpu_inverse_transform_l2(const double* c, int ndims, const uint64_t* shape, const double* const* coords,
                                  double* u) {
  return guarded([&] {
    require(u != nullptr && c != nullptr, "null argument");
    const Grid g = grid_from(ndims, shape, coords);
    ensure_device();
    inverse_transform_l2(context_for_current_device(), c, u, g);
  });
}

int mgrc_gpu_quantize(const double* c, int ndims, const uint64_t* shape, const double* const* coords,
                      const double* widths, int nwidths, int64_t* q, double* residuals, uint64_t* outliers) {
  return guarded([&] {
    require(c != nullptr && q != nullptr && widths != nullptr, "null argument");
    const Grid g = grid_from(ndims, shape, coords);
    ensure_device();
    const uint64_t o = quantize_coefficients(context_for_current_device(), c, g, widths, nwidths, q, residuals);
    if (outliers) *outliers = o;
  });
}

int mgrc_gpu_dequantize(const int64_t* q, int ndims, const uint64_t* shape, const double* const* coords,
                        const double* widths, int nwidths, double* c) {
  return guarded([&] {
    require(c != nullptr && q != nullptr && widths != nullptr, "null argument");
    const Grid g = grid_from(ndims, shape, coords);
    ensure_device();
    dequantize_coefficients(context_for_current_device(), q, g, widths, nwidths, c);
  });
}

int mgrc_gpu_compress_chunked(const void* data, int dtype, int ndims, const uint64_t* shape,
                              const double* const* coords, double tol, int norm, double smoothness, int mode,
                              int codec, uint64_t chunk_mem, uint8_t** out, uint64_t* out_len) {
  return guarded([&] {
    compress_chunked_impl(data, dtype, ndims, shape, coords, tol, norm, smoothness, mode, codec, chunk_mem, 1, out,
                          out_len);
  });
}

int mgrc_gpu_compress_chunked_multi(const void* data, int dtype, int ndims, const uint64_t* shape,
                                    const double* const* coords, double tol, int norm, double smoothness, int mode,
                                    int codec, uint64_t chunk_mem, int ngpus, uint8_t** out, uint64_t* out_len) {
  return guarded([&] {
    compress_chunked_impl(data, dtype, ndims, shape, coords, tol, norm, smoothness, mode, codec, chunk_mem, ngpus,
                          out, out_len);
  });
}

int mgrc_gpu_decompress_chunked(const uint8_t* in, uint64_t len, void** out, int* dtype, int* ndims,
                                uint64_t* shape) {
  return guarded([&] { decompress_chunked_impl(in, len, 1, out, dtype, ndims, shape); });
}

int mgrc_gpu_decompress_chunked_multi(const uint8_t* in, uint64_t len, int ngpus, void** out, int* dtype, int* ndims,
                                      uint64_t* shape) {
  return guarded([&] { decompress_chunked_impl(in, len, ngpus, out, dtype, ndims, shape); });
}

int mgrc_gpu_mdr_refactor(const double* u, int ndims, const uint64_t* shape, const double* const* coords,
                          uint32_t planes, void** store) {
  return guarded([&] {
    require(u != nullptr && store != nullptr, "null argument");
    const Grid g = grid_from(ndims, shape, coords);
    ensure_device();
    *store = new MdrStore(mdr_refactor(context_for_current_device(), u, g, planes));
  });
}

int mgrc_gpu_mdr_store_manifest(const void* store, mgrc_mdr_manifest* m, mgrc_mdr_segment* segs) {
  return guarded([&] {
    require(store != nullptr && m != nullptr, "null argument");
    const MdrManifest& s = static_cast<const MdrStore*>(store)->m;
    std::memset(m, 0, sizeof *m);
    m->ndims = s.grid.d;
    for (int a = 0; a < s.grid.d; ++a) m->shape[a] = s.grid.shape[a];
    m->nlevels = s.nlevels;
    m->planes = s.planes;
    for (int l = 0; l <= s.nlevels; ++l) {
      m->level_exponents[l] = s.exps[l];
      m->level_counts[l] = s.counts[l];
      for (uint32_t p = 0; segs && p < s.planes; ++p) {
        mgrc_mdr_segment& o = segs[static_cast<size_t>(l) * s.planes + p];
        o.bytes = s.seg[l][p].bytes;
        o.raw_bits = s.seg[l][p].raw_bits;
        o.crc32 = s.seg[l][p].crc;
      }
    }
    m->value_min = s.vmin;
    m->value_max = s.vmax;
    m->value_rms = s.vrms;
  });
}

int mgrc_gpu_mdr_store_segment(const void* store, uint32_t level, uint32_t plane, const uint8_t** data, uint64_t* len) {
  return guarded([&] {
    require(store != nullptr && data != nullptr && len != nullptr, "null argument");
    const auto& pl = static_cast<const MdrStore*>(store)->payload;
    if (level >= pl.size() || plane >= pl[level].size()) raise(Errc::invalid_state, "segment id out of range");
    *data = pl[level][plane].data();
    *len = pl[level][plane].size();
  });
}

void mgrc_gpu_mdr_store_free(void* store) { delete static_cast<MdrStore*>(store); }

int mgrc_gpu_mdr_request(const mgrc_mdr_manifest* m, const mgrc_mdr_segment* segs, double tol_abs, int norm,
                         double smoothness, const uint32_t* fetched, uint32_t* levels, uint32_t* planes, uint64_t cap,
                         uint64_t* n, uint64_t* total_bytes, double* predicted, int* satisfiable) {
  return guarded([&] {
    require(n != nullptr, "null argument");
    const MdrManifest mf = manifest_from(m, segs, nullptr);
    std::vector<uint32_t> f(mf.nlevels + 1, 0);
    if (fetched) f.assign(fetched, fetched + mf.nlevels + 1);
    const MdrRequest r = mdr_request(mf, tol_abs, to_spec(tol_abs, norm, smoothness, 0).norm, smoothness, f);
    *n = r.segs.size();
    for (size_t i = 0; i < r.segs.size() && i < cap; ++i) {
      if (levels) levels[i] = r.segs[i].first;
      if (planes) planes[i] = r.segs[i].second;
    }
    if (total_bytes) *total_bytes = r.bytes;
    if (predicted) *predicted = r.predicted;
    if (satisfiable) *satisfiable = r.satisfiable ? 1 : 0;
  });
}

int mgrc_gpu_mdr_session_new(const mgrc_mdr_manifest* m, const mgrc_mdr_segment* segs, const double* const* coords,
                             void** session) {
  return guarded([&] {
    require(session != nullptr, "null argument");
    *session = mdr_session_new(manifest_from(m, segs, coords));
  });
}

int mgrc_gpu_mdr_reconstruct(void* session, const uint32_t* levels, const uint32_t* planes, uint64_t n,
                             const uint8_t* const* payloads, const uint64_t* lens, int norm, double smoothness,
                             double* out, double* accrued, uint32_t* fetched_out) {
  return guarded([&] {
    require(session != nullptr && out != nullptr, "null argument");
    ensure_device();
    auto* ss = static_cast<MdrSession*>(session);
    std::vector<std::pair<uint32_t, uint32_t>> segs;
    std::vector<const uint8_t*> pl;
    std::vector<uint64_t> ln;
    for (uint64_t i = 0; i < n; ++i) {
      segs.push_back({levels[i], planes[i]});
      pl.push_back(payloads[i]);
      ln.push_back(lens[i]);
    }
    const double a = mdr_reconstruct(context_for_current_device(), *ss, segs, pl, ln,
                                     to_spec(1.0, norm, smoothness, 0).norm, smoothness, out);
    if (accrued) *accrued = a;
    if (fetched_out) {
      const auto& f = mdr_session_fetched(ss);
      for (size_t l = 0; l < f.size(); ++l) fetched_out[l] = f[l];
    }
  });
}

void mgrc_gpu_mdr_session_free(void* session) { mdr_session_free(static_cast<MdrSession*>(session)); }

}  // extern "C"
