// Host-side infrastructure shared by the CUDA translation units of the
// library: per-thread device contexts (stream + grow-only workspaces), the
// device copy of a grid hierarchy, CUDA-event phase timing and launch helpers.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "pipeline.hpp"

namespace mgrc_gpu {

using namespace dev;

#define CK(x)                                                                                        \
  do {                                                                                               \
    cudaError_t e_ = (x);                                                                            \
    if (e_ != cudaSuccess) raise(Errc::cuda, std::string(#x) + ": " + cudaGetErrorString(e_));       \
  } while (0)

inline thread_local unsigned long long g_launches = 0;  // kernels launched by this thread

inline thread_local CompressStats g_cstats{};

inline void check_launch(const char* what) {
  ++g_launches;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) raise(Errc::cuda, std::string(what) + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------------------
// workspace

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  template <typename T = void>
  T* get(size_t bytes) {
    if (bytes > cap) {
      if (p) cudaFree(p);
      p = nullptr;
      const size_t want = std::max(bytes, cap + cap / 4);
      if (cudaMalloc(&p, want) != cudaSuccess) {
        cudaGetLastError();
        cap = 0;
        if (cudaMalloc(&p, bytes) != cudaSuccess) {
          cudaGetLastError();
          p = nullptr;
          raise(Errc::cuda, "cudaMalloc of " + std::to_string(bytes) + " bytes failed");
        }
        cap = bytes;
      } else {
        cap = want;
      }
    }
    return static_cast<T*>(p);
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

struct PinnedBuf {
  void* p = nullptr;
  size_t cap = 0;
  template <typename T = void>
  T* get(size_t bytes) {
    if (bytes > cap) {
      if (p) cudaFreeHost(p);
      CK(cudaHostAlloc(&p, bytes, cudaHostAllocDefault));
      cap = bytes;
    }
    return static_cast<T*>(p);
  }
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
};

// Device copy of a hierarchy's tables: the finest grid (g, boxes) and the
// compact coarse box = the level-(L-1) box as a grid of its own (gc, cboxes)
// carrying the same stencils, on which the coarse part of the inverse runs.
struct DevHier {
  std::string key;
  Hierarchy h;
  DevBuf buf;
  GridDev g{};
  std::vector<BoxDev> boxes;   // per level, finest-grid indices
  GridDev gc{};                // coarse box (valid when h.L >= 1)
  std::vector<BoxDev> cboxes;  // per level 0..L-1, compact indices
  // L²-projection correction tables (transform.cu), built on first use
  DevBuf l2buf;
  std::vector<L2Axis> l2;      // [l * 4 + a], l = 1..L
  bool l2_ready = false;
};

struct Scratch {  // small device-side results read back at sync points
  Stats stats;
  QuantFlags qflags;
  unsigned long long red_bits;
  DecodeStatus dstat;
  unsigned int fix_changed;
  unsigned int raw_wide;
  unsigned long long hist[256];
  unsigned long long queues[4];  // dynamic work queues of the row kernels (zeroed per launch)
  double ssum;                   // running value of the exact serial sum
};

class Context {
 public:
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  bool profiling = false;
  std::vector<PhaseTime> profile;
  std::vector<cudaEvent_t> event_pool;  // timing events reused by Prof (creating them per call costs ~µs each)
  // workspace
  DevBuf ssmaps;
  PinnedBuf ssmaps_h;
  DevBuf in, zz, zc, r, e, v, bits, tiles, scan, seq, lut, codes, crc_tab, crc_a, crc_b, partial, lbws, tfst, tftab;
  DevBuf tftab2;  // decoder: per-tile prefix maps within their group, then the group maps
  DevBuf tfrec;  // decoder: per-subsequence, per-entry terminator counts (k_tfd_maps -> k_tfd_count)
  DevBuf l2a, l2b;  // dense level arrays of the L²-projection correction
  DevBuf scratch_d;
  PinnedBuf scratch_h, partial_h;
  PinnedBuf mdr_h;  // MDR refactor: a level's packed planes on their way to the host
  std::vector<std::unique_ptr<DevHier>> hiers;  // most recently used first (chunked slabs alternate shapes)
  cudaStream_t aux = nullptr;            // concurrent side work (decompress CRC)
  cudaEvent_t ev_in = nullptr, ev_crc = nullptr;
  CrcConsts crc_k{};
  bool crc_ready = false;

  Scratch* sd() { return scratch_d.get<Scratch>(sizeof(Scratch)); }
  Scratch* sh() { return scratch_h.get<Scratch>(sizeof(Scratch)); }

  ~Context() {
    for (cudaEvent_t e : event_pool) cudaEventDestroy(e);
    if (aux) cudaStreamDestroy(aux);
    if (ev_in) cudaEventDestroy(ev_in);
    if (ev_crc) cudaEventDestroy(ev_crc);
    if (own_stream && stream) cudaStreamDestroy(stream);
  }
};


// Named CUDA-event brackets on the context stream (profiling mode only).
class Prof {
 public:
  explicit Prof(Context& c) : c_(c) { c_.profile.clear(); }
  void begin(const char* name, double bytes = 0) {
    if (!c_.profiling) return;
    Rec r;
    r.name = name;
    r.bytes = bytes;
    r.a = take();
    r.b = take();
    cudaEventRecord(r.a, c_.stream);
    recs_.push_back(r);
  }
  void end() {
    if (!c_.profiling || recs_.empty()) return;
    cudaEventRecord(recs_.back().b, c_.stream);
  }
  ~Prof() {
    if (!c_.profiling) return;
    cudaStreamSynchronize(c_.stream);
    for (auto& r : recs_) {
      float ms = 0;
      cudaEventElapsedTime(&ms, r.a, r.b);
      c_.profile.push_back({r.name, ms, r.bytes});
      c_.event_pool.push_back(r.a);
      c_.event_pool.push_back(r.b);
    }
  }

 private:
  cudaEvent_t take() {
    if (c_.event_pool.empty()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      return e;
    }
    cudaEvent_t e = c_.event_pool.back();
    c_.event_pool.pop_back();
    return e;
  }
  struct Rec {
    std::string name;
    double bytes;
    cudaEvent_t a, b;
  };
  Context& c_;
  std::vector<Rec> recs_;
};

inline int num_sms() {
  static thread_local int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

inline int grid_blocks(uint64_t work_items, int threads, int per_sm = 8) {
  const int sms = num_sms();
  const uint64_t need = (work_items + threads - 1) / threads;
  return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>(need, static_cast<uint64_t>(sms) * per_sm)));
}

DevHier& device_hierarchy(Context& ctx, const Grid& grid);

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

inline Widths to_widths(const std::vector<double>& w) {
  Widths W{};
  for (size_t l = 0; l < w.size() && l < static_cast<size_t>(kMaxL); ++l) W.w[l] = w[l];
  return W;
}


// ---------------------------------------------------------------------------
// dispatch helpers over the dimension count

template <template <int> class F, class... Args>
void by_dim(int d, Args&&... args) {
  switch (d) {
    case 1: F<1>::run(args...); break;
    case 2: F<2>::run(args...); break;
    case 3: F<3>::run(args...); break;
    case 4: F<4>::run(args...); break;
    default: raise(Errc::too_many_dims, "unsupported dimension count");
  }
}

template <typename T>
void launch_stats(Context& ctx, const T* u, uint64_t n, Stats* out) {
  Stats init{~0ull, 0ull, 0u};
  CK(cudaMemcpyAsync(out, &init, sizeof init, cudaMemcpyHostToDevice, ctx.stream));
  k_stats<T><<<grid_blocks((n + 3) / 4, 256, 4), 256, 0, ctx.stream>>>(u, n, out, aligned16(u));
  check_launch("k_stats");
}

inline double key_to_double(unsigned long long k) {
  const unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  double d;
  std::memcpy(&d, &b, 8);
  return d;
}

}  // namespace mgrc_gpu
