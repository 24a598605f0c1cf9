// sm_100a kernels for the compress / decompress hot path.
//
// Arithmetic contract: the reference computes in plain IEEE
// double with no FMA contraction, and the order of the corner sum is part of
// the result.  Every floating-point operation below is an explicit
// round-to-nearest intrinsic (__dmul_rn / __dadd_rn / __dsub_rn / __ddiv_rn)
// in the reference's order, and the TU is additionally compiled with
// --fmad=false.  f32 data is widened to f64 on load (container.cpp:197-203).
//
// Layout: arrays are row-major, last axis fastest (grid.hpp:12-13).  Per-axis
// tables (level of each index, bracketing neighbours, weights) are tiny and
// live in L1/L2; the array traffic is streamed with 16-byte vector accesses.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace mgrc_gpu {
namespace dev {

constexpr int kMaxL = 64;

struct AxisTab {
  const uint8_t* lvl;
  const uint32_t* left;
  const uint32_t* right;
  const double* wl;
  const double* wr;
  // Compact level-(L-1) box ("coarse box"): every node with tag < L lies in
  // it, and so does every corner of a tag-L node.
  const uint32_t* cpos;   // finest index -> position in the level-(L-1) set (coarse indices only)
  const uint32_t* cl;     // tag-L-fresh index -> cpos[left]
  const uint32_t* cr;     // tag-L-fresh index -> cpos[right]
  const uint32_t* cset;   // position in the level-(L-1) set -> finest index
  const uint32_t* colc;   // uint2 per index: {cpos[i-1], cpos[i+1]} if fresh at L, else {cpos[i], 0xFFFFFFFF}
  const double* colw;     // double2 per index: {w_left, w_right} if fresh at L
};

struct GridDev {
  int d, L;
  uint32_t shape[4];
  uint64_t stride[4];
  uint64_t N;
  AxisTab ax[4];
  uint32_t cshape[4];    // coarse-box shape
  uint64_t cstride[4];
  uint64_t Nc;
};

struct BoxDev {  // level-l box: the tensor product of the level-l index sets
  const uint32_t* set[4];
  uint32_t n[4];
  uint64_t count;
};

struct Widths {
  double w[kMaxL];
};

// One axis of the L²-projection correction at level l (transform.cu): the
// level-l line (nl nodes: mass matrix rows lo/di/up, fresh flags, the fresh
// nodes' interpolation weights) and the level-(l-1) line (nc nodes: their
// positions kq in the level-l line, Thomas coefficients lo/cp/den).
struct L2Axis {
  const double *lo, *di, *up, *wl, *wr;
  const uint8_t* fresh;
  const uint32_t* kq;
  const double *clo, *cp, *den;
  uint32_t nl, nc;
  int refines;
};

__device__ __forceinline__ uint64_t zigzag(long long q) {
  return (static_cast<uint64_t>(q) << 1) ^ static_cast<uint64_t>(q >> 63);
}
__device__ __forceinline__ long long unzigzag(uint64_t z) {
  return static_cast<long long>(z >> 1) ^ -static_cast<long long>(z & 1u);
}

// Order-preserving key of a double (for atomicMin/Max on min/max).
__device__ __forceinline__ unsigned long long dkey(double x) {
  const unsigned long long b = __double_as_longlong(x);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ uint32_t bswap32(uint32_t x) { return __byte_perm(x, 0, 0x0123); }
__device__ __forceinline__ uint64_t umin64(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ uint64_t umax64(uint64_t a, uint64_t b) { return a > b ? a : b; }

// ---------------------------------------------------------------------------
// Multilinear corner interpolation of one node (transform.cpp:102-128).
// Fresh axes are the axes whose index is new at `tag`; corners are visited in
// binary order with bit k selecting the right neighbour of the k-th fresh
// axis (ascending axis order), w = Π w_axis starting from 1.0, and the sum
// starts at 0.0 and accumulates w·v.  Submasks of the fresh mask enumerated
// with s = (s - F) & F come out in exactly that increasing order.
template <int D, class Load>
__device__ __forceinline__ double interp(const GridDev& g, const uint32_t (&i)[4], int tag, Load load) {
  uint32_t F = 0;
  uint64_t base = 0;
  double wl[D], wr[D];
  uint64_t ol[D], orr[D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    wl[a] = wr[a] = 0.0;
    ol[a] = orr[a] = 0;
    if (__ldg(g.ax[a].lvl + i[a]) == tag) {
      F |= 1u << a;
      wl[a] = __ldg(g.ax[a].wl + i[a]);
      wr[a] = __ldg(g.ax[a].wr + i[a]);
      ol[a] = static_cast<uint64_t>(__ldg(g.ax[a].left + i[a])) * g.stride[a];
      orr[a] = static_cast<uint64_t>(__ldg(g.ax[a].right + i[a])) * g.stride[a];
    } else {
      base += static_cast<uint64_t>(i[a]) * g.stride[a];
    }
  }
  double acc = 0.0;
  uint32_t s = 0;
  do {
    double w = 1.0;
    uint64_t off = base;
#pragma unroll
    for (int a = 0; a < D; ++a)
      if ((F >> a) & 1u) {
        const bool right = (s >> a) & 1u;
        w = __dmul_rn(w, right ? wr[a] : wl[a]);
        off += right ? orr[a] : ol[a];
      }
    acc = __dadd_rn(acc, __dmul_rn(w, load(off)));
    s = (s - F) & F;
  } while (s);
  return acc;
}

template <int D>
__device__ __forceinline__ int node_tag(const GridDev& g, const uint32_t (&i)[4]) {
  int t = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) t = max(t, static_cast<int>(__ldg(g.ax[a].lvl + i[a])));
  return t;
}

template <int D>
__device__ __forceinline__ void decompose(const GridDev& g, uint64_t e, uint32_t (&i)[4]) {
#pragma unroll
  for (int a = D - 1; a > 0; --a) {
    const uint64_t q = e / g.shape[a];
    i[a] = static_cast<uint32_t>(e - q * g.shape[a]);
    e = q;
  }
  i[0] = static_cast<uint32_t>(e);
}

template <int D>
__device__ __forceinline__ void advance(const GridDev& g, uint32_t (&i)[4]) {
#pragma unroll
  for (int a = D - 1; a >= 0; --a) {
    if (++i[a] < g.shape[a]) return;
    i[a] = 0;
  }
}

// 4-element vector load/store helpers (16-byte transactions).
template <typename T>
__device__ __forceinline__ void load4(const T* p, double (&v)[4]);
template <>
__device__ __forceinline__ void load4<float>(const float* p, double (&v)[4]) {
  const float4 x = __ldg(reinterpret_cast<const float4*>(p));
  v[0] = x.x, v[1] = x.y, v[2] = x.z, v[3] = x.w;
}
template <>
__device__ __forceinline__ void load4<double>(const double* p, double (&v)[4]) {
  const double2 a = __ldg(reinterpret_cast<const double2*>(p));
  const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
  v[0] = a.x, v[1] = a.y, v[2] = b.x, v[3] = b.y;
}
__device__ __forceinline__ void store4(double* p, const double (&v)[4]) {
  reinterpret_cast<double2*>(p)[0] = make_double2(v[0], v[1]);
  reinterpret_cast<double2*>(p)[1] = make_double2(v[2], v[3]);
}
__device__ __forceinline__ void store4(float* p, const double (&v)[4]) {
  *reinterpret_cast<float4*>(p) = make_float4(__double2float_rn(v[0]), __double2float_rn(v[1]),
                                              __double2float_rn(v[2]), __double2float_rn(v[3]));
}
template <typename Z>
__device__ __forceinline__ void load4z(const Z* p, uint64_t (&z)[4]);
template <>
__device__ __forceinline__ void load4z<uint32_t>(const uint32_t* p, uint64_t (&z)[4]) {
  const uint4 x = __ldg(reinterpret_cast<const uint4*>(p));
  z[0] = x.x, z[1] = x.y, z[2] = x.z, z[3] = x.w;
}
template <>
__device__ __forceinline__ void load4z<unsigned long long>(const unsigned long long* p, uint64_t (&z)[4]) {
  const ulonglong2 a = __ldg(reinterpret_cast<const ulonglong2*>(p));
  const ulonglong2 b = __ldg(reinterpret_cast<const ulonglong2*>(p) + 1);
  z[0] = a.x, z[1] = a.y, z[2] = b.x, z[3] = b.y;
}
__device__ __forceinline__ void store4z(uint32_t* p, const uint64_t (&z)[4]) {
  *reinterpret_cast<uint4*>(p) = make_uint4(static_cast<uint32_t>(z[0]), static_cast<uint32_t>(z[1]),
                                            static_cast<uint32_t>(z[2]), static_cast<uint32_t>(z[3]));
}
__device__ __forceinline__ void store4z(unsigned long long* p, const uint64_t (&z)[4]) {
  reinterpret_cast<ulonglong2*>(p)[0] = make_ulonglong2(z[0], z[1]);
  reinterpret_cast<ulonglong2*>(p)[1] = make_ulonglong2(z[2], z[3]);
}

// ---------------------------------------------------------------------------
// K1: input statistics (exec.cpp:89-128): non-finite flag, min, max.
// min/max are order-independent; the constant-field value the reference
// stores (the last 4096-block's first element, see pipeline) is read apart.

struct Stats {
  unsigned long long min_key, max_key;
  unsigned int nonfinite;
};

template <typename T>
static __global__ void __launch_bounds__(256) k_stats(const T* __restrict__ u, uint64_t n, Stats* out, int vec_ok) {
  double mn = __longlong_as_double(0x7ff0000000000000ll), mx = -mn;
  unsigned bad = 0;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t n4 = vec_ok ? n / 4 : 0;
  if constexpr (sizeof(T) == 4) {  // f32: min / max in single precision (the widening is monotone and exact)
    float fmn = __int_as_float(0x7f800000), fmx = -fmn;
    const float4* u4 = reinterpret_cast<const float4*>(u);
    for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < n4; k += stride) {
      const float4 a = __ldg(u4 + k);
      bad |= !isfinite(a.x) | !isfinite(a.y) | !isfinite(a.z) | !isfinite(a.w);
      fmn = fminf(fminf(fmn, a.x), fminf(a.y, fminf(a.z, a.w)));
      fmx = fmaxf(fmaxf(fmx, a.x), fmaxf(a.y, fmaxf(a.z, a.w)));
    }
    mn = static_cast<double>(fmn);
    mx = static_cast<double>(fmx);
  } else {
    for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < n4; k += stride) {
      double v[4];
      load4<T>(u + 4 * k, v);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        bad |= !isfinite(v[j]);
        mn = fmin(mn, v[j]);
        mx = fmax(mx, v[j]);
      }
    }
  }
  for (uint64_t k = 4 * n4 + blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < n; k += stride) {
    const double v = static_cast<double>(u[k]);
    bad |= !isfinite(v);
    mn = fmin(mn, v);
    mx = fmax(mx, v);
  }
  unsigned long long kmn = dkey(mn), kmx = dkey(mx);
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    kmn = min(kmn, __shfl_xor_sync(0xffffffffu, kmn, o));
    kmx = max(kmx, __shfl_xor_sync(0xffffffffu, kmx, o));
    bad |= __shfl_xor_sync(0xffffffffu, bad, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&out->min_key, kmn);
    atomicMax(&out->max_key, kmx);
    if (bad) atomicOr(&out->nonfinite, 1u);
  }
}

// Exact 4096-block sums of squares (exec.cpp:47-71, :108-117): one thread
// per block, serial in index order, no FMA.  Partials are combined serially
// on the host, exactly as blocked_reduce does.
template <typename T>
static __global__ void __launch_bounds__(128) k_block_sumsq(const T* __restrict__ v, uint64_t n, double* __restrict__ partials,
                                                     int vec_ok) {
  const uint64_t b = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t nb = (n + 4095) / 4096;
  if (b >= nb) return;
  const uint64_t lo = b * 4096, hi = min(lo + 4096, n);
  double s = 0.0;
  uint64_t i = lo;
  if (hi - lo == 4096 && vec_ok) {
    for (; i < hi; i += 4) {
      double x[4];
      load4<T>(v + i, x);
#pragma unroll
      for (int j = 0; j < 4; ++j) s = __dadd_rn(s, __dmul_rn(x[j], x[j]));
    }
  }
  for (; i < hi; ++i) {
    const double x = static_cast<double>(v[i]);
    s = __dadd_rn(s, __dmul_rn(x, x));
  }
  partials[b] = s;
}

// ---------------------------------------------------------------------------
// Shared state of the quantising passes (rows.cuh): the forward sweep only
// ever reads coarse nodes that it has not yet modified (transform.cpp:65-67,
// L→1), so c(node) = u(node) − I(u)(node) with the node's own tag (SURVEY
// §0.3); quantisation follows quantize.cpp:105-123; codes are stored as
// zigzag(q) (Z = u32 with a "wide" flag, or u64) and the LEB128 bytes of
// zigzag(q) are histogrammed for the codebook (codec.cpp:445-449).
struct QuantFlags {
  unsigned long long overflow;  // |c/δ| ≥ 2^63 (quantize.cpp:113-116)
  unsigned int wide;            // some zz does not fit the u32 store
  unsigned int pad;
  unsigned long long rmax_bits; // max |r| over the coarse-box nodes (bits of a non-negative double)
  unsigned long long queue;     // row-segment work queue of the fused pass
};

__device__ __forceinline__ void flag_rmax(QuantFlags* f, double rmax) {
#pragma unroll
  for (int o = 16; o; o >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
  if ((threadIdx.x & 31) == 0 && rmax > 0.0)
    atomicMax(&f->rmax_bits, static_cast<unsigned long long>(__double_as_longlong(rmax)));
}

__device__ __forceinline__ void hist_flush(uint32_t* sh, uint32_t& sym, uint32_t& cnt) {
  if (cnt) atomicAdd(&sh[sym], cnt);
  cnt = 0;
}

__device__ __forceinline__ void hist_varint(uint32_t* sh, uint64_t z, uint32_t& sym, uint32_t& cnt) {
  for (;;) {
    const uint32_t b = z >= 0x80 ? static_cast<uint32_t>((z & 0x7F) | 0x80) : static_cast<uint32_t>(z);
    if (b != sym) {
      hist_flush(sh, sym, cnt);
      sym = b;
    }
    ++cnt;
    if (z < 0x80) return;
    z >>= 7;
  }
}

// continuation bytes of one code (z = code >> 7): rare, straight into the block histogram
__device__ __forceinline__ void hist_tail(uint32_t* sh, uint64_t z) {
  for (;;) {
    const uint32_t b = z >= 0x80 ? static_cast<uint32_t>((z & 0x7F) | 0x80) : static_cast<uint32_t>(z);
    atomicAdd(&sh[b], 1u);
    if (z < 0x80) return;
    z >>= 7;
  }
}

// ---------------------------------------------------------------------------
// Inverse transform, coarse → fine (transform.cpp:155-159).  Level l ≥ 1
// touches only nodes tagged l and reads only nodes of lower tag, which are
// final by then.  The per-node source value is either a residual (the
// a-posteriori check of container.cpp:93-119) or a dequantised code
// (decompress, quantize.cpp:134-158): v = src + 1.0·I(v).

struct SrcResidual {
  const double* r;
  __device__ __forceinline__ double operator()(uint64_t n, int) const { return r[n]; }
};

// Box pass for level l < L (and level 0): enumerates the level-l box with
// the level index sets and updates the nodes tagged l.
template <int D, class Src>
static __global__ void __launch_bounds__(256) k_inverse_box(GridDev g, BoxDev box, int l, Src src, double* v) {
  auto ld = [v](uint64_t off) { return v[off]; };
  const uint64_t step = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < box.count; p += step) {
    uint32_t i[4] = {0, 0, 0, 0};
    uint64_t q = p;
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
      const uint64_t qq = q / box.n[a];
      i[a] = __ldg(box.set[a] + (q - qq * box.n[a]));
      q = qq;
    }
    const int tag = node_tag<D>(g, i);
    if (tag != l) continue;
    uint64_t n = 0;
#pragma unroll
    for (int a = 0; a < D; ++a) n += static_cast<uint64_t>(i[a]) * g.stride[a];
    double val = src(n, l);
    if (l > 0) val = __dadd_rn(val, interp<D>(g, i, l, ld));
    v[n] = val;
  }
}

// Check epilogues of the fused pass: (n, e, source value widened, reduction).
struct ChkMaxAbs {
  static constexpr bool kNeedsE = true;  // max|e| (error_control.cpp:105, exec.cpp:75-87)
  __device__ __forceinline__ void operator()(uint64_t, double e, double, double& red) const {
    red = fmax(red, fabs(e));
  }
};
struct ChkCastMaxAbs {
  static constexpr bool kNeedsE = true;  // f32: max|src − (double)(float)(u − e)| (container.cpp:96-107)
  __device__ __forceinline__ void operator()(uint64_t, double e, double s, double& red) const {
    red = fmax(red, fabs(__dsub_rn(s, static_cast<double>(__double2float_rn(__dsub_rn(s, e))))));
  }
};
struct ChkStore {
  static constexpr bool kNeedsE = true;  // S(0): e stored for the ordered 4096-block RMS
  double* out;
  __device__ __forceinline__ void operator()(uint64_t n, double e, double, double&) const { out[n] = e; }
};
struct ChkCastStore {
  static constexpr bool kNeedsE = true;  // S(0), f32: the cast error stored
  double* out;
  __device__ __forceinline__ void operator()(uint64_t n, double e, double s, double&) const {
    out[n] = __dsub_rn(s, static_cast<double>(__double2float_rn(__dsub_rn(s, e))));
  }
};
// Bound pass: the a-posteriori error is not evaluated; the pass only tracks
// max|r| over the finest nodes (passed as e), see compress_t's accept bound.
struct ChkBound {
  static constexpr bool kNeedsE = false;
  __device__ __forceinline__ void operator()(uint64_t, double r, double, double& red) const {
    red = fmax(red, fabs(r));
  }
};
struct ChkLevelWeighted {
  static constexpr bool kNeedsE = true;  // S(s≠0): Σ 2^{2s(tag−L)} r² (error_control.cpp:72-100), r passed as e
  double* rstore;  // non-null on the certified fallback: every node's r, row-major, for the serial level sums
  __device__ __forceinline__ void operator()(uint64_t n, double r, double, double&) const {
    if (rstore) rstore[n] = r;
  }
};

// out[n] = r[n] if tag(n) == l else 0: the masked sequence whose SERIAL sum of squares equals the
// reference's level_sumsq[l] (error_control.cpp:77-90 adds v*v in row-major order over the tag-l nodes;
// the zero terms leave the running sum unchanged).
template <int D>
static __global__ void k_level_mask(GridDev g, const double* __restrict__ r, int l, double* __restrict__ out) {
  for (uint64_t n = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; n < g.N;
       n += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint32_t i[4] = {0, 0, 0, 0};
    decompose<D>(g, n, i);
    out[n] = node_tag<D>(g, i) == l ? r[n] : 0.0;
  }
}

// ---------------------------------------------------------------------------
// Decoupled look-back (single-pass prefix) helpers.  A tile publishes
// (flag << 62 | value): 1 = its own aggregate, 2 = inclusive prefix.
constexpr unsigned long long kLbAgg = 1ull << 62, kLbInc = 2ull << 62, kLbMask = (1ull << 62) - 1;

// Called by warp 0 of the tile; returns the exclusive prefix of tile t.
__device__ __forceinline__ unsigned long long lookback(unsigned long long* status, uint64_t t,
                                                       unsigned long long aggregate) {
  const int lane = threadIdx.x & 31;
  if (t == 0) {
    if (lane == 0) atomicExch(status, kLbInc | aggregate);
    return 0;
  }
  if (lane == 0) atomicExch(status + t, kLbAgg | aggregate);
  unsigned long long excl = 0;
  int64_t base = static_cast<int64_t>(t) - 1;
  for (;;) {
    const int64_t j = base - lane;
    unsigned long long v = kLbInc;  // beyond tile 0: acts as a zero inclusive
    if (j >= 0) {
      do {
        v = *reinterpret_cast<volatile unsigned long long*>(status + j);
      } while ((v >> 62) == 0);
    }
    // lanes ordered from nearest predecessor; find the first inclusive
    const unsigned inc_mask = __ballot_sync(0xffffffffu, (v >> 62) == 2);
    const int first_inc = inc_mask ? __ffs(inc_mask) - 1 : 32;
    unsigned long long contrib = lane <= first_inc ? (v & kLbMask) : 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) contrib += __shfl_xor_sync(0xffffffffu, contrib, o);
    excl += contrib;
    if (first_inc < 32) break;
    base -= 32;
  }
  if (lane == 0) atomicExch(status + t, kLbInc | (excl + aggregate));
  return excl;
}

// Single-pass exclusive scan of u64 counts (values < 2^62); out[n] = total.
// Tiles are claimed through a ticket so that predecessors always run first.
constexpr int kScanThreads = 256, kScanPer = 8, kScanTile = kScanThreads * kScanPer;

static __global__ void __launch_bounds__(kScanThreads) k_scan_lb(const unsigned long long* __restrict__ in,
                                                          unsigned long long* __restrict__ out, uint64_t n,
                                                          unsigned long long* status, unsigned int* ticket) {
  __shared__ unsigned long long wsum[kScanThreads / 32];
  __shared__ unsigned long long s_prefix;
  __shared__ uint32_t s_tile;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint64_t t = s_tile;
  const uint64_t base = t * kScanTile + threadIdx.x * kScanPer;
  unsigned long long v[kScanPer], mine = 0;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    v[k] = base + k < n ? in[base + k] : 0;
    mine += v[k];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (threadIdx.x == 0)
    for (int w = 1; w < kScanThreads / 32; ++w) wsum[w] += wsum[w - 1];
  __syncthreads();
  if (warp == 0) {
    const unsigned long long p = lookback(status, t, wsum[kScanThreads / 32 - 1]);
    if (lane == 0) s_prefix = p;
  }
  __syncthreads();
  unsigned long long run = s_prefix + (warp ? wsum[warp - 1] : 0) + incl - mine;
#pragma unroll
  for (int k = 0; k < kScanPer; ++k) {
    if (base + k < n) out[base + k] = run;
    run += v[k];
  }
  const uint64_t ntiles = (n + kScanTile - 1) / kScanTile;
  if (t == ntiles - 1 && threadIdx.x == 0) out[n] = s_prefix + wsum[kScanThreads / 32 - 1];
}

// ---------------------------------------------------------------------------
// Lossless stage.  Codec 2 codes every LEB128 byte of zigzag(q) with the
// canonical Huffman code (codec.cpp:399-418, MSB-first, zero padded); codec 1
// is the same packer with the identity 8-bit code.

#ifndef MGRC_PACK_THREADS
#define MGRC_PACK_THREADS 256
#endif
#ifndef MGRC_PACK_PER
#define MGRC_PACK_PER 16
#endif
constexpr int kPackThreads = MGRC_PACK_THREADS;
constexpr int kPackPerThread = MGRC_PACK_PER;  // a multiple of 4
constexpr int kPackTile = kPackThreads * kPackPerThread;  // values per tile
constexpr int kPackMaxWords = kPackTile * 150 / 32 + 2;   // ≤ 10 bytes × 15 bits per value

template <typename V>
__device__ __forceinline__ uint32_t varint_bits(V z, const uint8_t* len) {
  uint32_t b = 0;
  for (;;) {
    if (z < 0x80) return b + len[z];
    b += len[(z & 0x7F) | 0x80];
    z >>= 7;
  }
}

// Single-pass Huffman / varint packer: per-value bit counts → block scan →
// look-back for the tile's start bit → codes OR-ed into a shared-memory word
// image → interior words stored directly; the first and last word of the
// tile (possibly shared with a neighbour) go to edge slots merged by
// k_pack_edges.  Output words hold the stream MSB-first in memory byte order.
template <typename Z>
static __global__ void __launch_bounds__(kPackThreads) k_pack_lb(const Z* __restrict__ zz, uint64_t n,
                                                          const uint32_t* __restrict__ code_g,
                                                          const uint8_t* __restrict__ len_g,
                                                          unsigned long long* status, unsigned int* ticket,
                                                          unsigned long long* __restrict__ tile_start,
                                                          uint32_t* __restrict__ edge_first,
                                                          uint32_t* __restrict__ edge_last,
                                                          uint32_t* __restrict__ out, uint32_t cap_words) {
  extern __shared__ uint32_t words[];  // cap_words + 1: the tile's stream, packed from tile-relative bit 0
  __shared__ uint32_t cl[256];  // code << 4 | length: one lookup per byte
  __shared__ uint8_t len[256];
  __shared__ uint32_t wsum[kPackThreads / 32];
  __shared__ unsigned long long s_prefix;
  __shared__ uint32_t s_tile;
  for (int c = threadIdx.x; c < 256; c += blockDim.x) {
    cl[c] = code_g[c] << 4 | len_g[c];
    len[c] = len_g[c];
  }
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const uint64_t t = s_tile;
  const uint64_t base = t * static_cast<uint64_t>(kPackTile) + threadIdx.x * kPackPerThread;
  Z z[kPackPerThread];
  if constexpr (sizeof(Z) == 4) {
    if (base + kPackPerThread <= n) {  // 16-byte loads
#pragma unroll
      for (int q = 0; q < kPackPerThread / 4; ++q) {
        const uint4 a = __ldg(reinterpret_cast<const uint4*>(zz + base) + q);
        z[4 * q] = a.x, z[4 * q + 1] = a.y, z[4 * q + 2] = a.z, z[4 * q + 3] = a.w;
      }
    } else {
#pragma unroll
      for (int k = 0; k < kPackPerThread; ++k) z[k] = base + k < n ? zz[base + k] : Z(0);
    }
  } else {
#pragma unroll
    for (int k = 0; k < kPackPerThread; ++k) z[k] = base + k < n ? zz[base + k] : Z(0);
  }
  uint32_t mine = 0;  // ≤ kPackPerThread values × 150 bits
#pragma unroll
  for (int k = 0; k < kPackPerThread; ++k)
    if (base + k < n) mine += varint_bits(z[k], len);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (threadIdx.x == 0)
    for (int w = 1; w < kPackThreads / 32; ++w) wsum[w] += wsum[w - 1];
  __syncthreads();
  const uint32_t tile_total = wsum[kPackThreads / 32 - 1];
  const uint32_t p0 = (warp ? wsum[warp - 1] : 0) + incl - mine;
  // only the words two threads share need zeroing (the edge words of every range, ORed into), and the
  // word past the last one (read by the shifted store)
  if (mine) {
    words[p0 >> 5] = 0u;
    words[(p0 + mine - 1) >> 5] = 0u;
  }
  if (threadIdx.x == 0 && tile_total) words[((tile_total - 1) >> 5) + 1] = 0u;
  __syncthreads();
  // warp 0 looks back for the tile's global start bit while the other warps
  // already pack at tile-relative positions
  if (warp == 0) {
    const unsigned long long pfx = lookback(status, t, tile_total);
    if (lane == 0) s_prefix = pfx;
  }
  if (mine) {
    const uint32_t p1 = p0 + mine;
    const uint32_t w_first = p0 >> 5, w_last = (p1 - 1) >> 5;
    uint64_t acc = 0;            // bits left-aligned
    uint32_t nacc = p0 & 31;     // the first word starts mid-word
    uint32_t wi = w_first;
    auto put_word = [&](uint32_t word) {
      if (wi == w_first || wi == w_last) atomicOr(&words[wi], word);
      else words[wi] = word;
      ++wi;
    };
#pragma unroll
    for (int k = 0; k < kPackPerThread; ++k) {
      if (base + k >= n) break;
      Z v = z[k];
      for (;;) {
        const uint32_t sym = v >= 0x80 ? static_cast<uint32_t>((v & 0x7F) | 0x80) : static_cast<uint32_t>(v);
        const uint32_t e = cl[sym], l = e & 15u, c = e >> 4;
        acc |= static_cast<uint64_t>(c) << (64 - nacc - l);
        nacc += l;
        if (nacc >= 32) {
          put_word(static_cast<uint32_t>(acc >> 32));
          acc <<= 32;
          nacc -= 32;
        }
        if (v < 0x80) break;
        v >>= 7;
      }
    }
    if (nacc) put_word(static_cast<uint32_t>(acc >> 32));
  }
  __syncthreads();
  // store, shifted right by the global bit alignment of the tile
  const unsigned long long tile_start_bit = s_prefix;
  const uint32_t shift0 = static_cast<uint32_t>(tile_start_bit & 31);
  const uint32_t nwords = (shift0 + tile_total + 31) >> 5;
  const uint64_t gw0 = tile_start_bit >> 5;
  for (uint32_t w = threadIdx.x; w < nwords; w += blockDim.x) {
    const uint32_t hi = w ? words[w - 1] : 0u, lo = words[w];
    const uint32_t word = shift0 ? ((lo >> shift0) | (hi << (32 - shift0))) : lo;
    const uint32_t val = bswap32(word);
    if (w == 0) edge_first[t] = val;
    else if (w == nwords - 1) edge_last[t] = val;
    else out[gw0 + w] = val;
  }
  if (threadIdx.x == 0) {
    tile_start[t] = tile_start_bit;
    if (nwords <= 1) edge_last[t] = 0;
    if (nwords == 0) edge_first[t] = 0;
  }
}

// Merges the edge words: word W receives the OR of every tile's first / last
// word that falls on W (only neighbours can share a word: a full tile spans
// ≥ 2048 bits).  tile_start has ntiles+1 entries (the last = total bits).
static __global__ void k_pack_edges(const unsigned long long* __restrict__ tile_start, uint64_t ntiles,
                             const uint32_t* __restrict__ edge_first, const uint32_t* __restrict__ edge_last,
                             uint32_t* __restrict__ out) {
  const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (t >= ntiles) return;
  auto first_w = [&](uint64_t s) { return tile_start[s] >> 5; };
  auto last_w = [&](uint64_t s) {  // word of the tile's last bit (tile non-empty)
    return (tile_start[s + 1] - 1) >> 5;
  };
  auto nonempty = [&](uint64_t s) { return tile_start[s + 1] > tile_start[s]; };
  auto contrib = [&](uint64_t s, uint64_t W) -> uint32_t {
    if (!nonempty(s)) return 0;
    if (first_w(s) == W) return edge_first[s];
    if (last_w(s) == W) return edge_last[s];
    return 0;
  };
  if (!nonempty(t)) return;
  const uint64_t Ws[2] = {first_w(t), last_w(t)};
  for (int k = 0; k < 2; ++k) {
    if (k == 1 && Ws[1] == Ws[0]) break;
    const uint64_t W = Ws[k];
    uint32_t v = contrib(t, W);
    if (t > 0) v |= contrib(t - 1, W);
    if (t + 1 < ntiles) v |= contrib(t + 1, W);
    out[W] = v;
  }
}

// Codec 0 (raw little-endian int64, codec.cpp:437-441).
template <typename Z>
static __global__ void k_raw_encode(const Z* __restrict__ zz, uint64_t n, long long* __restrict__ out) {
  const uint64_t step = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < n; k += step)
    out[k] = unzigzag(static_cast<uint64_t>(zz[k]));
}

// ---------------------------------------------------------------------------
// CRC-32 (codec.cpp:14-28): slicing-by-4 per segment, then a GF(2) tree
// combine crc(A‖B) = crc(A)·x^{8|B|} ⊕ crc(B) (standard CRCs are affine, the
// init/xorout terms cancel).

__device__ __forceinline__ uint32_t gf2_mul(uint32_t a, uint32_t b) {
  uint32_t prod = 0;
#pragma unroll 8
  for (int i = 0; i < 32; ++i) {
    if (a & (0x80000000u >> i)) prod ^= b;
    b = (b & 1u) ? (b >> 1) ^ 0xEDB88320u : b >> 1;
  }
  return prod;
}

struct CrcConsts {
  uint32_t x8n[64];    // x^(8·2^k) mod P
  uint32_t lanec[32];  // x^(8·16·(31−l)) mod P: lane l's last 16-byte granule to the end of a warp chunk
};

__device__ __forceinline__ uint32_t crc_shift(uint32_t crc, uint64_t nbytes, const CrcConsts& k) {
  uint32_t m = 0;
  bool have = false;  // m = x^(8·nbytes) mod P, built from the set bits (no multiply by the identity)
  for (int b = 0; nbytes; ++b, nbytes >>= 1)
    if (nbytes & 1) {
      m = have ? gf2_mul(m, k.x8n[b]) : k.x8n[b];
      have = true;
    }
  return have ? gf2_mul(m, crc) : crc;
}

constexpr int kCrcThreads = 256;
constexpr int kCrcSeg = 1024;  // bytes per thread


static __global__ void __launch_bounds__(kCrcThreads) k_crc_blocks(const uint8_t* __restrict__ p, uint64_t n,
                                                            const uint32_t* __restrict__ tab_g, CrcConsts K,
                                                            uint32_t* __restrict__ blk_crc,
                                                            unsigned long long* __restrict__ blk_len) {
  __shared__ uint32_t tab[4][256];
  __shared__ uint32_t scrc[kCrcThreads];
  __shared__ unsigned long long slen[kCrcThreads];
  for (int t = threadIdx.x; t < 1024; t += blockDim.x) tab[t >> 8][t & 255] = tab_g[t];
  __syncthreads();
  const uint64_t lo = (blockIdx.x * static_cast<uint64_t>(kCrcThreads) + threadIdx.x) * kCrcSeg;
  const uint64_t hi = lo < n ? umin64(lo + kCrcSeg, n) : lo;
  uint32_t c = 0xFFFFFFFFu;
  uint64_t i = lo;
  if (hi - lo == kCrcSeg && (reinterpret_cast<uintptr_t>(p + lo) & 15) == 0) {
    // four interleaved 256-byte sub-streams (independent chains: 4x the ILP of one
    // dependent table walk), combined at the end with x^(8*256) = x8n[8]
    constexpr int kSub = 4, kSubBytes = kCrcSeg / kSub;
    uint32_t cs[kSub];
#pragma unroll
    for (int q = 0; q < kSub; ++q) cs[q] = 0xFFFFFFFFu;
    for (int off = 0; off < kSubBytes; off += 16) {
      uint4 wv[kSub];
#pragma unroll
      for (int q = 0; q < kSub; ++q) wv[q] = __ldg(reinterpret_cast<const uint4*>(p + lo + q * kSubBytes + off));
#pragma unroll
      for (int j = 0; j < 4; ++j) {
#pragma unroll
        for (int q = 0; q < kSub; ++q) {
          const uint32_t wj = j == 0 ? wv[q].x : j == 1 ? wv[q].y : j == 2 ? wv[q].z : wv[q].w;
          uint32_t cq = cs[q] ^ wj;
          cq = tab[3][cq & 255] ^ tab[2][(cq >> 8) & 255] ^ tab[1][(cq >> 16) & 255] ^ tab[0][cq >> 24];
          cs[q] = cq;
        }
      }
    }
    uint32_t acc = ~cs[0];
#pragma unroll
    for (int q = 1; q < kSub; ++q) acc = gf2_mul(K.x8n[8], acc) ^ ~cs[q];
    c = ~acc;  // back to the running-register convention of the tail loop below
    i = hi;
  }
  for (; i < hi; ++i) c = tab[0][(c ^ p[i]) & 255] ^ (c >> 8);
  scrc[threadIdx.x] = ~c;
  slen[threadIdx.x] = hi - lo;
  __syncthreads();
  for (int s = 1; s < kCrcThreads; s <<= 1) {
    uint32_t nc = 0;
    unsigned long long nl = 0;
    const bool act = (threadIdx.x % (2 * s)) == 0;
    if (act) {
      const unsigned long long lb = slen[threadIdx.x + s];
      nc = lb ? crc_shift(scrc[threadIdx.x], lb, K) ^ scrc[threadIdx.x + s] : scrc[threadIdx.x];
      nl = slen[threadIdx.x] + lb;
    }
    __syncthreads();
    if (act) {
      scrc[threadIdx.x] = nc;
      slen[threadIdx.x] = nl;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    blk_crc[blockIdx.x] = scrc[0];
    blk_len[blockIdx.x] = slen[0];
  }
}

// Coalesced CRC (the main path): the register is GF(2)-linear, so with
// raw(M) = register after M from 0, raw(A‖B) = raw(A)·x^(8|B|) ⊕ raw(B) and
// crc(M) = ~(0xFFFFFFFF·x^(8|M|) ⊕ raw(M)).  A warp owns a 16 KB chunk; lane l
// reads the 16-byte granules l, l+32, … (every load instruction is 512
// contiguous bytes), folds granule k into acc = acc·x^(8·512) ⊕ raw(granule)
// with a byte-sliced multiply table, and the lanes' sums are aligned to the
// chunk end and XOR-reduced.  The last CTA takes the sub-chunk tail (lanes
// own 512-byte pieces).  Output: raw (crc, len) per CTA for k_crc_fold.
constexpr int kCrcK = 32;                                   // granules per lane
constexpr uint64_t kCrcChunk = 32ull * 16 * kCrcK;          // bytes per warp chunk (16 KB = 2^14)
constexpr int kCrcWarps = 8;

__device__ __forceinline__ uint32_t crc_slice4(const uint32_t (*tab)[256], uint32_t c) {
  return tab[3][c & 255] ^ tab[2][(c >> 8) & 255] ^ tab[1][(c >> 16) & 255] ^ tab[0][c >> 24];
}

static __global__ void __launch_bounds__(kCrcWarps * 32) k_crc_coal(const uint8_t* __restrict__ p, uint64_t nchunks,
                                                             uint64_t tail, const uint32_t* __restrict__ tab_g,
                                                             CrcConsts K, uint32_t* __restrict__ blk_crc,
                                                             unsigned long long* __restrict__ blk_len) {
  __shared__ uint32_t tab[4][256], mt[4][256];
  __shared__ uint32_t wr[kCrcWarps];
  for (int t = threadIdx.x; t < 1024; t += blockDim.x) {
    tab[t >> 8][t & 255] = tab_g[t];
    mt[t >> 8][t & 255] = tab_g[1024 + t];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t nfull = (nchunks + kCrcWarps - 1) / kCrcWarps;  // CTAs over whole chunks
  if (blockIdx.x >= nfull) {  // the tail [nchunks·16 KB, +tail): warp 0, 512 bytes per lane, bytewise
    if (warp == 0) {
      const uint8_t* q = p + nchunks * kCrcChunk;
      const uint64_t a = umin64(tail, static_cast<uint64_t>(lane) * 512), b = umin64(tail, a + 512);
      uint32_t c = 0;
      for (uint64_t i = a; i < b; ++i) c = tab[0][(c ^ q[i]) & 255] ^ (c >> 8);
      c = crc_shift(c, tail - b, K);
#pragma unroll
      for (int o = 16; o; o >>= 1) c ^= __shfl_xor_sync(0xffffffffu, c, o);
      if (lane == 0) {
        blk_crc[blockIdx.x] = c;
        blk_len[blockIdx.x] = tail;
      }
    }
    return;
  }
  const uint64_t chunk = blockIdx.x * static_cast<uint64_t>(kCrcWarps) + warp;
  uint32_t res = 0;
  if (chunk < nchunks) {
    const uint4* g = reinterpret_cast<const uint4*>(p + chunk * kCrcChunk) + lane;
    uint32_t acc = 0;
#pragma unroll 8
    for (int k = 0; k < kCrcK; ++k) {
      const uint4 w = __ldg(g + 32 * k);
      uint32_t c = crc_slice4(tab, w.x);
      c = crc_slice4(tab, c ^ w.y);
      c = crc_slice4(tab, c ^ w.z);
      c = crc_slice4(tab, c ^ w.w);
      acc = crc_slice4(mt, acc) ^ c;  // crc_slice4 over mt = multiply by x^(8·512)
    }
    acc = gf2_mul(K.lanec[lane], acc);
#pragma unroll
    for (int o = 16; o; o >>= 1) acc ^= __shfl_xor_sync(0xffffffffu, acc, o);
    res = acc;
  }
  if (lane == 0) wr[warp] = res;
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t first = blockIdx.x * static_cast<uint64_t>(kCrcWarps);
    const int nw = static_cast<int>(umin64(kCrcWarps, nchunks - first));
    uint32_t a = wr[0];
    for (int i = 1; i < nw; ++i) a = gf2_mul(K.x8n[14], a) ^ wr[i];  // x^(8·2^14): one chunk
    blk_crc[blockIdx.x] = a;
    blk_len[blockIdx.x] = static_cast<unsigned long long>(nw) * kCrcChunk;
  }
}

// raw(M) -> crc(M) in place (one thread)
static __global__ void k_crc_finish(uint32_t* crc, const unsigned long long* len, CrcConsts K) {
  crc[0] = ~(crc_shift(0xFFFFFFFFu, len[0], K) ^ crc[0]);
}

// Folds per-block (crc, len) pairs; iterated until one pair remains.
static __global__ void __launch_bounds__(kCrcThreads) k_crc_fold(const uint32_t* __restrict__ in_crc,
                                                          const unsigned long long* __restrict__ in_len, uint64_t n,
                                                          CrcConsts K, uint32_t* __restrict__ out_crc,
                                                          unsigned long long* __restrict__ out_len) {
  __shared__ uint32_t scrc[kCrcThreads];
  __shared__ unsigned long long slen[kCrcThreads];
  const uint64_t i = blockIdx.x * static_cast<uint64_t>(kCrcThreads) + threadIdx.x;
  scrc[threadIdx.x] = i < n ? in_crc[i] : 0;
  slen[threadIdx.x] = i < n ? in_len[i] : 0;
  __syncthreads();
  for (int s = 1; s < kCrcThreads; s <<= 1) {
    uint32_t nc = 0;
    unsigned long long nl = 0;
    const bool act = (threadIdx.x % (2 * s)) == 0;
    if (act) {
      const unsigned long long lb = slen[threadIdx.x + s];
      nc = lb ? crc_shift(scrc[threadIdx.x], lb, K) ^ scrc[threadIdx.x + s] : scrc[threadIdx.x];
      nl = slen[threadIdx.x] + lb;
    }
    __syncthreads();
    if (act) {
      scrc[threadIdx.x] = nc;
      slen[threadIdx.x] = nl;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out_crc[blockIdx.x] = scrc[0];
    out_len[blockIdx.x] = slen[0];
  }
}

// ---------------------------------------------------------------------------
// Huffman decode (huff.cuh, huff_tf.cuh): the coded stream is cut into
// subsequences of kSeqBits bits (the unit of the transfer-function scan).

#ifndef MGRC_SEQ_BITS
#define MGRC_SEQ_BITS 1024
#endif
constexpr int kSeqBits = MGRC_SEQ_BITS;

struct DecodeStatus {
  unsigned long long end_bit;  // bit position after the N-th varint (ULLONG_MAX: not reached)
  unsigned int error;          // 1: varint overflow, 2: truncated value
  unsigned int wide;           // a value does not fit the u32 store
  unsigned int clean;          // only zero padding (< 8 bits) follows the N-th varint
};

// Codec 0 decode: raw little-endian int64 → zigzag.
template <typename Z>
static __global__ void k_raw_decode(const long long* __restrict__ in, uint64_t n, Z* __restrict__ zz, unsigned int* wide) {
  const uint64_t step = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  unsigned wd = 0;
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < n; k += step) {
    const uint64_t z = zigzag(in[k]);
    if (sizeof(Z) == 4 && z > 0xFFFFFFFFull) wd = 1;
    zz[k] = static_cast<Z>(z);
  }
  if (wd) atomicOr(wide, 1u);
}

template <typename T>
static __global__ void k_fill(T* __restrict__ out, uint64_t n, T value) {
  const uint64_t step = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t k = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; k < n; k += step) out[k] = value;
}

}  // namespace dev
}  // namespace mgrc_gpu
