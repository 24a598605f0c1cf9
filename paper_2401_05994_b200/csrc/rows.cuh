// Row-structured finest-level kernels (compress: k_fine_rows, decompress:
// k_recon_rows) and their coarse-box companions.
//
// The grid is walked as rows along the last (contiguous) axis.  For a row
// with outer multi-index o, every node (o, k) has tag max(t_o, lvl_last[k])
// where t_o = max_a lvl[a][o_a] over the outer axes.  Two kinds of node
// matter for the finest level L (7/8 of a 3-D grid):
//   * t_o == L: every node of the row is tagged L; the fresh outer axes F_o
//     are a per-row constant, so the outer corner rows, their offsets and the
//     outer weight products (multiplied in ascending axis order, as
//     transform.cpp:111-128 does) are computed ONCE per row;
//   * t_o < L and lvl_last[k] == L: tagged L with only the last axis fresh.
// Every other node is a coarse-box node (tag < L): its code and its
// a-posteriori error (compress) or its value (decompress) come from the
// compact coarse box, which the level-by-level kernels have finished.
//
// Corner order: the reference enumerates corners with bit k selecting the
// right neighbour of the k-th fresh axis (ascending); the last axis is the
// highest bit, so corners run (last: left, right) × (outer subsets in
// increasing bit order), and w = ((1·w_a0)·w_a1…)·w_last.  interp starts at
// 0.0 and accumulates fl(w·v); the update is v ± interp (transform.cpp:126-128).
#pragma once

#include "kernels.cuh"

// CTA shape of the warp-per-row kernels: 128 x 5 (20 warps/SM at <= 102
// registers) measured best for the fused pass among 64..288 threads x 2..9
// CTAs (1.09 ms vs 1.30 ms for 256 x 2 on 513^3 f32)
#ifndef MGRC_FINE_MINB
#define MGRC_FINE_MINB 5  // resident CTAs per SM the fused pass is compiled for
#endif
#ifndef MGRC_FINE_THREADS
#define MGRC_FINE_THREADS 128
#endif
#ifndef MGRC_RECON_THREADS
#define MGRC_RECON_THREADS 128  // with MGRC_RECON_MINB 7: 28 warps/SM, measured best of 96..256 x 3..8
#endif
#ifndef MGRC_RECON_MINB
#define MGRC_RECON_MINB 7
#endif
#ifndef MGRC_BOX_THREADS
#define MGRC_BOX_THREADS 128  // coarse-box row kernels (k_cq_warp, k_inv_warp)
#endif
#ifndef MGRC_BOX_MINB
#define MGRC_BOX_MINB 7
#endif

namespace mgrc_gpu {
namespace dev {

constexpr int kRowThreads = 256;
constexpr int kFineThreads = MGRC_FINE_THREADS;  // k_fine_warp CTA size
constexpr int kReconThreads = MGRC_RECON_THREADS;  // k_recon_warp CTA size
constexpr int kBoxThreads = MGRC_BOX_THREADS;
static_assert(kFineThreads % 32 == 0 && kReconThreads % 32 == 0 && kBoxThreads % 32 == 0, "whole warps");
// Resident CTAs per SM each variant is compiled (and launched) for: the measured
// best for the 3-D passes; fewer for the variants carrying more live state
// (the exact a-posteriori epilogues, 4-D rows with 8 corner rows) so that no
// variant spills.
template <int D, class Chk>
constexpr int fine_minb() { return D >= 4 ? 2 : (Chk::kNeedsE ? 4 : MGRC_FINE_MINB); }
template <int D>
constexpr int recon_minb() { return D >= 4 ? 4 : MGRC_RECON_MINB; }
template <int D>
constexpr int box_minb() { return D >= 4 ? 4 : MGRC_BOX_MINB; }
constexpr int kRowTileElems = 4096;  // nodes per CTA (rows × columns)
constexpr int kRowMaxR = 16;         // rows per CTA

struct RowMeta {
  uint64_t uoff[8];  // finest-grid offset of (corner row j, k = 0)
  uint64_t coff[8];  // compact offset of (corner row j, column 0) of the coarse box
  double w[8];       // outer weight product of corner row j
  uint64_t own;      // finest offset of (o, 0)
  uint64_t cown;     // compact offset of (o, 0) when every outer index is coarse
  int nsub;          // 2^|F_o| (1 when no outer axis is fresh at L)
  int all_fine;      // t_o == L: every node of the row is tagged L
};

struct RowTiling {
  uint64_t nrows;     // N / n_last
  uint32_t n_last;    // last-axis length
  uint32_t K;         // columns per tile
  uint32_t R;         // rows per tile
  uint32_t ncol_tiles;
  float invK;         // 1 / (columns in a full tile)
};

// Per-row metadata for rows [r0, r0 + R) built by threads t < R.
template <int D>
__device__ __forceinline__ void build_rows(const GridDev& g, const RowTiling& rt, uint64_t r0, uint32_t R,
                                           RowMeta* meta) {
  const uint32_t t = threadIdx.x;
  if (t >= R) return;
  RowMeta& m = meta[t];
  uint32_t o[4] = {0, 0, 0, 0};
  uint64_t q = r0 + t;
#pragma unroll
  for (int a = D - 2; a >= 0; --a) {
    const uint64_t qq = q / g.shape[a];
    o[a] = static_cast<uint32_t>(q - qq * g.shape[a]);
    q = qq;
  }
  int t_o = 0;
  uint32_t F = 0;
  uint64_t own = 0, cown = 0;
  bool all_coarse = true;
#pragma unroll
  for (int a = 0; a < D - 1; ++a) {
    const int la = __ldg(g.ax[a].lvl + o[a]);
    t_o = max(t_o, la);
    own += static_cast<uint64_t>(o[a]) * g.stride[a];
    if (g.L >= 1) {
      if (la == g.L) all_coarse = false;
      else cown += static_cast<uint64_t>(__ldg(g.ax[a].cpos + o[a])) * g.cstride[a];
    }
  }
  m.own = own;
  m.cown = all_coarse ? cown : ~0ull;
  m.all_fine = (g.L >= 1 && t_o == g.L) ? 1 : 0;
  if (m.all_fine) {
#pragma unroll
    for (int a = 0; a < D - 1; ++a)
      if (__ldg(g.ax[a].lvl + o[a]) == g.L) F |= 1u << a;
  }
  // corner rows: j enumerates the submasks of F in increasing order
  int j = 0;
  uint32_t s = 0;
  do {
    double w = 1.0;
    uint64_t uo = 0, co = 0;
#pragma unroll
    for (int a = 0; a < D - 1; ++a) {
      if ((F >> a) & 1u) {
        const bool right = (s >> a) & 1u;
        w = __dmul_rn(w, right ? __ldg(g.ax[a].wr + o[a]) : __ldg(g.ax[a].wl + o[a]));
        uo += static_cast<uint64_t>(right ? __ldg(g.ax[a].right + o[a]) : __ldg(g.ax[a].left + o[a])) * g.stride[a];
        co += static_cast<uint64_t>(right ? __ldg(g.ax[a].cr + o[a]) : __ldg(g.ax[a].cl + o[a])) * g.cstride[a];
      } else {
        uo += static_cast<uint64_t>(o[a]) * g.stride[a];
        if (g.L >= 1) co += static_cast<uint64_t>(__ldg(g.ax[a].cpos + o[a])) * g.cstride[a];
      }
    }
    m.uoff[j] = uo;
    m.coff[j] = co;
    m.w[j] = w;
    ++j;
    s = (s - F) & F;
  } while (s);
  m.nsub = j;
}

// Column descriptors of the last axis (host-built, see device_hierarchy):
//   colc[k] = {cpos[k-1], cpos[k+1]} when k is fresh at L (its bracketing
//             neighbours are always k-1 and k+1 at the finest level), else
//             {cpos[k], kNotFresh}
//   colw[k] = {w_left, w_right} when fresh at L.
constexpr uint32_t kNotFresh = 0xFFFFFFFFu;

// Corner-row data of one row, held in registers by the warp that owns it.
template <int NS>
struct RowRegs {
  uint64_t uoff[NS], coff[NS];
  double w[NS];
  uint64_t own, cown;
  int nsub, all_fine;
  __device__ __forceinline__ void load(const RowMeta& m) {
#pragma unroll
    for (int j = 0; j < NS; ++j) {
      uoff[j] = m.uoff[j];
      coff[j] = m.coff[j];
      w[j] = m.w[j];
    }
    own = m.own;
    cown = m.cown;
    nsub = m.nsub;
    all_fine = m.all_fine;
  }
};

// Σ_corners w·src in the reference's corner order for a compile-time number
// of outer corner rows M (≤ NS).  Non-fresh last axis: column kc of every
// corner row.  Fresh: columns kl then kr (last axis is the highest corner bit).
template <int M, int NS, class Ld>
__device__ __forceinline__ double interp_rows(const RowRegs<NS>& r, const uint64_t (&off)[NS], bool fresh,
                                              uint64_t kc, uint64_t kl, uint64_t kr, double wl, double wr, Ld ld) {
  double acc = 0.0;
  if (!fresh) {
#pragma unroll
    for (int j = 0; j < M; ++j) acc = __dadd_rn(acc, __dmul_rn(r.w[j], ld(off[j] + kc)));
  } else {
    double vl[M], vr[M];
#pragma unroll
    for (int j = 0; j < M; ++j) {
      vl[j] = ld(off[j] + kl);
      vr[j] = ld(off[j] + kr);
    }
#pragma unroll
    for (int j = 0; j < M; ++j) acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(r.w[j], wl), vl[j]));
#pragma unroll
    for (int j = 0; j < M; ++j) acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(r.w[j], wr), vr[j]));
  }
  return acc;
}

template <int NS, class Ld>
__device__ __forceinline__ double interp_any(const RowRegs<NS>& r, const uint64_t (&off)[NS], bool fresh, uint64_t kc,
                                             uint64_t kl, uint64_t kr, double wl, double wr, Ld ld) {
  // r.nsub is warp-uniform: no divergence
  if (NS >= 8 && r.nsub == 8) return interp_rows<(NS >= 8 ? 8 : 1), NS>(r, off, fresh, kc, kl, kr, wl, wr, ld);
  if (NS >= 4 && r.nsub == 4) return interp_rows<(NS >= 4 ? 4 : 1), NS>(r, off, fresh, kc, kl, kr, wl, wr, ld);
  if (NS >= 2 && r.nsub == 2) return interp_rows<(NS >= 2 ? 2 : 1), NS>(r, off, fresh, kc, kl, kr, wl, wr, ld);
  return interp_rows<1, NS>(r, off, fresh, kc, kl, kr, wl, wr, ld);
}

// Work split of a tile: units of one row × 64 columns (2 adjacent columns
// per lane: column parity, hence freshness, is uniform across the warp).
constexpr int kUnitCols = 64;

// ---------------------------------------------------------------------------
// Compress: coarse box residuals + codes (compact), then the fused row pass.

// r and zigzag(q) of every coarse-box node, compact layout.
template <int D, typename T, typename Z>
__global__ void __launch_bounds__(256) k_coarse_quant(GridDev g, Widths W, const T* __restrict__ u,
                                                      double* __restrict__ ec, Z* __restrict__ zc, QuantFlags* flags) {
  auto ld = [u](uint64_t off) { return static_cast<double>(__ldg(u + off)); };
  unsigned long long ovf = 0;
  unsigned wide = 0;
  double rmax = 0.0;
  const uint64_t step = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < g.Nc; j += step) {
    uint32_t i[4] = {0, 0, 0, 0};
    uint64_t q = j, n = 0;
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
      const uint64_t qq = q / g.cshape[a];
      i[a] = __ldg(g.ax[a].cset + (q - qq * g.cshape[a]));
      n += static_cast<uint64_t>(i[a]) * g.stride[a];
      q = qq;
    }
    const int tag = node_tag<D>(g, i);
    double c = static_cast<double>(u[n]);
    if (tag > 0) c = __dsub_rn(c, interp<D>(g, i, tag, ld));
    const double delta = W.w[tag];
    const double scaled = __ddiv_rn(c, delta);
    double r = 0.0;
    uint64_t z = 0;
    if (fabs(scaled) < 9223372036854775808.0) {
      const long long qv = __double2ll_rn(scaled);
      r = __dsub_rn(c, __dmul_rn(__ll2double_rn(qv), delta));
      z = zigzag(qv);
      if (sizeof(Z) == 4 && z > 0xFFFFFFFFull) wide = 1;
    } else {
      ++ovf;
    }
    ec[j] = r;
    zc[j] = static_cast<Z>(z);
    rmax = fmax(rmax, fabs(r));
  }
  flag_rmax(flags, rmax);
  if (ovf) atomicAdd(&flags->overflow, ovf);
  if (wide) atomicOr(&flags->wide, 1u);
}

// The fused pass over the finest grid, row by row: forward + quantise +
// zigzag store + varint histogram + a-posteriori check epilogue.  Coarse-box
// nodes take their code and error from (zc, ec).  Tiles are visited in a
// static grid-stride order (deterministic per-CTA partials for LW).
template <int D, typename T, typename Z, class Chk, bool LW>
__global__ void __launch_bounds__(kRowThreads) k_fine_rows(GridDev g, RowTiling rt, Widths W, const T* __restrict__ u,
                                                          Z* __restrict__ zz, unsigned long long* __restrict__ hist,
                                                          QuantFlags* flags, const double* __restrict__ ec,
                                                          const Z* __restrict__ zc, Chk chk,
                                                          unsigned long long* __restrict__ red_out, Widths lw,
                                                          double* __restrict__ partials) {
  constexpr int NS = 1 << (D - 1);
  __shared__ RowMeta meta[kRowMaxR];
  __shared__ uint32_t sh[256];
  __shared__ double sred[kRowThreads / 32];
  for (int t = threadIdx.x; t < 256; t += blockDim.x) sh[t] = 0;
  auto ldu = [u](uint64_t off) { return static_cast<double>(__ldg(u + off)); };
  auto lde = [ec](uint64_t off) { return __ldg(ec + off); };
  const AxisTab& ax = g.ax[D - 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t hsym = 0, hcnt = 0;
  unsigned long long ovf = 0;
  unsigned wide = 0;
  double red = 0.0;
  const double dL = W.w[g.L];
  const uint64_t ntiles = ((rt.nrows + rt.R - 1) / rt.R) * rt.ncol_tiles;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t row_tile = tile / rt.ncol_tiles;
    const uint32_t col_tile = static_cast<uint32_t>(tile - row_tile * rt.ncol_tiles);
    const uint64_t r0 = row_tile * rt.R;
    const uint32_t R = static_cast<uint32_t>(umin64(rt.R, rt.nrows - r0));
    const uint32_t k0 = col_tile * rt.K;
    const uint32_t Kt = min(rt.K, rt.n_last - k0);
    __syncthreads();  // previous tile's rows no longer in use
    build_rows<D>(g, rt, r0, R, meta);
    __syncthreads();
    const uint32_t nchunks = (Kt + kUnitCols - 1) / kUnitCols;
    for (uint32_t unit = warp; unit < R * nchunks; unit += kRowThreads / 32) {
      const uint32_t rr = unit / nchunks, ch = unit - rr * nchunks;
      RowRegs<NS> m;
      m.load(meta[rr]);
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        const uint32_t kk = ch * kUnitCols + 2 * lane + cc;
        if (kk >= Kt) continue;
        const uint32_t k = k0 + kk;
        const uint64_t n = m.own + k;
        const double src = static_cast<double>(__ldg(u + n));
        uint64_t z = 0;
        double e = 0.0, r = 0.0;
        int tag = 0;
        if (g.L == 0) {  // every node is level 0: c = u
          const double scaled = __ddiv_rn(src, W.w[0]);
          if (!(fabs(scaled) < 9223372036854775808.0)) {
            ++ovf;
          } else {
            const long long q = __double2ll_rn(scaled);
            r = __dsub_rn(src, __dmul_rn(__ll2double_rn(q), W.w[0]));
            z = zigzag(q);
          }
          e = r;
        } else {
          const uint2 cc2 = __ldg(reinterpret_cast<const uint2*>(ax.colc) + k);
          const bool fresh = cc2.y != kNotFresh;
          if (m.all_fine || fresh) {
            tag = g.L;
            double wl = 0.0, wr = 0.0;
            if (fresh) {
              const double2 ww = __ldg(reinterpret_cast<const double2*>(ax.colw) + k);
              wl = ww.x;
              wr = ww.y;
            }
            const double acc = interp_any<NS>(m, m.uoff, fresh, k, k - 1, k + 1, wl, wr, ldu);
            const double c = __dsub_rn(src, acc);
            const double scaled = __ddiv_rn(c, dL);
            if (!(fabs(scaled) < 9223372036854775808.0)) {
              ++ovf;
            } else {
              const long long q = __double2ll_rn(scaled);
              r = __dsub_rn(c, __dmul_rn(__ll2double_rn(q), dL));
              z = zigzag(q);
            }
            if (!LW) e = __dadd_rn(r, interp_any<NS>(m, m.coff, fresh, cc2.x, cc2.x, cc2.y, wl, wr, lde));
          } else {  // coarse-box node: finished by k_coarse_quant / the coarse inverse
            const uint64_t cj = m.cown + cc2.x;
            z = static_cast<uint64_t>(zc[cj]);
            if (!LW) {
              e = ec[cj];
            } else {  // the level-weighted estimator needs this node's tag and r
              uint32_t i[4] = {0, 0, 0, 0};
              decompose<D>(g, n, i);
              tag = node_tag<D>(g, i);
              r = ec[cj];
            }
          }
        }
        if (sizeof(Z) == 4 && z > 0xFFFFFFFFull) wide = 1;
        zz[n] = static_cast<Z>(z);
        hist_varint(sh, z, hsym, hcnt);
        if (LW) {
          red = __dadd_rn(red, __dmul_rn(lw.w[tag], __dmul_rn(r, r)));
          chk(n, r, src, red);
        } else {
          chk(n, e, src, red);
        }
      }
    }
  }
  hist_flush(sh, hsym, hcnt);
  if (ovf) atomicAdd(&flags->overflow, ovf);
  if (wide) atomicOr(&flags->wide, 1u);
  if (LW) {
#pragma unroll
    for (int o = 16; o; o >>= 1) red = __dadd_rn(red, __shfl_down_sync(0xffffffffu, red, o));
    if (lane == 0) sred[warp] = red;
  } else if (red_out) {
#pragma unroll
    for (int o = 16; o; o >>= 1) red = fmax(red, __shfl_xor_sync(0xffffffffu, red, o));
    if (lane == 0 && red > 0.0) atomicMax(red_out, static_cast<unsigned long long>(__double_as_longlong(red)));
  }
  __syncthreads();
  if (LW && threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kRowThreads / 32; ++w) t = __dadd_rn(t, sred[w]);
    partials[blockIdx.x] = t;
  }
  for (int t = threadIdx.x; t < 256; t += blockDim.x)
    if (sh[t]) atomicAdd(hist + t, static_cast<unsigned long long>(sh[t]));
}

// ---------------------------------------------------------------------------
// Quantisation q = round_half_even(c / δ) (quantize.cpp:105-123) without the
// IEEE division on the common path: t = c · fl(1/δ) differs from the exact
// quotient fl(c/δ) by at most 2^-51·|t|, so whenever t is farther than
// 2^-49·|t| from every half-integer both round to the same integer; otherwise
// (probability ~2^-48·|t|) and for |t| ≥ 2^50 the exact division decides.
// Returns false on overflow (|c/δ| ≥ 2^63, quantize.cpp:113-116).
__device__ __forceinline__ bool quantize_fast(double c, double delta, double inv, long long& q, double& r) {
  const double t = __dmul_rn(c, inv);
  const double at = fabs(t);
  if (at < 1125899906842624.0) {  // 2^50
    const double f = __dsub_rn(t, floor(t));
    if (fabs(__dsub_rn(f, 0.5)) > __dmul_rn(at, 1.7763568394002505e-15)) {  // 2^-49
      q = __double2ll_rn(t);
      r = __dsub_rn(c, __dmul_rn(__ll2double_rn(q), delta));
      return true;
    }
  }
  const double scaled = __ddiv_rn(c, delta);
  if (!(fabs(scaled) < 9223372036854775808.0)) return false;
  q = __double2ll_rn(scaled);
  r = __dsub_rn(c, __dmul_rn(__ll2double_rn(q), delta));
  return true;
}

// Per-lane first-byte counters of the code histogram: one byte per (symbol,
// lane), w[b][l/4] byte l%4, so a lane increments its own byte with a plain
// load/add/store (no atomics, at most 4-way bank conflicts: lanes of one
// word never conflict).  A lane adds at most 2 per unit (one per column), so
// the warp folds the counters into the block histogram every kUnits units.
struct LaneHist {
  static constexpr uint32_t kUnits = 127;
  uint32_t w[256][8];
  __device__ __forceinline__ void flush(uint32_t* sh, int lane) {
    __syncwarp();
#pragma unroll 1
    for (int b = lane; b < 256; b += 32) {
      uint32_t c = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        c = __dp4a(w[b][j], 0x01010101u, c);
        w[b][j] = 0u;
      }
      if (c) atomicAdd(&sh[b], c);
    }
    __syncwarp();
  }
};

// Fused finest-level pass, column-pair form.  Each lane owns columns (k, k+1)
// with k even: at the finest level an even column is never fresh and an odd
// one is fresh unless it is the last index, whose bracketing neighbours are
// k and k+2.  So the corner values of the odd column are the even column's
// (own lane) and the next lane's even column (warp shuffle), halving the
// gathers; the coarse-box errors are shared the same way.  Rows whose outer
// indices are all coarse (t_o < L) have their even column in the coarse box
// (code and error read from zc/ec) and only the last axis fresh on the odd
// one.  The number of outer corner rows M (1, 2, 4, 8) is warp-uniform and
// dispatched to a specialised body.  Same arithmetic, same order as
// transform.cpp:111-128.
template <typename T, typename Z, class Chk>
struct PairCtx {
  const GridDev* g;
  const T* __restrict__ u;
  Z* __restrict__ zz;
  const double* __restrict__ ec;
  const Z* __restrict__ zc;
  const uint4* colc4;
  const double2* colw;
  double dL, inv_L;
  Chk chk;
  uint32_t* sh;
  uint8_t* hl;         // this lane's column of the warp's first-byte counters: hl[32 * b] (LaneHist)
  unsigned long long ovf;
  unsigned wide;       // high halves of the codes OR-ed (u32 streams: any nonzero -> the wide fallback)
  double red;

  __device__ __forceinline__ uint64_t quant(double c, double& r) {
    long long q;
    if (!quantize_fast(c, dL, inv_L, q, r)) {
      ++ovf;
      r = 0.0;
      return 0;
    }
    return zigzag(q);
  }
  __device__ __forceinline__ void emit(uint64_t n, uint64_t z, double e, double src) {
    if constexpr (sizeof(Z) == 4) wide |= static_cast<unsigned>(z >> 32);
    zz[n] = static_cast<Z>(z);
    if (z < 0x80) {
      ++hl[32u * static_cast<uint32_t>(z)];
    } else {  // first byte into the lane counters, continuation bytes straight into the block histogram
      ++hl[32u * static_cast<uint32_t>((z & 0x7F) | 0x80)];
      hist_tail(sh, z >> 7);
    }
    chk(n, e, src, red);
  }
  __device__ __forceinline__ double ld(uint64_t i) const { return static_cast<double>(__ldg(u + i)); }

  // one row unit (64 columns) with M outer corner rows (M = 1: row not all-fine)
  template <int M, class Meta>
  __device__ __forceinline__ void unit(const Meta& m, uint32_t k0, uint32_t kk, uint32_t Kt, int lane) {
    constexpr bool kE = Chk::kNeedsE;
    const bool va = kk < Kt, vb = kk + 1 < Kt;
    const uint32_t k = k0 + min(kk, Kt - 1);
    const uint4 cc = __ldg(colc4 + (k >> 1));
    const bool fb = vb && cc.w != kNotFresh;
    const bool fine = M > 1;  // row all-fine (every node tagged L)
    const uint64_t own = m.own;
    const uint64_t n = own + k;
    const double sa = ld(n);
    const double sb = vb ? ld(n + 1) : 0.0;
    double wl = 0.0, wr = 0.0;
    if (fb) {
      const double2 ww = __ldg(colw + k + 1);
      wl = ww.x;
      wr = ww.y;
    }
    double U0[M], U2[M], E0[M], E2[M];
    const uint64_t cbase0 = fine ? 0 : m.cown;
#pragma unroll
    for (int j = 0; j < M; ++j) {
      U0[j] = fine ? ld(m.uoff[j] + k) : sa;
      if constexpr (kE) E0[j] = __ldg(ec + (fine ? m.coff[j] : cbase0) + cc.x);
    }
#pragma unroll
    for (int j = 0; j < M; ++j) {
      U2[j] = __shfl_down_sync(0xffffffffu, U0[j], 1);
      if constexpr (kE) E2[j] = __shfl_down_sync(0xffffffffu, E0[j], 1);
    }
    if (fb && (lane == 31 || kk + 2 >= Kt)) {  // column k+2 is not held by the next lane
#pragma unroll
      for (int j = 0; j < M; ++j) {
        U2[j] = ld((fine ? m.uoff[j] : own) + k + 2);
        if constexpr (kE) E2[j] = __ldg(ec + (fine ? m.coff[j] : cbase0) + cc.w);
      }
    }
    if (!va) return;
    // column k (even, never fresh)
    if (fine) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < M; ++j) acc = __dadd_rn(acc, __dmul_rn(m.w[j], U0[j]));
      double r;
      const uint64_t z = quant(__dsub_rn(sa, acc), r);
      if constexpr (kE) {
        double eacc = 0.0;
#pragma unroll
        for (int j = 0; j < M; ++j) eacc = __dadd_rn(eacc, __dmul_rn(m.w[j], E0[j]));
        emit(n, z, __dadd_rn(r, eacc), sa);
      } else {
        emit(n, z, r, sa);
      }
    } else {
      if constexpr (kE) emit(n, static_cast<uint64_t>(zc[cbase0 + cc.x]), E0[0], sa);
      else emit(n, static_cast<uint64_t>(zc[cbase0 + cc.x]), 0.0, sa);
    }
    if (!vb) return;
    // column k+1
    if (fb) {
      double wlj[M], wrj[M];
#pragma unroll
      for (int j = 0; j < M; ++j) {
        wlj[j] = __dmul_rn(m.w[j], wl);
        wrj[j] = __dmul_rn(m.w[j], wr);
      }
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < M; ++j) acc = __dadd_rn(acc, __dmul_rn(wlj[j], U0[j]));
#pragma unroll
      for (int j = 0; j < M; ++j) acc = __dadd_rn(acc, __dmul_rn(wrj[j], U2[j]));
      double r;
      const uint64_t z = quant(__dsub_rn(sb, acc), r);
      if constexpr (kE) {
        double eacc = 0.0;
#pragma unroll
        for (int j = 0; j < M; ++j) eacc = __dadd_rn(eacc, __dmul_rn(wlj[j], E0[j]));
#pragma unroll
        for (int j = 0; j < M; ++j) eacc = __dadd_rn(eacc, __dmul_rn(wrj[j], E2[j]));
        emit(n + 1, z, __dadd_rn(r, eacc), sb);
      } else {
        emit(n + 1, z, r, sb);
      }
    } else if (fine) {  // last index of an even-length axis, tagged L by the outer axes
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < M; ++j) acc = __dadd_rn(acc, __dmul_rn(m.w[j], ld(m.uoff[j] + k + 1)));
      double r;
      const uint64_t z = quant(__dsub_rn(sb, acc), r);
      if constexpr (kE) {
        double eacc = 0.0;
#pragma unroll
        for (int j = 0; j < M; ++j) eacc = __dadd_rn(eacc, __dmul_rn(m.w[j], __ldg(ec + m.coff[j] + cc.z)));
        emit(n + 1, z, __dadd_rn(r, eacc), sb);
      } else {
        emit(n + 1, z, r, sb);
      }
    } else {
      const uint64_t cj = cbase0 + cc.z;
      if constexpr (kE) emit(n + 1, static_cast<uint64_t>(zc[cj]), ec[cj], sb);
      else emit(n + 1, static_cast<uint64_t>(zc[cj]), 0.0, sb);
    }
  }
};


// Warp-per-row form of the fused pass: a warp takes row segments from a
// dynamic queue (no CTA barriers), builds the row's corner metadata itself
// (lane j computes outer corner row j, broadcast by shuffles), prefetches its
// next segment of u into L2 and walks the segment in 64-column units.
// (Keeping the next unit's gathers in registers while one is computed was
// measured slower: 128 registers and spills.)
template <int NS>
struct RowLite {                 // warp-uniform row metadata in registers
  uint64_t uoff[NS], coff[NS];
  double w[NS];
  uint64_t own, cown;
  int nsub, all_fine;
};

template <int D>
__device__ __forceinline__ void warp_row_meta(const GridDev& g, uint64_t row, RowLite<(1 << (D - 1))>& m) {
  const int lane = threadIdx.x & 31;
  uint32_t o[4] = {0, 0, 0, 0};
  uint64_t q = row;
#pragma unroll
  for (int a = D - 2; a >= 0; --a) {
    const uint64_t qq = q / g.shape[a];
    o[a] = static_cast<uint32_t>(q - qq * g.shape[a]);
    q = qq;
  }
  int t_o = 0;
  uint32_t F = 0;
  uint64_t own = 0, cown = 0;
  bool all_coarse = true;
  int lv[4] = {0, 0, 0, 0};
#pragma unroll
  for (int a = 0; a < D - 1; ++a) {
    lv[a] = __ldg(g.ax[a].lvl + o[a]);
    t_o = max(t_o, lv[a]);
    own += static_cast<uint64_t>(o[a]) * g.stride[a];
    if (lv[a] == g.L) all_coarse = false;
    else cown += static_cast<uint64_t>(__ldg(g.ax[a].cpos + o[a])) * g.cstride[a];
  }
  m.own = own;
  m.cown = all_coarse ? cown : ~0ull;
  m.all_fine = t_o == g.L ? 1 : 0;
  if (m.all_fine) {
#pragma unroll
    for (int a = 0; a < D - 1; ++a)
      if (lv[a] == g.L) F |= 1u << a;
  }
  const int nsub = 1 << __popc(F);
  m.nsub = nsub;
  // lane j < nsub: the j-th submask of F (increasing order) -> corner row j
  uint64_t uo = 0, co = 0;
  double w = 1.0;
  if (lane < nsub) {
    // expand the j-th submask: bit b of j selects the b-th fresh axis (ascending)
    int b = 0;
#pragma unroll
    for (int a = 0; a < D - 1; ++a) {
      if ((F >> a) & 1u) {
        const bool right = (lane >> b) & 1;
        ++b;
        w = __dmul_rn(w, right ? __ldg(g.ax[a].wr + o[a]) : __ldg(g.ax[a].wl + o[a]));
        uo += static_cast<uint64_t>(right ? __ldg(g.ax[a].right + o[a]) : __ldg(g.ax[a].left + o[a])) * g.stride[a];
        co += static_cast<uint64_t>(right ? __ldg(g.ax[a].cr + o[a]) : __ldg(g.ax[a].cl + o[a])) * g.cstride[a];
      } else {
        uo += static_cast<uint64_t>(o[a]) * g.stride[a];
        co += static_cast<uint64_t>(__ldg(g.ax[a].cpos + o[a])) * g.cstride[a];
      }
    }
  }
#pragma unroll
  for (int j = 0; j < (1 << (D - 1)); ++j) {
    m.uoff[j] = __shfl_sync(0xffffffffu, uo, j);
    m.coff[j] = __shfl_sync(0xffffffffu, co, j);
    m.w[j] = __shfl_sync(0xffffffffu, w, j);
  }
}

// Warp-wide dynamic work item (lane 0 takes a ticket, broadcast to the warp).
__device__ __forceinline__ uint64_t next_item(unsigned long long* queue) {
  uint64_t it = 0;
  if ((threadIdx.x & 31) == 0) it = atomicAdd(queue, 1ull);
  return __shfl_sync(0xffffffffu, it, 0);
}

// Registers of one 64-column unit (lane: columns k, k+1).
template <int M>
struct UnitLoads {
  uint4 cc;
  double sa, sb, wl, wr;
  double U0[M], E0[M];
};

template <int D, typename T, typename Z, class Chk>
__global__ void __launch_bounds__(kFineThreads, fine_minb<D, Chk>()) k_fine_warp(GridDev g, RowTiling rt, Widths W, double inv_L,
                                                             const T* __restrict__ u, Z* __restrict__ zz,
                                                             unsigned long long* __restrict__ hist, QuantFlags* flags,
                                                             const double* __restrict__ ec, const Z* __restrict__ zc,
                                                             Chk chk, unsigned long long* __restrict__ red_out,
                                                             unsigned long long* queue) {
  __shared__ uint32_t sh[256];
  __shared__ LaneHist lh[kFineThreads / 32];
  for (int t = threadIdx.x; t < 256; t += blockDim.x) sh[t] = 0;
  for (int t = threadIdx.x; t < kFineThreads / 32 * 256 * 8; t += blockDim.x) (&lh[0].w[0][0])[t] = 0u;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  LaneHist& myh = lh[threadIdx.x >> 5];
  uint32_t units = 0;
  PairCtx<T, Z, Chk> P;
  P.g = &g;
  P.u = u;
  P.zz = zz;
  P.ec = ec;
  P.zc = zc;
  P.colc4 = reinterpret_cast<const uint4*>(g.ax[D - 1].colc);
  P.colw = reinterpret_cast<const double2*>(g.ax[D - 1].colw);
  P.dL = W.w[g.L];
  P.inv_L = inv_L;
  P.chk = chk;
  P.sh = sh;
  P.hl = reinterpret_cast<uint8_t*>(&myh.w[0][0]) + lane;
  P.ovf = 0;
  P.wide = 0;
  P.red = 0.0;
  const uint64_t nitems = rt.nrows * rt.ncol_tiles;
  const uint64_t gw = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  // dynamic row-segment queue (load balance; every reduction here is order-independent)
  uint64_t item = 0;
  if (lane == 0) item = atomicAdd(queue, 1ull);
  item = __shfl_sync(0xffffffffu, item, 0);
  (void)gw;
  while (item < nitems) {
    const uint64_t row = item / rt.ncol_tiles;
    const uint32_t seg = static_cast<uint32_t>(item - row * rt.ncol_tiles);
    const uint32_t k0 = seg * rt.K;  // even
    const uint32_t Kt = min(rt.K, rt.n_last - k0);
    RowLite<(1 << (D - 1))> mm;
    warp_row_meta<D>(g, row, mm);
    {  // pull this warp's next row segment of u into L2 while this one is computed
      const uint64_t nitem = item + nwarps;  // roughly the segment this warp gets next
      if (nitem < nitems) {
        const uint64_t nrow = nitem / rt.ncol_tiles;
        const uint32_t nk0 = static_cast<uint32_t>(nitem - nrow * rt.ncol_tiles) * rt.K;
        const uint32_t nK = min(rt.K, rt.n_last - nk0);
        const char* base = reinterpret_cast<const char*>(u + nrow * rt.n_last + nk0);
        const uint32_t bytes = nK * static_cast<uint32_t>(sizeof(T));
        for (uint32_t off = lane * 128u; off < bytes; off += 32u * 128u)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(base + off));
      }
    }
    const uint32_t nchunks = (Kt + kUnitCols - 1) / kUnitCols;
    for (uint32_t ch = 0; ch < nchunks; ++ch) {
      const uint32_t kk = ch * kUnitCols + 2 * lane;
      if (!mm.all_fine) P.template unit<1>(mm, k0, kk, Kt, lane);
      else if (D >= 4 && mm.nsub == 8) P.template unit<(D >= 4 ? 8 : 2)>(mm, k0, kk, Kt, lane);
      else if (D >= 3 && mm.nsub == 4) P.template unit<(D >= 3 ? 4 : 2)>(mm, k0, kk, Kt, lane);
      else P.template unit<2>(mm, k0, kk, Kt, lane);
      if (++units == LaneHist::kUnits) {  // ≤ 2 counts per lane per unit: flush before a byte counter wraps
        myh.flush(sh, lane);
        units = 0;
      }
    }
    if (lane == 0) item = atomicAdd(queue, 1ull);
    item = __shfl_sync(0xffffffffu, item, 0);
  }
  myh.flush(sh, lane);
  if (P.ovf) atomicAdd(&flags->overflow, P.ovf);
  if (P.wide) atomicOr(&flags->wide, 1u);
  if (red_out) {
    double red = P.red;
#pragma unroll
    for (int o = 16; o; o >>= 1) red = fmax(red, __shfl_xor_sync(0xffffffffu, red, o));
    if (lane == 0 && red > 0.0) atomicMax(red_out, static_cast<unsigned long long>(__double_as_longlong(red)));
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 256; t += blockDim.x)
    if (sh[t]) atomicAdd(hist + t, static_cast<unsigned long long>(sh[t]));
}

// ---------------------------------------------------------------------------
// Decompress: dequantised coarse box (compact), then the row reconstruction.

template <int D, typename Z>
__global__ void __launch_bounds__(256) k_recon_coarse(GridDev g, Widths W, const Z* __restrict__ zz,
                                                      double* __restrict__ vc) {
  const uint64_t step = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; j < g.Nc; j += step) {
    uint32_t i[4] = {0, 0, 0, 0};
    uint64_t q = j, n = 0;
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
      const uint64_t qq = q / g.cshape[a];
      i[a] = __ldg(g.ax[a].cset + (q - qq * g.cshape[a]));
      n += static_cast<uint64_t>(i[a]) * g.stride[a];
      q = qq;
    }
    const int tag = node_tag<D>(g, i);
    vc[j] = __dmul_rn(__ll2double_rn(unzigzag(static_cast<uint64_t>(zz[n]))), W.w[tag]);
  }
}

struct OutF32 {
  float* p;
  __device__ __forceinline__ void operator()(uint64_t n, double v) const { p[n] = __double2float_rn(v); }
};
struct OutF64 {
  double* p;
  __device__ __forceinline__ void operator()(uint64_t n, double v) const { p[n] = v; }
};

// Final values of every node: tag-L nodes = q·δ_L + I(v_coarse); coarse-box
// nodes = their finished compact value (quantize.cpp:134-158,
// transform.cpp:155-159, container.cpp:252-259 narrowing).
template <int D, typename Z, class Out>
__global__ void __launch_bounds__(kRowThreads) k_recon_rows(GridDev g, RowTiling rt, Widths W,
                                                           const Z* __restrict__ zz, const double* __restrict__ vc,
                                                           Out out) {
  constexpr int NS = 1 << (D - 1);
  __shared__ RowMeta meta[kRowMaxR];
  const uint64_t row_tile = blockIdx.x / rt.ncol_tiles;
  const uint32_t col_tile = blockIdx.x - static_cast<uint32_t>(row_tile * rt.ncol_tiles);
  const uint64_t r0 = row_tile * rt.R;
  const uint32_t R = static_cast<uint32_t>(umin64(rt.R, rt.nrows - r0));
  const uint32_t k0 = col_tile * rt.K;
  const uint32_t Kt = min(rt.K, rt.n_last - k0);
  build_rows<D>(g, rt, r0, R, meta);
  __syncthreads();
  auto ldv = [vc](uint64_t off) { return __ldg(vc + off); };
  const AxisTab& ax = g.ax[D - 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double dL = W.w[g.L];
  const uint32_t nchunks = (Kt + kUnitCols - 1) / kUnitCols;
  for (uint32_t unit = warp; unit < R * nchunks; unit += kRowThreads / 32) {
    const uint32_t rr = unit / nchunks, ch = unit - rr * nchunks;
    RowRegs<NS> m;
    m.load(meta[rr]);
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      const uint32_t kk = ch * kUnitCols + 2 * lane + cc;
      if (kk >= Kt) continue;
      const uint32_t k = k0 + kk;
      const uint64_t n = m.own + k;
      double v;
      if (g.L == 0) {
        v = __dmul_rn(__ll2double_rn(unzigzag(static_cast<uint64_t>(zz[n]))), W.w[0]);
      } else {
        const uint2 cc2 = __ldg(reinterpret_cast<const uint2*>(ax.colc) + k);
        const bool fresh = cc2.y != kNotFresh;
        if (m.all_fine || fresh) {
          double wl = 0.0, wr = 0.0;
          if (fresh) {
            const double2 ww = __ldg(reinterpret_cast<const double2*>(ax.colw) + k);
            wl = ww.x;
            wr = ww.y;
          }
          const double base = __dmul_rn(__ll2double_rn(unzigzag(static_cast<uint64_t>(zz[n]))), dL);
          v = __dadd_rn(base, interp_any<NS>(m, m.coff, fresh, cc2.x, cc2.x, cc2.y, wl, wr, ldv));
        } else {
          v = vc[m.cown + cc2.x];
        }
      }
      out(n, v);
    }
  }
}

// Decompress finest level, warp-per-row column-pair form (see k_fine_warp):
// v = q·δ_L + Σ w·v_coarse over the corners, coarse-box nodes copied from vc.
template <typename Z, class Out>
struct ReconCtx {
  const Z* __restrict__ zz;
  const double* __restrict__ vc;
  const uint4* colc4;
  const double2* colw;
  double dL;
  Out out;

  template <int M>
  struct Ld {  // one unit's loads, issued ahead of its arithmetic
    uint4 cc;
    uint64_t za, zb;
    double2 ww;
    double V0[M];
    double V2x[M];  // column k+2 corners when the next lane does not hold them
  };

  template <int M, class Meta>
  __device__ __forceinline__ void load(const Meta& m, uint32_t k0, uint32_t kk, uint32_t Kt, int lane,
                                       Ld<M>& L) const {
    const bool vb = kk + 1 < Kt;
    const uint32_t k = k0 + min(kk, Kt - 1);
    const bool fine = M > 1;
    const uint64_t n = m.own + k;
    const uint64_t cbase0 = fine ? 0 : m.cown;
    L.cc = __ldg(colc4 + (k >> 1));
    const bool fb = vb && L.cc.w != kNotFresh;
    L.za = fine ? static_cast<uint64_t>(__ldg(zz + n)) : 0;
    L.zb = (fb || (vb && fine)) ? static_cast<uint64_t>(__ldg(zz + n + 1)) : 0;
    L.ww = fb ? __ldg(colw + k + 1) : make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 0; j < M; ++j) L.V0[j] = __ldg(vc + (fine ? m.coff[j] : cbase0) + L.cc.x);
    if (fb && (lane == 31 || kk + 2 >= Kt)) {
#pragma unroll
      for (int j = 0; j < M; ++j) L.V2x[j] = __ldg(vc + (fine ? m.coff[j] : cbase0) + L.cc.w);
    }
  }

  template <int M, class Meta>
  __device__ __forceinline__ void compute(const Meta& m, uint32_t k0, uint32_t kk, uint32_t Kt, int lane,
                                          const Ld<M>& L) const {
    const bool va = kk < Kt, vb = kk + 1 < Kt;
    const uint32_t k = k0 + min(kk, Kt - 1);
    const bool fb = vb && L.cc.w != kNotFresh;
    const bool fine = M > 1;
    const uint64_t n = m.own + k;
    const uint64_t cbase0 = fine ? 0 : m.cown;
    double V2[M];
#pragma unroll
    for (int j = 0; j < M; ++j) V2[j] = __shfl_down_sync(0xffffffffu, L.V0[j], 1);
    if (fb && (lane == 31 || kk + 2 >= Kt)) {
#pragma unroll
      for (int j = 0; j < M; ++j) V2[j] = L.V2x[j];
    }
    if (!va) return;
    if (fine) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < M; ++j) acc = __dadd_rn(acc, __dmul_rn(m.w[j], L.V0[j]));
      out(n, __dadd_rn(__dmul_rn(__ll2double_rn(unzigzag(L.za)), dL), acc));
    } else {
      out(n, L.V0[0]);
    }
    if (!vb) return;
    if (fb) {
      const double wl = L.ww.x, wr = L.ww.y;
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < M; ++j) acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(m.w[j], wl), L.V0[j]));
#pragma unroll
      for (int j = 0; j < M; ++j) acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(m.w[j], wr), V2[j]));
      out(n + 1, __dadd_rn(__dmul_rn(__ll2double_rn(unzigzag(L.zb)), dL), acc));
    } else if (fine) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < M; ++j) acc = __dadd_rn(acc, __dmul_rn(m.w[j], __ldg(vc + m.coff[j] + L.cc.z)));
      out(n + 1, __dadd_rn(__dmul_rn(__ll2double_rn(unzigzag(L.zb)), dL), acc));
    } else {
      out(n + 1, vc[cbase0 + L.cc.z]);
    }
  }

  // all units of one row segment, loads of unit i+1 in flight during unit i
  template <int M, class Meta>
  __device__ __forceinline__ void row(const Meta& m, uint32_t k0, uint32_t Kt, int lane) const {
    const uint32_t nchunks = (Kt + kUnitCols - 1) / kUnitCols;
    for (uint32_t ch = 0; ch < nchunks; ++ch) {
      const uint32_t kk = ch * kUnitCols + 2 * lane;
      Ld<M> cur;
      load<M>(m, k0, kk, Kt, lane, cur);
      compute<M>(m, k0, kk, Kt, lane, cur);
    }
  }
};

template <int D, typename Z, class Out>
__global__ void __launch_bounds__(kReconThreads, recon_minb<D>()) k_recon_warp(GridDev g, RowTiling rt, Widths W,
                                                              const Z* __restrict__ zz, const double* __restrict__ vc,
                                                              Out out, unsigned long long* queue) {
  const int lane = threadIdx.x & 31;
  ReconCtx<Z, Out> P;
  P.zz = zz;
  P.vc = vc;
  P.colc4 = reinterpret_cast<const uint4*>(g.ax[D - 1].colc);
  P.colw = reinterpret_cast<const double2*>(g.ax[D - 1].colw);
  P.dL = W.w[g.L];
  P.out = out;
  const uint64_t nitems = rt.nrows * rt.ncol_tiles;
  const uint64_t gw = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  const uint64_t nwarps = (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5;
  (void)gw;
  for (uint64_t item = next_item(queue); item < nitems; item = next_item(queue)) {
    const uint64_t row = item / rt.ncol_tiles;
    const uint32_t seg = static_cast<uint32_t>(item - row * rt.ncol_tiles);
    const uint32_t k0 = seg * rt.K;
    const uint32_t Kt = min(rt.K, rt.n_last - k0);
    RowLite<(1 << (D - 1))> mm;
    warp_row_meta<D>(g, row, mm);
    {  // pull this warp's next row segment of the codes into L2
      const uint64_t nitem = item + nwarps;
      if (nitem < nitems) {
        const uint64_t nrow = nitem / rt.ncol_tiles;
        const uint32_t nk0 = static_cast<uint32_t>(nitem - nrow * rt.ncol_tiles) * rt.K;
        const uint32_t nK = min(rt.K, rt.n_last - nk0);
        const char* base = reinterpret_cast<const char*>(zz + nrow * rt.n_last + nk0);
        const uint32_t bytes = nK * static_cast<uint32_t>(sizeof(Z));
        for (uint32_t off = lane * 128u; off < bytes; off += 32u * 128u)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(base + off));
      }
    }
    if (!mm.all_fine) P.template row<1>(mm, k0, Kt, lane);
    else if (D >= 4 && mm.nsub == 8) P.template row<(D >= 4 ? 8 : 2)>(mm, k0, Kt, lane);
    else if (D >= 3 && mm.nsub == 4) P.template row<(D >= 3 ? 4 : 2)>(mm, k0, Kt, lane);
    else P.template row<2>(mm, k0, Kt, lane);
  }
}

// ---------------------------------------------------------------------------
// In-place finest level of an inverse (v(tag-L node) += I(v)(node)) on a grid
// whose coarse values live in the same array — used on the compact coarse
// box, whose level L−1 is 7/8 of it in 3-D (transform.cpp:155-159).  Same
// column-pair structure as k_fine_warp: fresh indices at the finest level are
// the odd positions (minus the last), bracketed by k−1 and k+1.
template <int NS>
struct RowU {
  uint64_t uoff[NS];
  double w[NS];
  uint64_t own;
  int nsub, all_fine;
};

template <int D>
__device__ __forceinline__ void warp_row_meta_u(const GridDev& g, uint64_t row, RowU<(1 << (D - 1))>& m) {
  const int lane = threadIdx.x & 31;
  uint32_t o[4] = {0, 0, 0, 0};
  uint64_t q = row;
#pragma unroll
  for (int a = D - 2; a >= 0; --a) {
    const uint64_t qq = q / g.shape[a];
    o[a] = static_cast<uint32_t>(q - qq * g.shape[a]);
    q = qq;
  }
  uint32_t F = 0;
  uint64_t own = 0;
#pragma unroll
  for (int a = 0; a < D - 1; ++a) {
    if (__ldg(g.ax[a].lvl + o[a]) == g.L) F |= 1u << a;
    own += static_cast<uint64_t>(o[a]) * g.stride[a];
  }
  m.own = own;
  m.all_fine = F != 0;
  m.nsub = 1 << __popc(F);
  uint64_t uo = 0;
  double w = 1.0;
  if (lane < m.nsub) {
    int b = 0;
#pragma unroll
    for (int a = 0; a < D - 1; ++a) {
      if ((F >> a) & 1u) {
        const bool right = (lane >> b) & 1;
        ++b;
        w = __dmul_rn(w, right ? __ldg(g.ax[a].wr + o[a]) : __ldg(g.ax[a].wl + o[a]));
        uo += static_cast<uint64_t>(right ? __ldg(g.ax[a].right + o[a]) : __ldg(g.ax[a].left + o[a])) * g.stride[a];
      } else {
        uo += static_cast<uint64_t>(o[a]) * g.stride[a];
      }
    }
  }
#pragma unroll
  for (int j = 0; j < (1 << (D - 1)); ++j) {
    m.uoff[j] = __shfl_sync(0xffffffffu, uo, j);
    m.w[j] = __shfl_sync(0xffffffffu, w, j);
  }
}

template <int M, int NS>
__device__ __forceinline__ void inv_unit(const GridDev& g, const RowU<NS>& m, double* v, uint32_t k0, uint32_t kk,
                                         uint32_t Kt, int lane, int D) {
  const bool va = kk < Kt, vb = kk + 1 < Kt;
  const uint32_t k = k0 + min(kk, Kt - 1);
  const AxisTab& ax = g.ax[D - 1];
  const bool fb = vb && __ldg(ax.lvl + k + 1) == g.L;
  const bool fine = M > 1;
  const uint64_t n = m.own + k;
  double U0[M], U2[M];
#pragma unroll
  for (int j = 0; j < M; ++j) U0[j] = v[(fine ? m.uoff[j] : m.own) + k];
#pragma unroll
  for (int j = 0; j < M; ++j) U2[j] = __shfl_down_sync(0xffffffffu, U0[j], 1);
  if (fb && (lane == 31 || kk + 2 >= Kt)) {
#pragma unroll
    for (int j = 0; j < M; ++j) U2[j] = v[(fine ? m.uoff[j] : m.own) + k + 2];
  }
  if (!va) return;
  if (fine) {  // even column: tag L via the outer axes
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < M; ++j) acc = __dadd_rn(acc, __dmul_rn(m.w[j], U0[j]));
    v[n] = __dadd_rn(v[n], acc);
  }
  if (!vb) return;
  if (fb) {
    const double wl = __ldg(ax.wl + k + 1), wr = __ldg(ax.wr + k + 1);
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < M; ++j) acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(m.w[j], wl), U0[j]));
#pragma unroll
    for (int j = 0; j < M; ++j) acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(m.w[j], wr), U2[j]));
    v[n + 1] = __dadd_rn(v[n + 1], acc);
  } else if (fine) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < M; ++j) acc = __dadd_rn(acc, __dmul_rn(m.w[j], v[m.uoff[j] + k + 1]));
    v[n + 1] = __dadd_rn(v[n + 1], acc);
  }
}

template <int D>
__global__ void __launch_bounds__(kBoxThreads, box_minb<D>()) k_inv_warp(GridDev g, RowTiling rt, double* v,
                                                            unsigned long long* queue) {
  const int lane = threadIdx.x & 31;
  const uint64_t nitems = rt.nrows * rt.ncol_tiles;
  const uint64_t gw = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  (void)gw;
  for (uint64_t item = next_item(queue); item < nitems; item = next_item(queue)) {
    const uint64_t row = item / rt.ncol_tiles;
    const uint32_t seg = static_cast<uint32_t>(item - row * rt.ncol_tiles);
    const uint32_t k0 = seg * rt.K;
    const uint32_t Kt = min(rt.K, rt.n_last - k0);
    RowU<(1 << (D - 1))> mm;
    warp_row_meta_u<D>(g, row, mm);
    const uint32_t nchunks = (Kt + kUnitCols - 1) / kUnitCols;
    for (uint32_t ch = 0; ch < nchunks; ++ch) {
      const uint32_t kk = ch * kUnitCols + 2 * lane;
      if (!mm.all_fine) inv_unit<1>(g, mm, v, k0, kk, Kt, lane, D);
      else if (D >= 4 && mm.nsub == 8) inv_unit<(D >= 4 ? 8 : 2)>(g, mm, v, k0, kk, Kt, lane, D);
      else if (D >= 3 && mm.nsub == 4) inv_unit<(D >= 3 ? 4 : 2)>(g, mm, v, k0, kk, Kt, lane, D);
      else inv_unit<2>(g, mm, v, k0, kk, Kt, lane, D);
    }
  }
}

// ---------------------------------------------------------------------------
// Compress, coarse box: r and codes of its finest level (tag L−1, 7/8 of the
// box in 3-D) in column-pair form over the compact grid gc, reading u at the
// corresponding finest-grid positions (cset); the remaining nodes (tag ≤ L−2)
// by the generic gather over the level-(L−2) box (k_cq_box).
template <int NS>
struct RowCQ {
  uint64_t uoff[NS];  // finest-grid offsets of the corner rows
  double w[NS];
  uint64_t own_c, own_f;
  int nsub, all_fine;
};

template <int D>
__device__ __forceinline__ void warp_row_meta_cq(const GridDev& g, const GridDev& gc, uint64_t row,
                                                 RowCQ<(1 << (D - 1))>& m) {
  const int lane = threadIdx.x & 31;
  uint32_t o[4] = {0, 0, 0, 0};
  uint64_t q = row;
#pragma unroll
  for (int a = D - 2; a >= 0; --a) {
    const uint64_t qq = q / gc.shape[a];
    o[a] = static_cast<uint32_t>(q - qq * gc.shape[a]);
    q = qq;
  }
  uint32_t F = 0;
  uint64_t own_c = 0, own_f = 0;
#pragma unroll
  for (int a = 0; a < D - 1; ++a) {
    if (__ldg(gc.ax[a].lvl + o[a]) == gc.L) F |= 1u << a;
    own_c += static_cast<uint64_t>(o[a]) * gc.stride[a];
    own_f += static_cast<uint64_t>(__ldg(g.ax[a].cset + o[a])) * g.stride[a];
  }
  m.own_c = own_c;
  m.own_f = own_f;
  m.all_fine = F != 0;
  m.nsub = 1 << __popc(F);
  uint64_t uo = 0;
  double w = 1.0;
  if (lane < m.nsub) {
    int b = 0;
#pragma unroll
    for (int a = 0; a < D - 1; ++a) {
      uint32_t oc = o[a];
      if ((F >> a) & 1u) {
        const bool right = (lane >> b) & 1;
        ++b;
        w = __dmul_rn(w, right ? __ldg(gc.ax[a].wr + o[a]) : __ldg(gc.ax[a].wl + o[a]));
        oc = right ? __ldg(gc.ax[a].right + o[a]) : __ldg(gc.ax[a].left + o[a]);
      }
      uo += static_cast<uint64_t>(__ldg(g.ax[a].cset + oc)) * g.stride[a];
    }
  }
#pragma unroll
  for (int j = 0; j < (1 << (D - 1)); ++j) {
    m.uoff[j] = __shfl_sync(0xffffffffu, uo, j);
    m.w[j] = __shfl_sync(0xffffffffu, w, j);
  }
}

template <int M, int NS, typename T, typename Z>
__device__ __forceinline__ void cq_unit(const GridDev& g, const GridDev& gc, const RowCQ<NS>& m, const T* __restrict__ u,
                                        double* __restrict__ ec, Z* __restrict__ zc, double delta, double inv,
                                        uint32_t k0, uint32_t kk, uint32_t Kt, int lane, int D,
                                        unsigned long long& ovf, unsigned& wide, double& rmax) {
  const bool va = kk < Kt, vb = kk + 1 < Kt;
  const uint32_t k = k0 + min(kk, Kt - 1);
  const AxisTab& axc = gc.ax[D - 1];
  const uint32_t* cs = g.ax[D - 1].cset;
  const bool fb = vb && __ldg(axc.lvl + k + 1) == gc.L;
  const bool fine = M > 1;
  const uint32_t ck = __ldg(cs + k);
  double U0[M], U2[M];
#pragma unroll
  for (int j = 0; j < M; ++j) U0[j] = static_cast<double>(__ldg(u + (fine ? m.uoff[j] : m.own_f) + ck));
#pragma unroll
  for (int j = 0; j < M; ++j) U2[j] = __shfl_down_sync(0xffffffffu, U0[j], 1);
  if (fb && (lane == 31 || kk + 2 >= Kt)) {
    const uint32_t ck2 = __ldg(cs + k + 2);
#pragma unroll
    for (int j = 0; j < M; ++j) U2[j] = static_cast<double>(__ldg(u + (fine ? m.uoff[j] : m.own_f) + ck2));
  }
  if (!va) return;
  auto quant = [&](double c, uint64_t nc) {
    long long qv;
    double r;
    uint64_t z = 0;
    if (quantize_fast(c, delta, inv, qv, r)) {
      z = zigzag(qv);
      if (sizeof(Z) == 4 && z > 0xFFFFFFFFull) wide = 1;
    } else {
      ++ovf;
      r = 0.0;
    }
    ec[nc] = r;
    zc[nc] = static_cast<Z>(z);
    rmax = fmax(rmax, fabs(r));
  };
  if (fine) {  // even column, tag L−1 through the outer axes
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < M; ++j) acc = __dadd_rn(acc, __dmul_rn(m.w[j], U0[j]));
    quant(__dsub_rn(static_cast<double>(__ldg(u + m.own_f + ck)), acc), m.own_c + k);
  }
  if (!vb) return;
  const uint32_t ck1 = __ldg(cs + k + 1);
  if (fb) {
    const double wl = __ldg(axc.wl + k + 1), wr = __ldg(axc.wr + k + 1);
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < M; ++j) acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(m.w[j], wl), U0[j]));
#pragma unroll
    for (int j = 0; j < M; ++j) acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(m.w[j], wr), U2[j]));
    quant(__dsub_rn(static_cast<double>(__ldg(u + m.own_f + ck1)), acc), m.own_c + k + 1);
  } else if (fine) {
    double acc = 0.0;
#pragma unroll
    for (int j = 0; j < M; ++j)
      acc = __dadd_rn(acc, __dmul_rn(m.w[j], static_cast<double>(__ldg(u + m.uoff[j] + ck1))));
    quant(__dsub_rn(static_cast<double>(__ldg(u + m.own_f + ck1)), acc), m.own_c + k + 1);
  }
}

template <int D, typename T, typename Z>
__global__ void __launch_bounds__(kBoxThreads, box_minb<D>()) k_cq_warp(GridDev g, GridDev gc, RowTiling rt, Widths W, double inv,
                                                           const T* __restrict__ u, double* __restrict__ ec,
                                                           Z* __restrict__ zc, QuantFlags* flags,
                                                           unsigned long long* queue) {
  const int lane = threadIdx.x & 31;
  const double delta = W.w[gc.L];
  unsigned long long ovf = 0;
  unsigned wide = 0;
  double rmax = 0.0;
  const uint64_t nitems = rt.nrows * rt.ncol_tiles;
  const uint64_t gw = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5;
  (void)gw;
  for (uint64_t item = next_item(queue); item < nitems; item = next_item(queue)) {
    const uint64_t row = item / rt.ncol_tiles;
    const uint32_t seg = static_cast<uint32_t>(item - row * rt.ncol_tiles);
    const uint32_t k0 = seg * rt.K;
    const uint32_t Kt = min(rt.K, rt.n_last - k0);
    RowCQ<(1 << (D - 1))> mm;
    warp_row_meta_cq<D>(g, gc, row, mm);
    const uint32_t nchunks = (Kt + kUnitCols - 1) / kUnitCols;
    for (uint32_t ch = 0; ch < nchunks; ++ch) {
      const uint32_t kk = ch * kUnitCols + 2 * lane;
      if (!mm.all_fine) cq_unit<1>(g, gc, mm, u, ec, zc, delta, inv, k0, kk, Kt, lane, D, ovf, wide, rmax);
      else if (D >= 4 && mm.nsub == 8)
        cq_unit<(D >= 4 ? 8 : 2)>(g, gc, mm, u, ec, zc, delta, inv, k0, kk, Kt, lane, D, ovf, wide, rmax);
      else if (D >= 3 && mm.nsub == 4)
        cq_unit<(D >= 3 ? 4 : 2)>(g, gc, mm, u, ec, zc, delta, inv, k0, kk, Kt, lane, D, ovf, wide, rmax);
      else cq_unit<2>(g, gc, mm, u, ec, zc, delta, inv, k0, kk, Kt, lane, D, ovf, wide, rmax);
    }
  }
  flag_rmax(flags, rmax);
  if (ovf) atomicAdd(&flags->overflow, ovf);
  if (wide) atomicOr(&flags->wide, 1u);
}

// Nodes of tag ≤ L−2: generic gather over the level-(L−2) box (finest
// coordinates), results stored at their compact positions.
template <int D, typename T, typename Z>
__global__ void __launch_bounds__(256) k_cq_box(GridDev g, BoxDev box, Widths W, const T* __restrict__ u,
                                                double* __restrict__ ec, Z* __restrict__ zc, QuantFlags* flags) {
  auto ld = [u](uint64_t off) { return static_cast<double>(__ldg(u + off)); };
  unsigned long long ovf = 0;
  unsigned wide = 0;
  double rmax = 0.0;
  const uint64_t step = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < box.count; p += step) {
    uint32_t i[4] = {0, 0, 0, 0};
    uint64_t q = p, n = 0, nc = 0;
#pragma unroll
    for (int a = D - 1; a >= 0; --a) {
      const uint64_t qq = q / box.n[a];
      i[a] = __ldg(box.set[a] + (q - qq * box.n[a]));
      n += static_cast<uint64_t>(i[a]) * g.stride[a];
      nc += static_cast<uint64_t>(__ldg(g.ax[a].cpos + i[a])) * g.cstride[a];
      q = qq;
    }
    const int tag = node_tag<D>(g, i);
    double c = static_cast<double>(u[n]);
    if (tag > 0) c = __dsub_rn(c, interp<D>(g, i, tag, ld));
    const double delta = W.w[tag];
    const double scaled = __ddiv_rn(c, delta);
    double r = 0.0;
    uint64_t z = 0;
    if (fabs(scaled) < 9223372036854775808.0) {
      const long long qv = __double2ll_rn(scaled);
      r = __dsub_rn(c, __dmul_rn(__ll2double_rn(qv), delta));
      z = zigzag(qv);
      if (sizeof(Z) == 4 && z > 0xFFFFFFFFull) wide = 1;
    } else {
      ++ovf;
    }
    ec[nc] = r;
    zc[nc] = static_cast<Z>(z);
    rmax = fmax(rmax, fabs(r));
  }
  flag_rmax(flags, rmax);
  if (ovf) atomicAdd(&flags->overflow, ovf);
  if (wide) atomicOr(&flags->wide, 1u);
}

}  // namespace dev
}  // namespace mgrc_gpu
