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

namespace mgrc_gpu {
namespace dev {

constexpr int kRowThreads = 256;
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

// Column descriptor of a tag-L node on the last axis.
struct LastAxis {
  bool fresh;
  uint32_t kl, kr;    // finest columns of the bracketing neighbours (fresh)
  uint32_t ckl, ckr;  // their compact columns
  uint32_t ck;        // compact column (not fresh)
  double wl, wr;
};

__device__ __forceinline__ LastAxis last_axis(const GridDev& g, int D, uint32_t k) {
  const AxisTab& ax = g.ax[D - 1];
  LastAxis la;
  la.fresh = __ldg(ax.lvl + k) == g.L;
  if (la.fresh) {
    la.kl = __ldg(ax.left + k);
    la.kr = __ldg(ax.right + k);
    la.ckl = __ldg(ax.cl + k);
    la.ckr = __ldg(ax.cr + k);
    la.wl = __ldg(ax.wl + k);
    la.wr = __ldg(ax.wr + k);
    la.ck = 0;
  } else {
    la.kl = la.kr = la.ckl = la.ckr = 0;
    la.wl = la.wr = 0.0;
    la.ck = __ldg(ax.cpos + k);
  }
  return la;
}

// Σ_corners w·src over the finest grid (row offsets uoff) or the compact box
// (row offsets coff), in the reference's corner order.
template <class Ld>
__device__ __forceinline__ double row_interp(const RowMeta& m, const uint64_t* off, const LastAxis& la, uint32_t kcol,
                                             uint32_t kl, uint32_t kr, Ld ld) {
  double acc = 0.0;
  const int ns = m.nsub;
  if (!la.fresh) {
    for (int j = 0; j < ns; ++j) acc = __dadd_rn(acc, __dmul_rn(m.w[j], ld(off[j] + kcol)));
  } else {
    for (int j = 0; j < ns; ++j) acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(m.w[j], la.wl), ld(off[j] + kl)));
    for (int j = 0; j < ns; ++j) acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(m.w[j], la.wr), ld(off[j] + kr)));
  }
  return acc;
}

// Maps a tile-local element index to (row within tile, column).
__device__ __forceinline__ void tile_rc(uint32_t idx, uint32_t Kt, float invK, uint32_t& rr, uint32_t& kk) {
  rr = __float2uint_rz(__fmul_rn(static_cast<float>(idx), invK));
  int k = static_cast<int>(idx) - static_cast<int>(rr * Kt);
  if (k < 0) {
    --rr;
    k += Kt;
  } else if (k >= static_cast<int>(Kt)) {
    ++rr;
    k -= Kt;
  }
  kk = static_cast<uint32_t>(k);
}

// ---------------------------------------------------------------------------
// Compress: coarse box residuals + codes (compact), then the fused row pass.

// r and zigzag(q) of every coarse-box node, compact layout.
template <int D, typename T, typename Z>
__global__ void __launch_bounds__(256) k_coarse_quant(GridDev g, Widths W, const T* __restrict__ u,
                                                      double* __restrict__ ec, Z* __restrict__ zc, QuantFlags* flags) {
  auto ld = [u](uint64_t off) { return static_cast<double>(__ldg(u + off)); };
  unsigned long long ovf = 0;
  unsigned wide = 0;
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
  }
  if (ovf) atomicAdd(&flags->overflow, ovf);
  if (wide) atomicOr(&flags->wide, 1u);
}

// The fused pass over the finest grid, row by row: forward + quantise +
// zigzag store + varint histogram + a-posteriori check epilogue.  Coarse-box
// nodes take their code and error from (zc, ec).
template <int D, typename T, typename Z, class Chk, bool LW>
__global__ void __launch_bounds__(kRowThreads) k_fine_rows(GridDev g, RowTiling rt, Widths W, const T* __restrict__ u,
                                                          Z* __restrict__ zz, unsigned long long* __restrict__ hist,
                                                          QuantFlags* flags, const double* __restrict__ ec,
                                                          const Z* __restrict__ zc, Chk chk,
                                                          unsigned long long* __restrict__ red_out, Widths lw,
                                                          double* __restrict__ partials) {
  __shared__ RowMeta meta[kRowMaxR];
  __shared__ uint32_t sh[256];
  __shared__ double sred[kRowThreads / 32];
  for (int t = threadIdx.x; t < 256; t += blockDim.x) sh[t] = 0;
  auto ldu = [u](uint64_t off) { return static_cast<double>(__ldg(u + off)); };
  auto lde = [ec](uint64_t off) { return __ldg(ec + off); };
  uint32_t hsym = 0, hcnt = 0;
  unsigned long long ovf = 0;
  unsigned wide = 0;
  double red = 0.0;
  const uint64_t ntiles = ((rt.nrows + rt.R - 1) / rt.R) * rt.ncol_tiles;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {  // static, deterministic schedule
  const uint64_t row_tile = tile / rt.ncol_tiles;
  const uint32_t col_tile = static_cast<uint32_t>(tile - row_tile * rt.ncol_tiles);
  const uint64_t r0 = row_tile * rt.R;
  const uint32_t R = static_cast<uint32_t>(umin64(rt.R, rt.nrows - r0));
  const uint32_t k0 = col_tile * rt.K;
  const uint32_t Kt = min(rt.K, rt.n_last - k0);
  __syncthreads();  // previous tile's rows no longer in use
  build_rows<D>(g, rt, r0, R, meta);
  __syncthreads();
  const uint32_t E = R * Kt;
  const float invK = Kt == rt.K ? rt.invK : 1.0f / static_cast<float>(Kt);
  for (uint32_t idx = threadIdx.x; idx < E; idx += kRowThreads) {
    uint32_t rr, kk;
    tile_rc(idx, Kt, invK, rr, kk);
    const uint32_t k = k0 + kk;
    const RowMeta& m = meta[rr];
    const uint64_t n = m.own + k;
    const double src = static_cast<double>(__ldg(u + n));
    uint64_t z = 0;
    double e = 0.0, r = 0.0;
    int tag;
    if (g.L == 0) {  // every node is level 0: c = u
      tag = 0;
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
      const bool last_fine = __ldg(g.ax[D - 1].lvl + k) == g.L;
      if (m.all_fine || last_fine) {
        tag = g.L;
        const LastAxis la = last_axis(g, D, k);
        const double acc = row_interp(m, m.uoff, la, k, la.kl, la.kr, ldu);
        const double c = __dsub_rn(src, acc);
        const double delta = W.w[g.L];
        const double scaled = __ddiv_rn(c, delta);
        if (!(fabs(scaled) < 9223372036854775808.0)) {
          ++ovf;
        } else {
          const long long q = __double2ll_rn(scaled);
          r = __dsub_rn(c, __dmul_rn(__ll2double_rn(q), delta));
          z = zigzag(q);
        }
        if (!LW) e = __dadd_rn(r, row_interp(m, m.coff, la, la.ck, la.ckl, la.ckr, lde));
      } else {  // coarse-box node: finished by k_coarse_quant / the coarse inverse
        const uint64_t cj = m.cown + __ldg(g.ax[D - 1].cpos + k);
        z = static_cast<uint64_t>(zc[cj]);
        if (!LW) e = ec[cj];
        if (LW) {  // the level-weighted estimator needs this node's tag and r
          uint32_t i[4] = {0, 0, 0, 0};
          decompose<D>(g, n, i);
          tag = node_tag<D>(g, i);
          r = ec[cj];
        } else {
          tag = 0;
        }
      }
    }
    if (sizeof(Z) == 4 && z > 0xFFFFFFFFull) wide = 1;
    zz[n] = static_cast<Z>(z);
    hist_varint(sh, z, hsym, hcnt);
    if (LW) red = __dadd_rn(red, __dmul_rn(lw.w[tag], __dmul_rn(r, r)));
    else chk(n, e, src, red);
  }
  }  // tiles
  hist_flush(sh, hsym, hcnt);
  if (ovf) atomicAdd(&flags->overflow, ovf);
  if (wide) atomicOr(&flags->wide, 1u);
  if (LW) {
#pragma unroll
    for (int o = 16; o; o >>= 1) red = __dadd_rn(red, __shfl_down_sync(0xffffffffu, red, o));
    if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = red;
  } else if (red_out) {
#pragma unroll
    for (int o = 16; o; o >>= 1) red = fmax(red, __shfl_xor_sync(0xffffffffu, red, o));
    if ((threadIdx.x & 31) == 0 && red > 0.0)
      atomicMax(red_out, static_cast<unsigned long long>(__double_as_longlong(red)));
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
  const uint32_t E = R * Kt;
  const float invK = Kt == rt.K ? rt.invK : 1.0f / static_cast<float>(Kt);
  for (uint32_t idx = threadIdx.x; idx < E; idx += kRowThreads) {
    uint32_t rr, kk;
    tile_rc(idx, Kt, invK, rr, kk);
    const uint32_t k = k0 + kk;
    const RowMeta& m = meta[rr];
    const uint64_t n = m.own + k;
    double v;
    if (g.L == 0) {
      v = __dmul_rn(__ll2double_rn(unzigzag(static_cast<uint64_t>(zz[n]))), W.w[0]);
    } else if (m.all_fine || __ldg(g.ax[D - 1].lvl + k) == g.L) {
      const LastAxis la = last_axis(g, D, k);
      const double base = __dmul_rn(__ll2double_rn(unzigzag(static_cast<uint64_t>(zz[n]))), W.w[g.L]);
      v = __dadd_rn(base, row_interp(m, m.coff, la, la.ck, la.ckl, la.ckr, ldv));
    } else {
      v = vc[m.cown + __ldg(g.ax[D - 1].cpos + k)];
    }
    out(n, v);
  }
}

}  // namespace dev
}  // namespace mgrc_gpu
