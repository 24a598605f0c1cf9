// Multilevel decomposition / recomposition and the level-wise quantiser as
// entry points of their own (transform.hpp:24-30, quantize.hpp:32-42):
//
//   forward_transform   c(node) = u(node) − Σ_corners (Π w)·u(corner), the
//                       corners of the node's own tag level — ONE pass over the
//                       original data (the reference's fine→coarse sweep reads
//                       only coarse nodes that are still original)
//   inverse_transform   coarse → fine, one pass per level over the level-l box:
//                       v(node) = c(node) + Σ (Π w)·v(corner) for the nodes
//                       tagged l (transform.cpp:155-159)
//   quantize            q = rne(c/δ_tag), r = c − q·δ_tag, Overflow at
//                       |c/δ| ≥ 2^63, outliers |q| > 2^31−1 (quantize.cpp:72-132)
//   dequantize          c = (double)q·δ_tag (quantize.cpp:134-158)
//
// Arithmetic is the reference's, operation for operation (explicit _rn
// intrinsics, corner order of transform.cpp:111-128, no FMA), so
// coefficients, codes and residuals are bit-identical to the CPU library.
// All kernels walk rows of the (level-l) box: the outer indices and their tag
// are decoded once per row segment, the last axis runs across the threads, so
// the finest-level passes (the full grid) read and write coalesced rows.
#include <cuda_runtime.h>

#include <cmath>
#include <string>
#include <vector>

#include "context.hpp"
#include "kernels.cuh"
#include "pipeline.hpp"
#include "transform.hpp"

namespace mgrc_gpu {
namespace dev {

constexpr int kTfmThreads = 256;

// Box row iteration: element p of the box enumeration (row-major over the
// level-l index sets) → finest-grid multi-index i, flat index n.
template <int D>
struct BoxWalk {
  const GridDev& g;
  const BoxDev& b;
  __device__ __forceinline__ uint64_t locate(uint64_t p, uint32_t (&i)[4]) const {
    const uint32_t nk = b.n[D - 1];
    uint64_t row = p / nk;
    const uint32_t k = static_cast<uint32_t>(p - row * nk);
    i[D - 1] = __ldg(b.set[D - 1] + k);
#pragma unroll
    for (int a = D - 2; a >= 0; --a) {
      const uint64_t q = row / b.n[a];
      i[a] = __ldg(b.set[a] + static_cast<uint32_t>(row - q * b.n[a]));
      row = q;
    }
    uint64_t n = 0;
#pragma unroll
    for (int a = 0; a < D; ++a) n += static_cast<uint64_t>(i[a]) * g.stride[a];
    return n;
  }
};

// Forward transform over the whole grid (box = level L = every index).
template <int D>
__global__ void __launch_bounds__(kTfmThreads) k_forward(GridDev g, BoxDev box, const double* __restrict__ u,
                                                          double* __restrict__ c) {
  const BoxWalk<D> w{g, box};
  auto ld = [u](uint64_t off) { return __ldg(u + off); };
  const uint64_t step = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < box.count; p += step) {
    uint32_t i[4] = {0, 0, 0, 0};
    const uint64_t n = w.locate(p, i);
    const int tag = node_tag<D>(g, i);
    const double v = __ldg(u + n);
    c[n] = tag == 0 ? v : __dsub_rn(v, interp<D>(g, i, tag, ld));  // v + (−1.0)·I  (transform.cpp:130)
  }
}

// Inverse pass of level l over the level-l box: nodes tagged l get
// c + I(v) (corners are tagged < l, final by now); level 0 copies c.
template <int D>
__global__ void __launch_bounds__(kTfmThreads) k_inverse_level(GridDev g, BoxDev box, int l,
                                                                const double* __restrict__ c, double* v) {
  const BoxWalk<D> w{g, box};
  auto ld = [v](uint64_t off) { return v[off]; };
  const uint64_t step = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < box.count; p += step) {
    uint32_t i[4] = {0, 0, 0, 0};
    const uint64_t n = w.locate(p, i);
    if (node_tag<D>(g, i) != l) continue;
    const double cv = __ldg(c + n);
    v[n] = l == 0 ? cv : __dadd_rn(cv, interp<D>(g, i, l, ld));  // v + (+1.0)·I
  }
}


// ---------------------------------------------------------------------------
// Row forms over the full grid (the finest-level box, where almost all the
// bytes are): a warp per row, the lanes across the last axis (coalesced).
// The row's outer indices, their levels and the outer corner rows with their
// weight products are decoded once per row; per column the node's tag is
// max(outer tag, level of the column) and the stencil follows from it:
//   column level > outer tag: only the last axis is new (in-row neighbours);
//   column level = outer tag: the outer new axes and the last one (corner
//                             rows x left/right columns, last-axis bit highest);
//   column level < outer tag: the outer new axes only (corner rows, same column).
// Corner order, weight products and accumulation are transform.cpp:111-128's.
template <int D>
struct RowCorners {
  static constexpr int NS = 1 << (D - 1);
  uint64_t own, off[NS];
  double w[NS];
  int nsub, t_o;
};

template <int D>
__device__ __forceinline__ void row_corners(const GridDev& g, uint64_t row, int lvl, RowCorners<D>& m) {
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
  uint64_t own = 0;
  int lv[4] = {0, 0, 0, 0};
#pragma unroll
  for (int a = 0; a < D - 1; ++a) {
    lv[a] = __ldg(g.ax[a].lvl + o[a]);
    t_o = max(t_o, lv[a]);
    own += static_cast<uint64_t>(o[a]) * g.stride[a];
  }
  // lvl < 0: the forward pass (each node at its own tag); else the inverse pass of level lvl
  const int tl = lvl < 0 ? t_o : lvl;
#pragma unroll
  for (int a = 0; a < D - 1; ++a)
    if (lv[a] == tl && tl > 0) F |= 1u << a;
  m.own = own;
  m.t_o = t_o;
  m.nsub = 1 << __popc(F);
#pragma unroll
  for (int j = 0; j < RowCorners<D>::NS; ++j) {
    m.off[j] = 0;
    m.w[j] = 0.0;
    if (j >= m.nsub) continue;
    double w = 1.0;
    uint64_t uo = 0;
    int b = 0;
#pragma unroll
    for (int a = 0; a < D - 1; ++a) {
      if ((F >> a) & 1u) {
        const bool right = (j >> b) & 1;
        ++b;
        w = __dmul_rn(w, right ? __ldg(g.ax[a].wr + o[a]) : __ldg(g.ax[a].wl + o[a]));
        uo += static_cast<uint64_t>(right ? __ldg(g.ax[a].right + o[a]) : __ldg(g.ax[a].left + o[a])) * g.stride[a];
      } else {
        uo += static_cast<uint64_t>(o[a]) * g.stride[a];
      }
    }
    m.off[j] = uo;
    m.w[j] = w;
  }
}

// I(v) of node (row m, column k) at level `tag`; `lastfresh`: the column is new at `tag`.
template <int D, class Load>
__device__ __forceinline__ double row_interp(const GridDev& g, const RowCorners<D>& m, uint32_t k, bool lastfresh,
                                             bool outer, Load ld) {
  const AxisTab& t = g.ax[D - 1];
  double acc = 0.0;
  if (lastfresh) {
    const uint32_t kl = __ldg(t.left + k), kr = __ldg(t.right + k);
    const double wl = __ldg(t.wl + k), wr = __ldg(t.wr + k);
    if (!outer) return __dadd_rn(__dmul_rn(wl, ld(m.own + kl)), __dmul_rn(wr, ld(m.own + kr)));
#pragma unroll
    for (int j = 0; j < RowCorners<D>::NS; ++j)
      if (j < m.nsub) acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(m.w[j], wl), ld(m.off[j] + kl)));
#pragma unroll
    for (int j = 0; j < RowCorners<D>::NS; ++j)
      if (j < m.nsub) acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(m.w[j], wr), ld(m.off[j] + kr)));
  } else {
#pragma unroll
    for (int j = 0; j < RowCorners<D>::NS; ++j)
      if (j < m.nsub) acc = __dadd_rn(acc, __dmul_rn(m.w[j], ld(m.off[j] + k)));
  }
  return acc;
}

template <int D>
__global__ void __launch_bounds__(kTfmThreads) k_forward_rows(GridDev g, const double* __restrict__ u,
                                                               double* __restrict__ c) {
  const uint32_t n_last = g.shape[D - 1];
  const uint64_t nrows = g.N / n_last;
  const int lane = threadIdx.x & 31;
  auto ld = [u](uint64_t off) { return __ldg(u + off); };
  for (uint64_t row = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; row < nrows;
       row += (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5) {
    RowCorners<D> m;
    row_corners<D>(g, row, -1, m);
    for (uint32_t k = lane; k < n_last; k += 32) {
      const int lk = __ldg(g.ax[D - 1].lvl + k);
      const uint64_t n = m.own + k;
      const double v = __ldg(u + n);
      double out = v;
      if (lk > m.t_o) {  // only the last axis is new (tag = lk)
        out = __dsub_rn(v, row_interp<D>(g, m, k, true, false, ld));
      } else if (m.t_o > 0) {  // tag = t_o: the outer new axes, and the last if new at t_o
        out = __dsub_rn(v, row_interp<D>(g, m, k, lk == m.t_o, true, ld));
      }
      c[n] = out;
    }
  }
}

// The inverse pass of the finest level L over the full grid: nodes tagged L get c + I(v).
template <int D>
__global__ void __launch_bounds__(kTfmThreads) k_inverse_rows(GridDev g, const double* __restrict__ c, double* v) {
  const uint32_t n_last = g.shape[D - 1];
  const uint64_t nrows = g.N / n_last;
  const int lane = threadIdx.x & 31;
  const int L = g.L;
  auto ld = [v](uint64_t off) { return v[off]; };
  for (uint64_t row = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; row < nrows;
       row += (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5) {
    RowCorners<D> m;
    row_corners<D>(g, row, L, m);
    for (uint32_t k = lane; k < n_last; k += 32) {
      const int lk = __ldg(g.ax[D - 1].lvl + k);
      if (m.t_o < L && lk < L) continue;  // tag < L: written by a coarser pass
      const uint64_t n = m.own + k;
      v[n] = __dadd_rn(__ldg(c + n), row_interp<D>(g, m, k, lk == L, m.t_o == L, ld));
    }
  }
}

// The finest level of the L²-projection transform as rows: nodes tagged L
// get v ∓ I(v) in place (forward: sub; inverse: add) — k_interp_level's
// arithmetic for l = L with the row stencil of k_inverse_rows.
template <int D>
__global__ void __launch_bounds__(kTfmThreads) k_interp_rows(GridDev g, double* v, int sub) {
  const uint32_t n_last = g.shape[D - 1];
  const uint64_t nrows = g.N / n_last;
  const int lane = threadIdx.x & 31;
  const int L = g.L;
  auto ld = [v](uint64_t off) { return v[off]; };
  for (uint64_t row = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; row < nrows;
       row += (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5) {
    RowCorners<D> m;
    row_corners<D>(g, row, L, m);
    for (uint32_t k = lane; k < n_last; k += 32) {
      const int lk = __ldg(g.ax[D - 1].lvl + k);
      if (m.t_o < L && lk < L) continue;  // tag < L
      const uint64_t n = m.own + k;
      const double acc = row_interp<D>(g, m, k, lk == L, m.t_o == L, ld);
      v[n] = sub ? __dsub_rn(v[n], acc) : __dadd_rn(v[n], acc);
    }
  }
}

// The dense level-L array of the correction (the full grid): v at the nodes tagged L, zero elsewhere.
template <int D>
__global__ void __launch_bounds__(kTfmThreads) k_l2_gather_rows(GridDev g, const double* __restrict__ v,
                                                                 double* __restrict__ out) {
  const uint32_t n_last = g.shape[D - 1];
  const uint64_t nrows = g.N / n_last;
  const int lane = threadIdx.x & 31;
  const int L = g.L;
  for (uint64_t row = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) >> 5; row < nrows;
       row += (static_cast<uint64_t>(gridDim.x) * blockDim.x) >> 5) {
    int t_o = 0;
    uint64_t q = row;
#pragma unroll
    for (int a = D - 2; a >= 0; --a) {
      const uint64_t qq = q / g.shape[a];
      t_o = max(t_o, static_cast<int>(__ldg(g.ax[a].lvl + (q - qq * g.shape[a]))));
      q = qq;
    }
    const uint64_t own = row * n_last;
    for (uint32_t k = lane; k < n_last; k += 32) {
      const bool fine = t_o == L || __ldg(g.ax[D - 1].lvl + k) == L;
      out[own + k] = fine ? v[own + k] : 0.0;
    }
  }
}

struct QuantOut {
  unsigned long long overflow, outliers;
};

template <int D>
__global__ void __launch_bounds__(kTfmThreads) k_quantize(GridDev g, BoxDev box, Widths W,
                                                           const double* __restrict__ c, long long* __restrict__ q,
                                                           double* __restrict__ r, QuantOut* out) {
  const BoxWalk<D> w{g, box};
  unsigned long long ovf = 0, outl = 0;
  const uint64_t step = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < box.count; p += step) {
    uint32_t i[4] = {0, 0, 0, 0};
    const uint64_t n = w.locate(p, i);
    const double delta = W.w[node_tag<D>(g, i)];
    const double cv = __ldg(c + n);
    const double scaled = __ddiv_rn(cv, delta);
    if (!(fabs(scaled) < 9223372036854775808.0)) {  // quantize.cpp:113-116
      ++ovf;
      continue;
    }
    const long long qi = __double2ll_rn(scaled);  // = round_half_even for |x| < 2^63
    q[n] = qi;
    if (r) r[n] = __dsub_rn(cv, __dmul_rn(__ll2double_rn(qi), delta));
    if (qi > 2147483647LL || qi < -2147483648LL) ++outl;
  }
  if (ovf) atomicAdd(&out->overflow, ovf);
  if (outl) atomicAdd(&out->outliers, outl);
}

template <int D>
__global__ void __launch_bounds__(kTfmThreads) k_dequantize(GridDev g, BoxDev box, Widths W,
                                                             const long long* __restrict__ q,
                                                             double* __restrict__ c) {
  const BoxWalk<D> w{g, box};
  const uint64_t step = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < box.count; p += step) {
    uint32_t i[4] = {0, 0, 0, 0};
    const uint64_t n = w.locate(p, i);
    c[n] = __dmul_rn(__ll2double_rn(__ldg(q + n)), W.w[node_tag<D>(g, i)]);
  }
}


// ---------------------------------------------------------------------------
// L²-projection correction (opt-in; MGARD's decomposition):
// after the level-l coefficients are formed, the coarse values receive
// z = M_{l-1}^{-1} R M_l c, axis by axis (oracle/l2proj.py states the
// algorithm and the operation order this follows).

// v[node] = v[node] ± I(v)(node) in place for the nodes tagged l.
template <int D>
__global__ void __launch_bounds__(kTfmThreads) k_interp_level(GridDev g, BoxDev box, int l, int sub, double* v) {
  const BoxWalk<D> w{g, box};
  auto ld = [v](uint64_t off) { return v[off]; };
  const uint64_t step = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < box.count; p += step) {
    uint32_t i[4] = {0, 0, 0, 0};
    const uint64_t n = w.locate(p, i);
    if (node_tag<D>(g, i) != l) continue;
    const double acc = interp<D>(g, i, l, ld);
    v[n] = sub ? __dsub_rn(v[n], acc) : __dadd_rn(v[n], acc);
  }
}

// Dense level-l array (row-major over the level sets): the coefficients of
// the nodes tagged l, zero at the coarse nodes.
template <int D>
__global__ void __launch_bounds__(kTfmThreads) k_l2_gather(GridDev g, BoxDev box, int l, const double* __restrict__ v,
                                                            double* __restrict__ out) {
  const BoxWalk<D> w{g, box};
  const uint64_t step = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < box.count; p += step) {
    uint32_t i[4] = {0, 0, 0, 0};
    const uint64_t n = w.locate(p, i);
    out[p] = node_tag<D>(g, i) == l ? v[n] : 0.0;
  }
}

// v[node] = v[node] ± z for the nodes of the level-(l-1) box (z dense over it).
template <int D>
__global__ void __launch_bounds__(kTfmThreads) k_l2_scatter(GridDev g, BoxDev box, int sub,
                                                             const double* __restrict__ z, double* v) {
  const BoxWalk<D> w{g, box};
  const uint64_t step = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t p = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; p < box.count; p += step) {
    uint32_t i[4] = {0, 0, 0, 0};
    const uint64_t n = w.locate(p, i);
    v[n] = sub ? __dsub_rn(v[n], z[p]) : __dadd_rn(v[n], z[p]);
  }
}

// One axis of the correction, one thread per line: mass-matrix row, the
// restriction onto the coarse positions, the Thomas sweeps of the coarse mass
// matrix.  A: dense with `nl` along the axis, B: dense with `nc` along it;
// `inner` = product of the later dimensions (the axis stride in both), so
// consecutive threads touch consecutive addresses (coalesced unless the axis
// is the last one, where L1 serves the reuse along the line).
__device__ __forceinline__ double l2_mass(const L2Axis& t, const double* __restrict__ a, uint64_t inner, uint32_t k) {
  // ((lo_k v_{k-1} + di_k v_k) + up_k v_{k+1}), end terms absent (oracle/l2proj.py _axis_correction)
  double f = __dmul_rn(__ldg(t.di + k), a[k * inner]);
  if (k > 0) f = __dadd_rn(__dmul_rn(__ldg(t.lo + k), a[(k - 1) * inner]), f);
  if (k + 1 < t.nl) f = __dadd_rn(f, __dmul_rn(__ldg(t.up + k), a[(k + 1) * inner]));
  return f;
}

__global__ void __launch_bounds__(256) k_l2_line(L2Axis t, const double* __restrict__ A, double* __restrict__ B,
                                                 uint64_t nlines, uint64_t inner) {
  const uint64_t line = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  if (line >= nlines) return;
  const uint64_t o = line / inner, ii = line - o * inner;
  const double* a = A + o * t.nl * inner + ii;
  double* b = B + o * t.nc * inner + ii;
  // restriction + Thomas forward sweep: dp_q = (r_q - lo_q dp_{q-1}) / den_q
  double dp = 0.0;
  uint32_t mk = ~0u;  // the last mass row computed (a fresh node between two coarse ones is needed twice)
  double mv = 0.0;
  auto mass = [&](uint32_t k) {
    if (k != mk) {
      mk = k;
      mv = l2_mass(t, a, inner, k);
    }
    return mv;
  };
  for (uint32_t q = 0; q < t.nc; ++q) {
    const uint32_t k = __ldg(t.kq + q);
    double r;
    if (k > 0 && __ldg(t.fresh + k - 1)) {
      const double ml = mass(k - 1);
      r = __dadd_rn(l2_mass(t, a, inner, k), __dmul_rn(__ldg(t.wr + k - 1), ml));
    } else {
      r = l2_mass(t, a, inner, k);
    }
    if (k + 1 < t.nl && __ldg(t.fresh + k + 1))
      r = __dadd_rn(r, __dmul_rn(__ldg(t.wl + k + 1), mass(k + 1)));
    dp = q == 0 ? __ddiv_rn(r, __ldg(t.den)) : __ddiv_rn(__dsub_rn(r, __dmul_rn(__ldg(t.clo + q), dp)), __ldg(t.den + q));
    b[q * inner] = dp;
  }
  // back substitution: x_q = dp_q - cp_q x_{q+1}
  double x = dp;
  for (int q = static_cast<int>(t.nc) - 2; q >= 0; --q) {
    x = __dsub_rn(b[q * inner], __dmul_rn(__ldg(t.cp + q), x));
    b[q * inner] = x;
  }
}

}  // namespace dev

namespace {

int blocks_for(uint64_t n) { return grid_blocks(n, kTfmThreads, 16); }

struct Fwd {
  template <int D>
  struct L {
    static void run(cudaStream_t s, const GridDev& g, const BoxDev& b, const double* u, double* c) {
      (void)b;
      k_forward_rows<D><<<blocks_for(g.N / g.shape[D - 1] * 32), kTfmThreads, 0, s>>>(g, u, c);
      check_launch("k_forward_rows");
    }
  };
};
struct InvRows {
  template <int D>
  struct L {
    static void run(cudaStream_t s, const GridDev& g, const double* c, double* v) {
      k_inverse_rows<D><<<blocks_for(g.N / g.shape[D - 1] * 32), kTfmThreads, 0, s>>>(g, c, v);
      check_launch("k_inverse_rows");
    }
  };
};
struct Inv {
  template <int D>
  struct L {
    static void run(cudaStream_t s, const GridDev& g, const BoxDev& b, int l, const double* c, double* v) {
      k_inverse_level<D><<<blocks_for(b.count), kTfmThreads, 0, s>>>(g, b, l, c, v);
      check_launch("k_inverse_level");
    }
  };
};
struct Quant {
  template <int D>
  struct L {
    static void run(cudaStream_t s, const GridDev& g, const BoxDev& b, const Widths& W, const double* c,
                    long long* q, double* r, QuantOut* o) {
      k_quantize<D><<<blocks_for(b.count), kTfmThreads, 0, s>>>(g, b, W, c, q, r, o);
      check_launch("k_quantize");
    }
  };
};
struct Dequant {
  template <int D>
  struct L {
    static void run(cudaStream_t s, const GridDev& g, const BoxDev& b, const Widths& W, const long long* q,
                    double* c) {
      k_dequantize<D><<<blocks_for(b.count), kTfmThreads, 0, s>>>(g, b, W, q, c);
      check_launch("k_dequantize");
    }
  };
};


struct InterpLevel {
  template <int D>
  struct L {
    static void run(cudaStream_t s, const GridDev& g, const BoxDev& b, int l, int sub, double* v) {
      if (l == g.L) {  // the finest level (7/8 of the nodes in 3-D): rows
        k_interp_rows<D><<<blocks_for(g.N / g.shape[D - 1] * 32), kTfmThreads, 0, s>>>(g, v, sub);
        check_launch("k_interp_rows");
        return;
      }
      k_interp_level<D><<<blocks_for(b.count), kTfmThreads, 0, s>>>(g, b, l, sub, v);
      check_launch("k_interp_level");
    }
  };
};
struct L2Gather {
  template <int D>
  struct L {
    static void run(cudaStream_t s, const GridDev& g, const BoxDev& b, int l, const double* v, double* out) {
      if (l == g.L) {
        k_l2_gather_rows<D><<<blocks_for(g.N / g.shape[D - 1] * 32), kTfmThreads, 0, s>>>(g, v, out);
        check_launch("k_l2_gather_rows");
        return;
      }
      k_l2_gather<D><<<blocks_for(b.count), kTfmThreads, 0, s>>>(g, b, l, v, out);
      check_launch("k_l2_gather");
    }
  };
};
struct L2Scatter {
  template <int D>
  struct L {
    static void run(cudaStream_t s, const GridDev& g, const BoxDev& b, int sub, const double* z, double* v) {
      k_l2_scatter<D><<<blocks_for(b.count), kTfmThreads, 0, s>>>(g, b, sub, z, v);
      check_launch("k_l2_scatter");
    }
  };
};

// Device tables of the correction for every level and axis (oracle/l2proj.py
// _level_tables, the same double expressions).
void l2_tables(Context& ctx, DevHier& dh) {
  if (dh.l2_ready) return;
  const Hierarchy& h = dh.h;
  const int d = h.grid.d, L = h.L;
  std::vector<uint8_t> host;
  auto align = [](size_t x) { return (x + 15) & ~size_t{15}; };
  auto put = [&](const void* p, size_t n) {
    const size_t off = host.size();
    host.resize(align(off + n), 0);
    if (n) std::memcpy(&host[off], p, n);
    return off;
  };
  struct Off {
    size_t lo, di, up, wl, wr, fresh, kq, clo, cp, den;
    uint32_t nl, nc;
    int refines;
  };
  std::vector<Off> offs(static_cast<size_t>(L + 1) * 4);
  auto mass = [](const std::vector<double>& x, std::vector<double>& lo, std::vector<double>& di,
                 std::vector<double>& up) {
    const size_t n = x.size();
    lo.assign(n, 0.0), di.assign(n, 0.0), up.assign(n, 0.0);
    for (size_t k = 0; k < n; ++k) {
      const double hp = k > 0 ? x[k] - x[k - 1] : 0.0;
      const double hn = k + 1 < n ? x[k + 1] - x[k] : 0.0;
      lo[k] = hp / 6.0;
      di[k] = (hp + hn) / 3.0;
      up[k] = hn / 6.0;
    }
  };
  for (int l = 1; l <= L; ++l)
    for (int a = 0; a < d; ++a) {
      const auto& S = h.sets[a][l];
      const auto& Sc = h.sets[a][l - 1];
      Off& o = offs[static_cast<size_t>(l) * 4 + a];
      o.nl = static_cast<uint32_t>(S.size());
      o.nc = static_cast<uint32_t>(Sc.size());
      o.refines = S.size() > Sc.size();
      std::vector<double> x(S.size()), xc(Sc.size());
      for (size_t k = 0; k < S.size(); ++k) x[k] = h.grid.coords[a][S[k]];
      for (size_t k = 0; k < Sc.size(); ++k) xc[k] = h.grid.coords[a][Sc[k]];
      std::vector<double> lo, di, up, clo, cdi, cup;
      mass(x, lo, di, up);
      mass(xc, clo, cdi, cup);
      std::vector<uint8_t> fresh(S.size(), 0);
      std::vector<double> wl(S.size(), 0.0), wr(S.size(), 0.0);
      std::vector<uint32_t> kq;
      for (size_t k = 0; k < S.size(); ++k) {
        if (h.lvl[a][S[k]] == l) {
          fresh[k] = 1;
          wl[k] = h.wl[a][S[k]];
          wr[k] = h.wr[a][S[k]];
        } else {
          kq.push_back(static_cast<uint32_t>(k));
        }
      }
      std::vector<double> cp(Sc.size()), den(Sc.size());
      den[0] = cdi[0];
      cp[0] = cup[0] / den[0];
      for (size_t k = 1; k < Sc.size(); ++k) {
        den[k] = cdi[k] - clo[k] * cp[k - 1];
        cp[k] = cup[k] / den[k];
      }
      o.lo = put(lo.data(), 8 * lo.size());
      o.di = put(di.data(), 8 * di.size());
      o.up = put(up.data(), 8 * up.size());
      o.wl = put(wl.data(), 8 * wl.size());
      o.wr = put(wr.data(), 8 * wr.size());
      o.fresh = put(fresh.data(), fresh.size());
      o.kq = put(kq.data(), 4 * kq.size());
      o.clo = put(clo.data(), 8 * clo.size());
      o.cp = put(cp.data(), 8 * cp.size());
      o.den = put(den.data(), 8 * den.size());
    }
  uint8_t* dp = dh.l2buf.get<uint8_t>(std::max<size_t>(host.size(), 16));
  CK(cudaMemcpyAsync(dp, host.data(), host.size(), cudaMemcpyHostToDevice, ctx.stream));
  CK(cudaStreamSynchronize(ctx.stream));
  dh.l2.assign(static_cast<size_t>(L + 1) * 4, L2Axis{});
  for (int l = 1; l <= L; ++l)
    for (int a = 0; a < d; ++a) {
      const Off& o = offs[static_cast<size_t>(l) * 4 + a];
      L2Axis& t = dh.l2[static_cast<size_t>(l) * 4 + a];
      auto P64 = [&](size_t x) { return reinterpret_cast<const double*>(dp + x); };
      t.lo = P64(o.lo), t.di = P64(o.di), t.up = P64(o.up), t.wl = P64(o.wl), t.wr = P64(o.wr);
      t.fresh = dp + o.fresh;
      t.kq = reinterpret_cast<const uint32_t*>(dp + o.kq);
      t.clo = P64(o.clo), t.cp = P64(o.cp), t.den = P64(o.den);
      t.nl = o.nl, t.nc = o.nc, t.refines = o.refines;
    }
  dh.l2_ready = true;
}

// z_l (dense over the level-(l-1) box) from the coefficients of the nodes tagged l; returns its buffer.
const double* l2_correction(Context& ctx, DevHier& dh, int l, const double* v) {
  cudaStream_t s = ctx.stream;
  const int d = dh.h.grid.d;
  uint64_t dims[kMaxDims] = {1, 1, 1, 1};
  for (int a = 0; a < d; ++a) dims[a] = dh.h.sets[a][l].size();
  const uint64_t n = dh.boxes[l].count;
  double* A = ctx.l2a.get<double>(n * 8);
  double* B = ctx.l2b.get<double>(n * 8);
  by_dim<L2Gather::L>(d, s, dh.g, dh.boxes[l], l, v, A);
  for (int a = 0; a < d; ++a) {
    const L2Axis& t = dh.l2[static_cast<size_t>(l) * 4 + a];
    if (!t.refines) continue;
    uint64_t inner = 1, lines = 1;
    for (int b = 0; b < d; ++b)
      if (b != a) lines *= dims[b];
    for (int b = a + 1; b < d; ++b) inner *= dims[b];
    k_l2_line<<<static_cast<unsigned>((lines + 255) / 256), 256, 0, s>>>(t, A, B, lines, inner);
    check_launch("k_l2_line");
    dims[a] = t.nc;
    std::swap(A, B);
  }
  return A;
}

// A caller array as a device pointer: device arrays are used in place, host
// arrays are staged through the context buffer `buf` (uploaded when `in`).
template <typename T>
T* staged(Context& ctx, DevBuf& buf, const void* p, uint64_t n, bool in) {
  if (is_device_pointer(p)) return static_cast<T*>(const_cast<void*>(p));
  T* d = buf.get<T>(std::max<uint64_t>(n, 1) * sizeof(T));
  if (in) CK(cudaMemcpyAsync(d, p, n * sizeof(T), cudaMemcpyHostToDevice, ctx.stream));
  return d;
}

void download(Context& ctx, void* dst, const void* src, uint64_t bytes) {
  if (dst != src) CK(cudaMemcpyAsync(dst, src, bytes, is_device_pointer(dst) ? cudaMemcpyDeviceToDevice
                                                                               : cudaMemcpyDeviceToHost,
                                     ctx.stream));
}

Widths widths_of(const DevHier& dh, const double* widths, int nwidths) {
  if (nwidths != dh.h.L + 1) raise(Errc::shape_mismatch, "budget does not match the hierarchy");
  for (int l = 0; l < nwidths; ++l)
    if (!(widths[l] > 0.0)) raise(Errc::invalid_state, "bin widths must be > 0");
  Widths W{};
  for (int l = 0; l < nwidths; ++l) W.w[l] = widths[l];
  return W;
}

}  // namespace

void forward_transform(Context& ctx, const double* u, double* c, const Grid& grid) {
  Prof prof(ctx);
  cudaStream_t s = ctx.stream;
  const uint64_t N = grid.count();
  const double* du = staged<double>(ctx, ctx.in, u, N, true);
  // any_non_finite (transform.cpp:170)
  Scratch* sd = ctx.sd();
  Scratch* sh = ctx.sh();
  launch_stats(ctx, du, N, &sd->stats);
  CK(cudaMemcpyAsync(&sh->stats, &sd->stats, sizeof(Stats), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (sh->stats.nonfinite) raise(Errc::non_finite_input, "input contains NaN or Inf");
  DevHier& dh = device_hierarchy(ctx, grid);
  double* dc = staged<double>(ctx, ctx.v, c, N, false);
  if (static_cast<const void*>(dc) == static_cast<const void*>(du))
    raise(Errc::invalid_argument, "forward_transform: output aliases the input");
  prof.begin("forward", static_cast<double>(N) * 16);
  by_dim<Fwd::L>(grid.d, s, dh.g, dh.boxes[dh.h.L], du, dc);
  prof.end();
  download(ctx, c, dc, N * 8);
  CK(cudaStreamSynchronize(s));
}

void inverse_transform(Context& ctx, const double* c, double* u, const Grid& grid) {
  Prof prof(ctx);
  cudaStream_t s = ctx.stream;
  const uint64_t N = grid.count();
  const double* dc = staged<double>(ctx, ctx.in, c, N, true);
  DevHier& dh = device_hierarchy(ctx, grid);
  double* du = staged<double>(ctx, ctx.v, u, N, false);
  if (du == dc) raise(Errc::invalid_argument, "inverse_transform: output aliases the coefficients");
  prof.begin("inverse", static_cast<double>(N) * 16);
  for (int l = 0; l < dh.h.L; ++l) by_dim<Inv::L>(grid.d, s, dh.g, dh.boxes[l], l, dc, du);
  if (dh.h.L >= 1) by_dim<InvRows::L>(grid.d, s, dh.g, dc, du);  // the finest level: rows of the full grid
  else by_dim<Inv::L>(grid.d, s, dh.g, dh.boxes[0], 0, dc, du);
  prof.end();
  download(ctx, u, du, N * 8);
  CK(cudaStreamSynchronize(s));
}

uint64_t quantize_coefficients(Context& ctx, const double* c, const Grid& grid, const double* widths, int nwidths,
                               int64_t* q, double* r) {
  Prof prof(ctx);
  cudaStream_t s = ctx.stream;
  const uint64_t N = grid.count();
  DevHier& dh = device_hierarchy(ctx, grid);
  const Widths W = widths_of(dh, widths, nwidths);
  const double* dc = staged<double>(ctx, ctx.in, c, N, true);
  auto* dq = staged<long long>(ctx, ctx.zz, q, N, false);
  double* dr = r ? staged<double>(ctx, ctx.r, r, N, false) : nullptr;
  auto* o = ctx.partial.get<QuantOut>(sizeof(QuantOut));
  CK(cudaMemsetAsync(o, 0, sizeof(QuantOut), s));
  prof.begin("quantize", static_cast<double>(N) * (r ? 24 : 16));
  by_dim<Quant::L>(grid.d, s, dh.g, dh.boxes[dh.h.L], W, dc, dq, dr, o);
  prof.end();
  QuantOut ho{};
  CK(cudaMemcpyAsync(&ho, o, sizeof ho, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (ho.overflow)
    raise(Errc::overflow, std::to_string(ho.overflow) + " coefficients exceed the 63-bit symbol range");
  download(ctx, q, dq, N * 8);
  if (r) download(ctx, r, dr, N * 8);
  CK(cudaStreamSynchronize(s));
  return ho.outliers;
}

void dequantize_coefficients(Context& ctx, const int64_t* q, const Grid& grid, const double* widths, int nwidths,
                             double* c) {
  Prof prof(ctx);
  cudaStream_t s = ctx.stream;
  const uint64_t N = grid.count();
  DevHier& dh = device_hierarchy(ctx, grid);
  const Widths W = widths_of(dh, widths, nwidths);
  const auto* dq = staged<long long>(ctx, ctx.zz, q, N, true);
  double* dc = staged<double>(ctx, ctx.v, c, N, false);
  prof.begin("dequantize", static_cast<double>(N) * 16);
  by_dim<Dequant::L>(grid.d, s, dh.g, dh.boxes[dh.h.L], W, dq, dc);
  prof.end();
  download(ctx, c, dc, N * 8);
  CK(cudaStreamSynchronize(s));
}


void forward_transform_l2(Context& ctx, const double* u, double* c, const Grid& grid) {
  Prof prof(ctx);
  cudaStream_t s = ctx.stream;
  const uint64_t N = grid.count();
  const double* du = staged<double>(ctx, ctx.in, u, N, true);
  Scratch* sd = ctx.sd();
  Scratch* sh = ctx.sh();
  launch_stats(ctx, du, N, &sd->stats);
  CK(cudaMemcpyAsync(&sh->stats, &sd->stats, sizeof(Stats), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (sh->stats.nonfinite) raise(Errc::non_finite_input, "input contains NaN or Inf");
  DevHier& dh = device_hierarchy(ctx, grid);
  l2_tables(ctx, dh);
  double* v = staged<double>(ctx, ctx.v, c, N, false);
  if (static_cast<const void*>(v) == static_cast<const void*>(du))
    raise(Errc::invalid_argument, "forward_transform: output aliases the input");
  prof.begin("forward_l2", static_cast<double>(N) * 16);
  CK(cudaMemcpyAsync(v, du, N * 8, cudaMemcpyDeviceToDevice, s));
  for (int l = dh.h.L; l >= 1; --l) {  // oracle/l2proj.py forward_l2
    by_dim<InterpLevel::L>(grid.d, s, dh.g, dh.boxes[l], l, 1, v);
    const double* z = l2_correction(ctx, dh, l, v);
    by_dim<L2Scatter::L>(grid.d, s, dh.g, dh.boxes[l - 1], 0, z, v);
  }
  prof.end();
  download(ctx, c, v, N * 8);
  CK(cudaStreamSynchronize(s));
}

void inverse_transform_l2(Context& ctx, const double* c, double* u, const Grid& grid) {
  Prof prof(ctx);
  cudaStream_t s = ctx.stream;
  const uint64_t N = grid.count();
  const double* dc = staged<double>(ctx, ctx.in, c, N, true);
  DevHier& dh = device_hierarchy(ctx, grid);
  l2_tables(ctx, dh);
  double* v = staged<double>(ctx, ctx.v, u, N, false);
  if (v == dc) raise(Errc::invalid_argument, "inverse_transform: output aliases the coefficients");
  prof.begin("inverse_l2", static_cast<double>(N) * 16);
  CK(cudaMemcpyAsync(v, dc, N * 8, cudaMemcpyDeviceToDevice, s));
  for (int l = 1; l <= dh.h.L; ++l) {  // oracle/l2proj.py inverse_l2
    const double* z = l2_correction(ctx, dh, l, v);
    by_dim<L2Scatter::L>(grid.d, s, dh.g, dh.boxes[l - 1], 1, z, v);
    by_dim<InterpLevel::L>(grid.d, s, dh.g, dh.boxes[l], l, 0, v);
  }
  prof.end();
  download(ctx, u, v, N * 8);
  CK(cudaStreamSynchronize(s));
}

}  // namespace mgrc_gpu
