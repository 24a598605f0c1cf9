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

}  // namespace dev

namespace {

int blocks_for(uint64_t n) { return grid_blocks(n, kTfmThreads, 16); }

struct Fwd {
  template <int D>
  struct L {
    static void run(cudaStream_t s, const GridDev& g, const BoxDev& b, const double* u, double* c) {
      k_forward<D><<<blocks_for(b.count), kTfmThreads, 0, s>>>(g, b, u, c);
      check_launch("k_forward");
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
  for (int l = 0; l <= dh.h.L; ++l) by_dim<Inv::L>(grid.d, s, dh.g, dh.boxes[l], l, dc, du);
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

}  // namespace mgrc_gpu
