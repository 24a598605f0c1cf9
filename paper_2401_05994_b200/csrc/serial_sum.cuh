// Exact parallel reproduction of a SERIAL IEEE-754 double sum
//     s_{i+1} = fl(s_i + p_i),  p_i = fl(v_i · v_i) (SQ) or v_i,  p_i ≥ 0,
// the order the reference uses for the CLI's whole-file Σu² (tools/mgrc.cpp:
// 197-233: `sumsq += v * v`, no FMA) and for the serial combine of 4096-block
// partials (exec.cpp:68-70), so the normalised tolerance τ = tol·√(Σ/N) — and
// with it every header byte — is bit-identical without a host loop.
//
// While s stays in one binade [2^e, 2^(e+1)) it is an integer m·ulp
// (ulp = 2^(e-52), m ∈ [2^52, 2^53)) and fl(s + p) = (m + inc)·ulp with
// inc = round-half-even(p/ulp) relative to m's parity: x = p/ulp (exact,
// power-of-two scaling), f = ⌊x⌋; inc = f if x−f < ½, f+1 if > ½, and on a
// tie f or f+1 whichever makes m+inc even.  So one element is a map on the
// parity of m: (inc when m even, inc when m odd), and maps compose
// associatively: (X∘Y)_P = X_P + Y_{(P+X_P) mod 2}.  A block's composed map
// tells whether m reaches 2^53 (binade crossing, detected exactly because
// the increments are ≥ 0) inside it; the host walks the block maps, the one
// crossing block is summed serially by one thread, and the sweep restarts in
// the next binade (≈ log2(Σ/p̄) crossings in total).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace mgrc_gpu {
namespace dev {

constexpr int kSsThreads = 256;
constexpr int kSsPerThread = 4;                           // consecutive elements per lane per step
constexpr int kSsWarpSpan = 32 * kSsPerThread;            // 128 elements per warp step
constexpr int kSsBlock = 32768;                           // elements per block map
constexpr unsigned long long kSsSat = 1ull << 62;         // saturated (certain crossing)

struct SsMap {
  unsigned long long t[2];  // total increment for start parity 0 / 1 (saturating at kSsSat)
};

__device__ __forceinline__ unsigned long long ss_sat_add(unsigned long long a, unsigned long long b) {
  const unsigned long long c = a + b;
  return (c >= kSsSat || c < a) ? kSsSat : c;
}

__device__ __forceinline__ SsMap ss_compose(const SsMap& x, const SsMap& y) {
  SsMap r;
  r.t[0] = ss_sat_add(x.t[0], y.t[(x.t[0] & 1ull)]);
  r.t[1] = ss_sat_add(x.t[1], y.t[((1ull + x.t[1]) & 1ull)]);
  return r;
}

template <typename T, bool SQ>
__device__ __forceinline__ double ss_term(T v) {
  const double x = static_cast<double>(v);
  return SQ ? __dmul_rn(x, x) : x;
}

// Map of one term p in the binade whose ulp is 2^(52-e): `scale` = 2^(52-e),
// `big` = 2^53 (x ≥ big cannot stay in the binade).
__device__ __forceinline__ SsMap ss_elem(double p, double scale) {
  SsMap m;
  const double x = __dmul_rn(p, scale);
  if (!(x < 9007199254740992.0)) {  // ≥ 2^53 (or NaN): crossing for sure
    m.t[0] = m.t[1] = kSsSat;
    return m;
  }
  const double f = floor(x);
  const double fr = __dsub_rn(x, f);
  const unsigned long long fi = static_cast<unsigned long long>(f);
  if (fr < 0.5) {
    m.t[0] = m.t[1] = fi;
  } else if (fr > 0.5) {
    m.t[0] = m.t[1] = fi + 1;
  } else {  // tie: round half to even on m + inc
    m.t[0] = (fi & 1ull) ? fi + 1 : fi;  // m even: m + fi even iff fi even
    m.t[1] = (fi & 1ull) ? fi : fi + 1;  // m odd
  }
  return m;
}

// One map per block of kSsBlock terms of v[lo, hi).
template <typename T, bool SQ>
static __global__ void __launch_bounds__(kSsThreads) k_ss_blocks(const T* __restrict__ v, uint64_t lo, uint64_t hi,
                                                          double scale, SsMap* __restrict__ out) {
  __shared__ SsMap wm[kSsThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int kWarpElems = kSsBlock / (kSsThreads / 32);
  const uint64_t b0 = lo + static_cast<uint64_t>(blockIdx.x) * kSsBlock;
  const uint64_t w0 = b0 + static_cast<uint64_t>(warp) * kWarpElems;
  const uint64_t w1 = w0 + kWarpElems < hi ? w0 + kWarpElems : hi;
  SsMap acc{{0ull, 0ull}};  // identity
  for (uint64_t c = w0; c < w1; c += kSsWarpSpan) {
    SsMap mine{{0ull, 0ull}};
    const uint64_t e0 = c + static_cast<uint64_t>(lane) * kSsPerThread;
#pragma unroll
    for (int k = 0; k < kSsPerThread; ++k)
      if (e0 + k < w1) mine = ss_compose(mine, ss_elem(ss_term<T, SQ>(__ldg(v + e0 + k)), scale));
    // ordered warp reduction: lane 0 ends with lanes 0..31 composed in order
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      SsMap y;
      y.t[0] = __shfl_down_sync(0xffffffffu, mine.t[0], o);
      y.t[1] = __shfl_down_sync(0xffffffffu, mine.t[1], o);
      if ((lane & (2 * o - 1)) == 0 && lane + o < 32) mine = ss_compose(mine, y);
    }
    if (lane == 0) acc = ss_compose(acc, mine);
  }
  if (lane == 0) wm[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    SsMap m = wm[0];
    for (int w = 1; w < kSsThreads / 32; ++w) m = ss_compose(m, wm[w]);
    out[blockIdx.x] = m;
  }
}

// Serial continuation on one thread: s = fl(s + p_i) for i in [lo, hi).
template <typename T, bool SQ>
static __global__ void k_ss_serial(const T* __restrict__ v, uint64_t lo, uint64_t hi, double* __restrict__ s) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  double acc = *s;
  for (uint64_t i = lo; i < hi; ++i) acc = __dadd_rn(acc, ss_term<T, SQ>(v[i]));
  *s = acc;
}

}  // namespace dev
}  // namespace mgrc_gpu
