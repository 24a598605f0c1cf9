// Decomposition / recomposition and the level-wise quantiser as standalone
// device operations (transform.hpp:24-30, quantize.hpp:32-42 of the
// reference).  Arrays are host or device pointers (detected per call), f64,
// row-major over `grid`.
#pragma once

#include <cstdint>

#include "host.hpp"

namespace mgrc_gpu {

class Context;

// forward_transform (transform.cpp:163-178): NonFiniteInput on NaN/Inf.
void forward_transform(Context& ctx, const double* u, double* c, const Grid& grid);
// inverse_transform (transform.cpp:180-191).
void inverse_transform(Context& ctx, const double* c, double* u, const Grid& grid);
// The decomposition / recomposition with MGARD's L²-projection correction
// (opt-in, not in the reference: SPEC.md:12; oracle/l2proj.py).
void forward_transform_l2(Context& ctx, const double* u, double* c, const Grid& grid);
void inverse_transform_l2(Context& ctx, const double* c, double* u, const Grid& grid);
// quantize (quantize.cpp:72-132): Overflow when |c/δ| ≥ 2^63; returns the
// outlier count (|q| > 2^31 − 1).  r may be null.
uint64_t quantize_coefficients(Context& ctx, const double* c, const Grid& grid, const double* widths, int nwidths,
                               int64_t* q, double* r);
// dequantize (quantize.cpp:134-158).
void dequantize_coefficients(Context& ctx, const int64_t* q, const Grid& grid, const double* widths, int nwidths,
                             double* c);

}  // namespace mgrc_gpu
