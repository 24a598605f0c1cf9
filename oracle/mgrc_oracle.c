/*
 * TEST INFRASTRUCTURE ONLY — not part of the product.
 *
 * CPU restatement (plain C, single thread) of the reference compress /
 * decompress hot path (`/root/reference/proj`).  It is the *checker* for the
 * sm_100a implementation in `paper_2401_05994_b200/`: only `tests/`,
 * `__graft_entry__.smoke()` and the `cpu_baseline` leg of `bench.py` may load
 * it.  Every function cites the reference file:line it restates.
 *
 * Parity pinning: this restatement is checked against (a) the reference's
 * own known-answer tests (tests/test_grid.cpp, tests/test_transform.cpp,
 * SPEC.md examples) and (b) the reference library itself, compiled from its
 * sources by oracle/Makefile into oracle/_ref/libmgrc_ref.so, through the
 * committed golden fixtures under tests/golden/ (see tests/test_oracle.py).
 *
 * Build: gcc -O2 -ffp-contract=off (no FMA contraction: the reference's
 * Release build has no -march, so it never contracts).
 *
 * The exported C API (oc_*) is shared with oracle/ref_capi.cpp so that the
 * tests can run the same checks against either implementation.
 */
#include <math.h>
#include <stdarg.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define MAXD 4
#define MAXL 64

/* errc ordinals (error.hpp:11-31) + 1; 0 = ok. */
enum {
  OC_OK = 0,
  OC_INVALID_SHAPE = 1,
  OC_TOO_MANY_DIMS,
  OC_LEVEL_OUT_OF_RANGE,
  OC_SHAPE_MISMATCH,
  OC_NON_FINITE_INPUT,
  OC_DEGENERATE_DATA,
  OC_OVERFLOW,
  OC_UNKNOWN_CODEC,
  OC_CORRUPT_STREAM,
  OC_BAD_MAGIC,
  OC_UNSUPPORTED_VERSION,
  OC_CHECKSUM_MISMATCH,
  OC_TOLERANCE_UNREACHABLE,
  OC_PLANE_COUNT_OUT_OF_RANGE,
  OC_UNSATISFIABLE_TOLERANCE,
  OC_INVALID_STATE,
  OC_PREFIX_VIOLATION,
  OC_BUDGET_TOO_SMALL,
  OC_IO_ERROR,
};

static _Thread_local char g_err[512];

static int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

const char* oc_last_error(void) { return g_err; }
void oc_free(void* p) { free(p); }
int oc_set_threads(int n) { (void)n; return 0; } /* scalar port */
const char* oc_impl(void) { return "restatement"; }

/* ------------------------------------------------------------------------ */
/* byte buffer                                                              */

typedef struct {
  uint8_t* p;
  uint64_t n, cap;
} buf_t;

static void bput(buf_t* b, uint8_t v) {
  if (b->n == b->cap) {
    b->cap = b->cap ? b->cap * 2 : 256;
    b->p = (uint8_t*)realloc(b->p, b->cap);
  }
  b->p[b->n++] = v;
}
/* bytes.hpp:17-35, little-endian byte by byte */
static void put_u16(buf_t* b, uint16_t v) { bput(b, (uint8_t)v); bput(b, (uint8_t)(v >> 8)); }
static void put_u32(buf_t* b, uint32_t v) { for (int i = 0; i < 4; ++i) bput(b, (uint8_t)(v >> (8 * i))); }
static void put_u64(buf_t* b, uint64_t v) { for (int i = 0; i < 8; ++i) bput(b, (uint8_t)(v >> (8 * i))); }
static void put_f64(buf_t* b, double v) { uint64_t u; memcpy(&u, &v, 8); put_u64(b, u); }
static void put_bytes(buf_t* b, const uint8_t* s, uint64_t n) { for (uint64_t i = 0; i < n; ++i) bput(b, s[i]); }

/* bytes.hpp:38-74: bounds-checked reader, failures are CorruptStream */
typedef struct {
  const uint8_t* p;
  uint64_t n, pos;
  int bad;
} rd_t;

static const uint8_t* take(rd_t* r, uint64_t k) {
  if (r->bad || k > r->n - r->pos) { r->bad = 1; return NULL; }
  const uint8_t* o = r->p + r->pos;
  r->pos += k;
  return o;
}
static uint8_t get_u8(rd_t* r) { const uint8_t* b = take(r, 1); return b ? b[0] : 0; }
static uint16_t get_u16(rd_t* r) { const uint8_t* b = take(r, 2); return b ? (uint16_t)(b[0] | (b[1] << 8)) : 0; }
static uint32_t get_u32(rd_t* r) {
  const uint8_t* b = take(r, 4);
  uint32_t v = 0;
  if (b) for (int i = 3; i >= 0; --i) v = (v << 8) | b[i];
  return v;
}
static uint64_t get_u64(rd_t* r) {
  const uint8_t* b = take(r, 8);
  uint64_t v = 0;
  if (b) for (int i = 7; i >= 0; --i) v = (v << 8) | b[i];
  return v;
}
static double get_f64(rd_t* r) { uint64_t u = get_u64(r); double d; memcpy(&d, &u, 8); return d; }

/* ------------------------------------------------------------------------ */
/* grid + hierarchy (grid.cpp)                                              */

typedef struct {
  int d;
  uint64_t shape[MAXD];
  double* coords[MAXD];
  int explicit_coords;
} grid_t;

typedef struct {
  grid_t g;
  int L;
  uint64_t* sets[MAXL + 1][MAXD]; /* level_index_sets (grid.hpp:41-42) */
  uint64_t set_n[MAXL + 1][MAXD];
  uint8_t* axis_level[MAXD];      /* grid.hpp:43-44 */
  uint64_t node_counts[MAXL + 1]; /* grid.hpp:45-47 */
} hier_t;

static uint64_t grid_count(const grid_t* g) {
  uint64_t n = 1;
  for (int a = 0; a < g->d; ++a) n *= g->shape[a];
  return n;
}

/* grid.cpp:20-31 */
static int validate_shape(int d, const uint64_t* shape) {
  if (d < 1) return fail(OC_INVALID_SHAPE, "InvalidShape: grid needs at least one axis");
  if (d > MAXD) return fail(OC_TOO_MANY_DIMS, "TooManyDims: grid has %d axes, max is 4", d);
  for (int a = 0; a < d; ++a)
    if (shape[a] < 2) return fail(OC_INVALID_SHAPE, "InvalidShape: axis %d has %llu nodes, need at least 2", a, (unsigned long long)shape[a]);
  return 0;
}

static void grid_free(grid_t* g) {
  for (int a = 0; a < MAXD; ++a) { free(g->coords[a]); g->coords[a] = NULL; }
}

/* grid.cpp:56-98 (make_grid with / without coordinates) */
static int make_grid(grid_t* g, int d, const uint64_t* shape, const double* coords) {
  memset(g, 0, sizeof *g);
  int rc = validate_shape(d, shape);
  if (rc) return rc;
  g->d = d;
  uint64_t off = 0;
  for (int a = 0; a < d; ++a) {
    g->shape[a] = shape[a];
    g->coords[a] = (double*)malloc(shape[a] * sizeof(double));
    for (uint64_t i = 0; i < shape[a]; ++i)
      g->coords[a][i] = coords ? coords[off + i] : (double)i;
    if (coords) {
      for (uint64_t i = 0; i + 1 < shape[a]; ++i)
        if (!(g->coords[a][i] < g->coords[a][i + 1])) {
          grid_free(g);
          return fail(OC_INVALID_SHAPE, "InvalidShape: axis %d coordinates are not strictly increasing", a);
        }
      if (!isfinite(g->coords[a][0]) || !isfinite(g->coords[a][shape[a] - 1])) {
        grid_free(g);
        return fail(OC_INVALID_SHAPE, "InvalidShape: axis %d has non-finite coordinates", a);
      }
    }
    off += shape[a];
  }
  g->explicit_coords = coords != NULL;
  return 0;
}

static void hier_free(hier_t* h) {
  for (int a = 0; a < MAXD; ++a) {
    free(h->axis_level[a]);
    h->axis_level[a] = NULL;
  }
  /* sets alias chain storage owned per (level, axis): free unique pointers */
  for (int a = 0; a < h->g.d; ++a) {
    uint64_t* prev = NULL;
    for (int l = h->L; l >= 0; --l) {
      if (h->sets[l][a] != prev) free(h->sets[l][a]);
      prev = h->sets[l][a];
      h->sets[l][a] = NULL;
    }
  }
}

/* grid.cpp:44-52: keep even positions, plus the last when the size is even */
static uint64_t coarsen(const uint64_t* fine, uint64_t n, uint64_t* out) {
  if (n <= 2) { memcpy(out, fine, n * sizeof *out); return n; }
  uint64_t k = 0;
  for (uint64_t p = 0; p < n; p += 2) out[k++] = fine[p];
  if (n % 2 == 0) out[k++] = fine[n - 1];
  return k;
}

/* grid.cpp:100-153 */
static int build_hierarchy(hier_t* h, const grid_t* g) {
  memset(h, 0, sizeof *h);
  h->g = *g;
  const int d = g->d;
  uint64_t* chain[MAXD][MAXL + 1];
  uint64_t chain_n[MAXD][MAXL + 1];
  int chain_len[MAXD];
  int L = 0;
  for (int a = 0; a < d; ++a) {
    chain[a][0] = (uint64_t*)malloc(g->shape[a] * sizeof(uint64_t));
    for (uint64_t i = 0; i < g->shape[a]; ++i) chain[a][0][i] = i;
    chain_n[a][0] = g->shape[a];
    int k = 0;
    while (chain_n[a][k] > 2) {
      chain[a][k + 1] = (uint64_t*)malloc((chain_n[a][k] / 2 + 2) * sizeof(uint64_t));
      chain_n[a][k + 1] = coarsen(chain[a][k], chain_n[a][k], chain[a][k + 1]);
      ++k;
    }
    chain_len[a] = k + 1;
    if (k > L) L = k;
  }
  h->L = L;
  for (int l = 0; l <= L; ++l)
    for (int a = 0; a < d; ++a) {
      int steps = L - l < chain_len[a] - 1 ? L - l : chain_len[a] - 1;
      h->sets[l][a] = chain[a][steps];
      h->set_n[l][a] = chain_n[a][steps];
    }
  for (int a = 0; a < d; ++a) {
    h->axis_level[a] = (uint8_t*)malloc(g->shape[a]);
    memset(h->axis_level[a], L, g->shape[a]);
    for (int l = L; l >= 0; --l)
      for (uint64_t p = 0; p < h->set_n[l][a]; ++p) h->axis_level[a][h->sets[l][a][p]] = (uint8_t)l;
  }
  uint64_t prev = 0;
  for (int l = 0; l <= L; ++l) {
    uint64_t box = 1;
    for (int a = 0; a < d; ++a) box *= h->set_n[l][a];
    h->node_counts[l] = box - prev;
    prev = box;
  }
  return 0;
}

/* grid.hpp:52-59 */
static int level_tag(const hier_t* h, const uint64_t* idx) {
  int t = 0;
  for (int a = 0; a < h->g.d; ++a)
    if (h->axis_level[a][idx[a]] > t) t = h->axis_level[a][idx[a]];
  return t;
}

/* ------------------------------------------------------------------------ */
/* multilevel transform (transform.cpp)                                     */

typedef struct {
  uint64_t n;
  const uint64_t* idx;
  uint8_t* fresh;
  uint64_t* left;
  uint64_t* right;
  double* wl;
  double* wr;
} stencil_t;

/* transform.cpp:27-63 */
static void build_axis_stencil(const hier_t* h, int level, int axis, stencil_t* s) {
  const uint64_t* set = h->sets[level][axis];
  const double* x = h->g.coords[axis];
  const uint64_t n = h->set_n[level][axis];
  s->n = n;
  s->idx = set;
  s->fresh = (uint8_t*)calloc(n, 1);
  s->left = (uint64_t*)calloc(n, 8);
  s->right = (uint64_t*)calloc(n, 8);
  s->wl = (double*)calloc(n, 8);
  s->wr = (double*)calloc(n, 8);
  uint64_t* next_coarse = (uint64_t*)malloc(n * 8);
  for (uint64_t p = 0; p < n; ++p) next_coarse[p] = set[n - 1];
  for (uint64_t p = n; p-- > 0;) {
    if (h->axis_level[axis][set[p]] < level) next_coarse[p] = set[p];
    else if (p + 1 < n) next_coarse[p] = next_coarse[p + 1];
  }
  uint64_t prev_coarse = set[0];
  for (uint64_t p = 0; p < n; ++p) {
    const uint64_t i = set[p];
    if (h->axis_level[axis][i] < level) { prev_coarse = i; continue; }
    s->fresh[p] = 1;
    s->left[p] = prev_coarse;
    s->right[p] = next_coarse[p];
    const double xl = x[s->left[p]], xr = x[s->right[p]];
    s->wl[p] = (xr - x[i]) / (xr - xl);
    s->wr[p] = (x[i] - xl) / (xr - xl);
  }
  free(next_coarse);
}

static void free_stencil(stencil_t* s) {
  free(s->fresh); free(s->left); free(s->right); free(s->wl); free(s->wr);
}

/* transform.cpp:68-143: values[node] += sign * I_{l-1}(node) for new nodes */
static void apply_level(double* values, const hier_t* h, int level, double sign) {
  const int d = h->g.d;
  stencil_t st[MAXD];
  memset(st, 0, sizeof st);
  uint64_t stride[MAXD];
  stride[d - 1] = 1;
  for (int a = d - 1; a-- > 0;) stride[a] = stride[a + 1] * h->g.shape[a + 1];
  for (int a = 0; a < d; ++a) build_axis_stencil(h, level, a, &st[a]);
  uint64_t nrows = 1;
  for (int a = 0; a + 1 < d; ++a) nrows *= st[a].n;
  const uint64_t inner = st[d - 1].n;
  for (uint64_t row = 0; row < nrows; ++row) {
    uint64_t pos[MAXD] = {0, 0, 0, 0};
    uint64_t r = row;
    for (int a = d - 1; a-- > 0;) { pos[a] = r % st[a].n; r /= st[a].n; }
    uint64_t base = 0;
    int outer_new = 0;
    for (int a = 0; a + 1 < d; ++a) {
      base += st[a].idx[pos[a]] * stride[a];
      outer_new |= st[a].fresh[pos[a]] != 0;
    }
    const stencil_t* in = &st[d - 1];
    for (uint64_t p = 0; p < inner; ++p) {
      if (!(outer_new || in->fresh[p])) continue;
      pos[d - 1] = p;
      int new_axes[MAXD], n_new = 0;
      uint64_t fixed = 0;
      for (int a = 0; a < d; ++a) {
        if (st[a].fresh[pos[a]]) new_axes[n_new++] = a;
        else fixed += st[a].idx[pos[a]] * stride[a];
      }
      double interp = 0.0;
      for (uint64_t corner = 0; corner < (1ull << n_new); ++corner) {
        double w = 1.0;
        uint64_t off = fixed;
        for (int k = 0; k < n_new; ++k) {
          const int a = new_axes[k];
          const uint64_t q = pos[a];
          if ((corner >> k) & 1u) { w *= st[a].wr[q]; off += st[a].right[q] * stride[a]; }
          else { w *= st[a].wl[q]; off += st[a].left[q] * stride[a]; }
        }
        interp += w * values[off];
      }
      values[base + in->idx[p] * stride[d - 1]] += sign * interp;
    }
  }
  for (int a = 0; a < d; ++a) free_stencil(&st[a]);
}

/* transform.cpp:149-159 */
static void forward_inplace(double* v, const hier_t* h) {
  for (int l = h->L; l >= 1; --l) apply_level(v, h, l, -1.0);
}
static void inverse_inplace(double* v, const hier_t* h) {
  for (int l = 1; l <= h->L; ++l) apply_level(v, h, l, +1.0);
}

/* ------------------------------------------------------------------------ */
/* deterministic reductions (exec.cpp:47-128): 4096-element blocks reduced   */
/* serially, partials combined serially                                     */

#define RBLOCK 4096

static double max_abs(const double* v, uint64_t n) {
  double acc = 0.0;
  for (uint64_t lo = 0; lo < n; lo += RBLOCK) {
    uint64_t hi = lo + RBLOCK < n ? lo + RBLOCK : n;
    double m = 0.0;
    for (uint64_t i = lo; i < hi; ++i) { double a = fabs(v[i]); if (a > m) m = a; }
    acc = acc > m ? acc : m;
  }
  return acc;
}

static void minmax(const double* v, uint64_t n, double* mn, double* mx) {
  double amin = n ? v[0] : 0.0, amax = n ? v[0] : 0.0;
  for (uint64_t lo = 0; lo < n; lo += RBLOCK) {
    uint64_t hi = lo + RBLOCK < n ? lo + RBLOCK : n;
    double bmin = v[lo], bmax = v[lo];
    for (uint64_t i = lo; i < hi; ++i) { if (v[i] < bmin) bmin = v[i]; if (v[i] > bmax) bmax = v[i]; }
    amin = amin < bmin ? amin : bmin;
    amax = amax > bmax ? amax : bmax;
  }
  *mn = amin;
  *mx = amax;
}

static double sum_squares(const double* v, uint64_t n) {
  double acc = 0.0;
  for (uint64_t lo = 0; lo < n; lo += RBLOCK) {
    uint64_t hi = lo + RBLOCK < n ? lo + RBLOCK : n;
    double s = 0.0;
    for (uint64_t i = lo; i < hi; ++i) s += v[i] * v[i];
    acc = acc + s;
  }
  return acc;
}

static int any_non_finite(const double* v, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) if (!isfinite(v[i])) return 1;
  return 0;
}

/* ------------------------------------------------------------------------ */
/* quantize (quantize.cpp)                                                  */

/* quantize.cpp:14-23 */
double oc_round_half_even(double x) {
  if (!(fabs(x) < 4503599627370496.0)) return x;
  const double f = floor(x);
  const double frac = x - f;
  if (frac > 0.5) return f + 1.0;
  if (frac < 0.5) return f;
  return fmod(f, 2.0) == 0.0 ? f : f + 1.0;
}

/* per-node tag for flat index (quantize.cpp:30-68 walks rows; same tag) */
static void flat_tags(const hier_t* h, uint8_t* tags) {
  const int d = h->g.d;
  uint64_t idx[MAXD] = {0, 0, 0, 0};
  const uint64_t n = grid_count(&h->g);
  for (uint64_t f = 0; f < n; ++f) {
    tags[f] = (uint8_t)level_tag(h, idx);
    for (int a = d; a-- > 0;) {
      if (++idx[a] < h->g.shape[a]) break;
      idx[a] = 0;
    }
  }
}

/* quantize.cpp:72-132 */
static int quantize(const hier_t* h, const double* c, const double* widths, int64_t* q, double* res, uint64_t* outliers) {
  const uint64_t n = grid_count(&h->g);
  for (int l = 0; l <= h->L; ++l)
    if (!(widths[l] > 0.0)) return fail(OC_INVALID_STATE, "InvalidState: bin widths must be > 0");
  uint8_t* tags = (uint8_t*)malloc(n);
  flat_tags(h, tags);
  const double limit = 9223372036854775808.0;
  uint64_t overflow = 0, outl = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const double delta = widths[tags[i]];
    const double scaled = c[i] / delta;
    if (!(fabs(scaled) < limit)) { ++overflow; continue; }
    const int64_t qq = (int64_t)oc_round_half_even(scaled);
    q[i] = qq;
    res[i] = c[i] - (double)qq * delta;
    if (qq > 2147483647LL || qq < -2147483648LL) ++outl;
  }
  free(tags);
  if (outliers) *outliers = outl;
  if (overflow) return fail(OC_OVERFLOW, "Overflow: %llu coefficients exceed the 63-bit symbol range", (unsigned long long)overflow);
  return 0;
}

/* quantize.cpp:134-158 */
static void dequantize(const hier_t* h, const int64_t* q, const double* widths, double* c) {
  const uint64_t n = grid_count(&h->g);
  uint8_t* tags = (uint8_t*)malloc(n);
  flat_tags(h, tags);
  for (uint64_t i = 0; i < n; ++i) c[i] = (double)q[i] * widths[tags[i]];
  free(tags);
}

/* ------------------------------------------------------------------------ */
/* error control (error_control.cpp)                                        */

/* error_control.cpp:25-40 */
static int absolute_tolerance(const double* u, uint64_t n, double tol, int norm, int mode, double* out) {
  if (!(tol > 0.0)) return fail(OC_INVALID_STATE, "InvalidState: tolerance must be > 0");
  if (n == 0) return fail(OC_SHAPE_MISMATCH, "ShapeMismatch: empty array");
  if (mode == 0) { *out = tol; return 0; }
  if (norm == 0) {
    double mn, mx;
    minmax(u, n, &mn, &mx);
    const double range = mx - mn;
    if (range == 0.0) return fail(OC_DEGENERATE_DATA, "DegenerateData: relative bound on a constant field");
    *out = tol * range;
    return 0;
  }
  const double r = sqrt(sum_squares(u, n) / (double)n);
  if (r == 0.0) return fail(OC_DEGENERATE_DATA, "DegenerateData: relative bound on a zero field");
  *out = tol * r;
  return 0;
}

/* error_control.cpp:42-60 */
static int bin_widths(double tau, int norm, double s, int d, int L, double* w) {
  if (!(tau > 0.0)) return fail(OC_INVALID_STATE, "InvalidState: absolute tolerance must be > 0");
  const double Ld = (double)L;
  const double cells = ldexp(1.0, d);
  if (norm == 0) {
    const double delta = 2.0 * tau / (1.0 + Ld * cells);
    for (int l = 0; l <= L; ++l) w[l] = delta;
  } else {
    const double base = 2.0 * tau / sqrt((Ld + 1.0) * cells);
    for (int l = 0; l <= L; ++l) w[l] = base * exp2(s * (Ld - (double)l));
  }
  return 0;
}

/* error_control.cpp:62-108 */
static double achieved_error(const hier_t* h, const double* res, int norm, double s) {
  const uint64_t n = grid_count(&h->g);
  if (norm == 1 && s != 0.0) {
    double level_sumsq[MAXL + 1];
    memset(level_sumsq, 0, sizeof level_sumsq);
    uint64_t idx[MAXD] = {0, 0, 0, 0};
    for (uint64_t f = 0; f < n; ++f) {
      const int tag = level_tag(h, idx);
      level_sumsq[tag] += res[f] * res[f];
      for (int a = h->g.d; a-- > 0;) {
        if (++idx[a] < h->g.shape[a]) break;
        idx[a] = 0;
      }
    }
    double acc = 0.0;
    const double L = (double)h->L;
    for (int l = 0; l <= h->L; ++l) acc += exp2(2.0 * s * ((double)l - L)) * level_sumsq[l];
    return sqrt(acc / (double)n);
  }
  double* e = (double*)malloc(n * 8);
  memcpy(e, res, n * 8);
  if (h->L > 0) inverse_inplace(e, h);
  double v = norm == 0 ? max_abs(e, n) : sqrt(sum_squares(e, n) / (double)n);
  free(e);
  return v;
}

/* ------------------------------------------------------------------------ */
/* lossless codec (codec.cpp)                                               */

/* codec.cpp:14-28 */
uint32_t oc_crc32(const uint8_t* data, uint64_t n) {
  static uint32_t table[256];
  static int init = 0;
  if (!init) {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1u) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      table[i] = c;
    }
    init = 1;
  }
  uint32_t c = 0xFFFFFFFFu;
  for (uint64_t i = 0; i < n; ++i) c = table[(c ^ data[i]) & 0xFFu] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

#define MAX_CODE_LEN 15
#define KRAFT_ONE (1u << MAX_CODE_LEN)

/* codec.cpp:35-50 */
static uint64_t zigzag(int64_t v) { return ((uint64_t)v << 1) ^ (uint64_t)(v >> 63); }
static int64_t unzigzag(uint64_t u) { return (int64_t)(u >> 1) ^ -(int64_t)(u & 1u); }
static void put_varint(buf_t* b, uint64_t u) {
  while (u >= 0x80u) { bput(b, (uint8_t)u | 0x80u); u >>= 7; }
  bput(b, (uint8_t)u);
}

/* codec.cpp:100-192: deterministic Huffman lengths + 15-bit Kraft repair.
 * The reference's priority queue pops the minimum (freq, key); keys are
 * unique so a linear scan for the two minima is the same schedule. */
static int build_lengths(const uint64_t* freq, uint8_t* lengths) {
  memset(lengths, 0, 256);
  int symbols[256], ns = 0;
  for (int s = 0; s < 256; ++s) if (freq[s] > 0) symbols[ns++] = s;
  if (ns == 0) return 0;
  if (ns == 1) { lengths[symbols[0]] = 1; return 0; }
  uint64_t nf[512];
  int nkey[512], nleft[512], nright[512], alive[512];
  int nn = 0;
  for (int i = 0; i < ns; ++i) {
    nf[nn] = freq[symbols[i]]; nkey[nn] = symbols[i]; nleft[nn] = nright[nn] = -1; alive[nn] = 1; ++nn;
  }
  int next_key = 256, live = ns;
  while (live > 1) {
    int pick[2];
    for (int t = 0; t < 2; ++t) {
      int best = -1;
      for (int i = 0; i < nn; ++i) {
        if (!alive[i]) continue;
        if (best < 0 || nf[i] < nf[best] || (nf[i] == nf[best] && nkey[i] < nkey[best])) best = i;
      }
      alive[best] = 0;
      pick[t] = best;
    }
    nf[nn] = nf[pick[0]] + nf[pick[1]]; nkey[nn] = next_key++; nleft[nn] = pick[0]; nright[nn] = pick[1]; alive[nn] = 1; ++nn;
    --live;
  }
  /* depth-first depth assignment (codec.cpp:143-155) */
  int stack_n[512], stack_d[512], sp = 0;
  stack_n[sp] = nn - 1; stack_d[sp] = 0; ++sp;
  while (sp > 0) {
    --sp;
    const int n = stack_n[sp], depth = stack_d[sp];
    if (nleft[n] < 0) { lengths[nkey[n]] = (uint8_t)(depth > 255 ? 255 : depth); continue; }
    stack_n[sp] = nleft[n]; stack_d[sp] = depth + 1; ++sp;
    stack_n[sp] = nright[n]; stack_d[sp] = depth + 1; ++sp;
  }
  /* clamp, then restore Kraft equality (codec.cpp:157-190) */
  uint64_t kraft = 0;
  for (int i = 0; i < ns; ++i) {
    uint8_t* len = &lengths[symbols[i]];
    if (*len > MAX_CODE_LEN) *len = MAX_CODE_LEN;
    kraft += KRAFT_ONE >> *len;
  }
  while (kraft > KRAFT_ONE) {
    int pick = -1;
    for (int i = 0; i < ns; ++i) {
      const int s = symbols[i], len = lengths[s];
      if (len < MAX_CODE_LEN && (pick < 0 || len > lengths[pick] || (len == lengths[pick] && s > pick))) pick = s;
    }
    kraft -= KRAFT_ONE >> (lengths[pick] + 1);
    ++lengths[pick];
  }
  while (kraft < KRAFT_ONE) {
    int pick = -1;
    for (int i = 0; i < ns; ++i) {
      const int s = symbols[i], len = lengths[s];
      if (len > 1 && kraft + (KRAFT_ONE >> len) <= KRAFT_ONE && (pick < 0 || len > lengths[pick])) pick = s;
    }
    if (pick < 0) return fail(OC_CORRUPT_STREAM, "CorruptStream: internal: kraft repair failed");
    kraft += KRAFT_ONE >> lengths[pick];
    --lengths[pick];
  }
  return 0;
}

/* codec.cpp:195-220 */
static void canonical_codes(const uint8_t* lengths, uint32_t* codes, int* max_len, int* nsym) {
  uint16_t bl_count[MAX_CODE_LEN + 1] = {0};
  *max_len = 0;
  *nsym = 0;
  for (int s = 0; s < 256; ++s)
    if (lengths[s]) { ++bl_count[lengths[s]]; ++*nsym; if (lengths[s] > *max_len) *max_len = lengths[s]; }
  uint32_t next_code[MAX_CODE_LEN + 2] = {0};
  uint32_t code = 0;
  for (int len = 1; len <= *max_len; ++len) {
    code = (code + bl_count[len - 1]) << 1;
    next_code[len] = code;
  }
  for (int s = 0; s < 256; ++s) codes[s] = lengths[s] ? next_code[lengths[s]]++ : 0;
}

/* codec.cpp:399-418 */
static int huffman_pack(const uint8_t* in, uint64_t n, buf_t* out) {
  uint64_t freq[256] = {0};
  for (uint64_t i = 0; i < n; ++i) ++freq[in[i]];
  uint8_t lengths[256];
  int rc = build_lengths(freq, lengths);
  if (rc) return rc;
  uint32_t codes[256];
  int max_len, nsym;
  canonical_codes(lengths, codes, &max_len, &nsym);
  if (nsym == 0) { put_u16(out, 0); bput(out, 0); return 0; }
  put_u16(out, (uint16_t)nsym); /* codec.cpp:310-317 */
  bput(out, (uint8_t)max_len);
  for (int s = 0; s < 256; s += 2) bput(out, (uint8_t)((lengths[s] & 0x0Fu) | (lengths[s + 1] << 4)));
  if (nsym == 1) return 0;
  /* MSB-first BitWriter (codec.cpp:222-247) */
  uint8_t acc = 0;
  int nbits = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const uint32_t code = codes[in[i]];
    for (int b = lengths[in[i]] - 1; b >= 0; --b) {
      acc = (uint8_t)((acc << 1) | ((code >> b) & 1u));
      if (++nbits == 8) { bput(out, acc); acc = 0; nbits = 0; }
    }
  }
  if (nbits > 0) bput(out, (uint8_t)(acc << (8 - nbits)));
  return 0;
}

/* byte sources for the varint reader (codec.cpp:54-74, :354-395) */
typedef struct {
  int huffman;
  const uint8_t* bits;
  uint64_t nbytes;
  uint64_t byte_pos;
  int bit_pos;
  int nsym;
  /* canonical decoder tables (codec.cpp:251-308) */
  uint8_t sorted_sym[256];
  uint32_t first_code[MAX_CODE_LEN + 1];
  uint32_t first_index[MAX_CODE_LEN + 1];
  uint32_t count[MAX_CODE_LEN + 1];
  int max_len;
} src_t;

static int src_next(src_t* s, uint8_t* out) {
  if (!s->huffman) {
    if (s->byte_pos >= s->nbytes) return fail(OC_CORRUPT_STREAM, "CorruptStream: truncated varint stream");
    *out = s->bits[s->byte_pos++];
    return 0;
  }
  if (s->nsym == 0) return fail(OC_CORRUPT_STREAM, "CorruptStream: read past empty Huffman stream");
  if (s->nsym == 1) { *out = s->sorted_sym[0]; return 0; }
  uint32_t code = 0;
  for (int len = 1; len <= s->max_len; ++len) {
    if (s->byte_pos >= s->nbytes) return fail(OC_CORRUPT_STREAM, "CorruptStream: Huffman stream truncated");
    const uint32_t bit = (s->bits[s->byte_pos] >> (7 - s->bit_pos)) & 1u;
    if (++s->bit_pos == 8) { s->bit_pos = 0; ++s->byte_pos; }
    code = (code << 1) | bit;
    if (s->count[len] != 0 && code - s->first_code[len] < s->count[len]) {
      *out = s->sorted_sym[s->first_index[len] + (code - s->first_code[len])];
      return 0;
    }
  }
  return fail(OC_CORRUPT_STREAM, "CorruptStream: invalid Huffman code");
}

static int src_exhausted_clean(const src_t* s) {
  if (!s->huffman) return s->byte_pos == s->nbytes;
  if (s->bit_pos == 0) return s->byte_pos == s->nbytes;
  if (s->byte_pos + 1 != s->nbytes) return 0;
  return (uint8_t)(s->bits[s->byte_pos] << s->bit_pos) == 0;
}

/* codec.cpp:325-352 + HuffmanDecoder ctor :253-285 */
static int huffman_source(src_t* s, const uint8_t* packed, uint64_t n) {
  memset(s, 0, sizeof *s);
  s->huffman = 1;
  rd_t r = {packed, n, 0, 0};
  s->nsym = get_u16(&r);
  if (s->nsym == 0) {
    if (get_u8(&r) != 0 || r.bad) return fail(OC_CORRUPT_STREAM, "CorruptStream: nonzero max length for empty table");
  } else {
    const int max_len = get_u8(&r);
    if (r.bad) return fail(OC_CORRUPT_STREAM, "CorruptStream: truncated stream");
    if (max_len == 0 || max_len > MAX_CODE_LEN) return fail(OC_CORRUPT_STREAM, "CorruptStream: Huffman max code length out of range");
    uint8_t lengths[256];
    int nonzero = 0, observed = 0;
    for (int sy = 0; sy < 256; sy += 2) {
      const uint8_t b = get_u8(&r);
      lengths[sy] = b & 0x0F;
      lengths[sy + 1] = b >> 4;
      if (lengths[sy]) { ++nonzero; if (lengths[sy] > observed) observed = lengths[sy]; }
      if (lengths[sy + 1]) { ++nonzero; if (lengths[sy + 1] > observed) observed = lengths[sy + 1]; }
    }
    if (r.bad) return fail(OC_CORRUPT_STREAM, "CorruptStream: truncated stream");
    if (nonzero != s->nsym) return fail(OC_CORRUPT_STREAM, "CorruptStream: Huffman symbol count mismatch");
    if (observed != max_len) return fail(OC_CORRUPT_STREAM, "CorruptStream: Huffman max code length mismatch");
    /* sorted (len, symbol) */
    int k = 0;
    uint16_t bl_count[MAX_CODE_LEN + 1] = {0};
    for (int len = 1; len <= MAX_CODE_LEN; ++len)
      for (int sy = 0; sy < 256; ++sy)
        if (lengths[sy] == len) { s->sorted_sym[k++] = (uint8_t)sy; ++bl_count[len]; }
    uint64_t kraft = 0;
    for (int sy = 0; sy < 256; ++sy) if (lengths[sy]) kraft += KRAFT_ONE >> lengths[sy];
    if (k >= 2 && kraft != KRAFT_ONE) return fail(OC_CORRUPT_STREAM, "CorruptStream: Huffman table violates Kraft equality");
    if (k == 1) {
      int len1 = 0;
      for (int sy = 0; sy < 256; ++sy) if (lengths[sy]) len1 = lengths[sy];
      if (len1 != 1) return fail(OC_CORRUPT_STREAM, "CorruptStream: degenerate Huffman table");
    }
    s->max_len = max_len;
    uint32_t code = 0, index = 0;
    for (int len = 1; len <= max_len; ++len) {
      code <<= 1;
      s->first_code[len] = code;
      s->first_index[len] = index;
      s->count[len] = bl_count[len];
      code += bl_count[len];
      index += bl_count[len];
    }
  }
  s->bits = packed + r.pos;
  s->nbytes = n - r.pos;
  return 0;
}

/* codec.cpp:76-86 */
static int read_varint(src_t* s, uint64_t* out) {
  uint64_t v = 0;
  for (int shift = 0; shift < 64; shift += 7) {
    uint8_t b;
    int rc = src_next(s, &b);
    if (rc) return rc;
    if (shift == 63 && (b & 0xFEu)) return fail(OC_CORRUPT_STREAM, "CorruptStream: varint overflows 64 bits");
    v |= (uint64_t)(b & 0x7Fu) << shift;
    if ((b & 0x80u) == 0) { *out = v; return 0; }
  }
  return fail(OC_CORRUPT_STREAM, "CorruptStream: varint continuation too long");
}

/* codec.cpp:431-453 */
static int lossless_encode(const int64_t* v, uint64_t n, int codec, buf_t* out) {
  if (codec == 0) {
    for (uint64_t i = 0; i < n; ++i) put_u64(out, (uint64_t)v[i]);
    return 0;
  }
  if (codec == 1) {
    for (uint64_t i = 0; i < n; ++i) put_varint(out, zigzag(v[i]));
    return 0;
  }
  if (codec == 2) {
    buf_t vb = {0};
    for (uint64_t i = 0; i < n; ++i) put_varint(&vb, zigzag(v[i]));
    int rc = huffman_pack(vb.p, vb.n, out);
    free(vb.p);
    return rc;
  }
  return fail(OC_UNKNOWN_CODEC, "UnknownCodec: codec %d", codec);
}

/* codec.cpp:455-485 */
static int lossless_decode(const uint8_t* p, uint64_t len, uint64_t count, int codec, int64_t* out) {
  if (codec == 0) {
    if (len != count * 8) return fail(OC_CORRUPT_STREAM, "CorruptStream: raw payload length mismatch");
    rd_t r = {p, len, 0, 0};
    for (uint64_t i = 0; i < count; ++i) out[i] = (int64_t)get_u64(&r);
    return 0;
  }
  src_t s;
  if (codec == 1) {
    memset(&s, 0, sizeof s);
    s.bits = p;
    s.nbytes = len;
  } else if (codec == 2) {
    int rc = huffman_source(&s, p, len);
    if (rc) return rc;
  } else {
    return fail(OC_UNKNOWN_CODEC, "UnknownCodec: codec %d", codec);
  }
  for (uint64_t i = 0; i < count; ++i) {
    uint64_t u = 0;
    int rc = read_varint(&s, &u);
    if (rc) return rc;
    out[i] = unzigzag(u);
  }
  if (!src_exhausted_clean(&s))
    return fail(OC_CORRUPT_STREAM, codec == 1 ? "CorruptStream: trailing bytes after varint stream" : "CorruptStream: trailing bits after Huffman stream");
  return 0;
}

/* ------------------------------------------------------------------------ */
/* container (container.cpp)                                                */

static const char MAGIC[4] = {'M', 'G', 'R', 'C'};
#define SHRINK_PASSES 10
#define BOUND_SLACK (1.0 - 1e-9)

/* container.cpp:28-55 */
static void append_header(buf_t* out, const grid_t* g, int dtype, int constant, double tol, int norm, double s, int mode,
                          const double* widths, int nw, int codec, uint64_t payload_len, uint32_t crc) {
  put_bytes(out, (const uint8_t*)MAGIC, 4);
  put_u16(out, 1);
  uint8_t flags = 0;
  if (constant) flags |= 1u;
  if (g->explicit_coords) flags |= 2u;
  bput(out, flags);
  bput(out, (uint8_t)dtype);
  bput(out, (uint8_t)g->d);
  for (int a = 0; a < g->d; ++a) put_u64(out, g->shape[a]);
  if (g->explicit_coords)
    for (int a = 0; a < g->d; ++a) {
      put_u64(out, g->shape[a]);
      for (uint64_t i = 0; i < g->shape[a]; ++i) put_f64(out, g->coords[a][i]);
    }
  bput(out, (uint8_t)mode);
  bput(out, (uint8_t)norm);
  put_f64(out, norm == 1 ? s : 0.0);
  put_f64(out, tol);
  bput(out, (uint8_t)(nw - 1));
  for (int l = 0; l < nw; ++l) put_f64(out, widths[l]);
  bput(out, (uint8_t)codec);
  put_u64(out, payload_len);
  put_u32(out, crc);
}

/* container.cpp:71-131 (+ f32 wrapper :197-203, constant :57-69) */
static int compress_f64(const double* u, const grid_t* g, double tol, int norm, double s, int mode, int codec, int dtype,
                        const float* f32src, buf_t* out) {
  const uint64_t n = grid_count(g);
  if (any_non_finite(u, n)) return fail(OC_NON_FINITE_INPUT, "NonFiniteInput: input contains NaN or Inf");
  if (!(tol > 0.0)) return fail(OC_INVALID_STATE, "InvalidState: tolerance must be > 0");
  double mn, mx;
  minmax(u, n, &mn, &mx);
  if (mx == mn) {
    buf_t pl = {0};
    put_f64(&pl, mx);
    const double dummy = 0.0;
    append_header(out, g, dtype, 1, tol, norm, s, mode, &dummy, 1, codec, pl.n, oc_crc32(pl.p, pl.n));
    put_bytes(out, pl.p, pl.n);
    free(pl.p);
    return 0;
  }
  double tau = 0.0;
  int rc = absolute_tolerance(u, n, tol, norm, mode, &tau);
  if (rc) return rc;
  hier_t h;
  build_hierarchy(&h, g);
  double* c = (double*)malloc(n * 8);
  memcpy(c, u, n * 8);
  if (h.L > 0) forward_inplace(c, &h);
  double widths[MAXL + 1];
  bin_widths(tau, norm, s, g->d, h.L, widths);
  int64_t* q = (int64_t*)malloc(n * 8);
  double* res = (double*)malloc(n * 8);
  int accepted = 0;
  for (int pass = 0; pass < SHRINK_PASSES && !rc; ++pass) {
    rc = quantize(&h, c, widths, q, res, NULL);
    if (rc) break;
    double achieved;
    if (dtype == 0 && !(norm == 1 && s != 0.0)) {
      double* e = (double*)malloc(n * 8);
      memcpy(e, res, n * 8);
      if (h.L > 0) inverse_inplace(e, &h);
      for (uint64_t i = 0; i < n; ++i) e[i] = (double)f32src[i] - (double)(float)(u[i] - e[i]);
      achieved = norm == 0 ? max_abs(e, n) : sqrt(sum_squares(e, n) / (double)n);
      free(e);
    } else {
      achieved = achieved_error(&h, res, norm, s);
    }
    if (achieved <= tau * BOUND_SLACK) { accepted = 1; break; }
    for (int l = 0; l <= h.L; ++l) widths[l] *= 0.5;
  }
  if (!rc && !accepted) rc = fail(OC_TOLERANCE_UNREACHABLE, "ToleranceUnreachable: bin shrink loop exhausted after 10 passes");
  if (!rc) {
    buf_t pl = {0};
    rc = lossless_encode(q, n, codec, &pl);
    if (!rc) {
      append_header(out, g, dtype, 0, tol, norm, s, mode, widths, h.L + 1, codec, pl.n, oc_crc32(pl.p, pl.n));
      put_bytes(out, pl.p, pl.n);
    }
    free(pl.p);
  }
  free(c); free(q); free(res);
  hier_free(&h);
  return rc;
}

int oc_compress(const void* data, int dtype, int ndims, const uint64_t* shape, const double* coords, double tol, int norm,
                double s, int mode, int codec, uint8_t** out, uint64_t* out_len) {
  grid_t g;
  int rc = make_grid(&g, ndims, shape, coords);
  if (rc) return rc;
  const uint64_t n = grid_count(&g);
  buf_t ob = {0};
  if (dtype == 0) {
    const float* f = (const float*)data;
    double* w = (double*)malloc(n * 8);
    for (uint64_t i = 0; i < n; ++i) w[i] = (double)f[i];
    rc = compress_f64(w, &g, tol, norm, s, mode, codec, 0, f, &ob);
    free(w);
  } else {
    rc = compress_f64((const double*)data, &g, tol, norm, s, mode, codec, 1, NULL, &ob);
  }
  grid_free(&g);
  if (rc) { free(ob.p); return rc; }
  *out = ob.p;
  *out_len = ob.n;
  return 0;
}

/* ContainerInfo (container.hpp:37-51) flattened for the C API */
typedef struct {
  uint16_t version;
  uint8_t constant_field, coords_present, dtype, ndims, nlevels, codec_id;
  uint64_t shape[MAXD];
  uint8_t mode, norm;
  double smoothness, tol;
  double bin_widths[MAXL + 1];
  uint64_t payload_len;
  uint32_t checksum;
  uint64_t header_size;
} oc_info;

/* container.cpp:133-188; coords (if present) returned through *coords */
static int parse_header(rd_t* r, oc_info* info, double** coords) {
  memset(info, 0, sizeof *info);
  if (coords) *coords = NULL;
  const uint8_t* m = take(r, 4);
  if (!m) return fail(OC_CORRUPT_STREAM, "CorruptStream: truncated stream");
  if (memcmp(m, MAGIC, 4) != 0) return fail(OC_BAD_MAGIC, "BadMagic: not an MGRC container");
#define CHK() do { if (r->bad) { if (coords) { free(*coords); *coords = NULL; } return fail(OC_CORRUPT_STREAM, "CorruptStream: truncated stream"); } } while (0)
  info->version = get_u16(r); CHK();
  if (info->version != 1) return fail(OC_UNSUPPORTED_VERSION, "UnsupportedVersion: container version %u", info->version);
  const uint8_t flags = get_u8(r); CHK();
  if (flags & ~0x03u) return fail(OC_CORRUPT_STREAM, "CorruptStream: unknown header flags");
  info->constant_field = (flags & 1u) != 0;
  info->coords_present = (flags & 2u) != 0;
  const uint8_t dt = get_u8(r); CHK();
  if (dt > 1) return fail(OC_CORRUPT_STREAM, "CorruptStream: unknown element type");
  info->dtype = dt;
  const uint8_t nd = get_u8(r); CHK();
  if (nd < 1 || nd > MAXD) return fail(OC_CORRUPT_STREAM, "CorruptStream: dimension count out of range");
  info->ndims = nd;
  uint64_t count = 1;
  uint64_t total_axes = 0;
  for (int a = 0; a < nd; ++a) {
    const uint64_t sz = get_u64(r); CHK();
    if (sz < 2) return fail(OC_CORRUPT_STREAM, "CorruptStream: axis shorter than 2 nodes");
    if (sz > (1ull << 40) / count) return fail(OC_CORRUPT_STREAM, "CorruptStream: implausible shape");
    count *= sz;
    info->shape[a] = sz;
    total_axes += sz;
  }
  if (info->coords_present) {
    double* cs = (double*)malloc(total_axes * 8);
    if (coords) *coords = cs;
    uint64_t off = 0;
    for (int a = 0; a < nd; ++a) {
      const uint64_t k = get_u64(r);
      if (r->bad) { free(cs); if (coords) *coords = NULL; return fail(OC_CORRUPT_STREAM, "CorruptStream: truncated stream"); }
      if (k != info->shape[a]) { free(cs); if (coords) *coords = NULL; return fail(OC_CORRUPT_STREAM, "CorruptStream: coordinate count mismatch"); }
      for (uint64_t i = 0; i < k; ++i) cs[off + i] = get_f64(r);
      off += k;
    }
    if (!coords) free(cs);
    if (r->bad) { if (coords) { free(*coords); *coords = NULL; } return fail(OC_CORRUPT_STREAM, "CorruptStream: truncated stream"); }
  }
  const uint8_t mode = get_u8(r); CHK();
  if (mode > 1) { if (coords) { free(*coords); *coords = NULL; } return fail(OC_CORRUPT_STREAM, "CorruptStream: unknown error-bound mode"); }
  info->mode = mode;
  const uint8_t norm = get_u8(r); CHK();
  if (norm > 1) { if (coords) { free(*coords); *coords = NULL; } return fail(OC_CORRUPT_STREAM, "CorruptStream: unknown norm"); }
  info->norm = norm;
  info->smoothness = get_f64(r);
  info->tol = get_f64(r);
  info->nlevels = get_u8(r); CHK();
  for (int l = 0; l <= info->nlevels; ++l) info->bin_widths[l] = get_f64(r);
  info->codec_id = get_u8(r); CHK();
  if (info->codec_id > 2) { if (coords) { free(*coords); *coords = NULL; } return fail(OC_CORRUPT_STREAM, "CorruptStream: unknown codec id"); }
  info->payload_len = get_u64(r);
  info->checksum = get_u32(r); CHK();
  info->header_size = r->pos;
#undef CHK
  return 0;
}

int oc_inspect(const uint8_t* in, uint64_t len, oc_info* info) {
  rd_t r = {in, len, 0, 0};
  return parse_header(&r, info, NULL);
}

/* container.cpp:210-261 */
int oc_decompress(const uint8_t* in, uint64_t len, void** out, int* dtype, int* ndims, uint64_t* shape) {
  rd_t r = {in, len, 0, 0};
  oc_info info;
  double* coords = NULL;
  int rc = parse_header(&r, &info, &coords);
  if (rc) return rc;
  if (info.payload_len != len - r.pos) { free(coords); return fail(OC_CORRUPT_STREAM, "CorruptStream: payload length mismatch"); }
  const uint8_t* payload = in + r.pos;
  if (oc_crc32(payload, info.payload_len) != info.checksum) { free(coords); return fail(OC_CHECKSUM_MISMATCH, "ChecksumMismatch: payload checksum failed"); }
  uint64_t count = 1;
  for (int a = 0; a < info.ndims; ++a) count *= info.shape[a];
  double* values = (double*)malloc(count * 8);
  if (info.constant_field) {
    if (info.payload_len != 8) { free(coords); free(values); return fail(OC_CORRUPT_STREAM, "CorruptStream: constant payload must be 8 bytes"); }
    rd_t p = {payload, 8, 0, 0};
    const double v = get_f64(&p);
    for (uint64_t i = 0; i < count; ++i) values[i] = v;
  } else {
    grid_t g;
    rc = make_grid(&g, info.ndims, info.shape, info.coords_present ? coords : NULL);
    if (rc) { free(coords); free(values); return rc; }
    hier_t h;
    build_hierarchy(&h, &g);
    if (info.nlevels != h.L) { hier_free(&h); grid_free(&g); free(coords); free(values); return fail(OC_CORRUPT_STREAM, "CorruptStream: level count does not match the shape"); }
    int64_t* q = (int64_t*)malloc(count * 8);
    rc = lossless_decode(payload, info.payload_len, count, info.codec_id, q);
    if (!rc) {
      dequantize(&h, q, info.bin_widths, values);
      if (h.L > 0) inverse_inplace(values, &h);
    }
    free(q);
    hier_free(&h);
    grid_free(&g);
    if (rc) { free(coords); free(values); return rc; }
  }
  free(coords);
  *dtype = info.dtype;
  *ndims = info.ndims;
  for (int a = 0; a < info.ndims; ++a) shape[a] = info.shape[a];
  if (info.dtype == 0) {
    float* f = (float*)malloc(count * 4);
    for (uint64_t i = 0; i < count; ++i) f[i] = (float)values[i];
    free(values);
    *out = f;
  } else {
    *out = values;
  }
  return 0;
}

/* container.cpp:263-299 */
int oc_describe(const uint8_t* in, uint64_t len, char** text) {
  oc_info info;
  int rc = oc_inspect(in, len, &info);
  if (rc) return rc;
  char* s = (char*)malloc(4096 + 32 * (MAXL + 1));
  int k = 0;
  k += sprintf(s + k, "format: mgrc-container\nversion: %u\nconstant_field: %d\ncoords_present: %d\ndtype: %s\nndims: %d\nshape: ",
               info.version, info.constant_field, info.coords_present, info.dtype == 0 ? "f32" : "f64", info.ndims);
  for (int a = 0; a < info.ndims; ++a) k += sprintf(s + k, a ? "x%llu" : "%llu", (unsigned long long)info.shape[a]);
  k += sprintf(s + k, "\nmode: %s\nnorm: %s\ns: %.17g\ntol: %.17g\nnlevels: %d\nbin_widths: ", info.mode == 0 ? "abs" : "rel",
               info.norm == 0 ? "inf" : "s", info.smoothness, info.tol, info.nlevels);
  for (int l = 0; l <= info.nlevels; ++l) k += sprintf(s + k, l ? ",%.17g" : "%.17g", info.bin_widths[l]);
  k += sprintf(s + k, "\ncodec: %d\nheader_bytes: %llu\npayload_bytes: %llu\ncrc32: %u\n", info.codec_id,
               (unsigned long long)info.header_size, (unsigned long long)info.payload_len, info.checksum);
  *text = s;
  return 0;
}

/* ------------------------------------------------------------------------ */
/* component-level entry points used by the parity tests                    */

static int with_hier(int ndims, const uint64_t* shape, const double* coords, grid_t* g, hier_t* h) {
  int rc = make_grid(g, ndims, shape, coords);
  if (rc) return rc;
  build_hierarchy(h, g);
  return 0;
}

/* hierarchy summary: nlevels, axis_level (concatenated), level node counts,
 * level sizes [(L+1) x ndims] */
int oc_hierarchy(int ndims, const uint64_t* shape, const double* coords, int* nlevels, uint8_t* axis_level,
                 uint64_t* node_counts, uint64_t* level_sizes, int cap_levels) {
  grid_t g;
  hier_t h;
  int rc = with_hier(ndims, shape, coords, &g, &h);
  if (rc) return rc;
  *nlevels = h.L;
  uint64_t off = 0;
  for (int a = 0; a < ndims; ++a) {
    if (axis_level) memcpy(axis_level + off, h.axis_level[a], shape[a]);
    off += shape[a];
  }
  for (int l = 0; l <= h.L && l < cap_levels; ++l) {
    if (node_counts) node_counts[l] = h.node_counts[l];
    if (level_sizes) for (int a = 0; a < ndims; ++a) level_sizes[l * ndims + a] = h.set_n[l][a];
  }
  hier_free(&h);
  grid_free(&g);
  return 0;
}

int oc_level_set(int ndims, const uint64_t* shape, int level, int axis, uint64_t* out, uint64_t* n) {
  grid_t g;
  hier_t h;
  int rc = with_hier(ndims, shape, NULL, &g, &h);
  if (rc) return rc;
  if (level < 0 || level > h.L) { hier_free(&h); grid_free(&g); return fail(OC_LEVEL_OUT_OF_RANGE, "LevelOutOfRange: level %d of %d", level, h.L); }
  *n = h.set_n[level][axis];
  if (out) memcpy(out, h.sets[level][axis], *n * 8);
  hier_free(&h);
  grid_free(&g);
  return 0;
}

int oc_forward(int ndims, const uint64_t* shape, const double* coords, const double* u, double* c) {
  grid_t g;
  hier_t h;
  int rc = with_hier(ndims, shape, coords, &g, &h);
  if (rc) return rc;
  const uint64_t n = grid_count(&g);
  if (any_non_finite(u, n)) { hier_free(&h); grid_free(&g); return fail(OC_NON_FINITE_INPUT, "NonFiniteInput: input contains NaN or Inf"); }
  memcpy(c, u, n * 8);
  if (h.L > 0) forward_inplace(c, &h);
  hier_free(&h);
  grid_free(&g);
  return 0;
}

int oc_inverse(int ndims, const uint64_t* shape, const double* coords, const double* c, double* u) {
  grid_t g;
  hier_t h;
  int rc = with_hier(ndims, shape, coords, &g, &h);
  if (rc) return rc;
  memcpy(u, c, grid_count(&g) * 8);
  if (h.L > 0) inverse_inplace(u, &h);
  hier_free(&h);
  grid_free(&g);
  return 0;
}

int oc_quantize(int ndims, const uint64_t* shape, const double* coords, const double* c, const double* widths, int64_t* q,
                double* res, uint64_t* outliers) {
  grid_t g;
  hier_t h;
  int rc = with_hier(ndims, shape, coords, &g, &h);
  if (rc) return rc;
  rc = quantize(&h, c, widths, q, res, outliers);
  hier_free(&h);
  grid_free(&g);
  return rc;
}

int oc_dequantize(int ndims, const uint64_t* shape, const double* coords, const int64_t* q, const double* widths, double* c) {
  grid_t g;
  hier_t h;
  int rc = with_hier(ndims, shape, coords, &g, &h);
  if (rc) return rc;
  dequantize(&h, q, widths, c);
  hier_free(&h);
  grid_free(&g);
  return 0;
}

int oc_absolute_tolerance(const double* u, uint64_t n, double tol, int norm, double s, int mode, double* out) {
  (void)s;
  return absolute_tolerance(u, n, tol, norm, mode, out);
}

int oc_bin_widths(double tau, int norm, double s, int ndims, int nlevels, double* out) {
  return bin_widths(tau, norm, s, ndims, nlevels, out);
}

int oc_achieved_error(int ndims, const uint64_t* shape, const double* coords, const double* res, int norm, double s, double* out) {
  grid_t g;
  hier_t h;
  int rc = with_hier(ndims, shape, coords, &g, &h);
  if (rc) return rc;
  *out = achieved_error(&h, res, norm, s);
  hier_free(&h);
  grid_free(&g);
  return 0;
}

double oc_sum_squares(const double* v, uint64_t n) { return sum_squares(v, n); }

int oc_huffman_pack(const uint8_t* in, uint64_t n, uint8_t** out, uint64_t* out_len) {
  buf_t b = {0};
  int rc = huffman_pack(in, n, &b);
  if (rc) { free(b.p); return rc; }
  *out = b.p;
  *out_len = b.n;
  return 0;
}

int oc_huffman_unpack(const uint8_t* in, uint64_t n, uint64_t count, uint8_t* out) {
  src_t s;
  int rc = huffman_source(&s, in, n);
  if (rc) return rc;
  for (uint64_t i = 0; i < count; ++i) {
    rc = src_next(&s, &out[i]);
    if (rc) return rc;
  }
  if (!src_exhausted_clean(&s)) return fail(OC_CORRUPT_STREAM, "CorruptStream: trailing data after Huffman stream");
  return 0;
}

int oc_huffman_lengths(const uint64_t* freq, uint8_t* lengths) { return build_lengths(freq, lengths); }

int oc_lossless_encode(const int64_t* v, uint64_t n, int codec, uint8_t** out, uint64_t* out_len) {
  buf_t b = {0};
  int rc = lossless_encode(v, n, codec, &b);
  if (rc) { free(b.p); return rc; }
  *out = b.p;
  *out_len = b.n;
  return 0;
}

int oc_lossless_decode(const uint8_t* p, uint64_t len, uint64_t count, int codec, int64_t* out) {
  return lossless_decode(p, len, count, codec, out);
}

/* ------------------------------------------------------------------------ */
/* chunking (chunking.cpp) + CLI multiblock (tools/mgrc.cpp)                */

static void split_axis(uint64_t n, uint64_t k, uint64_t* ranges /* 2k */) {
  const uint64_t base = n / k, extra = n % k;
  uint64_t at = 0;
  for (uint64_t i = 0; i < k; ++i) {
    const uint64_t len = base + (i < extra ? 1 : 0);
    ranges[2 * i] = at;
    ranges[2 * i + 1] = at + len;
    at += len;
  }
}

/* chunking.cpp:38-110.  axis_ranges[a] = list of [begin,end); the ranges are
 * returned per block in row-major block order: out[(b*ndims + a)*2 + {0,1}] */
int oc_plan_chunks(int ndims, const uint64_t* shape, int dtype, uint64_t budget, uint64_t* nblocks, uint64_t* out,
                   uint64_t cap_blocks) {
  if (ndims < 1 || ndims > MAXD) return fail(OC_INVALID_SHAPE, "InvalidShape: unsupported dimension count");
  for (int a = 0; a < ndims; ++a)
    if (shape[a] < 2) return fail(OC_INVALID_SHAPE, "InvalidShape: axis shorter than 2 nodes");
  const uint64_t unit = dtype == 0 ? 4 : 8;
  uint64_t total = unit;
  for (int a = 0; a < ndims; ++a) total *= shape[a];
  uint64_t* ranges[MAXD];
  uint64_t nr[MAXD];
  for (int a = 0; a < ndims; ++a) { ranges[a] = NULL; nr[a] = 0; }
  int rc = 0;
  if (total <= budget) {
    for (int a = 0; a < ndims; ++a) { ranges[a] = (uint64_t*)malloc(16); ranges[a][0] = 0; ranges[a][1] = shape[a]; nr[a] = 1; }
  } else {
    uint64_t floor_bytes = unit;
    for (int a = 0; a < ndims; ++a) floor_bytes *= 17;
    if (budget < floor_bytes) return fail(OC_BUDGET_TOO_SMALL, "BudgetTooSmall: budget %llu is below one 17^%d block (%llu bytes)",
                                          (unsigned long long)budget, ndims, (unsigned long long)floor_bytes);
    uint64_t prefix = 1;
    for (int a = 0; a < ndims; ++a) {
      uint64_t tail = unit;
      for (int b = a + 1; b < ndims; ++b) tail *= shape[b];
      const uint64_t cap = budget / (prefix * tail);
      if (cap >= shape[a]) {
        for (int b = a; b < ndims; ++b) { ranges[b] = (uint64_t*)malloc(16); ranges[b][0] = 0; ranges[b][1] = shape[b]; nr[b] = 1; }
        break;
      }
      const uint64_t want = cap >= 2 ? cap : 2;
      uint64_t k = (shape[a] + want - 1) / want;
      if (k > shape[a] / 2) k = shape[a] / 2;
      if (k < 1) k = 1;
      ranges[a] = (uint64_t*)malloc(16 * k);
      split_axis(shape[a], k, ranges[a]);
      nr[a] = k;
      uint64_t max_len = 0;
      for (uint64_t i = 0; i < k; ++i) if (ranges[a][2 * i + 1] - ranges[a][2 * i] > max_len) max_len = ranges[a][2 * i + 1] - ranges[a][2 * i];
      prefix *= max_len;
      if (prefix * tail <= budget && a + 1 < ndims) {
        for (int b = a + 1; b < ndims; ++b) { ranges[b] = (uint64_t*)malloc(16); ranges[b][0] = 0; ranges[b][1] = shape[b]; nr[b] = 1; }
        break;
      }
    }
    uint64_t worst = unit;
    for (int a = 0; a < ndims; ++a) {
      uint64_t max_len = 0;
      for (uint64_t i = 0; i < nr[a]; ++i) if (ranges[a][2 * i + 1] - ranges[a][2 * i] > max_len) max_len = ranges[a][2 * i + 1] - ranges[a][2 * i];
      worst *= max_len;
    }
    if (worst > budget) rc = fail(OC_BUDGET_TOO_SMALL, "BudgetTooSmall: budget cannot hold a minimal block of this shape");
  }
  if (!rc) {
    uint64_t nb = 1;
    for (int a = 0; a < ndims; ++a) nb *= nr[a];
    *nblocks = nb;
    if (out && nb <= cap_blocks) {
      for (uint64_t b = 0; b < nb; ++b) {
        uint64_t index = b; /* ChunkPlan::block, chunking.cpp:10-17 */
        for (int a = ndims; a-- > 0;) {
          const uint64_t j = index % nr[a];
          index /= nr[a];
          out[(b * ndims + a) * 2] = ranges[a][2 * j];
          out[(b * ndims + a) * 2 + 1] = ranges[a][2 * j + 1];
        }
      }
    }
  }
  for (int a = 0; a < ndims; ++a) free(ranges[a]);
  return rc;
}

/* tools/mgrc.cpp:363-484 (run_compress), restated without file I/O: the
 * array is in memory, blocks are compressed in plan order with a shared
 * absolute tolerance (REL normalised over the whole array by the CLI's
 * serial scan, :197-233), each block carrying its coordinate slice, and the
 * multiblock file is u32 count | u64 offsets | containers (:258-275). */
int oc_compress_chunked(const void* data, int dtype, int ndims, const uint64_t* shape, const double* coords, double tol,
                        int norm, double s, int mode, int codec, uint64_t chunk_mem, uint8_t** out, uint64_t* out_len) {
  uint64_t nb = 0;
  const uint64_t budget = chunk_mem > 0 ? chunk_mem : UINT64_MAX;
  int rc = oc_plan_chunks(ndims, shape, dtype, budget, &nb, NULL, 0);
  if (rc) return rc;
  uint64_t* plan = (uint64_t*)malloc(nb * ndims * 16);
  oc_plan_chunks(ndims, shape, dtype, budget, &nb, plan, nb);
  uint64_t count = 1;
  for (int a = 0; a < ndims; ++a) count *= shape[a];
  const uint64_t unit = dtype == 0 ? 4 : 8;
  uint8_t** blocks = (uint8_t**)calloc(nb, sizeof(uint8_t*));
  uint64_t* blens = (uint64_t*)calloc(nb, 8);
  if (nb == 1) {
    rc = oc_compress(data, dtype, ndims, shape, coords, tol, norm, s, mode, codec, &blocks[0], &blens[0]);
  } else {
    double btol = tol;
    if (mode == 1) {
      double mn = 0, mx = 0, sumsq = 0;
      for (uint64_t i = 0; i < count; ++i) {
        const double v = dtype == 0 ? (double)((const float*)data)[i] : ((const double*)data)[i];
        if (!isfinite(v)) { rc = fail(OC_NON_FINITE_INPUT, "NonFiniteInput: input contains NaN or Inf"); break; }
        if (i == 0 || v < mn) mn = v;
        if (i == 0 || v > mx) mx = v;
        sumsq += v * v;
      }
      const double nrm = norm == 0 ? mx - mn : sqrt(sumsq / (double)count);
      if (!rc && nrm == 0.0) rc = fail(OC_DEGENERATE_DATA, "DegenerateData: relative bound on a constant file");
      btol = tol * nrm;
    }
    uint64_t stride[MAXD];
    stride[ndims - 1] = 1;
    for (int a = ndims - 1; a-- > 0;) stride[a] = stride[a + 1] * shape[a + 1];
    uint64_t coff[MAXD];
    uint64_t at = 0;
    for (int a = 0; a < ndims; ++a) { coff[a] = at; at += shape[a]; }
    for (uint64_t b = 0; b < nb && !rc; ++b) {
      uint64_t bshape[MAXD], bn = 1, nc = 0;
      for (int a = 0; a < ndims; ++a) { bshape[a] = plan[(b * ndims + a) * 2 + 1] - plan[(b * ndims + a) * 2]; bn *= bshape[a]; nc += bshape[a]; }
      double* bc = (double*)malloc(nc * 8);
      uint64_t k = 0;
      for (int a = 0; a < ndims; ++a)
        for (uint64_t i = plan[(b * ndims + a) * 2]; i < plan[(b * ndims + a) * 2 + 1]; ++i)
          bc[k++] = coords ? coords[coff[a] + i] : (double)i;
      uint8_t* bd = (uint8_t*)malloc(bn * unit);
      uint64_t idx[MAXD] = {0, 0, 0, 0};
      for (uint64_t f = 0; f < bn; ++f) { /* read_block (mgrc.cpp:91-145) */
        uint64_t src = 0;
        for (int a = 0; a < ndims; ++a) src += (plan[(b * ndims + a) * 2] + idx[a]) * stride[a];
        memcpy(bd + f * unit, (const uint8_t*)data + src * unit, unit);
        for (int a = ndims; a-- > 0;) { if (++idx[a] < bshape[a]) break; idx[a] = 0; }
      }
      rc = oc_compress(bd, dtype, ndims, bshape, bc, btol, norm, s, 0, codec, &blocks[b], &blens[b]);
      free(bd);
      free(bc);
    }
  }
  if (!rc) {
    buf_t ob = {0};
    put_u32(&ob, (uint32_t)nb);
    uint64_t off = 4 + 8 * nb;
    for (uint64_t b = 0; b < nb; ++b) { put_u64(&ob, off); off += blens[b]; }
    for (uint64_t b = 0; b < nb; ++b) put_bytes(&ob, blocks[b], blens[b]);
    *out = ob.p;
    *out_len = ob.n;
  }
  for (uint64_t b = 0; b < nb; ++b) free(blocks[b]);
  free(blocks);
  free(blens);
  free(plan);
  return rc;
}

/* ------------------------------------------------------------------------ */
/* test fields (tests/support/test_support.hpp)                             */

/* test_support.hpp:43-62 */
void oc_multisine(int ndims, const uint64_t* shape, double* u) {
  const double tau = 2.0 * 3.14159265358979323846;
  uint64_t n = 1;
  for (int a = 0; a < ndims; ++a) n *= shape[a];
  uint64_t idx[MAXD] = {0, 0, 0, 0};
  for (uint64_t f = 0; f < n; ++f) {
    double t[4] = {0, 0, 0, 0};
    for (int a = 0; a < ndims; ++a) t[a] = (double)idx[a] / (double)(shape[a] - 1);
    u[f] = sin(tau * (1.0 * t[0] + 0.7 * t[1] + 0.4 * t[2])) + 0.5 * sin(tau * (3.0 * t[0] + 2.2 * t[1])) +
           0.25 * sin(tau * (7.0 * t[0] + 5.0 * t[3])) + 1.5 * t[0];
    for (int a = ndims; a-- > 0;) { if (++idx[a] < shape[a]) break; idx[a] = 0; }
  }
}

/* std::mt19937_64 (pinned by the C++ standard) + test_support.hpp:18-34 */
typedef struct { uint64_t mt[312]; int i; } mt64_t;

static void mt64_seed(mt64_t* m, uint64_t seed) {
  m->mt[0] = seed;
  for (int i = 1; i < 312; ++i) m->mt[i] = 6364136223846793005ULL * (m->mt[i - 1] ^ (m->mt[i - 1] >> 62)) + (uint64_t)i;
  m->i = 312;
}

static uint64_t mt64_next(mt64_t* m) {
  if (m->i >= 312) {
    for (int i = 0; i < 312; ++i) {
      const uint64_t x = (m->mt[i] & 0xFFFFFFFF80000000ULL) | (m->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      m->mt[i] = m->mt[(i + 156) % 312] ^ xa;
    }
    m->i = 0;
  }
  uint64_t y = m->mt[m->i++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

void oc_mt19937_64(uint64_t seed, uint64_t n, uint64_t* out) {
  mt64_t m;
  mt64_seed(&m, seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = mt64_next(&m);
}

/* random_field (test_support.hpp:64-70): lo + (hi-lo) * uniform() */
void oc_random_field(uint64_t n, uint64_t seed, double lo, double hi, double* out) {
  mt64_t m;
  mt64_seed(&m, seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = lo + (hi - lo) * ((double)(mt64_next(&m) >> 11) * 0x1.0p-53);
}

/* multisine_noisy (test_support.hpp:72-77) */
void oc_multisine_noisy(int ndims, const uint64_t* shape, uint64_t seed, double noise, double* out) {
  oc_multisine(ndims, shape, out);
  uint64_t n = 1;
  for (int a = 0; a < ndims; ++a) n *= shape[a];
  mt64_t m;
  mt64_seed(&m, seed);
  for (uint64_t i = 0; i < n; ++i) out[i] += noise * (-1.0 + 2.0 * ((double)(mt64_next(&m) >> 11) * 0x1.0p-53));
}
