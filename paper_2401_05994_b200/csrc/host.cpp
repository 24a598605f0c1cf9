// Host-side pieces of the B200 path (see host.hpp).  All O(Σ shape) / O(256)
// work; the array itself is only ever touched by the sm_100a kernels.
#include "host.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>

namespace mgrc_gpu {

const char* errc_name(Errc c) {
  static const char* names[] = {"InvalidShape", "TooManyDims", "LevelOutOfRange", "ShapeMismatch", "NonFiniteInput",
                                "DegenerateData", "Overflow", "UnknownCodec", "CorruptStream", "BadMagic",
                                "UnsupportedVersion", "ChecksumMismatch", "ToleranceUnreachable",
                                "PlaneCountOutOfRange", "UnsatisfiableTolerance", "InvalidState", "PrefixViolation",
                                "BudgetTooSmall", "IoError"};
  const int i = static_cast<int>(c);
  if (i >= 1 && i <= 19) return names[i - 1];
  if (c == Errc::cuda) return "CudaError";
  if (c == Errc::invalid_argument) return "InvalidArgument";
  return "UnknownError";
}

// ---------------------------------------------------------------------------
// grid + hierarchy

static void validate_shape(int d, const uint64_t* shape) {  // grid.cpp:20-31
  if (d < 1) raise(Errc::invalid_shape, "grid needs at least one axis");
  if (d > kMaxDims) raise(Errc::too_many_dims, "grid has " + std::to_string(d) + " axes, max is 4");
  for (int a = 0; a < d; ++a)
    if (shape[a] < 2)
      raise(Errc::invalid_shape, "axis " + std::to_string(a) + " has " + std::to_string(shape[a]) +
                                     " nodes, need at least 2");
}

Grid make_grid(int d, const uint64_t* shape, const double* const* coords) {
  validate_shape(d, shape);
  Grid g;
  g.d = d;
  for (int a = 0; a < d; ++a) {
    if (shape[a] >= (uint64_t{1} << 32)) raise(Errc::invalid_shape, "axis longer than 2^32 nodes");
    g.shape[a] = shape[a];
    g.coords[a].resize(shape[a]);
    for (uint64_t i = 0; i < shape[a]; ++i) g.coords[a][i] = coords ? coords[a][i] : static_cast<double>(i);
    if (coords) {  // grid.cpp:81-88
      for (uint64_t i = 0; i + 1 < shape[a]; ++i)
        if (!(g.coords[a][i] < g.coords[a][i + 1]))
          raise(Errc::invalid_shape, "axis " + std::to_string(a) + " coordinates are not strictly increasing");
      if (!std::isfinite(g.coords[a].front()) || !std::isfinite(g.coords[a].back()))
        raise(Errc::invalid_shape, "axis " + std::to_string(a) + " has non-finite coordinates");
    }
  }
  g.explicit_coords = coords != nullptr;
  return g;
}

// One coarsening step of grid.cpp:44-52: even positions, plus the last
// position when the set size is even; size-2 sets are fixed points.
static std::vector<uint32_t> coarsen(const std::vector<uint32_t>& fine) {
  const size_t n = fine.size();
  if (n <= 2) return fine;
  std::vector<uint32_t> c;
  c.reserve(n / 2 + 1);
  for (size_t p = 0; p < n; p += 2) c.push_back(fine[p]);
  if ((n & 1) == 0) c.push_back(fine[n - 1]);
  return c;
}

Hierarchy build_hierarchy(const Grid& g) {
  Hierarchy h;
  h.grid = g;
  const int d = g.d;
  std::vector<std::vector<uint32_t>> chain[kMaxDims];  // finest first
  int L = 0;
  for (int a = 0; a < d; ++a) {
    std::vector<uint32_t> s(g.shape[a]);
    for (uint64_t i = 0; i < g.shape[a]; ++i) s[i] = static_cast<uint32_t>(i);
    chain[a].push_back(std::move(s));
    while (chain[a].back().size() > 2) chain[a].push_back(coarsen(chain[a].back()));
    L = std::max(L, static_cast<int>(chain[a].size()) - 1);
  }
  if (L > kMaxLevels - 1) raise(Errc::invalid_shape, "too many levels");
  h.L = L;
  for (int a = 0; a < d; ++a) {
    h.sets[a].resize(L + 1);
    const int clen = static_cast<int>(chain[a].size());
    for (int l = 0; l <= L; ++l) h.sets[a][l] = chain[a][std::min(L - l, clen - 1)];  // grid.cpp:126-128
    // axis_level: coarsest membership wins (grid.cpp:134-140).
    h.lvl[a].assign(g.shape[a], static_cast<uint8_t>(L));
    for (int l = L; l >= 0; --l)
      for (uint32_t i : h.sets[a][l]) h.lvl[a][i] = static_cast<uint8_t>(l);
    // Stencil of every index at its own level (transform.cpp:27-63): the
    // bracketing coarse neighbours inside the level-l set.  Positions 0 and
    // n-1 of the set are always coarse, so both neighbours exist.
    h.left[a].assign(g.shape[a], 0);
    h.right[a].assign(g.shape[a], 0);
    h.wl[a].assign(g.shape[a], 0.0);
    h.wr[a].assign(g.shape[a], 0.0);
    const std::vector<double>& x = g.coords[a];
    for (int l = 1; l <= L; ++l) {
      const auto& set = h.sets[a][l];
      uint32_t prev = set[0];
      for (size_t p = 0; p < set.size(); ++p) {
        const uint32_t i = set[p];
        if (h.lvl[a][i] < l) {
          prev = i;
          continue;
        }
        size_t q = p + 1;
        while (h.lvl[a][set[q]] >= l) ++q;  // next coarse position
        const uint32_t nxt = set[q];
        h.left[a][i] = prev;
        h.right[a][i] = nxt;
        const double xl = x[prev], xr = x[nxt];
        h.wl[a][i] = (xr - x[i]) / (xr - xl);
        h.wr[a][i] = (x[i] - xl) / (xr - xl);
      }
    }
  }
  h.node_counts.assign(L + 1, 0);
  uint64_t prev_box = 0;
  for (int l = 0; l <= L; ++l) {
    const uint64_t b = h.box(l);
    h.node_counts[l] = b - prev_box;
    prev_box = b;
  }
  return h;
}

std::vector<double> initial_bin_widths(double tau_abs, const ErrorSpec& spec, int d, int L) {
  if (!(tau_abs > 0.0)) raise(Errc::invalid_state, "absolute tolerance must be > 0");
  const double Ld = static_cast<double>(L);
  const double cells = std::ldexp(1.0, d);  // 2^d
  std::vector<double> w(L + 1);
  if (spec.norm == Norm::inf) {
    const double delta = 2.0 * tau_abs / (1.0 + Ld * cells);
    std::fill(w.begin(), w.end(), delta);
  } else {
    const double base = 2.0 * tau_abs / std::sqrt((Ld + 1.0) * cells);
    for (int l = 0; l <= L; ++l) w[l] = base * std::exp2(spec.smoothness * (Ld - static_cast<double>(l)));
  }
  return w;
}

// ---------------------------------------------------------------------------
// little-endian byte helpers (bytes.hpp)

namespace {
void put8(std::vector<uint8_t>& o, uint8_t v) { o.push_back(v); }
void put16(std::vector<uint8_t>& o, uint16_t v) {
  o.push_back(static_cast<uint8_t>(v));
  o.push_back(static_cast<uint8_t>(v >> 8));
}
void put32(std::vector<uint8_t>& o, uint32_t v) {
  for (int i = 0; i < 4; ++i) o.push_back(static_cast<uint8_t>(v >> (8 * i)));
}
void put64(std::vector<uint8_t>& o, uint64_t v) {
  for (int i = 0; i < 8; ++i) o.push_back(static_cast<uint8_t>(v >> (8 * i)));
}
void putf64(std::vector<uint8_t>& o, double v) {
  uint64_t u;
  std::memcpy(&u, &v, 8);
  put64(o, u);
}

struct Reader {
  const uint8_t* p;
  uint64_t n, pos = 0;
  const uint8_t* take(uint64_t k) {
    if (k > n - pos) raise(Errc::corrupt_stream, "truncated stream");
    const uint8_t* r = p + pos;
    pos += k;
    return r;
  }
  uint8_t u8() { return *take(1); }
  uint16_t u16() {
    const uint8_t* b = take(2);
    return static_cast<uint16_t>(b[0] | (b[1] << 8));
  }
  uint32_t u32() {
    const uint8_t* b = take(4);
    return static_cast<uint32_t>(b[0]) | (static_cast<uint32_t>(b[1]) << 8) | (static_cast<uint32_t>(b[2]) << 16) |
           (static_cast<uint32_t>(b[3]) << 24);
  }
  uint64_t u64() {
    const uint8_t* b = take(8);
    uint64_t v = 0;
    for (int i = 7; i >= 0; --i) v = (v << 8) | b[i];
    return v;
  }
  double f64() {
    const uint64_t u = u64();
    double d;
    std::memcpy(&d, &u, 8);
    return d;
  }
};
}  // namespace

void append_header(std::vector<uint8_t>& out, const Grid& g, DType dtype, bool constant, const ErrorSpec& spec,
                   const std::vector<double>& widths, Codec codec, uint64_t payload_len, uint32_t crc) {
  const char magic[4] = {'M', 'G', 'R', 'C'};
  out.insert(out.end(), magic, magic + 4);
  put16(out, 1);
  put8(out, static_cast<uint8_t>((constant ? 1u : 0u) | (g.explicit_coords ? 2u : 0u)));
  put8(out, static_cast<uint8_t>(dtype));
  put8(out, static_cast<uint8_t>(g.d));
  for (int a = 0; a < g.d; ++a) put64(out, g.shape[a]);
  if (g.explicit_coords)
    for (int a = 0; a < g.d; ++a) {
      put64(out, g.coords[a].size());
      for (double x : g.coords[a]) putf64(out, x);
    }
  put8(out, static_cast<uint8_t>(spec.mode));
  put8(out, static_cast<uint8_t>(spec.norm));
  putf64(out, spec.norm == Norm::s ? spec.smoothness : 0.0);
  putf64(out, spec.tol);
  put8(out, static_cast<uint8_t>(widths.size() - 1));
  for (double w : widths) putf64(out, w);
  put8(out, static_cast<uint8_t>(codec));
  put64(out, payload_len);
  put32(out, crc);
}

ContainerInfo parse_header(const uint8_t* p, uint64_t n) {
  Reader r{p, n};
  ContainerInfo info;
  const uint8_t* m = r.take(4);
  if (std::memcmp(m, "MGRC", 4) != 0) raise(Errc::bad_magic, "not an MGRC container");
  info.version = r.u16();
  if (info.version != 1) raise(Errc::unsupported_version, "container version " + std::to_string(info.version));
  const uint8_t flags = r.u8();
  if (flags & ~(0x03u | kFlagL2Projection)) raise(Errc::corrupt_stream, "unknown header flags");
  info.constant_field = flags & 1u;
  info.coords_present = (flags & 2u) != 0;
  info.l2_projection = (flags & kFlagL2Projection) != 0;
  const uint8_t dt = r.u8();
  if (dt > 1) raise(Errc::corrupt_stream, "unknown element type");
  info.dtype = static_cast<DType>(dt);
  const uint8_t nd = r.u8();
  if (nd < 1 || nd > kMaxDims) raise(Errc::corrupt_stream, "dimension count out of range");
  info.ndims = nd;
  uint64_t count = 1;
  for (int a = 0; a < nd; ++a) {
    const uint64_t s = r.u64();
    if (s < 2) raise(Errc::corrupt_stream, "axis shorter than 2 nodes");
    if (s > (uint64_t{1} << 40) / count) raise(Errc::corrupt_stream, "implausible shape");
    count *= s;
    info.shape[a] = s;
  }
  if (info.coords_present)
    for (int a = 0; a < nd; ++a) {
      const uint64_t k = r.u64();
      if (k != info.shape[a]) raise(Errc::corrupt_stream, "coordinate count mismatch");
      if (k * 8 > r.n - r.pos) raise(Errc::corrupt_stream, "truncated stream");
      info.coords[a].resize(k);
      for (auto& x : info.coords[a]) x = r.f64();
    }
  const uint8_t mode = r.u8();
  if (mode > 1) raise(Errc::corrupt_stream, "unknown error-bound mode");
  info.spec.mode = static_cast<Mode>(mode);
  const uint8_t norm = r.u8();
  if (norm > 1) raise(Errc::corrupt_stream, "unknown norm");
  info.spec.norm = static_cast<Norm>(norm);
  info.spec.smoothness = r.f64();
  info.spec.tol = r.f64();
  info.nlevels = r.u8();
  info.bin_widths.resize(static_cast<size_t>(info.nlevels) + 1);
  for (auto& w : info.bin_widths) w = r.f64();
  info.codec_id = r.u8();
  if (info.codec_id > 2) raise(Errc::corrupt_stream, "unknown codec id");
  info.payload_len = r.u64();
  info.checksum = r.u32();
  info.header_size = r.pos;
  return info;
}

static std::string g17(double v) {
  char b[40];
  std::snprintf(b, sizeof b, "%.17g", v);
  return b;
}

std::string describe(const ContainerInfo& info) {
  std::string s;
  auto line = [&s](const char* k, const std::string& v) {
    s += k;
    s += ": ";
    s += v;
    s += '\n';
  };
  line("format", "mgrc-container");
  line("version", std::to_string(info.version));
  line("constant_field", info.constant_field ? "1" : "0");
  line("coords_present", info.coords_present ? "1" : "0");
  if (info.l2_projection) line("l2_projection", "1");
  line("dtype", info.dtype == DType::f32 ? "f32" : "f64");
  line("ndims", std::to_string(info.ndims));
  std::string sh;
  for (int a = 0; a < info.ndims; ++a) sh += (a ? "x" : "") + std::to_string(info.shape[a]);
  line("shape", sh);
  line("mode", info.spec.mode == Mode::abs ? "abs" : "rel");
  line("norm", info.spec.norm == Norm::inf ? "inf" : "s");
  line("s", g17(info.spec.smoothness));
  line("tol", g17(info.spec.tol));
  line("nlevels", std::to_string(info.nlevels));
  std::string w;
  for (size_t l = 0; l < info.bin_widths.size(); ++l) w += (l ? "," : "") + g17(info.bin_widths[l]);
  line("bin_widths", w);
  line("codec", std::to_string(info.codec_id));
  line("header_bytes", std::to_string(info.header_size));
  line("payload_bytes", std::to_string(info.payload_len));
  line("crc32", std::to_string(info.checksum));
  return s;
}

// ---------------------------------------------------------------------------
// Huffman codebook

// Code lengths with the reference's deterministic schedule
// (codec.cpp:100-192): repeatedly merge the two minimum (freq, key) nodes,
// leaves keyed by symbol, internal nodes by creation order 256, 257, ...
// Implemented as the two-queue construction: leaves sorted by (freq, symbol)
// and internal nodes in creation order (their (freq, key) is non-decreasing),
// so each front is its queue's minimum and leaves win equal-freq ties
// (key < 256) — the same merge sequence as the reference's binary heap.
static std::array<uint8_t, 256> huffman_lengths(const uint64_t* freq) {
  std::array<uint8_t, 256> len{};
  std::vector<int> leaves;
  for (int s = 0; s < 256; ++s)
    if (freq[s]) leaves.push_back(s);
  if (leaves.empty()) return len;
  if (leaves.size() == 1) {
    len[leaves[0]] = 1;
    return len;
  }
  std::stable_sort(leaves.begin(), leaves.end(), [&](int a, int b) { return freq[a] < freq[b]; });
  const int nl = static_cast<int>(leaves.size());
  // node ids: 0..nl-1 leaves (in sorted order), nl.. internal
  std::vector<uint64_t> w(2 * nl);
  std::vector<int> parent(2 * nl, -1);
  for (int i = 0; i < nl; ++i) w[i] = freq[leaves[i]];
  int li = 0, ii = nl, next = nl;
  auto pop = [&]() {
    if (li < nl && (ii >= next || w[li] <= w[ii])) return li++;
    return ii++;
  };
  while (next < 2 * nl - 1) {
    const int a = pop(), b = pop();
    w[next] = w[a] + w[b];
    parent[a] = parent[b] = next;
    ++next;
  }
  std::vector<int> depth(2 * nl - 1, 0);
  for (int n = 2 * nl - 3; n >= 0; --n) depth[n] = depth[parent[n]] + 1;  // parents are created after children
  for (int i = 0; i < nl; ++i) len[leaves[i]] = static_cast<uint8_t>(std::min(depth[i], 255));

  // Length limit 15, then Kraft equality restored (codec.cpp:157-190).
  constexpr uint32_t one = 1u << kMaxCodeLen;
  uint64_t kraft = 0;
  for (int s : leaves) {
    if (len[s] > kMaxCodeLen) len[s] = kMaxCodeLen;
    kraft += one >> len[s];
  }
  while (kraft > one) {  // deepen the longest extendable code, largest symbol on ties
    int pick = -1;
    for (int s = 255; s >= 0; --s)
      if (freq[s] && len[s] < kMaxCodeLen && (pick < 0 || len[s] > len[pick])) pick = s;
    kraft -= one >> (len[pick] + 1);
    ++len[pick];
  }
  while (kraft < one) {  // shorten the deepest code that still fits, smallest symbol on ties
    int pick = -1;
    for (int s = 0; s < 256; ++s)
      if (freq[s] && len[s] > 1 && kraft + (one >> len[s]) <= one && (pick < 0 || len[s] > len[pick])) pick = s;
    if (pick < 0) raise(Errc::corrupt_stream, "internal: kraft repair failed");
    kraft += one >> len[pick];
    --len[pick];
  }
  return len;
}

static void assign_canonical(CodeTable& t) {  // codec.cpp:195-220
  int bl_count[kMaxCodeLen + 2] = {0};
  t.max_len = 0;
  t.nsym = 0;
  for (int s = 0; s < 256; ++s)
    if (t.lengths[s]) {
      ++bl_count[t.lengths[s]];
      ++t.nsym;
      t.max_len = std::max<int>(t.max_len, t.lengths[s]);
    }
  uint32_t next[kMaxCodeLen + 2] = {0};
  uint32_t code = 0;
  for (int l = 1; l <= t.max_len; ++l) {
    code = (code + bl_count[l - 1]) << 1;
    next[l] = code;
  }
  for (int s = 0; s < 256; ++s) t.codes[s] = t.lengths[s] ? next[t.lengths[s]]++ : 0;
}

CodeTable build_code_table(const uint64_t* freq) {
  CodeTable t;
  t.lengths = huffman_lengths(freq);
  assign_canonical(t);
  return t;
}

void write_table_header(std::vector<uint8_t>& out, const CodeTable& t) {
  if (t.nsym == 0) {  // codec.cpp:407-411
    put16(out, 0);
    put8(out, 0);
    return;
  }
  put16(out, static_cast<uint16_t>(t.nsym));
  put8(out, static_cast<uint8_t>(t.max_len));
  for (int s = 0; s < 256; s += 2) put8(out, static_cast<uint8_t>((t.lengths[s] & 0x0F) | (t.lengths[s + 1] << 4)));
}

CodeTable read_table_header(const uint8_t* p, uint64_t n, uint64_t* consumed) {
  Reader r{p, n};
  CodeTable t;
  t.nsym = r.u16();
  if (t.nsym == 0) {  // codec.cpp:328-332
    if (r.u8() != 0) raise(Errc::corrupt_stream, "nonzero max length for empty table");
    *consumed = r.pos;
    return t;
  }
  const int max_len = r.u8();
  if (max_len == 0 || max_len > kMaxCodeLen) raise(Errc::corrupt_stream, "Huffman max code length out of range");
  int nonzero = 0, observed = 0;
  for (int s = 0; s < 256; s += 2) {
    const uint8_t b = r.u8();
    t.lengths[s] = b & 0x0F;
    t.lengths[s + 1] = b >> 4;
    for (int k = 0; k < 2; ++k)
      if (t.lengths[s + k]) {
        ++nonzero;
        observed = std::max<int>(observed, t.lengths[s + k]);
      }
  }
  if (nonzero != t.nsym) raise(Errc::corrupt_stream, "Huffman symbol count mismatch");
  if (observed != max_len) raise(Errc::corrupt_stream, "Huffman max code length mismatch");
  // HuffmanDecoder constructor checks (codec.cpp:265-270)
  constexpr uint32_t one = 1u << kMaxCodeLen;
  uint64_t kraft = 0;
  int only_len = 0;
  for (int s = 0; s < 256; ++s)
    if (t.lengths[s]) {
      kraft += one >> t.lengths[s];
      only_len = t.lengths[s];
    }
  if (nonzero >= 2 && kraft != one) raise(Errc::corrupt_stream, "Huffman table violates Kraft equality");
  if (nonzero == 1 && only_len != 1) raise(Errc::corrupt_stream, "degenerate Huffman table");
  assign_canonical(t);
  *consumed = r.pos;
  return t;
}

std::vector<uint16_t> build_decode_lut(const CodeTable& t) {
  std::vector<uint16_t> lut(size_t{1} << t.max_len, 0);
  for (int s = 0; s < 256; ++s) {
    const int l = t.lengths[s];
    if (!l) continue;
    const uint32_t lo = t.codes[s] << (t.max_len - l), hi = (t.codes[s] + 1) << (t.max_len - l);
    for (uint32_t k = lo; k < hi; ++k) lut[k] = static_cast<uint16_t>(s | (l << 8) | ((s < 0x80 ? 1 : 0) << 12));
  }
  return lut;
}

// ---------------------------------------------------------------------------
// CRC-32 (IEEE, reflected 0xEDB88320) and GF(2) combination

static const uint32_t* crc_table() {
  // magic static: initialised once, thread-safe (concurrent compress calls share it)
  static const std::array<uint32_t, 256> t = [] {
    std::array<uint32_t, 256> a{};
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1u) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      a[i] = c;
    }
    return a;
  }();
  return t.data();
}

uint32_t crc32_host(const uint8_t* p, uint64_t n, uint32_t crc) {
  const uint32_t* t = crc_table();
  uint32_t c = ~crc;
  for (uint64_t i = 0; i < n; ++i) c = t[(c ^ p[i]) & 0xFFu] ^ (c >> 8);
  return ~c;
}

// Product of two polynomials mod P in the reflected bit order (bit 31 = x^0).
uint32_t crc32_mul(uint32_t a, uint32_t b) {
  uint32_t prod = 0;
  for (int i = 0; i < 32; ++i) {
    if (a & (0x80000000u >> i)) prod ^= b;
    b = (b & 1u) ? (b >> 1) ^ 0xEDB88320u : b >> 1;
  }
  return prod;
}

void crc32_x8n_table(uint32_t* t64) {
  uint32_t p = crc32_mul(0x00800000u, 0x80000000u);  // x^8
  for (int k = 0; k < 64; ++k) {
    t64[k] = p;  // x^(8·2^k)
    p = crc32_mul(p, p);
  }
}

uint32_t crc32_x8n(uint64_t nbytes) {
  static const std::array<uint32_t, 64> t = [] {
    std::array<uint32_t, 64> a{};
    crc32_x8n_table(a.data());
    return a;
  }();
  uint32_t p = 0x80000000u;  // 1
  for (int k = 0; nbytes; ++k, nbytes >>= 1)
    if (nbytes & 1) p = crc32_mul(p, t[k]);
  return p;
}

// Standard (init ~0, xorout ~0) CRCs are affine in the data; the affine
// parts cancel and crc(A‖B) = crc(A)·x^(8|B|) ⊕ crc(B).
uint32_t crc32_combine(uint32_t a, uint32_t b, uint64_t len_b) { return crc32_mul(crc32_x8n(len_b), a) ^ b; }

// ---------------------------------------------------------------------------
// chunk planner (chunking.cpp:10-110)

std::vector<Range> ChunkPlan::block(uint64_t index) const {
  std::vector<Range> out(d);
  for (int a = d - 1; a >= 0; --a) {
    out[a] = axis_ranges[a][index % axis_ranges[a].size()];
    index /= axis_ranges[a].size();
  }
  return out;
}

static std::vector<Range> split_axis(uint64_t n, uint64_t k) {  // near-equal, longer first
  std::vector<Range> r(k);
  uint64_t at = 0;
  for (uint64_t i = 0; i < k; ++i) {
    const uint64_t len = n / k + (i < n % k ? 1 : 0);
    r[i] = {at, at + len};
    at += len;
  }
  return r;
}

ChunkPlan plan_chunks(int d, const uint64_t* shape, DType dtype, uint64_t budget) {
  if (d < 1 || d > kMaxDims) raise(Errc::invalid_shape, "unsupported dimension count");
  for (int a = 0; a < d; ++a)
    if (shape[a] < 2) raise(Errc::invalid_shape, "axis shorter than 2 nodes");
  const uint64_t unit = dtype_size(dtype);
  uint64_t total = unit;
  for (int a = 0; a < d; ++a) total *= shape[a];
  ChunkPlan plan;
  plan.d = d;
  auto whole_from = [&](int a0) {
    for (int b = a0; b < d; ++b) plan.axis_ranges[b] = {{0, shape[b]}};
  };
  if (total <= budget) {
    whole_from(0);
    return plan;
  }
  uint64_t floor_bytes = unit;
  for (int a = 0; a < d; ++a) floor_bytes *= 17;
  if (budget < floor_bytes)
    raise(Errc::budget_too_small, "budget " + std::to_string(budget) + " is below one 17^" + std::to_string(d) +
                                      " block (" + std::to_string(floor_bytes) + " bytes)");
  uint64_t prefix = 1;
  for (int a = 0; a < d; ++a) {
    uint64_t tail = unit;
    for (int b = a + 1; b < d; ++b) tail *= shape[b];
    const uint64_t cap = budget / (prefix * tail);
    if (cap >= shape[a]) {
      whole_from(a);
      break;
    }
    const uint64_t want = cap >= 2 ? cap : 2;
    uint64_t k = (shape[a] + want - 1) / want;
    k = std::min<uint64_t>(k, shape[a] / 2);
    k = std::max<uint64_t>(k, 1);
    plan.axis_ranges[a] = split_axis(shape[a], k);
    prefix *= plan.axis_ranges[a][0].length();  // longest range comes first
    if (prefix * tail <= budget && a + 1 < d) {
      whole_from(a + 1);
      break;
    }
  }
  uint64_t worst = unit;
  for (int a = 0; a < d; ++a) {
    uint64_t m = 0;
    for (const auto& r : plan.axis_ranges[a]) m = std::max(m, r.length());
    worst *= m;
  }
  if (worst > budget) raise(Errc::budget_too_small, "budget cannot hold a minimal block of this shape");
  return plan;
}

}  // namespace mgrc_gpu
