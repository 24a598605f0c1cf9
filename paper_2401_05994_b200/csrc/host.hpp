// Host-side (CPU) pieces of the B200 compress/decompress path: the parts that
// are O(Σ shape) or O(256) and therefore never touch the array itself —
// grid hierarchy + per-axis stencil tables, error-control formulas, the
// container header, the Huffman codebook (lengths + canonical codes), the
// chunk planner and the multiblock framing.  Each function cites the
// reference routine whose behaviour it reproduces (paths relative to
// /root/reference/proj).
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace mgrc_gpu {

constexpr int kMaxDims = 4;      // grid.hpp:10
constexpr int kMaxLevels = 64;
constexpr int kMaxCodeLen = 15;  // codec.cpp:32
constexpr int kHuffTableBytes = 3 + 128;  // u16 nsym | u8 maxlen | 128 nibble bytes (codec.cpp:310-317)

// errc (error.hpp:11-31); C-ABI status = ordinal + 1, 0 = ok.
enum class Errc : int {
  invalid_shape = 1, too_many_dims, level_out_of_range, shape_mismatch, non_finite_input, degenerate_data, overflow,
  unknown_codec, corrupt_stream, bad_magic, unsupported_version, checksum_mismatch, tolerance_unreachable,
  plane_count_out_of_range, unsatisfiable_tolerance, invalid_state, prefix_violation, budget_too_small, io_error,
  cuda = 100, invalid_argument = 101,
};

const char* errc_name(Errc c);  // error.cpp:5-28

class Error : public std::runtime_error {
 public:
  Error(Errc c, const std::string& msg) : std::runtime_error(std::string(errc_name(c)) + ": " + msg), code_(c) {}
  Errc code() const { return code_; }

 private:
  Errc code_;
};

[[noreturn]] inline void raise(Errc c, const std::string& msg) { throw Error(c, msg); }

enum class DType : uint8_t { f32 = 0, f64 = 1 };
enum class Norm : uint8_t { inf = 0, s = 1 };
enum class Mode : uint8_t { abs = 0, rel = 1 };
enum class Codec : uint8_t { raw = 0, varint = 1, huffman = 2 };

inline size_t dtype_size(DType t) { return t == DType::f32 ? 4 : 8; }

struct ErrorSpec {  // error_control.hpp:15-25
  double tol = 0.0;
  Norm norm = Norm::inf;
  double smoothness = 0.0;
  Mode mode = Mode::abs;
};

// TensorGrid (grid.hpp:15-23): shape + per-axis coordinates.
struct Grid {
  int d = 0;
  uint64_t shape[kMaxDims] = {1, 1, 1, 1};
  std::vector<double> coords[kMaxDims];
  bool explicit_coords = false;
  uint64_t count() const {
    uint64_t n = 1;
    for (int a = 0; a < d; ++a) n *= shape[a];
    return n;
  }
};

// make_grid (grid.cpp:56-98).  coords == nullptr → 0..n-1 per axis.
Grid make_grid(int d, const uint64_t* shape, const double* const* coords);

// GridHierarchy (grid.hpp:35-60, grid.cpp:100-153) flattened into the
// per-axis tables the kernels consume.  Every finest index i of axis a is
// "fresh" at exactly one level, lvl[a][i]; the stencil of transform.cpp:27-63
// (bracketing coarse neighbours + coordinate weights) is therefore a function
// of i alone and is stored once per axis index.
struct Hierarchy {
  Grid grid;
  int L = 0;
  std::vector<uint8_t> lvl[kMaxDims];                   // axis_level
  std::vector<uint32_t> left[kMaxDims], right[kMaxDims];
  std::vector<double> wl[kMaxDims], wr[kMaxDims];
  std::vector<std::vector<uint32_t>> sets[kMaxDims];    // sets[a][l] = level_index_sets[l][a]
  std::vector<uint64_t> node_counts;                    // level_node_counts
  uint64_t box(int l) const {
    uint64_t n = 1;
    for (int a = 0; a < grid.d; ++a) n *= sets[a][l].size();
    return n;
  }
};

Hierarchy build_hierarchy(const Grid& g);

// error_control.cpp:42-60
std::vector<double> initial_bin_widths(double tau_abs, const ErrorSpec& spec, int d, int L);

// ---- container header (container.cpp:28-55, :133-188) --------------------
// Header flag of containers of the L²-corrected decomposition (our extension;
// the reference rejects unknown flags, container.cpp:143).
constexpr uint8_t kFlagL2Projection = 0x04;

struct ContainerInfo {  // container.hpp:37-51
  uint16_t version = 1;
  bool constant_field = false;
  bool coords_present = false;
  bool l2_projection = false;  // flag 0x04
  DType dtype = DType::f64;
  int ndims = 0;
  uint64_t shape[kMaxDims] = {0, 0, 0, 0};
  std::vector<double> coords[kMaxDims];
  ErrorSpec spec;
  int nlevels = 0;
  std::vector<double> bin_widths;
  uint8_t codec_id = 0;
  uint64_t payload_len = 0;
  uint32_t checksum = 0;
  uint64_t header_size = 0;
};

void append_header(std::vector<uint8_t>& out, const Grid& g, DType dtype, bool constant, const ErrorSpec& spec,
                   const std::vector<double>& widths, Codec codec, uint64_t payload_len, uint32_t crc);
ContainerInfo parse_header(const uint8_t* p, uint64_t n);
std::string describe(const ContainerInfo& info);  // container.cpp:263-299

// ---- canonical Huffman codebook (codec.cpp:100-220, :310-352) ------------
struct CodeTable {
  std::array<uint8_t, 256> lengths{};
  std::array<uint32_t, 256> codes{};
  int max_len = 0;
  int nsym = 0;
};
CodeTable build_code_table(const uint64_t* freq);  // build_lengths + canonical_codes
void write_table_header(std::vector<uint8_t>& out, const CodeTable& t);
// Parses + validates the table header exactly like read_table_header and the
// HuffmanDecoder constructor; returns the lengths.  Throws CorruptStream.
CodeTable read_table_header(const uint8_t* p, uint64_t n, uint64_t* consumed);
// Decode LUT: 2^max_len entries, entry = symbol | (length << 8) | (symbol < 0x80) << 12.
std::vector<uint16_t> build_decode_lut(const CodeTable& t);

// ---- CRC-32 (codec.cpp:14-28) host helpers ---------------------------------
uint32_t crc32_host(const uint8_t* p, uint64_t n, uint32_t crc = 0);
uint32_t crc32_mul(uint32_t a, uint32_t b);       // a·b mod P (reflected)
uint32_t crc32_x8n(uint64_t nbytes);              // x^(8n) mod P
uint32_t crc32_combine(uint32_t crc_a, uint32_t crc_b, uint64_t len_b);
void crc32_x8n_table(uint32_t* t64);              // x^(8·2^k), k = 0..63

// ---- chunking (chunking.cpp:10-110) + multiblock (tools/mgrc.cpp) ---------
struct Range {
  uint64_t begin = 0, end = 0;
  uint64_t length() const { return end - begin; }
};
struct ChunkPlan {
  int d = 0;
  std::vector<Range> axis_ranges[kMaxDims];
  uint64_t block_count() const {
    uint64_t n = 1;
    for (int a = 0; a < d; ++a) n *= axis_ranges[a].size();
    return n;
  }
  std::vector<Range> block(uint64_t index) const;  // chunking.cpp:10-17
};
ChunkPlan plan_chunks(int d, const uint64_t* shape, DType dtype, uint64_t budget);

}  // namespace mgrc_gpu
