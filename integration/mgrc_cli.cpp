// mgrc-gpu: the reference command-line tool (tools/mgrc.cpp) for the
// compress / decompress / inspect subcommands, on the B200 path through the
// C-ABI (include/mgrc_gpu.h) only.  Same options, same raw-file conventions
// (headerless little-endian, row-major, last axis fastest), same multiblock
// file (u32 count | u64 offsets | containers, mgrc.cpp:258-275), same
// messages and exit status (0 ok, 1 on an mgrc error: "error: <what>").
//
//   mgrc-gpu compress   --input F --output F --shape 513x513x513 --tol 1e-4
//                       [--dtype f32|f64] [--s inf|<s>] [--mode abs|rel]
//                       [--codec 0..2] [--chunk-mem 4GiB] [--coords F] [--device N] [--gpus N]
//   mgrc-gpu decompress --input F --output F [--device N] [--gpus N]
//   mgrc-gpu inspect    PATH
//
// refactor / recompose (MDR stores, refactor.cpp) are SURVEY §8(f) row f2 and
// are rejected with an error.  Raw input is read straight into a page-locked
// buffer (mgrc_gpu_host_alloc) so the host->device staging runs at PCIe rate.
#include <fcntl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cinttypes>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "mgrc_gpu.h"

namespace {

struct Fail : std::runtime_error {  // an mgrc error: printed as "error: <what>", exit 1
  using std::runtime_error::runtime_error;
};
struct Usage : std::runtime_error {  // argument error (CLI11 prints and exits non-zero)
  using std::runtime_error::runtime_error;
};

// errc_name (error.cpp:5-28) for errors raised by the tool itself
const char* errc_name(int code) {
  static const char* names[] = {"",
                                "InvalidShape",
                                "TooManyDims",
                                "LevelOutOfRange",
                                "ShapeMismatch",
                                "NonFiniteInput",
                                "DegenerateData",
                                "Overflow",
                                "UnknownCodec",
                                "CorruptStream",
                                "BadMagic",
                                "UnsupportedVersion",
                                "ChecksumMismatch",
                                "ToleranceUnreachable",
                                "PlaneCountOutOfRange",
                                "UnsatisfiableTolerance",
                                "InvalidState",
                                "PrefixViolation",
                                "BudgetTooSmall",
                                "IoError"};
  return code >= 1 && code <= 19 ? names[code] : "Error";
}

[[noreturn]] void raise(int code, const std::string& msg) { throw Fail(std::string(errc_name(code)) + ": " + msg); }

void check(int rc) {
  if (rc != MGRC_OK) throw Fail(mgrc_gpu_last_error());
}

// parse_shape (mgrc.cpp:37-50): "129x129"
std::vector<uint64_t> parse_shape(const std::string& text) {
  std::vector<uint64_t> shape;
  size_t at = 0;
  while (at < text.size()) {
    size_t next = text.find('x', at);
    if (next == std::string::npos) next = text.size();
    const std::string part = text.substr(at, next - at);
    if (part.empty() || part.find_first_not_of("0123456789") != std::string::npos)
      raise(MGRC_E_INVALID_SHAPE, "bad --shape");
    shape.push_back(std::strtoull(part.c_str(), nullptr, 10));
    at = next + 1;
  }
  if (shape.empty()) raise(MGRC_E_INVALID_SHAPE, "bad --shape");
  return shape;
}

// CLI::AsSizeValue(false) (mgrc.cpp:878-879): a number with an optional unit;
// k/kb/kib = 1024, m/mb/mib = 1024^2, ... (case-insensitive).
uint64_t parse_size(const std::string& text) {
  size_t i = 0;
  while (i < text.size() && (std::isdigit(static_cast<unsigned char>(text[i])) || text[i] == '.')) ++i;
  if (i == 0) throw Usage("--chunk-mem: not a size: " + text);
  const double num = std::strtod(text.substr(0, i).c_str(), nullptr);
  std::string unit;
  for (size_t k = i; k < text.size(); ++k)
    if (!std::isspace(static_cast<unsigned char>(text[k]))) unit += static_cast<char>(std::tolower(text[k]));
  static const std::map<std::string, int> pw = {{"", 0},   {"b", 0},   {"k", 1},   {"kb", 1},  {"kib", 1},
                                                {"m", 2},  {"mb", 2},  {"mib", 2}, {"g", 3},   {"gb", 3},
                                                {"gib", 3}, {"t", 4},  {"tb", 4},  {"tib", 4}, {"p", 5},
                                                {"pb", 5}, {"pib", 5}, {"e", 6},   {"eb", 6},  {"eib", 6}};
  const auto it = pw.find(unit);
  if (it == pw.end()) throw Usage("--chunk-mem: unknown unit: " + text);
  double v = num;
  for (int k = 0; k < it->second; ++k) v *= 1024.0;
  return static_cast<uint64_t>(v);
}

uint64_t file_size(const std::string& p) {
  struct stat st;
  if (::stat(p.c_str(), &st) != 0) raise(MGRC_E_IO_ERROR, "cannot stat " + p);
  return static_cast<uint64_t>(st.st_size);
}

// A page-locked buffer when one can be had (plain heap memory otherwise: only
// the staging rate differs, the compute path is the same).
struct HostBuf {
  void* p = nullptr;
  bool pinned = false;
  uint64_t n = 0;
  explicit HostBuf(uint64_t bytes) : n(bytes) {
    if (mgrc_gpu_host_alloc(bytes, &p) == MGRC_OK) {
      pinned = true;
    } else {
      p = std::malloc(bytes ? bytes : 1);
      if (!p) raise(MGRC_E_IO_ERROR, "out of host memory");
    }
  }
  ~HostBuf() {
    if (pinned) mgrc_gpu_host_free(p);
    else std::free(p);
  }
  uint8_t* data() { return static_cast<uint8_t*>(p); }
};

// A raw input file mapped read-only: the multiblock compress reads it block by
// block in file order (the reference's read_block, mgrc.cpp:91-145), so host
// memory stays bounded by the page cache instead of holding the whole file.
struct MappedFile {
  void* p = MAP_FAILED;
  uint64_t n = 0;
  MappedFile(const std::string& path, uint64_t bytes) : n(bytes) {
    const int fd = ::open(path.c_str(), O_RDONLY);
    if (fd < 0) raise(MGRC_E_IO_ERROR, "cannot read " + path);
    p = ::mmap(nullptr, bytes, PROT_READ, MAP_PRIVATE, fd, 0);
    ::close(fd);
    if (p == MAP_FAILED) raise(MGRC_E_IO_ERROR, "cannot map " + path);
    ::madvise(p, bytes, MADV_SEQUENTIAL);
  }
  ~MappedFile() {
    if (p != MAP_FAILED) ::munmap(p, n);
  }
  const uint8_t* data() const { return static_cast<const uint8_t*>(p); }
};

void read_exact(const std::string& path, uint8_t* dst, uint64_t n) {
  const int fd = ::open(path.c_str(), O_RDONLY);
  if (fd < 0) raise(MGRC_E_IO_ERROR, "cannot read " + path);
  uint64_t got = 0;
  while (got < n) {
    const ssize_t r = ::read(fd, dst + got, static_cast<size_t>(std::min<uint64_t>(n - got, 1ull << 30)));
    if (r < 0 && errno == EINTR) continue;
    if (r <= 0) {
      ::close(fd);
      raise(MGRC_E_IO_ERROR, "short read from " + path);
    }
    got += static_cast<uint64_t>(r);
  }
  ::close(fd);
}

void write_all(const std::string& path, const uint8_t* src, uint64_t n) {
  const int fd = ::open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (fd < 0) raise(MGRC_E_IO_ERROR, "cannot write " + path);
  uint64_t put = 0;
  while (put < n) {
    const ssize_t w = ::write(fd, src + put, static_cast<size_t>(std::min<uint64_t>(n - put, 1ull << 30)));
    if (w < 0 && errno == EINTR) continue;
    if (w <= 0) {
      ::close(fd);
      raise(MGRC_E_IO_ERROR, "short write to " + path);
    }
    put += static_cast<uint64_t>(w);
  }
  if (::close(fd) != 0) raise(MGRC_E_IO_ERROR, "short write to " + path);
}

struct Args {
  std::map<std::string, std::string> opt;
  std::vector<std::string> pos;
  bool has(const std::string& k) const { return opt.count(k) != 0; }
  std::string get(const std::string& k, const std::string& dflt = "") const {
    const auto it = opt.find(k);
    return it == opt.end() ? dflt : it->second;
  }
  std::string need(const std::string& k) const {
    if (!has(k)) throw Usage(k + " is required");
    return get(k);
  }
};

Args parse_args(int argc, char** argv, int from, const std::vector<std::string>& known) {
  Args a;
  for (int i = from; i < argc; ++i) {
    std::string t = argv[i];
    if (t.rfind("--", 0) == 0) {
      std::string k = t, v;
      const size_t eq = t.find('=');
      if (eq != std::string::npos) {
        k = t.substr(0, eq);
        v = t.substr(eq + 1);
      } else {
        if (i + 1 >= argc) throw Usage(k + " needs a value");
        v = argv[++i];
      }
      bool ok = false;
      for (const auto& n : known) ok = ok || n == k;
      if (!ok) throw Usage("unknown option " + k);
      a.opt[k] = v;
    } else {
      a.pos.push_back(t);
    }
  }
  return a;
}

void select_device(const Args& a) {
  if (a.has("--device")) check(mgrc_gpu_set_device(std::atoi(a.get("--device").c_str())));
}

// --gpus N: the blocks are spread over N GPUs of this process (mgrc_gpu_*_chunked_multi)
int gpus(const Args& a) { return a.has("--gpus") ? std::max(1, std::atoi(a.get("--gpus").c_str())) : 1; }

// run_compress (mgrc.cpp:363-484)
int run_compress(const Args& a) {
  if (!a.pos.empty()) throw Usage("unexpected argument " + a.pos[0]);
  const std::string input = a.need("--input"), output = a.need("--output"), shape_text = a.need("--shape");
  const std::string tol_text = a.need("--tol");
  const std::string dtype_text = a.get("--dtype", "f64"), s_text = a.get("--s", "inf"),
                    mode_text = a.get("--mode", "abs");
  if (dtype_text != "f32" && dtype_text != "f64") throw Usage("--dtype: not in {f32, f64}");
  if (mode_text != "abs" && mode_text != "rel") throw Usage("--mode: not in {abs, rel}");
  const int codec = a.has("--codec") ? std::atoi(a.get("--codec").c_str()) : 2;
  if (codec < 0 || codec > 2) throw Usage("--codec: not in [0 - 2]");
  const double tol = std::strtod(tol_text.c_str(), nullptr);
  const uint64_t chunk_mem = a.has("--chunk-mem") ? parse_size(a.get("--chunk-mem")) : 0;
  // parse_spec (mgrc.cpp:52-64)
  int norm = MGRC_NORM_INF;
  double s = 0.0;
  if (s_text != "inf") {
    norm = MGRC_NORM_S;
    s = std::strtod(s_text.c_str(), nullptr);
  }
  const int mode = mode_text == "rel" ? MGRC_MODE_REL : MGRC_MODE_ABS;
  const int dtype = dtype_text == "f32" ? MGRC_DTYPE_F32 : MGRC_DTYPE_F64;
  const std::vector<uint64_t> shape = parse_shape(shape_text);
  if (shape.size() > 4) raise(MGRC_E_TOO_MANY_DIMS, "grid has " + std::to_string(shape.size()) + " axes, max is 4");
  uint64_t count = 1;
  for (uint64_t n : shape) count *= n;
  const uint64_t unit = dtype == MGRC_DTYPE_F32 ? 4 : 8;
  const uint64_t expect = count * unit;
  const uint64_t have = file_size(input);
  if (have != expect)
    raise(MGRC_E_INVALID_SHAPE, "size mismatch: " + input + " has " + std::to_string(have) + " bytes, shape " +
                                    shape_text + " needs " + std::to_string(expect));
  // load_coords (mgrc.cpp:235-256): concatenated per-axis f64
  std::vector<std::vector<double>> coords;
  std::vector<const double*> cptr;
  if (a.has("--coords")) {
    const std::string cp = a.get("--coords");
    uint64_t total = 0;
    for (uint64_t n : shape) total += n;
    const uint64_t cb = file_size(cp);
    if (cb != total * 8)
      raise(MGRC_E_INVALID_SHAPE, "coordinate file must hold " + std::to_string(total) + " f64 values");
    std::vector<double> all(total);
    read_exact(cp, reinterpret_cast<uint8_t*>(all.data()), cb);
    uint64_t at = 0;
    for (uint64_t n : shape) {
      coords.emplace_back(all.begin() + static_cast<std::ptrdiff_t>(at),
                          all.begin() + static_cast<std::ptrdiff_t>(at + n));
      at += n;
    }
    for (auto& c : coords) cptr.push_back(c.data());
  }
  select_device(a);
  // one container: the whole array is uploaded, read it into pinned memory (PCIe rate); several blocks:
  // stream them from the mapped file
  std::unique_ptr<HostBuf> whole;
  std::unique_ptr<MappedFile> mapped;
  const uint8_t* src = nullptr;
  if (chunk_mem > 0 && expect > chunk_mem) {
    mapped = std::make_unique<MappedFile>(input, expect);
    src = mapped->data();
  } else {
    whole = std::make_unique<HostBuf>(expect);
    read_exact(input, whole->data(), expect);
    src = whole->data();
  }
  uint8_t* out = nullptr;
  uint64_t out_len = 0;
  check(mgrc_gpu_compress_chunked_multi(src, dtype, static_cast<int>(shape.size()), shape.data(),
                                        cptr.empty() ? nullptr : cptr.data(), tol, norm, s, mode, codec, chunk_mem,
                                        gpus(a), &out, &out_len));
  const uint32_t nblocks = out_len >= 4 ? (uint32_t(out[0]) | uint32_t(out[1]) << 8 | uint32_t(out[2]) << 16 |
                                           uint32_t(out[3]) << 24)
                                        : 0;
  try {
    write_all(output, out, out_len);
  } catch (...) {
    mgrc_gpu_free(out);
    throw;
  }
  mgrc_gpu_free(out);
  const uint64_t out_bytes = file_size(output);
  std::fprintf(stderr, "compressed %s (%" PRIu64 " bytes) -> %s (%" PRIu64 " bytes), %zu block(s), ratio %.3f\n",
               input.c_str(), expect, output.c_str(), out_bytes, static_cast<size_t>(nblocks),
               static_cast<double>(expect) / static_cast<double>(out_bytes));
  return 0;
}

// run_decompress (mgrc.cpp:490-542)
int run_decompress(const Args& a) {
  if (!a.pos.empty()) throw Usage("unexpected argument " + a.pos[0]);
  const std::string input = a.need("--input"), output = a.need("--output");
  select_device(a);
  const uint64_t n = file_size(input);
  HostBuf in(n);
  read_exact(input, in.data(), n);
  void* out = nullptr;
  int dtype = 0, nd = 0;
  uint64_t shape[4] = {0, 0, 0, 0};
  check(mgrc_gpu_decompress_chunked_multi(in.data(), n, gpus(a), &out, &dtype, &nd, shape));
  uint64_t count = 1;
  for (int k = 0; k < nd; ++k) count *= shape[k];
  try {
    write_all(output, static_cast<const uint8_t*>(out), count * (dtype == MGRC_DTYPE_F32 ? 4 : 8));
  } catch (...) {
    mgrc_gpu_free(out);
    throw;
  }
  mgrc_gpu_free(out);
  return 0;
}

// run_inspect (mgrc.cpp:829-855), multiblock files (MDR store directories are row f2)
int run_inspect(const Args& a) {
  if (a.pos.size() != 1) throw Usage("inspect takes one path");
  const std::string path = a.pos[0];
  struct stat st;
  if (::stat(path.c_str(), &st) == 0 && S_ISDIR(st.st_mode))
    raise(MGRC_E_IO_ERROR, "refactored stores (directories) are not supported by the B200 path: " + path);
  const uint64_t n = file_size(path);
  std::vector<uint8_t> f(n);
  read_exact(path, f.data(), n);
  // split_multiblock (mgrc.cpp:277-293)
  auto rd = [&](uint64_t at, int bytes) {
    if (at + static_cast<uint64_t>(bytes) > n) raise(MGRC_E_CORRUPT_STREAM, "truncated stream");
    uint64_t v = 0;
    for (int i = bytes - 1; i >= 0; --i) v = (v << 8) | f[at + static_cast<uint64_t>(i)];
    return v;
  };
  const uint64_t count = rd(0, 4);
  if (count == 0) raise(MGRC_E_CORRUPT_STREAM, "no blocks");
  std::vector<uint64_t> off(count);
  for (uint64_t i = 0; i < count; ++i) off[i] = rd(4 + 8 * i, 8);
  const uint64_t pos = 4 + 8 * count;
  std::vector<std::pair<uint64_t, uint64_t>> blocks(count);
  for (uint64_t i = 0; i < count; ++i) {
    const uint64_t b = off[i], e = i + 1 < count ? off[i + 1] : n;
    if (b < pos || e > n || b > e) raise(MGRC_E_CORRUPT_STREAM, "bad block offsets");
    blocks[i] = {b, e - b};
  }
  std::string text = "format: mgrc-multiblock\nblocks: " + std::to_string(count) + "\n";
  for (uint64_t i = 0; i < count; ++i) {
    char* d = nullptr;
    check(mgrc_gpu_describe(f.data() + blocks[i].first, blocks[i].second, &d));
    text += "--- block " + std::to_string(i) + " ---\n";
    text += d;
    mgrc_gpu_free(d);
  }
  std::fputs(text.c_str(), stdout);
  return 0;
}

void usage(FILE* f) {
  std::fputs(
      "mgrc-gpu: error-bounded compression of raw floating-point arrays on the B200 path\n"
      "usage:\n"
      "  mgrc-gpu compress --input F --output F --shape AxBxC --tol T [--dtype f32|f64] [--s inf|S]\n"
      "                    [--mode abs|rel] [--codec 0..2] [--chunk-mem SIZE] [--coords F] [--device N] [--gpus N]\n"
      "  mgrc-gpu decompress --input F --output F [--device N] [--gpus N]\n"
      "  mgrc-gpu inspect PATH\n",
      f);
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    usage(stderr);
    return 106;  // CLI11: a subcommand is required
  }
  const std::string sub = argv[1];
  if (sub == "-h" || sub == "--help") {
    usage(stdout);
    return 0;
  }
  try {
    if (sub == "compress")
      return run_compress(parse_args(argc, argv, 2,
                                     {"--input", "--output", "--shape", "--dtype", "--tol", "--s", "--mode", "--codec",
                                      "--chunk-mem", "--coords", "--device", "--gpus"}));
    if (sub == "decompress") return run_decompress(parse_args(argc, argv, 2, {"--input", "--output", "--device", "--gpus"}));
    if (sub == "inspect") return run_inspect(parse_args(argc, argv, 2, {}));
    if (sub == "refactor" || sub == "recompose")
      raise(MGRC_E_INVALID_STATE, sub + " (MDR stores, refactor.cpp) is not part of the B200 path");
    throw Usage("unknown subcommand " + sub);
  } catch (const Usage& e) {
    std::fprintf(stderr, "%s\n", e.what());
    usage(stderr);
    return 109;  // CLI11 parse errors exit non-zero without "error:"
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
}
