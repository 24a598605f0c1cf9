// Minimal reference-API client: the reference library's own code (grid,
// codec, error, ... compiled from /root/reference/proj/src) with
// container.cpp replaced by integration/container_gpu.cpp, so the calls below
// are the reference's public API running on the B200 path.
//
//   mgrc_gpu_driver compress <in.raw> <f32|f64> <tol> <inf|s> <s> <abs|rel> <out.mgrc> <n0> [n1 ...]
//   mgrc_gpu_driver decompress <in.mgrc> <out.raw>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "mgrc/container.hpp"
#include "mgrc/error.hpp"

static std::vector<char> slurp(const char* p) {
  std::ifstream f(p, std::ios::binary);
  return std::vector<char>((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
}

int main(int argc, char** argv) {
  try {
    if (argc >= 10 && std::string(argv[1]) == "compress") {
      const auto raw = slurp(argv[2]);
      const bool f32 = std::string(argv[3]) == "f32";
      mgrc::ErrorSpec spec;
      spec.tol = std::atof(argv[4]);
      spec.norm = std::string(argv[5]) == "inf" ? mgrc::Norm::inf : mgrc::Norm::s;
      spec.smoothness = std::atof(argv[6]);
      spec.mode = std::string(argv[7]) == "abs" ? mgrc::Mode::abs : mgrc::Mode::rel;
      std::vector<std::size_t> shape;
      for (int i = 9; i < argc; ++i) shape.push_back(std::strtoull(argv[i], nullptr, 10));
      const auto grid = mgrc::make_grid(shape);
      mgrc::CompressedContainer c;
      if (f32)
        c = mgrc::compress(std::span<const float>(reinterpret_cast<const float*>(raw.data()), raw.size() / 4), grid,
                           spec, mgrc::Codec::huffman);
      else
        c = mgrc::compress(std::span<const double>(reinterpret_cast<const double*>(raw.data()), raw.size() / 8),
                           grid, spec, mgrc::Codec::huffman);
      std::ofstream(argv[8], std::ios::binary).write(reinterpret_cast<const char*>(c.bytes.data()), c.bytes.size());
      std::printf("%s", mgrc::describe(mgrc::inspect(c.bytes)).c_str());
      return 0;
    }
    if (argc == 4 && std::string(argv[1]) == "decompress") {
      const auto blob = slurp(argv[2]);
      const auto d = mgrc::decompress(std::span<const std::uint8_t>(
          reinterpret_cast<const std::uint8_t*>(blob.data()), blob.size()));
      std::ofstream out(argv[3], std::ios::binary);
      if (d.dtype == mgrc::DType::f32)
        out.write(reinterpret_cast<const char*>(d.f32().data()), d.f32().size() * 4);
      else
        out.write(reinterpret_cast<const char*>(d.f64().data()), d.f64().size() * 8);
      return 0;
    }
    std::fprintf(stderr, "usage: see integration/driver.cpp\n");
    return 2;
  } catch (const mgrc::error& e) {
    std::fprintf(stderr, "mgrc::error: %s\n", e.what());
    return 1;
  }
}
