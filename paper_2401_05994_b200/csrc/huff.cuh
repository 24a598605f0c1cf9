// Huffman decode primitives over shared-memory staged stream words.
//
// The coded stream (codec.cpp:399-418: MSB-first canonical codes of the
// zigzag+LEB128 bytes, no sync points, no symbol count) is staged by tiles
// into shared memory with coalesced loads, byte-swapped to big-endian words;
// threads decode from there through a 64-bit bit buffer with 32-bit
// tile-local bit positions (the decoder itself: huff_tf.cuh).
//
// Decode LUT entry (u16, 2^maxlen entries): sym | len << 8 | (sym < 0x80) << 12.
#pragma once

#include "kernels.cuh"

namespace mgrc_gpu {
namespace dev {

constexpr int kTailWords = 32;  // look-ahead staged past a tile (open codewords / varints)
__host__ __device__ constexpr int stage_idx(int w) { return w + (w >> 5); }  // one pad word per 32

__device__ __forceinline__ uint32_t lut_len(uint32_t ent) { return (ent >> 8) & 15u; }
__device__ __forceinline__ uint32_t lut_term(uint32_t ent) { return (ent >> 12) & 1u; }

// Decode LUT in shared memory (G = false) or read through L1 from global
// memory (G = true: long codes, 2^maxlen entries would cost the CTA its
// occupancy — a 15-bit table is 64 KB).
template <bool G>
struct Lut {
  const uint16_t* p;
  __device__ __forceinline__ uint32_t operator[](uint32_t i) const {
    if constexpr (G) return __ldg(p + i);
    else return p[i];
  }
};
#ifndef MGRC_SMEM_LUT_MAXLEN
#define MGRC_SMEM_LUT_MAXLEN 12
#endif
constexpr int kSmemLutMaxLen = MGRC_SMEM_LUT_MAXLEN;  // longer tables stay in global memory

// Stages words [w0, w0 + nwords) of the stream (zero beyond nw).
__device__ __forceinline__ void stage_words(const uint32_t* __restrict__ w, uint64_t nw, uint64_t w0, uint32_t* sm,
                                            int nwords) {
  for (int i = threadIdx.x; i < nwords; i += blockDim.x) {
    const uint64_t gw = w0 + i;
    sm[stage_idx(i)] = gw < nw ? bswap32(__ldg(w + gw)) : 0u;
  }
}

// 64-bit MSB-first bit buffer over staged words; ≥ 33 valid bits after refill().
struct BitReader {
  const uint32_t* sm;
  uint64_t buf;
  int nbits;
  int nextw;
  __device__ __forceinline__ void init(const uint32_t* s, uint32_t local_bit) {
    sm = s;
    const int wi = static_cast<int>(local_bit >> 5), sh = static_cast<int>(local_bit & 31);
    buf = ((static_cast<uint64_t>(s[stage_idx(wi)]) << 32) | s[stage_idx(wi + 1)]) << sh;
    nbits = 64 - sh;
    nextw = wi + 2;
  }
  __device__ __forceinline__ void refill() {
    if (nbits <= 32) {
      buf |= static_cast<uint64_t>(sm[stage_idx(nextw)]) << (32 - nbits);
      nbits += 32;
      ++nextw;
    }
  }
  __device__ __forceinline__ uint32_t peek(int maxlen) const {
    return static_cast<uint32_t>(buf >> 32) >> (32 - maxlen);
  }
  __device__ __forceinline__ void consume(uint32_t l) {
    buf <<= l;
    nbits -= static_cast<int>(l);
  }
};

}  // namespace dev
}  // namespace mgrc_gpu
