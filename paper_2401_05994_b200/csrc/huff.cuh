// Self-synchronising parallel Huffman decode of the varint byte stream,
// shared-memory staged.
//
// The coded stream (codec.cpp:399-418: MSB-first canonical codes of the
// zigzag+LEB128 bytes, no sync points, no symbol count) is cut into
// subsequences of kSeqBits bits; a CTA owns kDecThreads consecutive
// subsequences.  The CTA stages its bit range (plus a warm-up prefix and a
// look-ahead tail) into shared memory with coalesced loads, byte-swapped to
// big-endian words; every thread then decodes from shared memory through a
// 64-bit bit buffer with 32-bit CTA-local bit positions.
//
// Decode LUT entry (u16, 2^maxlen entries): sym | len << 8 | (sym < 0x80) << 12.
#pragma once

#include "kernels.cuh"

namespace mgrc_gpu {
namespace dev {

constexpr int kWarmBits = 1024;  // warm-up decoded before each subsequence's nominal start
constexpr int kSyncWarm = 8;     // overlap subsequences per sync CTA (never published)
constexpr int kSyncReal = kDecThreads - kSyncWarm;
constexpr int kStageWords = kDecThreads * kSeqBits / 32;
constexpr int kTailWords = 32;   // look-ahead past the last subsequence (open codewords / varints)
constexpr int kStageTotal = kWarmBits / 32 + kStageWords + kTailWords + 4;
__host__ __device__ constexpr int stage_idx(int w) { return w + (w >> 5); }  // one pad word per 32
constexpr int kStageSmemWords = stage_idx(kStageTotal) + 2;

__device__ __forceinline__ uint32_t lut_len(uint32_t ent) { return (ent >> 8) & 15u; }
__device__ __forceinline__ uint32_t lut_term(uint32_t ent) { return (ent >> 12) & 1u; }

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

// Skip codewords until the first boundary >= target; returns it.  tl: local
// stream end (a codeword that would run past it stops the walk).
__device__ __forceinline__ uint32_t walk_to(BitReader& br, const uint16_t* lut, int maxlen, uint32_t p,
                                            uint32_t target, uint32_t tl) {
  while (p < target) {
    br.refill();
    const uint32_t l = lut_len(lut[br.peek(maxlen)]);
    if (p + l > tl) break;
    p += l;
    br.consume(l);
  }
  return p;
}

// Count codewords / varint terminators starting in [p, end); returns the exit.
__device__ __forceinline__ uint32_t count_to(BitReader& br, const uint16_t* lut, int maxlen, uint32_t p, uint32_t end,
                                             uint32_t tl, uint32_t& nterm, uint32_t& last_ent) {
  uint32_t nt = 0, last = 0;
  if (end + 16 <= tl) {  // no codeword can run past the stream end: two symbols per refill
    while (p < end) {
      br.refill();
      uint32_t ent = lut[br.peek(maxlen)];
      uint32_t l = lut_len(ent);
      p += l;
      nt += lut_term(ent);
      last = ent;
      br.consume(l);
      if (p >= end) break;
      ent = lut[br.peek(maxlen)];
      l = lut_len(ent);
      p += l;
      nt += lut_term(ent);
      last = ent;
      br.consume(l);
    }
  } else {
    while (p < end) {
      br.refill();
      const uint32_t ent = lut[br.peek(maxlen)];
      const uint32_t l = lut_len(ent);
      if (p + l > tl) break;
      p += l;
      nt += lut_term(ent);
      last = ent;
      br.consume(l);
    }
  }
  nterm = nt;
  last_ent = last;
  return p;
}

// Pass 1: every subsequence j is decoded from kWarmBits before its nominal
// start S_j (a prefix code resynchronises within a few codewords; SURVEY
// Appendix A measures p99 < 3.1 kbit, mean ≈ 0.1–0.3 kbit); its start F_j is
// the first codeword boundary >= S_j and its exit E_j the first boundary >=
// S_j + kSeqBits.  Inside the CTA E_{j-1} == F_j is checked; the (rare)
// mismatching subsequences are compacted into a list and re-decoded from
// E_{j-1} until consistent.  Subsequence 0 starts at bit 0, so consistency at
// every boundary (CTA edges: k_huff_fix_s) proves every F_j is a true
// codeword boundary.
__global__ void __launch_bounds__(kDecThreads) k_huff_sync_s(const uint32_t* __restrict__ w, uint64_t nw, uint64_t T,
                                                             const uint16_t* __restrict__ lut_g, int maxlen,
                                                             uint64_t nseq, SeqInfo* __restrict__ seq) {
  extern __shared__ uint32_t dyn[];
  uint32_t* sm = dyn;
  uint16_t* lut = reinterpret_cast<uint16_t*>(dyn + kStageSmemWords);
  __shared__ uint32_t sexit[kDecThreads], sstart[kDecThreads];
  __shared__ int bad[kDecThreads];
  __shared__ int nbad;
  const int lutn = 1 << maxlen;
  for (int k = threadIdx.x; k < lutn; k += blockDim.x) lut[k] = lut_g[k];
  // thread t <-> subsequence j = c·kSyncReal - kSyncWarm + t: the first
  // kSyncWarm threads re-decode the predecessor CTA's last subsequences
  // (never published) so that the CTA's first published start is true unless a
  // desynchronisation outlasts kSyncWarm subsequences (then k_huff_fix_s).
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * kSyncReal - kSyncWarm;
  const uint64_t base = j0 > 0 ? static_cast<uint64_t>(j0) * kSeqBits - kWarmBits : 0;  // word aligned
  stage_words(w, nw, base >> 5, sm, kStageTotal);
  __syncthreads();
  const uint32_t tl = static_cast<uint32_t>(umin64(T - base, 0x7FFFFFFFu));
  const int64_t js = j0 + static_cast<int64_t>(threadIdx.x);
  const bool valid = js >= 0 && static_cast<uint64_t>(js) < nseq;
  const uint64_t j = valid ? static_cast<uint64_t>(js) : 0;
  uint32_t F = 0, E = 0, nterm = 0, last = 0, end = 0;
  if (valid) {
    const uint32_t S = static_cast<uint32_t>(j * kSeqBits - base);
    end = min(S + static_cast<uint32_t>(kSeqBits), tl);
    const uint32_t from = S >= kWarmBits ? S - kWarmBits : 0;
    BitReader br;
    br.init(sm, from);
    F = walk_to(br, lut, maxlen, from, S, tl);
    E = count_to(br, lut, maxlen, F, end, tl, nterm, last);
  }
  sexit[threadIdx.x] = E;
  sstart[threadIdx.x] = F;
  for (;;) {
    if (threadIdx.x == 0) nbad = 0;
    __syncthreads();
    if (valid && threadIdx.x > 0 && js > 0 && sexit[threadIdx.x - 1] != sstart[threadIdx.x])
      bad[atomicAdd(&nbad, 1)] = threadIdx.x;
    __syncthreads();
    const int nb = nbad;
    if (nb == 0) break;
    int t = -1;
    uint32_t from = 0;
    if (threadIdx.x < nb) {
      t = bad[threadIdx.x];
      from = sexit[t - 1];
    }
    __syncthreads();
    if (t >= 0) {  // compacted re-decode of subsequence t from its predecessor's exit
      const uint64_t jj = static_cast<uint64_t>(j0 + t);
      const uint32_t e2 = min(static_cast<uint32_t>(jj * kSeqBits - base) + static_cast<uint32_t>(kSeqBits), tl);
      BitReader br;
      br.init(sm, from);
      uint32_t nt2, last2;
      const uint32_t ex = count_to(br, lut, maxlen, from, e2, tl, nt2, last2);
      sexit[t] = ex;
      sstart[t] = from;
      SeqInfo s2;
      s2.start = base + from;
      s2.exit = base + ex;
      s2.nsym = 0;
      s2.nterm = nt2;
      s2.last_cont = (last2 & 0xFF) >= 0x80;
      s2.pad = 0;
      if (t >= kSyncWarm) seq[jj] = s2;
    }
    __syncthreads();
  }
  if (valid && threadIdx.x >= kSyncWarm && sstart[threadIdx.x] == F && sexit[threadIdx.x] == E) {  // never re-decoded
    SeqInfo s;
    s.start = base + F;
    s.exit = base + E;
    s.nsym = 0;
    s.nterm = nterm;
    s.last_cont = (last & 0xFF) >= 0x80;
    s.pad = 0;
    seq[j] = s;
  }
}

// CTA-edge consistency: one 32-thread CTA per edge b (first subsequence j =
// b·kDecThreads).  When E_{j-1} != F_j, the following subsequences are staged
// and re-decoded (thread 0, from shared memory) until a subsequence's exit is
// unchanged.  *changed tells the host to run another round (an edge fix can
// change the exit of a CTA's last subsequence, i.e. the next edge).
constexpr int kFixSeqs = 4;  // subsequences staged per round
constexpr int kFixWords = kFixSeqs * kSeqBits / 32 + kTailWords + 4;

__global__ void __launch_bounds__(32) k_huff_fix_s(const uint32_t* __restrict__ w, uint64_t nw, uint64_t T,
                                                   const uint16_t* __restrict__ lut_g, int maxlen, uint64_t nseq,
                                                   SeqInfo* seq, unsigned int* changed) {
  extern __shared__ uint32_t dyn[];
  uint32_t* sm = dyn;
  uint16_t* lut = reinterpret_cast<uint16_t*>(dyn + stage_idx(kFixWords) + 2);
  __shared__ int s_go;
  __shared__ unsigned long long s_from;
  const uint64_t b = blockIdx.x + 1;  // edge b: first published subsequence of sync CTA b
  uint64_t j = b * kSyncReal;
  const uint64_t jend = umin64(j + kSyncReal, nseq);
  if (j >= nseq) return;
  bool lut_ready = false;
  while (j < jend) {
    if (threadIdx.x == 0) {
      const unsigned long long pe = *reinterpret_cast<volatile unsigned long long*>(&seq[j - 1].exit);
      s_go = pe != seq[j].start;
      s_from = pe;
    }
    __syncthreads();
    if (!s_go) break;
    if (!lut_ready) {
      const int lutn = 1 << maxlen;
      for (int k = threadIdx.x; k < lutn; k += blockDim.x) lut[k] = lut_g[k];
      lut_ready = true;
    }
    const uint64_t base = (s_from >> 5) << 5;
    stage_words(w, nw, base >> 5, sm, kFixWords);
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t tl = static_cast<uint32_t>(umin64(T - base, 0x7FFFFFFFu));
      uint64_t jj = j;
      uint32_t from = static_cast<uint32_t>(s_from - base);
      // re-decode up to kFixSeqs subsequences inside the staged window
      for (int r = 0; r < kFixSeqs && jj < jend; ++r, ++jj) {
        const uint64_t e64 = umin64((jj + 1) * kSeqBits, T);
        if (e64 - base > static_cast<uint64_t>(kFixSeqs) * kSeqBits) break;  // beyond the window: next round
        BitReader br;
        br.init(sm, from);
        uint32_t nt, last;
        const uint32_t ex = count_to(br, lut, maxlen, from, static_cast<uint32_t>(e64 - base), tl, nt, last);
        const SeqInfo old = seq[jj];
        SeqInfo s;
        s.start = base + from;
        s.exit = base + ex;
        s.nsym = 0;
        s.nterm = nt;
        s.last_cont = (last & 0xFF) >= 0x80;
        s.pad = 0;
        seq[jj] = s;
        __threadfence();
        atomicOr(changed, 1u);
        if (old.exit == s.exit) {  // resynchronised: the rest of the CTA is consistent
          jj = jend;
          break;
        }
        from = ex;
      }
      s_from = jj;  // reuse as "next j"
    }
    __syncthreads();
    j = s_from;
    __syncthreads();
  }
}

// Pass 2: re-decode each synchronised subsequence and assemble the varints
// that START in it (an open value is finished by decoding on, ≤ 10 bytes).
// Values beyond N (decoded zero padding) are never stored, as the reference
// never reads them (codec.cpp:475-481).  Stores are staged per thread in
// 32-byte aligned chunks and written as 16-byte vectors.
template <typename Z>
__global__ void __launch_bounds__(kDecThreads) k_huff_emit_s(const uint32_t* __restrict__ w, uint64_t nw, uint64_t T,
                                                             const uint16_t* __restrict__ lut_g, int maxlen,
                                                             uint64_t nseq, const SeqInfo* __restrict__ seq,
                                                             const unsigned long long* __restrict__ term_off,
                                                             uint64_t N, Z* __restrict__ zz, DecodeStatus* st) {
  constexpr int CH = 32 / sizeof(Z);  // values per 32-byte chunk
  extern __shared__ uint32_t dyn[];
  uint32_t* sm = dyn;
  uint16_t* lut = reinterpret_cast<uint16_t*>(dyn + kStageSmemWords);
  __shared__ __align__(16) Z slot[kDecThreads][CH];
  const int lutn = 1 << maxlen;
  for (int k = threadIdx.x; k < lutn; k += blockDim.x) lut[k] = lut_g[k];
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kDecThreads * kSeqBits;
  stage_words(w, nw, base >> 5, sm, kStageTotal);
  __syncthreads();
  const uint64_t j = blockIdx.x * static_cast<uint64_t>(kDecThreads) + threadIdx.x;
  if (j >= nseq) return;
  const SeqInfo s = seq[j];
  bool skipping = j > 0 && seq[j - 1].last_cont;
  uint64_t k = term_off[j];
  if (k >= N && !skipping) return;
  const uint64_t k_first = k + (skipping ? 1 : 0);
  Z* my = slot[threadIdx.x];
  auto flush = [&](uint64_t upto) {  // values [chunk start, upto) of the current chunk
    const uint64_t c0 = (upto - 1) & ~static_cast<uint64_t>(CH - 1);
    if (c0 >= k_first && upto - c0 == CH) {
      const uint4* src = reinterpret_cast<const uint4*>(my);
      uint4* dst = reinterpret_cast<uint4*>(zz + c0);
      dst[0] = src[0];
      dst[1] = src[1];
    } else {
      for (uint64_t q = umax64(c0, k_first); q < upto; ++q) zz[q] = my[q & (CH - 1)];
    }
  };
  const uint32_t tl = static_cast<uint32_t>(umin64(T - base, 0x7FFFFFFFu));
  uint32_t p = static_cast<uint32_t>(s.start - base);
  const uint32_t ex = static_cast<uint32_t>(s.exit - base);
  uint64_t acc = 0;
  int nb = 0;
  unsigned err = 0, wide = 0;
  BitReader br;
  br.init(sm, p);
  for (;;) {
    if (p >= ex && nb == 0) break;
    if (k >= N) break;
    br.refill();
    const uint32_t ent = lut[br.peek(maxlen)];
    const uint32_t l = lut_len(ent);
    if (p + l > tl) {  // stream ends inside an open value
      err = 2;
      break;
    }
    const uint32_t b = ent & 0xFF;
    p += l;
    br.consume(l);
    if (skipping) {
      if (b < 0x80) {
        skipping = false;
        ++k;
      }
      continue;
    }
    if (nb == 9 && (b & 0xFE)) {  // varint overflows 64 bits (codec.cpp:80-81)
      err = 1;
      break;
    }
    acc |= static_cast<uint64_t>(b & 0x7F) << (7 * nb);
    ++nb;
    if (b < 0x80) {
      if (sizeof(Z) == 4 && acc > 0xFFFFFFFFull) wide = 1;
      my[k & (CH - 1)] = static_cast<Z>(acc);
      if (((k + 1) & (CH - 1)) == 0) flush(k + 1);
      if (k == N - 1) {  // exhausted_clean (codec.cpp:370-375)
        st->end_bit = base + p;
        const uint32_t rest = tl - p;
        br.refill();
        st->clean = rest < 8 && (rest == 0 || (static_cast<uint32_t>(br.buf >> 32) >> (32 - rest)) == 0);
      }
      ++k;
      acc = 0;
      nb = 0;
    }
  }
  if ((k & (CH - 1)) != 0 && k > k_first) flush(k);
  if (err) atomicMax(&st->error, err);
  if (wide) atomicOr(&st->wide, 1u);
}

}  // namespace dev
}  // namespace mgrc_gpu
