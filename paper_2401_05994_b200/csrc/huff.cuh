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

#ifndef MGRC_WARM_BITS
#define MGRC_WARM_BITS 512
#endif
constexpr int kWarmBits = MGRC_WARM_BITS;  // warm-up decoded before each subsequence's nominal start
#ifndef MGRC_SYNC_WARM
#define MGRC_SYNC_WARM 16
#endif
constexpr int kSyncWarm = MGRC_SYNC_WARM;  // overlap subsequences per sync CTA (never published)
#ifndef MGRC_SYNC_THREADS
#define MGRC_SYNC_THREADS 128
#endif
constexpr int kSyncThreads = MGRC_SYNC_THREADS;  // subsequences (threads) per sync CTA
constexpr int kSyncReal = kSyncThreads - kSyncWarm;
#ifndef MGRC_SYNC_ROUNDS
#define MGRC_SYNC_ROUNDS (1 << 20)
#endif
constexpr int kSyncRounds = MGRC_SYNC_ROUNDS;  // in-CTA resynchronisation rounds; longer chains go to the tables
#ifndef MGRC_EMIT_THREADS
#define MGRC_EMIT_THREADS 128
#endif
constexpr int kEmitThreads = MGRC_EMIT_THREADS;  // subsequences (threads) per emit CTA
constexpr int kStageWords = kEmitThreads * kSeqBits / 32;
constexpr int kTailWords = 32;   // look-ahead past the last subsequence (open codewords / varints)
constexpr int kStageTotal = kWarmBits / 32 + kStageWords + kTailWords + 4;
__host__ __device__ constexpr int stage_idx(int w) { return w + (w >> 5); }  // one pad word per 32
constexpr int kStageSmemWords = stage_idx(kStageTotal) + 2;
constexpr int kSyncStageTotal = kWarmBits / 32 + kSyncThreads * kSeqBits / 32 + kTailWords + 4;
constexpr int kSyncSmemWords = stage_idx(kSyncStageTotal) + 2;

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

// Skip codewords until the first boundary >= target; returns it.  tl: local
// stream end (a codeword that would run past it stops the walk).
template <class LT>
__device__ __forceinline__ uint32_t walk_to(BitReader& br, const LT& lut, int maxlen, uint32_t p,
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
template <class LT>
__device__ __forceinline__ uint32_t count_to(BitReader& br, const LT& lut, int maxlen, uint32_t p, uint32_t end,
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
template <bool G>
__global__ void __launch_bounds__(kSyncThreads) k_huff_sync_s(const uint32_t* __restrict__ w, uint64_t nw, uint64_t T,
                                                             const uint16_t* __restrict__ lut_g, int maxlen,
                                                             uint64_t nseq, SeqInfo* __restrict__ seq,
                                                             unsigned int* capped) {
  extern __shared__ uint32_t dyn[];
  uint32_t* sm = dyn;
  uint16_t* lut_s = reinterpret_cast<uint16_t*>(dyn + kSyncSmemWords);
  __shared__ uint32_t sexit[kSyncThreads], sstart[kSyncThreads];
  __shared__ int bad[kSyncThreads];
  __shared__ int nbad;
  const int lutn = 1 << maxlen;
  if (!G)
    for (int k = threadIdx.x; k < lutn; k += blockDim.x) lut_s[k] = lut_g[k];
  const Lut<G> lut{G ? lut_g : lut_s};
  // thread t <-> subsequence j = c·kSyncReal - kSyncWarm + t: the first
  // kSyncWarm threads re-decode the predecessor CTA's last subsequences
  // (never published) so that the CTA's first published start is true unless a
  // desynchronisation outlasts kSyncWarm subsequences (then k_huff_fix_s).
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * kSyncReal - kSyncWarm;
  const uint64_t base = j0 > 0 ? static_cast<uint64_t>(j0) * kSeqBits - kWarmBits : 0;  // word aligned
  stage_words(w, nw, base >> 5, sm, kSyncStageTotal);
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
  // in-CTA re-decode rounds, capped: a chain still open after kSyncRounds is
  // left inconsistent and resolved by the transfer-table windows (host loop)
  for (int round = 0;; ++round) {
    if (threadIdx.x == 0) nbad = 0;
    __syncthreads();
    if (valid && threadIdx.x > 0 && js > 0 && sexit[threadIdx.x - 1] != sstart[threadIdx.x])
      bad[atomicAdd(&nbad, 1)] = threadIdx.x;
    __syncthreads();
    const int nb = nbad;
    if (nb == 0) break;
    if (round == kSyncRounds) {  // leave the rest to the transfer-table windows
      if (threadIdx.x == 0) atomicOr(capped, 1u);
      break;
    }
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
#ifndef MGRC_FIX_WALK
#define MGRC_FIX_WALK kSyncReal
#endif
constexpr int kFixWalk = MGRC_FIX_WALK;  // subsequences one edge walk may rewrite (longer chains go to the tables)
constexpr int kFixWords = kFixSeqs * kSeqBits / 32 + kTailWords + 4;

__global__ void __launch_bounds__(32) k_huff_fix_s(const uint32_t* __restrict__ w, uint64_t nw, uint64_t T,
                                                   const uint16_t* __restrict__ lut_g, int maxlen, uint64_t nseq,
                                                   SeqInfo* seq, unsigned int* changed) {
  extern __shared__ uint32_t dyn[];
  uint32_t* sm = dyn;
  uint16_t* lut_s = reinterpret_cast<uint16_t*>(dyn + stage_idx(kFixWords) + 2);
  const Lut<false> lut{lut_s};
  __shared__ int s_go;
  __shared__ unsigned long long s_from;
  const uint64_t b = blockIdx.x + 1;  // edge b: first published subsequence of sync CTA b
  uint64_t j = b * kSyncReal;
  const uint64_t jend = umin64(j + kFixWalk, nseq);
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
      for (int k = threadIdx.x; k < lutn; k += blockDim.x) lut_s[k] = lut_g[k];
      lut_ready = true;
    }
    const uint64_t base = (s_from >> 5) << 5;
    stage_words(w, nw, base >> 5, sm, kFixWords);
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t tl = static_cast<uint32_t>(umin64(T - base, 0x7FFFFFFFu));
      uint64_t jj = j;
      bool conv = false;
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
          conv = true;
          break;
        }
        from = ex;
      }
      if (conv) {
        jj = jend;
      } else if (jj >= jend && jend < umin64((b + 1) * kSyncReal, nseq)) {
        atomicOr(changed, 2u);  // stopped at the walk cap inside the CTA: the tables take over
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
template <typename Z, bool G>
__global__ void __launch_bounds__(kEmitThreads) k_huff_emit_s(const uint32_t* __restrict__ w, uint64_t nw, uint64_t T,
                                                             const uint16_t* __restrict__ lut_g, int maxlen,
                                                             uint64_t nseq, const SeqInfo* __restrict__ seq,
                                                             const unsigned long long* __restrict__ term_off,
                                                             uint64_t N, Z* __restrict__ zz, DecodeStatus* st) {
  constexpr int CH = 32 / sizeof(Z);  // values per 32-byte chunk
  extern __shared__ uint32_t dyn[];
  uint32_t* sm = dyn;
  uint16_t* lut_s = reinterpret_cast<uint16_t*>(dyn + kStageSmemWords);
  __shared__ __align__(16) Z slot[kEmitThreads][CH];
  const int lutn = 1 << maxlen;
  if (!G)
    for (int k = threadIdx.x; k < lutn; k += blockDim.x) lut_s[k] = lut_g[k];
  const Lut<G> lut{G ? lut_g : lut_s};
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kEmitThreads * kSeqBits;
  stage_words(w, nw, base >> 5, sm, kStageTotal);
  __syncthreads();
  const uint64_t j = blockIdx.x * static_cast<uint64_t>(kEmitThreads) + threadIdx.x;
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
  const bool near_end = ex + 256 >= tl;  // only then can a codeword run past the stream end
  unsigned err = 0, wide = 0;
  BitReader br;
  br.init(sm, p);
  if (skipping) {  // the value open at the start began in the previous subsequence: skip to its end
    for (;;) {
      br.refill();
      const uint32_t ent = lut[br.peek(maxlen)];
      const uint32_t l = lut_len(ent);
      if (p + l > tl) {
        err = 2;
        break;
      }
      p += l;
      br.consume(l);
      if (lut_term(ent)) {
        ++k;
        break;
      }
    }
  }
  // values stored by this thread: indices k .. ; `room` of them before N
  const uint64_t room64 = k < N ? N - k : 0;
  const uint32_t room = static_cast<uint32_t>(umin64(room64, 0xFFFFFFFFu));
  const uint32_t k_lo = static_cast<uint32_t>(k);  // low bits for the chunk slots
  uint32_t kk = 0;
  uint64_t acc = 0;
  uint32_t sh = 0;  // 7 × bytes of the open value
  while (!err) {
    if (p >= ex && sh == 0) break;
    if (kk >= room) break;
    br.refill();
    const uint32_t ent = lut[br.peek(maxlen)];
    const uint32_t l = lut_len(ent);
    if (near_end && p + l > tl) {  // stream ends inside an open value
      err = 2;
      break;
    }
    p += l;
    br.consume(l);
    if (sh == 63 && (ent & 0xFEu)) {  // varint overflows 64 bits (codec.cpp:80-81)
      err = 1;
      break;
    }
    acc |= static_cast<uint64_t>(ent & 0x7Fu) << sh;
    if (!lut_term(ent)) {
      sh += 7;
      continue;
    }
    if (sizeof(Z) == 4 && (acc >> 32)) wide = 1;
    const uint32_t ki = k_lo + kk;
    my[ki & (CH - 1)] = static_cast<Z>(acc);
    if (((ki + 1) & (CH - 1)) == 0) flush(k + kk + 1);
    if (kk + 1 == room && room64 <= 0xFFFFFFFFu) {  // the N-th value: exhausted_clean (codec.cpp:370-375)
      st->end_bit = base + p;
      const uint32_t rest = tl - p;
      br.refill();
      st->clean = rest < 8 && (rest == 0 || (static_cast<uint32_t>(br.buf >> 32) >> (32 - rest)) == 0);
    }
    ++kk;
    acc = 0;
    sh = 0;
  }
  k += kk;
  if ((k & (CH - 1)) != 0 && k > k_first) flush(k);
  if (err) atomicMax(&st->error, err);
  if (wide) atomicOr(&st->wide, 1u);
}

// ---------------------------------------------------------------------------
// Long desynchronisation chains (periodic stretches of the stream can keep a
// decoder out of phase for megabits, e.g. long runs of one multi-bit code):
// instead of walking them serially, tabulate for every subsequence of a
// window the decode from EVERY entry offset o < maxlen — exit offset into the
// next subsequence, terminators, last-continues — and compose the tables with
// a parallel scan from the window's known true entry.  The decode from o = 0
// is recorded as boundary / terminator bitmaps; the other offsets are walked
// until they land on a recorded boundary (then both coincide).
constexpr int kTfOffs = 16;
constexpr int kTfThreads = 64;
constexpr int kTfStage = kTfThreads * kSeqBits / 32 + kTailWords + 4;
constexpr int kTfMapStride = kSeqBits / 32 + 1;

struct TfTab {
  uint8_t ex[kTfOffs];    // exit - S_{j+1}
  uint16_t nt[kTfOffs];   // varint terminators
  uint32_t lc;            // bit o: last codeword continues a varint
};

__device__ __forceinline__ uint32_t tf_terms_before(const uint32_t* Mm, uint32_t rel) {
  uint32_t c = 0;
  const uint32_t wq = rel >> 5;
  for (uint32_t w = 0; w < wq; ++w) c += __popc(Mm[w]);
  return c + __popc(Mm[wq] & ((1u << (rel & 31)) - 1u));
}

constexpr uint64_t kTfWin = 512;  // subsequences per window in the first round (later rounds: ×4 per round)

// grid: (window, CTA within the window); window w covers [starts[w], starts[w] + wlen) ∩ [0, nseq)
template <bool G>
__global__ void __launch_bounds__(kTfThreads) k_tf_tables(const uint32_t* __restrict__ w, uint64_t nw, uint64_t T,
                                                          const uint16_t* __restrict__ lut_g, int maxlen,
                                                          const unsigned long long* __restrict__ starts,
                                                          uint64_t nseq, TfTab* __restrict__ tabs_all, uint32_t wlen) {
  const uint32_t ctas_per_win = wlen / kTfThreads;
  const uint64_t win = blockIdx.x / ctas_per_win;
  const uint64_t j_first = starts[win];
  const uint64_t count = umin64(wlen, nseq - j_first);
  TfTab* tabs = tabs_all + win * wlen;
  extern __shared__ uint32_t dyn[];
  uint32_t* sm = dyn;                                              // staged words
  uint32_t* maps = sm + stage_idx(kTfStage) + 2;                   // B0 | M0 | B1 | M1 per thread
  uint16_t* lut_s = reinterpret_cast<uint16_t*>(maps + 4 * kTfThreads * kTfMapStride);
  const Lut<G> lut{G ? lut_g : lut_s};
  const int lutn = 1 << maxlen;
  if (!G)
    for (int k = threadIdx.x; k < lutn; k += blockDim.x) lut_s[k] = lut_g[k];
  const uint64_t j0 = j_first + static_cast<uint64_t>(blockIdx.x % ctas_per_win) * kTfThreads;
  if (j0 >= j_first + count) return;
  const uint64_t base = j0 * kSeqBits;
  stage_words(w, nw, base >> 5, sm, kTfStage);
  __syncthreads();
  const uint64_t j = j0 + threadIdx.x;
  if (j >= j_first + count || j >= nseq) return;
  const uint32_t tl = static_cast<uint32_t>(umin64(T - base, 0x7FFFFFFFu));
  const uint32_t S = threadIdx.x * kSeqBits;
  const uint32_t end = min(S + static_cast<uint32_t>(kSeqBits), tl);
  const bool last_seq = j + 1 == nseq;
  // two recorded tracks: the decode from offset 0, and the first offset that does
  // not merge into it (periodic stretches usually have exactly two phases)
  uint32_t* B[2] = {maps + threadIdx.x * kTfMapStride, maps + (2 * kTfThreads + threadIdx.x) * kTfMapStride};
  uint32_t* M[2] = {maps + (kTfThreads + threadIdx.x) * kTfMapStride,
                    maps + (3 * kTfThreads + threadIdx.x) * kTfMapStride};
  uint32_t tex[2] = {0, 0}, tn[2] = {0, 0}, tlc[2] = {0, 0};
  int ntracks = 0;
  auto record = [&](uint32_t from, int k) {  // full decode from `from`, recorded as track k
    uint32_t* Bm = B[k];
    uint32_t* Mm = M[k];
    for (int q = 0; q < kSeqBits / 32; ++q) Bm[q] = Mm[q] = 0u;
    uint32_t p = from, last = 0, n = 0;
    BitReader br;
    br.init(sm, p);
    while (p < end) {
      br.refill();
      const uint32_t ent = lut[br.peek(maxlen)];
      const uint32_t l = lut_len(ent);
      if (p + l > tl) break;
      const uint32_t rel = p - S;
      Bm[rel >> 5] |= 1u << (rel & 31);
      Mm[rel >> 5] |= lut_term(ent) << (rel & 31);
      n += lut_term(ent);
      last = lut_term(ent) ^ 1u;
      p += l;
      br.consume(l);
    }
    tex[k] = p;
    tn[k] = n;
    tlc[k] = p > from ? last : 0u;
  };
  record(S, 0);
  ntracks = 1;
  TfTab t;
  t.lc = 0;
  for (int o = 0; o < kTfOffs; ++o) {
    uint32_t eo = tex[0], no = tn[0], lco = tlc[0];
    if (o > 0 && o < maxlen) {
      if (S + o >= end) {
        eo = S + o;
        no = 0;
        lco = 0;
      } else {
        uint32_t q = S + o, walked = 0, lastw = 0;
        int hit = -1;
        bool any = false;
        BitReader bo;
        bo.init(sm, q);
        while (q < end) {
          const uint32_t rel = q - S;
          if ((B[0][rel >> 5] >> (rel & 31)) & 1u) {
            hit = 0;
            break;
          }
          if (ntracks > 1 && ((B[1][rel >> 5] >> (rel & 31)) & 1u)) {
            hit = 1;
            break;
          }
          bo.refill();
          const uint32_t ent = lut[bo.peek(maxlen)];
          const uint32_t l = lut_len(ent);
          if (q + l > tl) break;
          walked += lut_term(ent);
          lastw = lut_term(ent) ^ 1u;
          any = true;
          q += l;
          bo.consume(l);
        }
        if (hit >= 0) {
          eo = tex[hit];
          no = walked + (tn[hit] - tf_terms_before(M[hit], q - S));
          lco = tlc[hit];
        } else {
          eo = q;
          no = walked;
          lco = any ? lastw : 0u;
          if (ntracks == 1) {  // keep this phase as the second recorded track
            record(S + o, 1);
            ntracks = 2;
          }
        }
      }
    }
    t.ex[o] = last_seq ? 0 : static_cast<uint8_t>(min(eo - end, 255u));
    t.nt[o] = static_cast<uint16_t>(no);
    t.lc |= lco << o;
  }
  tabs[j - j_first] = t;
}

// One CTA: compose the window's tables from the true entry offset of its first
// subsequence and rewrite every subsequence's (start, exit, nterm, last_cont).
constexpr int kTfResolveThreads = 512;

// grid: one CTA per window
__global__ void __launch_bounds__(kTfResolveThreads) k_tf_resolve(const TfTab* __restrict__ tabs_all,
                                                                  const unsigned long long* __restrict__ starts,
                                                                  uint64_t nseq, uint64_t T, SeqInfo* seq,
                                                                  uint32_t wlen) {
  const uint64_t j_first = starts[blockIdx.x];
  const uint64_t count = umin64(wlen, nseq - j_first);
  const TfTab* tabs = tabs_all + static_cast<uint64_t>(blockIdx.x) * wlen;
  __shared__ uint8_t maps[kTfResolveThreads][kTfOffs];
  __shared__ uint8_t tmp[kTfResolveThreads][kTfOffs];
  const int t = threadIdx.x;
  const uint64_t per = (count + kTfResolveThreads - 1) / kTfResolveThreads;
  const uint64_t a = umin64(count, t * per), b = umin64(count, a + per);
  // 1. compose this thread's chunk: map o -> entry offset after the chunk
  uint8_t f[kTfOffs];
#pragma unroll
  for (int o = 0; o < kTfOffs; ++o) f[o] = static_cast<uint8_t>(o);
  for (uint64_t i = a; i < b; ++i) {
    const TfTab& tb = tabs[i];
#pragma unroll
    for (int o = 0; o < kTfOffs; ++o) f[o] = tb.ex[f[o] & 15];
  }
#pragma unroll
  for (int o = 0; o < kTfOffs; ++o) maps[t][o] = f[o];
  __syncthreads();
  // 2. inclusive scan of the chunk maps (Hillis–Steele; composition is associative)
  for (int d = 1; d < kTfResolveThreads; d <<= 1) {
    if (t >= d) {
#pragma unroll
      for (int o = 0; o < kTfOffs; ++o) tmp[t][o] = maps[t][maps[t - d][o] & 15];
    } else {
#pragma unroll
      for (int o = 0; o < kTfOffs; ++o) tmp[t][o] = maps[t][o];
    }
    __syncthreads();
#pragma unroll
    for (int o = 0; o < kTfOffs; ++o) maps[t][o] = tmp[t][o];
    __syncthreads();
  }
  // 3. true entry offset of the window, then of this chunk; rewrite the entries
  const uint64_t S0 = j_first * kSeqBits;
  const uint32_t e_in = static_cast<uint32_t>(
      (j_first > 0 ? *reinterpret_cast<volatile unsigned long long*>(&seq[j_first - 1].exit) : 0ull) - S0);
  uint32_t o = t == 0 ? e_in : maps[t - 1][e_in & 15];
  for (uint64_t i = a; i < b; ++i) {
    const TfTab& tb = tabs[i];
    const uint64_t j = j_first + i;
    const uint64_t Sj = j * kSeqBits;
    SeqInfo s;
    s.start = Sj + o;
    const uint32_t ex = tb.ex[o & 15];
    s.exit = j + 1 == nseq ? T : (j + 1) * kSeqBits + ex;
    s.nsym = 0;
    s.nterm = tb.nt[o & 15];
    s.last_cont = (tb.lc >> (o & 15)) & 1u;
    s.pad = 0;
    seq[j] = s;
    o = ex;
  }
}

// Positions j (1..nseq-1) with seq[j-1].exit != seq[j].start (first `cap`).
__global__ void k_seq_mismatch(const SeqInfo* __restrict__ seq, uint64_t nseq, unsigned long long* list,
                               unsigned int* nlist, unsigned int cap) {
  const uint64_t j = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x + 1;
  if (j >= nseq) return;
  if (seq[j - 1].exit != seq[j].start) {
    const unsigned k = atomicAdd(nlist, 1u);
    if (k < cap) list[k] = j;
  }
}

}  // namespace dev
}  // namespace mgrc_gpu
