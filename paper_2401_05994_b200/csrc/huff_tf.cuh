// One-pass Huffman decode of the varint byte stream by transfer functions.
//
// The reference decodes serially from bit 0 (codec.cpp:354-395); the stream
// has no sync points.  Cut it into subsequences of kSeqBits bits; the first
// codeword boundary at or after a subsequence's nominal start S lies in
// [S, S + maxlen), so a subsequence's parse is described by its TRANSFER
// FUNCTION over the maxlen possible entry offsets: entry e -> exit offset into
// the next subsequence (a map of 16 nibbles, one 64-bit word; 15 = the parse
// ran into the stream end).  Maps compose associatively, so the true path is
// found by a scan — no serial chains, however long a stream stays out of
// phase (periodic stretches keep parses desynchronised for megabits).
//
// Six launches; the three stream passes give each warp a tile of kTfdTile
// consecutive subsequences staged in shared memory (coalesced, byte-swapped):
//   K1 k_tfd_maps   every lane evaluates its subsequence's map: one cursor per
//                   entry, always advancing the smallest position, so all live
//                   cursors lie within maxlen bits of it (a 16-bit occupancy
//                   mask) and two parses that meet are at the same position at
//                   some step and merge (union-find on 4-bit cursor ids, all in
//                   registers); a lone cursor finishes by a plain walk; a warp
//                   scan composes the maps across the tile;
//   K2 k_tfd_tiles  scans the tile maps in groups of 256 tiles, and
//      k_tfd_groups one CTA scans the group maps: the true entry of every
//                   group (tile 0 starts at bit 0), hence of every tile;
//   K3 k_tfd_count  the true path's terminator count and open-varint flag,
//                   gathered from K1's per-entry records (K1 counts
//                   terminators per cursor as it decodes);
//   K4 k_scan_lb    exclusive scan of the terminator counts: value offsets;
//   K5 k_tfd_emit   every lane decodes its subsequence again and writes the
//                   zigzag codes of the varints that start in it (an open value
//                   is finished by decoding on, <= 10 bytes), stopping at the
//                   N-th value; the first error in stream order, the end of the
//                   N-th varint and the padding check follow codec.cpp:75-86
//                   and :370-375.
// The passes have no cross-CTA waits: tiles of very different cost (parses
// that stay apart for megabits) cannot stall their successors.
#pragma once

#include "huff.cuh"

namespace mgrc_gpu {
namespace dev {

constexpr int kTfdThreads = 128;  // threads per CTA: 4 independent warp tiles sharing the decode table
constexpr int kTfdTile = 32;      // subsequences per tile (one warp): the look-back unit
constexpr int kTfdStage = kTfdTile * kSeqBits / 32 + kTailWords + 4;
constexpr int kTfdStageSmem = stage_idx(kTfdStage) + 2;
constexpr int kTfdWarpSmem = kTfdStageSmem;  // words per warp tile
constexpr unsigned long long kNibId = 0xFEDCBA9876543210ull;  // identity map of 16 nibbles
constexpr uint32_t kDeadEx = 15u;                              // "the parse ran into the stream end"

__device__ __forceinline__ uint32_t nib(unsigned long long m, uint32_t i) {
  return static_cast<uint32_t>(m >> (4u * i)) & 15u;
}
__device__ __forceinline__ unsigned long long nib_set(unsigned long long m, uint32_t i, uint32_t v) {
  return (m & ~(15ull << (4u * i))) | (static_cast<unsigned long long>(v) << (4u * i));
}
// 4 nibbles (16 bits) -> 4 bytes
__device__ __forceinline__ uint32_t nib4_to_bytes(uint32_t x) {
  x &= 0xFFFFu;
  x = (x | (x << 8)) & 0x00FF00FFu;
  return (x | (x << 4)) & 0x0F0F0F0Fu;
}
// first f, then g: r[e] = g[f[e]], 16 table lookups as byte permutes (the low
// 3 bits of f[e] pick among 8 bytes of g, its bit 3 the half).  Nibble 15 of
// every map is 15 (dead), so dead stays dead; entries >= ne are not used.
__device__ __forceinline__ unsigned long long nib_then(unsigned long long f, unsigned long long g, int ne) {
  (void)ne;
  const uint32_t glo = static_cast<uint32_t>(g), ghi = static_cast<uint32_t>(g >> 32);
  const uint32_t G0 = nib4_to_bytes(glo), G1 = nib4_to_bytes(glo >> 16);
  const uint32_t G2 = nib4_to_bytes(ghi), G3 = nib4_to_bytes(ghi >> 16);
  unsigned long long r = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t sx = static_cast<uint32_t>(f >> (16 * i)) & 0xFFFFu;
    const uint32_t sel = sx & 0x7777u;
    const uint32_t lo = __byte_perm(G0, G1, sel), hi = __byte_perm(G2, G3, sel);
    const uint32_t mask = nib4_to_bytes((sx & 0x8888u) >> 3) * 0xFFu;
    uint32_t b = (lo & ~mask) | (hi & mask);  // 4 result bytes, each < 16
    b = (b | (b >> 4)) & 0x00FF00FFu;
    b = (b | (b >> 8)) & 0xFFFFu;
    r |= static_cast<unsigned long long>(b) << (16 * i);
  }
  return r;
}

// the true path through one subsequence (k_tfd_count -> k_tfd_emit)
struct TfdSeq {
  uint8_t entry;  // first codeword boundary at or after S (offset; kDeadEx: the stream ended before)
  uint8_t exit;   // first boundary at or after the next S (offset; kDeadEx: stream end)
  uint8_t lc;     // its last codeword continues a varint
  uint8_t pad;
};

// A warp stages its tile [base, base + kTfdStage words) of the stream.
__device__ __forceinline__ void tfd_stage(const uint32_t* __restrict__ w, uint64_t nw, uint64_t base, uint32_t* sm,
                                          int lane) {
  for (int i = lane; i < kTfdStage; i += 32) {
    const uint64_t gw = (base >> 5) + i;
    sm[stage_idx(i)] = gw < nw ? bswap32(__ldg(w + gw)) : 0u;
  }
  __syncwarp();
}

// Exit map of one subsequence [S, end).
//
// Live cursors are kept as a 64-bit map `r` of 16 nibbles over the positions
// [base, base + 16): nibble i = 1 + id of the cursor at base + i (0: none).
// The smallest cursor (nibble 0) is always the one decoded; its codeword of
// length l <= 15 lands on nibble l — occupied means two parses met (merge:
// union-find parent of the cursor id) — and the map is rebased to the next
// smallest cursor by one shift.  Everything stays in registers.
//
// Parses that have not met after kTfdMergeBits are usually out of phase over
// a periodic stretch and will not meet soon: the survivors then walk on one by
// one with the plain two-codewords-per-refill loop (parses that would still
// meet simply reach the same exit).
#ifndef MGRC_TFD_MERGE_BITS
#define MGRC_TFD_MERGE_BITS 64
#endif
constexpr uint32_t kTfdMergeBits = MGRC_TFD_MERGE_BITS;

// Walk one parse from p to its exit (>= end); ~0u: it ran into the stream end.
// nt: terminators of the codewords walked; last: the last codeword's entry (0: none).
template <bool NEAR_END, class LT>
__device__ __forceinline__ uint32_t tfd_walk(const uint32_t* sm, const LT& lut, int maxlen, uint32_t p, uint32_t end,
                                             uint32_t tl, uint32_t& nt, uint32_t& last) {
  BitReader br;
  br.init(sm, p);
  if (!NEAR_END) {  // no codeword can run past the stream end: two per refill
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
    return p;
  }
  while (p < end) {
    br.refill();
    const uint32_t ent = lut[br.peek(maxlen)];
    const uint32_t l = lut_len(ent);
    if (p + l > tl) return ~0u;
    p += l;
    nt += lut_term(ent);
    last = ent;
    br.consume(l);
  }
  return p;
}

// The merging part: returns the live cursors (nibble map r over [base, base +
// 16)) and the union-find parents; the survivors are walked by the warp.
//
// Terminator counts ride along (the value offsets, replacing a second decode
// of the stream): cnt[id] (shared memory, one int16 per (id, lane)) counts the
// terminators cursor id decoded; when id merges into the cursor it met, its
// counter becomes the difference to that cursor's count at the meeting point,
// so an entry's count is the root's final count plus the differences along
// its union-find path.  `last` holds, per id, whether its last codeword was a
// terminator (bit id) and whether it decoded any (bit 16 + id).
struct TfdCursors {
  unsigned long long r, parent;
  uint32_t base, last;
};
template <bool NEAR_END, class LT>
__device__ __forceinline__ TfdCursors tfd_merge(const uint32_t* sm, const LT& lut, int maxlen, int ne, uint32_t S,
                                                uint32_t end, uint32_t tl, int16_t* cnt) {
  uint32_t base = S;
  unsigned long long r = 0;
  for (int e = 0; e < ne; ++e) r |= static_cast<unsigned long long>(e + 1) << (4 * e);
  unsigned long long parent = kNibId;  // union-find parent of each cursor id
  uint32_t occ = (1u << ne) - 1u;  // bit i: a cursor at base + i (mirror of r's nonzero nibbles)
  BitReader br;
  br.init(sm, base);
  uint32_t last = 0;
  for (int e = 0; e < ne; ++e) cnt[32 * e] = 0;
  const uint32_t mend = min(end, S + kTfdMergeBits);
  while ((occ & (occ - 1u)) && base < mend) {
    const uint32_t id = static_cast<uint32_t>(r) & 15u;
    br.refill();
    const uint32_t ent = lut[br.peek(maxlen)];
    const uint32_t l = lut_len(ent);
    r &= ~15ull;
    occ &= ~1u;
    if (NEAR_END && base + l > tl) {
      // the stream ends inside this codeword: the cursor dies (its count and last codeword stand)
    } else {
      const uint32_t t = lut_term(ent);
      if (t) ++cnt[32 * (id - 1u)];
      last = (last & ~(1u << (id - 1u))) | (t << (id - 1u)) | (1u << (15u + id));
      if ((occ >> l) & 1u) {  // two parses met: merge (counter -> difference to the met cursor's)
        const uint32_t other = (static_cast<uint32_t>(r >> (4u * l)) & 15u) - 1u;
        parent = nib_set(parent, id - 1u, other);
        cnt[32 * (id - 1u)] -= cnt[32 * other];
      } else {
        r |= static_cast<unsigned long long>(id) << (4u * l);
        occ |= 1u << l;
      }
    }
    if (!occ) break;
    const uint32_t sh = static_cast<uint32_t>(__ffs(static_cast<int>(occ)) - 1);
    occ >>= sh;
    r >>= 4u * sh;
    base += sh;
    br.consume(sh);
  }
  return TfdCursors{r, parent, base, last};
}

// Survivor walks of a warp, balanced across its lanes: every lane queues its
// live cursors that are still before their end (position, end, lane, id) in
// shared memory, the 32 lanes walk the queue together, and each lane reads its
// cursors' exits back (one byte per (lane, id)).  A queue overflow is walked
// by its owner.
#ifndef MGRC_TFD_JOBS
#define MGRC_TFD_JOBS 128
#endif
constexpr uint32_t kTfdJobs = MGRC_TFD_JOBS;  // queued walks per warp
struct TfdWarpQueue {
  unsigned long long job[kTfdJobs];
  uint8_t exit[32][16];
  uint16_t tail[32][16];  // the walk's terminators | its last codeword was a terminator << 13 | decoded any << 14
  int16_t cnt[16][32];    // per-cursor terminator counters (tfd_merge)
};
static_assert(kTfdTile * kSeqBits + 32 * kTailWords < (1 << 16), "walk jobs hold tile-local bit positions in 16 bits");
__device__ __forceinline__ unsigned long long tfd_job(uint32_t p, uint32_t end, uint32_t lane, uint32_t id, bool near) {
  return p | (static_cast<unsigned long long>(end) << 16) | (static_cast<unsigned long long>(lane) << 32) |
         (static_cast<unsigned long long>(id) << 37) | (static_cast<unsigned long long>(near) << 41);
}
template <class LT>
__device__ __forceinline__ uint32_t tfd_walk_exit(const uint32_t* sm, const LT& lut, int maxlen, uint32_t p,
                                                  uint32_t end, uint32_t tl, bool near, uint32_t& tail) {
  uint32_t nt = 0, last = 0;
  const uint32_t x = near ? tfd_walk<true>(sm, lut, maxlen, p, end, tl, nt, last)
                          : tfd_walk<false>(sm, lut, maxlen, p, end, tl, nt, last);
  tail = nt | (last ? (lut_term(last) << 13) | (1u << 14) : 0u);
  return x == ~0u ? kDeadEx : min(x - end, 14u);
}

// Exit map of one subsequence [S, end) of every lane (live: it has a map to
// compute); warp-synchronous.  rec (4 words): per entry e, 16 bits at 16e =
// its parse's terminator count | (its last codeword continues a varint) << 15.
template <class LT>
__device__ __forceinline__ unsigned long long tfd_map_warp(const uint32_t* sm, const LT& lut, int maxlen, int ne,
                                                           uint32_t S, uint32_t end, uint32_t tl, bool live,
                                                           TfdWarpQueue& wq, int lane, unsigned long long* rec) {
  int16_t* cnt = &wq.cnt[0][lane];
  TfdCursors cs{0ull, kNibId, S, 0u};
  if (live) cs = end + 32 >= tl ? tfd_merge<true>(sm, lut, maxlen, ne, S, end, tl, cnt)
                                : tfd_merge<false>(sm, lut, maxlen, ne, S, end, tl, cnt);
  const bool near = end + 32 >= tl;
  unsigned long long exit_of = ~0ull;  // id -> exit offset (15: dead)
  uint32_t last = cs.last;
  uint32_t nj = 0;  // cursors still before the end
  {
    uint32_t i = 0;
    for (unsigned long long r = cs.r; r; r >>= 4, ++i) nj += (static_cast<uint32_t>(r) & 15u) != 0 && cs.base + i < end;
  }
  uint32_t off = nj;  // inclusive warp scan -> exclusive offset
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t h = __shfl_up_sync(0xffffffffu, off, d);
    if (lane >= d) off += h;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, off, 31);
  off -= nj;
  // a survivor's walk adds its terminators to the cursor's counter and may replace its last codeword
  auto add_tail = [&](uint32_t id0, uint32_t tail) {
    cnt[32 * id0] += static_cast<int16_t>(tail & 0x1FFFu);
    if (tail & (1u << 14)) last = (last & ~(1u << id0)) | (((tail >> 13) & 1u) << id0) | (1u << (16u + id0));
  };
  {
    uint32_t q = off, i = 0;
    for (unsigned long long r = cs.r; r; r >>= 4, ++i) {
      const uint32_t id = static_cast<uint32_t>(r) & 15u;
      if (!id) continue;
      const uint32_t p = cs.base + i;
      if (p >= end) {
        exit_of = nib_set(exit_of, id - 1u, min(p - end, 14u));
        continue;
      }
      if (q < kTfdJobs) {
        wq.job[q] = tfd_job(p, end, static_cast<uint32_t>(lane), id - 1u, near);
      } else {
        uint32_t tail;
        exit_of = nib_set(exit_of, id - 1u, tfd_walk_exit(sm, lut, maxlen, p, end, tl, near, tail));
        add_tail(id - 1u, tail);
      }
      ++q;
    }
  }
  __syncwarp();
  const uint32_t nq = min(total, kTfdJobs);
  for (uint32_t q = lane; q < nq; q += 32) {
    const unsigned long long jb = wq.job[q];
    const uint32_t p = static_cast<uint32_t>(jb) & 0xFFFFu, e = static_cast<uint32_t>(jb >> 16) & 0xFFFFu;
    const uint32_t jl = (jb >> 32) & 31u, jid = (jb >> 37) & 15u;
    uint32_t tail;
    wq.exit[jl][jid] = static_cast<uint8_t>(tfd_walk_exit(sm, lut, maxlen, p, e, tl, (jb >> 41) & 1u, tail));
    wq.tail[jl][jid] = static_cast<uint16_t>(tail);
  }
  __syncwarp();
  {
    uint32_t q = off, i = 0;
    for (unsigned long long r = cs.r; r; r >>= 4, ++i) {
      const uint32_t id = static_cast<uint32_t>(r) & 15u;
      if (!id) continue;
      if (cs.base + i >= end) continue;
      if (q < kTfdJobs) {
        exit_of = nib_set(exit_of, id - 1u, wq.exit[lane][id - 1u]);
        add_tail(id - 1u, wq.tail[lane][id - 1u]);
      }
      ++q;
    }
  }
  unsigned long long f = ~0ull;
  unsigned long long rw[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    if (e >= ne) break;
    uint32_t q = e;
    int32_t c = cnt[32 * e];
    for (uint32_t pq = nib(cs.parent, q); pq != q; pq = nib(cs.parent, q)) {
      q = pq;
      c += cnt[32 * q];
    }
    f = nib_set(f, e, nib(exit_of, q));
    const uint32_t lc = ((last >> (16u + q)) & 1u) & (((last >> q) & 1u) ^ 1u);
    rw[e >> 2] |= static_cast<unsigned long long>(static_cast<uint32_t>(c) | (lc << 15)) << (16u * (e & 3));
  }
  __syncwarp();  // the queue and the counters are reused by the next call
  if (live && rec) {
    rec[0] = rw[0];
    rec[1] = rw[1];
    rec[2] = rw[2];
    rec[3] = rw[3];
  }
  return f;
}

// K1: exit maps, scanned within the tile: gmap[j] = map of subsequences
// [tile start, j] (entry of the tile -> exit of j).
template <bool G>
static __global__ void __launch_bounds__(kTfdThreads) k_tfd_maps(const uint32_t* __restrict__ w, uint64_t nw, uint64_t T,
                                                          const uint16_t* __restrict__ lut_g, int maxlen, int ne,
                                                          uint64_t nseq, unsigned long long* __restrict__ gmap,
                                                          unsigned long long* __restrict__ rec) {
  extern __shared__ uint32_t dyn[];
  __shared__ TfdWarpQueue wqs[kTfdThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint16_t* lut_s = reinterpret_cast<uint16_t*>(dyn + (kTfdThreads / 32) * kTfdWarpSmem);
  uint32_t* sm = dyn + wid * kTfdWarpSmem;
  if (!G)
    for (int k = threadIdx.x; k < (1 << maxlen); k += kTfdThreads) lut_s[k] = lut_g[k];
  __syncthreads();
  const Lut<G> lut{G ? lut_g : lut_s};
  const uint64_t c = static_cast<uint64_t>(blockIdx.x) * (kTfdThreads / 32) + wid;
  if (c * kTfdTile >= nseq) return;
  const uint64_t base = c * kTfdTile * kSeqBits;
  tfd_stage(w, nw, base, sm, lane);
  const uint32_t tl = static_cast<uint32_t>(umin64(T - base, 0x7FFFFFFFu));
  const uint64_t j = c * kTfdTile + lane;
  const uint32_t S = static_cast<uint32_t>(lane) * kSeqBits;
  const uint32_t end = min(S + static_cast<uint32_t>(kSeqBits), tl);
  // the last subsequence ends the stream (all dead); identity past it
  const unsigned long long m = tfd_map_warp(sm, lut, maxlen, ne, S, end, tl, j < nseq, wqs[wid], lane, rec + 4 * j);
  unsigned long long g = j < nseq ? (j + 1 < nseq ? m : ~0ull) : kNibId;
#pragma unroll
  for (int d = 1; d < kTfdTile; d <<= 1) {
    const unsigned long long h = __shfl_up_sync(0xffffffffu, g, d);
    if (lane >= d) g = nib_then(h, g, ne);
  }
  if (j < nseq) gmap[j] = g;
}

// K2: the true entry of every tile, in two launches.  K2a: each CTA scans the
// maps of kTfdGroup consecutive tiles (warp shuffles, then the warp
// aggregates): tpre[i] = map of the tiles [group start, i]; gagg = the
// group's map.  K2b (one CTA) scans the group maps: each thread composes the
// maps of its chunk, a block scan combines the chunks, and each thread walks
// its chunk from the true entry (group 0 starts at offset 0) — gentry[g].
// K3 then reads a tile's entry as tpre[i-1] applied to its group's entry.
constexpr int kTfdGroup = 256;
static __global__ void __launch_bounds__(kTfdGroup) k_tfd_tiles(const unsigned long long* __restrict__ gmap,
                                                               uint64_t nseq, uint64_t ntile, int ne,
                                                               unsigned long long* __restrict__ tpre,
                                                               unsigned long long* __restrict__ gagg) {
  __shared__ unsigned long long wagg[kTfdGroup / 32];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const uint64_t i = static_cast<uint64_t>(blockIdx.x) * kTfdGroup + t;
  unsigned long long m = i < ntile ? gmap[umin64(i * kTfdTile + kTfdTile - 1, nseq - 1)] : kNibId;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned long long h = __shfl_up_sync(0xffffffffu, m, d);
    if (lane >= d) m = nib_then(h, m, ne);
  }
  if (lane == 31) wagg[wid] = m;
  __syncthreads();
  if (wid == 0) {  // exclusive prefixes of the warp aggregates
    unsigned long long x = lane < kTfdGroup / 32 ? wagg[lane] : kNibId;
#pragma unroll
    for (int d = 1; d < kTfdGroup / 32; d <<= 1) {
      const unsigned long long h = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x = nib_then(h, x, ne);
    }
    const unsigned long long ex = __shfl_up_sync(0xffffffffu, x, 1);
    __syncwarp();
    if (lane < kTfdGroup / 32) wagg[lane] = lane ? ex : kNibId;
  }
  __syncthreads();
  if (wid) m = nib_then(wagg[wid], m, ne);
  if (i < ntile) tpre[i] = m;
  if (t == kTfdGroup - 1) gagg[blockIdx.x] = m;  // identity past the last tile
}

constexpr int kTfdScanThreads = 1024;
static __global__ void __launch_bounds__(kTfdScanThreads) k_tfd_groups(const unsigned long long* __restrict__ gagg,
                                                                uint64_t ngroup, int ne,
                                                                uint8_t* __restrict__ gentry) {
  __shared__ unsigned long long sm[kTfdScanThreads];
  const int t = threadIdx.x;
  const uint64_t per = (ngroup + kTfdScanThreads - 1) / kTfdScanThreads;
  const uint64_t a = umin64(ngroup, t * per), b = umin64(ngroup, a + per);
  unsigned long long f = kNibId;
  for (uint64_t i = a; i < b; ++i) f = nib_then(f, gagg[i], ne);
  sm[t] = f;
  __syncthreads();
  for (int d = 1; d < kTfdScanThreads; d <<= 1) {  // inclusive Hillis-Steele
    const unsigned long long h = t >= d ? sm[t - d] : kNibId;
    __syncthreads();
    if (t >= d) sm[t] = nib_then(h, sm[t], ne);
    __syncthreads();
  }
  uint32_t e = t > 0 ? nib(sm[t - 1], 0) : 0u;
  for (uint64_t i = a; i < b; ++i) {
    gentry[i] = static_cast<uint8_t>(e);
    if (e != kDeadEx) e = nib(gagg[i], e);
  }
}

// K3: the true path through every subsequence: entry and exit from the maps,
// terminator count and open-varint flag from the maps pass's per-entry records.
static __global__ void __launch_bounds__(256) k_tfd_count(uint64_t nseq, const unsigned long long* __restrict__ gmap,
                                                          const unsigned long long* __restrict__ tpre,
                                                          const uint8_t* __restrict__ gentry,
                                                          const unsigned long long* __restrict__ rec,
                                                          TfdSeq* __restrict__ seqs, unsigned long long* __restrict__ cnt) {
  const uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= nseq) return;
  const uint64_t c = j / kTfdTile;
  const uint32_t ge = gentry[c / kTfdGroup];
  const uint32_t e = (ge == kDeadEx || c % kTfdGroup == 0) ? ge : nib(tpre[c - 1], ge);  // the tile's entry
  const uint32_t entry = e == kDeadEx ? kDeadEx : (j % kTfdTile ? nib(gmap[j - 1], e) : e);
  const uint32_t exo = e == kDeadEx ? kDeadEx : nib(gmap[j], e);
  TfdSeq q{static_cast<uint8_t>(entry), static_cast<uint8_t>(exo), 0, 0};
  uint32_t nterm = 0;
  if (entry != kDeadEx) {
    const uint32_t r = static_cast<uint32_t>(rec[4 * j + (entry >> 2)] >> (16u * (entry & 3u))) & 0xFFFFu;
    nterm = r & 0x7FFFu;
    q.lc = static_cast<uint8_t>(r >> 15);
  }
  seqs[j] = q;
  cnt[j] = nterm;
}

// The varints of one subsequence: `nv` values starting at index k_first (the
// first one at bit p, after the skip of a value begun earlier); NE: the
// stream end is within reach (codewords may run past it).
template <bool NE, typename Z, class LT>
__device__ __forceinline__ void tfd_emit_values(const uint32_t* sm, const LT& lut, int maxlen, uint32_t p,
                                                uint32_t tl, bool skipping, uint64_t k_first, uint32_t nv,
                                                bool has_last, uint64_t base, Z* __restrict__ zz, Z* my,
                                                DecodeStatus* st, unsigned long long* first_err) {
  constexpr int CH = 32 / sizeof(Z);  // values per 32-byte output chunk
  auto flush = [&](uint64_t upto) {   // values [chunk start, upto) of the current chunk
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
  BitReader br;
  br.init(sm, p);
  if (skipping) {  // the value open at the entry began in the previous subsequence: skip to its end
    for (;;) {
      br.refill();
      const uint32_t ent = lut[br.peek(maxlen)];
      const uint32_t l = lut_len(ent);
      if (NE && p + l > tl) return;  // truncated inside that value: its owner (the previous lane) reports it
      p += l;
      br.consume(l);
      if (lut_term(ent)) break;
    }
  }
  uint32_t err = 0, err_at = 0, wide = 0, v = 0;
  uint32_t ki = static_cast<uint32_t>(k_first);  // low bits pick the chunk slot
  for (; v < nv; ++v) {
    br.refill();
    uint32_t ent = lut[br.peek(maxlen)];
    uint32_t l = lut_len(ent);
    if (NE && p + l > tl) {
      err = 2, err_at = tl;
      break;
    }
    p += l;
    br.consume(l);
    // a terminator carries its whole symbol: < 0x80 for varint bytes, any byte for a raw byte stream
    // (decode table built with every symbol terminating, mdr.cu)
    uint64_t acc = ent & (lut_term(ent) ? 0xFFu : 0x7Fu);
    if (!lut_term(ent)) {  // continuation bytes (codec.cpp:75-86)
      for (uint32_t sh = 7;; sh += 7) {
        br.refill();
        ent = lut[br.peek(maxlen)];
        l = lut_len(ent);
        if (NE && p + l > tl) {
          err = 2, err_at = tl;
          break;
        }
        if (sh == 63 && (ent & 0xFEu)) {  // varint overflows 64 bits (codec.cpp:80-81)
          err = 1, err_at = p;
          break;
        }
        p += l;
        br.consume(l);
        acc |= static_cast<uint64_t>(ent & 0x7Fu) << sh;
        if (lut_term(ent)) break;
      }
      if (err) break;
      if (sizeof(Z) == 4 && (acc >> 32)) wide = 1;
    }
    my[ki & (CH - 1)] = static_cast<Z>(acc);
    ++ki;
    if ((ki & (CH - 1)) == 0) flush(k_first + v + 1);
  }
  const uint64_t kend = k_first + v;
  if ((kend & (CH - 1)) != 0 && kend > k_first) flush(kend);
  if (!err && has_last) {  // the N-th value ends here: exhausted_clean (codec.cpp:370-375)
    st->end_bit = base + p;
    const uint32_t rest = tl - p;
    br.refill();
    st->clean = rest < 8 && (rest == 0 || (static_cast<uint32_t>(br.buf >> 32) >> (32 - rest)) == 0);
  }
  if (err) atomicMin(first_err, ((base + err_at) << 2) | err);  // the first error in stream order
  if (wide) atomicOr(&st->wide, 1u);
}

// K5: decode every subsequence along the true path and write the zigzag codes
// of the varints that start in it.
template <typename Z, bool G>
static __global__ void __launch_bounds__(kTfdThreads) k_tfd_emit(const uint32_t* __restrict__ w, uint64_t nw, uint64_t T,
                                                          const uint16_t* __restrict__ lut_g, int maxlen,
                                                          uint64_t nseq, uint64_t N, const TfdSeq* __restrict__ seqs,
                                                          const unsigned long long* __restrict__ cnt,
                                                          const unsigned long long* __restrict__ toff,
                                                          Z* __restrict__ zz, DecodeStatus* st,
                                                          unsigned long long* first_err) {
  constexpr int CH = 32 / sizeof(Z);
  extern __shared__ uint32_t dyn[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint16_t* lut_s = reinterpret_cast<uint16_t*>(dyn + (kTfdThreads / 32) * kTfdWarpSmem);
  uint32_t* sm = dyn + wid * kTfdWarpSmem;
  __shared__ __align__(16) Z slot[kTfdThreads][CH];
  if (!G)
    for (int k = threadIdx.x; k < (1 << maxlen); k += kTfdThreads) lut_s[k] = lut_g[k];
  __syncthreads();
  const Lut<G> lut{G ? lut_g : lut_s};
  const uint64_t c = static_cast<uint64_t>(blockIdx.x) * (kTfdThreads / 32) + wid;
  if (c * kTfdTile >= nseq) return;
  const uint64_t base = c * kTfdTile * kSeqBits;
  tfd_stage(w, nw, base, sm, lane);
  const uint64_t j = c * kTfdTile + lane;
  if (j >= nseq) return;
  const uint32_t tl = static_cast<uint32_t>(umin64(T - base, 0x7FFFFFFFu));
  const uint32_t S = static_cast<uint32_t>(lane) * kSeqBits;
  const TfdSeq q = seqs[j];
  if (q.entry == kDeadEx) return;  // the true path already ran into the stream end (reported by its owner)
  const uint32_t ex = (j + 1 == nseq || q.exit == kDeadEx) ? tl : S + kSeqBits + q.exit;
  const bool skipping = j > 0 && seqs[j - 1].lc != 0;
  const uint64_t k_first = toff[j] + (skipping ? 1 : 0);
  if (k_first >= N) return;  // every value that starts here is past the N-th (never read, codec.cpp:475-481)
  // values that start here: the terminators in [entry, exit), less the one
  // closing a value begun earlier, plus the value left open at the exit
  const uint64_t nstart = cnt[j] - (skipping ? 1 : 0) + q.lc;
  const bool has_last = k_first + nstart >= N;
  const uint32_t nv = static_cast<uint32_t>(umin64(nstart, N - k_first));
  if (ex + 256 >= tl)
    tfd_emit_values<true>(sm, lut, maxlen, S + q.entry, tl, skipping, k_first, nv, has_last, base, zz,
                          slot[threadIdx.x], st, first_err);
  else
    tfd_emit_values<false>(sm, lut, maxlen, S + q.entry, tl, skipping, k_first, nv, has_last, base, zz,
                           slot[threadIdx.x], st, first_err);
}

}  // namespace dev
}  // namespace mgrc_gpu
