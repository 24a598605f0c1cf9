// Offline model of the self-synchronising Huffman decode (huff.cuh) on a real
// container: sync-distance distribution from arbitrary bit offsets and the
// per-CTA round structure of k_huff_sync_s for a given warm-up length.
// Build: g++ -O2 -std=c++17 -I paper_2401_05994_b200/csrc scripts/sync_sim.cpp
//        paper_2401_05994_b200/csrc/host.cpp -o /tmp/sync_sim
// Run:   /tmp/sync_sim container.mgrc [warm_bits ...]
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iterator>
#include <vector>

#include "host.hpp"

using namespace mgrc_gpu;

static const uint8_t* B;
static uint64_t T;
static int ML;
static std::vector<uint16_t> LUT;

static inline uint32_t peek32(uint64_t p) {
  const uint64_t byte = p >> 3;
  uint64_t v = 0;
  for (int k = 0; k < 8; ++k) v = (v << 8) | (byte + k < T / 8 ? B[byte + k] : 0);
  return static_cast<uint32_t>((v << (p & 7)) >> 32);
}
static inline uint32_t len_at(uint64_t p) { return (LUT[peek32(p) >> (32 - ML)] >> 8) & 15u; }
static inline uint32_t term_at(uint64_t p) { return (LUT[peek32(p) >> (32 - ML)] >> 12) & 1u; }

int main(int argc, char** argv) {
  std::ifstream f(argv[1], std::ios::binary);
  std::vector<uint8_t> c((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
  ContainerInfo info = parse_header(c.data(), c.size());
  const uint8_t* pay = c.data() + info.header_size;
  uint64_t cons = 0;
  CodeTable tab = read_table_header(pay, info.payload_len, &cons);
  LUT = build_decode_lut(tab);
  ML = tab.max_len;
  B = pay + cons;
  T = (info.payload_len - cons) * 8;
  std::printf("body %.1f MB, maxlen %d, nsym %d\n", T / 8e6, ML, tab.nsym);
  // true boundaries
  std::vector<uint8_t> bd((T >> 3) + 1, 0);
  uint64_t nsym = 0;
  for (uint64_t p = 0; p < T;) {
    bd[p >> 3] |= 1u << (p & 7);
    const uint32_t l = len_at(p);
    if (p + l > T) break;
    p += l;
    ++nsym;
  }
  auto isb = [&](uint64_t p) { return (bd[p >> 3] >> (p & 7)) & 1u; };
  std::printf("symbols %llu, mean code length %.3f bits\n", (unsigned long long)nsym, double(T) / nsym);
  // multi-symbol spans: codewords that fit entirely in a window of wb bits
  for (int wb = ML; wb <= 16; ++wb) {
    uint64_t looks = 0;
    for (uint64_t p = 0; p < T;) {
      const uint32_t v = peek32(p) >> (32 - wb);
      uint32_t used = 0;
      for (;;) {
        const uint32_t l = (LUT[((v << used) & ((1u << wb) - 1)) >> (wb - ML)] >> 8) & 15u;
        if (used + l > uint32_t(wb)) break;
        used += l;
      }
      if (p + used > T || used == 0) break;
      p += used;
      ++looks;
    }
    std::printf("span window %d bits: %.3f symbols per lookup\n", wb, double(nsym) / looks);
  }
  const uint64_t S = 1024, nseq = (T + S - 1) / S;
  // sync distance from each nominal start
  std::vector<uint32_t> dist(nseq);
  for (uint64_t j = 0; j < nseq; ++j) {
    uint64_t p = j * S, d = 0;
    while (p < T && !isb(p)) {
      const uint32_t l = len_at(p);
      p += l;
      d += l;
    }
    dist[j] = static_cast<uint32_t>(std::min<uint64_t>(d, 0xFFFFFFFFu));
  }
  std::vector<uint32_t> sd = dist;
  std::sort(sd.begin(), sd.end());
  auto pct = [&](double q) { return sd[std::min<size_t>(sd.size() - 1, size_t(q * sd.size()))]; };
  double mean = 0;
  for (auto x : sd) mean += x;
  mean /= sd.size();
  std::printf("sync distance: mean %.1f p50 %u p90 %u p99 %u p99.9 %u p99.99 %u max %u\n", mean, pct(.5), pct(.9),
              pct(.99), pct(.999), pct(.9999), sd.back());
  for (int W : {64, 128, 256, 512, 1024, 2048, 4096}) {
    uint64_t n = 0;
    for (auto x : sd) n += x > uint32_t(W);
    std::printf("  P(dist > %4d) = %.5f\n", W, double(n) / nseq);
  }
  if (!std::getenv("NOTF")) // transfer-table model: track 0 from S, other entry offsets walked until they
  // land on a recorded track (two recorded tracks at most, as k_tf_tables)
  {
    uint64_t c0 = 0, c1 = 0, cw = 0, third = 0, third_sym = 0, distinct_hist[17] = {0};
    std::vector<uint8_t> b0(S + 64), b1(S + 64);
    for (uint64_t j = 0; j + 1 < nseq; ++j) {
      const uint64_t s = j * S, end = s + S;
      std::fill(b0.begin(), b0.end(), 0);
      uint64_t p = s;
      while (p < end) { b0[p - s] = 1; p += len_at(p); ++c0; }
      const uint64_t e0 = p;
      bool two = false;
      uint64_t e1 = 0;
      int distinct = 1;
      for (int o = 1; o < ML; ++o) {
        uint64_t q = s + o, n = 0;
        int hit = -1;
        while (q < end) {
          if (b0[q - s]) { hit = 0; break; }
          if (two && b1[q - s]) { hit = 1; break; }
          q += len_at(q);
          ++n;
        }
        cw += n;
        if (hit < 0) {
          if (!two) {
            std::fill(b1.begin(), b1.end(), 0);
            uint64_t r = s + o;
            while (r < end) { b1[r - s] = 1; r += len_at(r); ++c1; }
            e1 = r;
            two = true;
            ++distinct;
          } else {
            ++third;
            third_sym += n;
            if (q != e0 && q != e1) ++distinct;
          }
        }
      }
      distinct_hist[std::min(distinct, 16)]++;
    }
    std::printf("TF model: symbols/seq track0 %.1f track1 %.1f walks %.1f third-phase walks %llu (%.1f sym/seq)\n",
                double(c0) / nseq, double(c1) / nseq, double(cw) / nseq, (unsigned long long)third,
                double(third_sym) / nseq);
    std::printf("  recorded+distinct phases hist:");
    for (int k = 1; k < 8; ++k) std::printf(" %d:%llu", k, (unsigned long long)distinct_hist[k]);
    std::printf("\n");
  }
  // CTA model: 128 threads, first 8 re-decode the predecessor's last subsequences
  const int SLOTS = std::getenv("SLOTS") ? std::atoi(std::getenv("SLOTS")) : 0;
  const int PLAIN = std::getenv("PLAIN") ? std::atoi(std::getenv("PLAIN")) : 3;
  const int K = std::getenv("KWIN") ? std::atoi(std::getenv("KWIN")) : 8;
  for (int ai = 2; ai < argc; ++ai) {
    const int W = std::atoi(argv[ai]);
    const int NT = 128, WARM = 8, REAL = NT - WARM;
    const uint64_t nblk = (nseq + REAL - 1) / REAL;
    uint64_t rounds_hist[8] = {0}, total_redo = 0, total_redo_warps = 0, init_sym = 0, bad_edges = 0;
    uint64_t max_rounds = 0, cta_open = 0, sum_rounds = 0;
    std::vector<int> edge_walk;
    for (uint64_t b = 0; b < nblk; ++b) {
      const int64_t j0 = int64_t(b) * REAL - WARM;
      uint64_t F[NT], E[NT];
      bool valid[NT];
      for (int t = 0; t < NT; ++t) {
        const int64_t js = j0 + t;
        valid[t] = js >= 0 && uint64_t(js) < nseq;
        F[t] = E[t] = 0;
        if (!valid[t]) continue;
        const uint64_t s = uint64_t(js) * S, end = std::min(s + S, T);
        uint64_t p = s >= uint64_t(W) ? s - W : 0;
        while (p < s) { const uint32_t l = len_at(p); if (p + l > T) break; p += l; ++init_sym; }
        F[t] = p;
        while (p < end) { const uint32_t l = len_at(p); if (p + l > T) break; p += l; ++init_sym; }
        E[t] = p;
      }
      uint64_t r = 0;
      for (;; ++r) {
        std::vector<int> bad;
        for (int t = 1; t < NT; ++t)
          if (valid[t] && j0 + t > 0 && E[t - 1] != F[t]) bad.push_back(t);
        if (bad.empty()) break;
        if (SLOTS > 0 && r >= uint64_t(PLAIN)) {
          std::vector<char> claim(NT, 0);
          int used = 0;
          for (int t : bad) {
            for (int u = t; u < NT && u < t + K && used < SLOTS; ++u)
              if (!claim[u] && valid[u]) { claim[u] = 1; ++used; }
            if (used >= SLOTS) break;
          }
          total_redo += used;
          total_redo_warps += (used * 16 + 31) / 32;
          for (int t = 1; t < NT; ++t) {
            if (!claim[t] || E[t - 1] == F[t]) continue;
            const uint64_t end = std::min(uint64_t(j0 + t) * S + S, T);
            uint64_t p = E[t - 1];
            F[t] = p;
            while (p < end) { const uint32_t l = len_at(p); if (p + l > T) break; p += l; }
            E[t] = p;
          }
          continue;
        }
        total_redo += bad.size();
        total_redo_warps += (bad.size() + 31) / 32;
        std::vector<uint64_t> from(bad.size());
        for (size_t k = 0; k < bad.size(); ++k) from[k] = E[bad[k] - 1];
        for (size_t k = 0; k < bad.size(); ++k) {
          const int t = bad[k];
          const uint64_t end = std::min(uint64_t(j0 + t) * S + S, T);
          uint64_t p = from[k];
          while (p < end) { const uint32_t l = len_at(p); if (p + l > T) break; p += l; }
          F[t] = from[k];
          E[t] = p;
        }
        if (r > 100000) { ++cta_open; break; }
      }
      sum_rounds += r;
      rounds_hist[std::min<uint64_t>(r, 7)]++;
      max_rounds = std::max(max_rounds, r);
      // edge correctness: first published start must be a true boundary; the
      // fix walk re-decodes from the true entry until an exit matches
      if (b > 0 && valid[WARM] && !isb(F[WARM])) {
        ++bad_edges;
        uint64_t p = uint64_t(j0 + WARM) * S;
        while (!isb(p)) ++p;  // true entry (first boundary >= S)
        int walked = 0;
        for (int t = WARM; t < NT && valid[t]; ++t) {
          const uint64_t end = std::min(uint64_t(j0 + t) * S + S, T);
          while (p < end) { const uint32_t l = len_at(p); if (p + l > T) break; p += l; }
          ++walked;
          if (p == E[t]) break;
        }
        edge_walk.push_back(walked);
      }
    }
    std::printf("W=%d: CTAs %llu, init symbols/seq %.1f, redo seqs %llu (%.4f/seq), redo warp-rounds/CTA %.3f, "
                "max rounds %llu, bad edges %llu, mean rounds %.2f\n  rounds hist:", W, (unsigned long long)nblk, double(init_sym) / nseq,
                (unsigned long long)total_redo, double(total_redo) / nseq, double(total_redo_warps) / nblk,
                (unsigned long long)max_rounds, (unsigned long long)bad_edges, double(sum_rounds) / nblk);
    for (int k = 0; k < 8; ++k) std::printf(" %d:%llu", k, (unsigned long long)rounds_hist[k]);
    std::printf("\n");
    std::sort(edge_walk.begin(), edge_walk.end());
    std::printf("  edge walks (subsequences):");
    for (size_t k = 0; k < edge_walk.size(); k += std::max<size_t>(1, edge_walk.size() / 12)) std::printf(" %d", edge_walk[k]);
    if (!edge_walk.empty()) std::printf(" max %d", edge_walk.back());
    std::printf("\n");
  }
}
