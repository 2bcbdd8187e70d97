// cs_schedule.cpp -- owner schedule for the CountSketch register-bin kernel.
//
// CountSketch has no reference implementation; the draw
// protocol is documented in countsketch.cu.  The schedule is a pure function
// of the operator's buckets h(i) and signs sigma(i), built once per operator:
//
//   * the kernel runs CS_THREADS threads per CTA and every thread OWNS the
//     buckets b with b % CS_THREADS == thread, holding their bins in registers
//     (slot j = b / CS_THREADS), so no two threads ever update the same bin;
//   * a T-row tile (T <= 4096) of one column is staged in shared memory; the rows of
//     warp w (rows whose bucket's owner lives in warp w) are processed in
//     "iterations": in each iteration a lane handles at most one of its rows;
//   * the rows of each half-warp form a bipartite multigraph (lane, r mod 16)
//     -- r mod 16 is the shared-memory bank pair of the staged double -- and an
//     iteration must be a matching so that the 16 lanes' 8-byte reads hit 16
//     distinct bank pairs.  Bipartite edge colouring (Koenig: Delta colours,
//     alternating-path recolouring) gives the fewest iterations.
//
// Section of one tile (bytes, 16-byte multiple):
//   u16 hdr[64]: hdr[w] = first iteration of warp w, hdr[32] = total
//   u16 ent[total][32]: ent[it][lane] = row | slot << 12 | negative << 14 | 1 << 15
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

#include "nsk_internal.hpp"

namespace nsk {

namespace {

constexpr int MAXC = 32;  // colours per half-warp (Delta ~ 8-10 at 3-4 rows per lane and tile)

// Edge-colours ne edges (L[e] in [0,16), R[e] in [0,16)); returns the colour
// count or -1 if more than MAXC would be needed.
int color_half(int ne, const uint8_t* L, const uint8_t* R, uint8_t* col) {
  int16_t atL[16][MAXC], atR[16][MAXC];
  std::memset(atL, 0xFF, sizeof atL);
  std::memset(atR, 0xFF, sizeof atR);
  int ncol = 0;
  std::vector<int> path;
  for (int e = 0; e < ne; ++e) {
    const int u = L[e], v = R[e];
    int a = 0, b = 0;
    while (a < MAXC && atL[u][a] >= 0) ++a;
    while (b < MAXC && atR[v][b] >= 0) ++b;
    if (a == MAXC || b == MAXC) return -1;
    if (atR[v][a] >= 0) {
      // a is used at v: swap a/b along the alternating path that starts at v
      // with its a-edge; it cannot reach u (u has no a-edge), and afterwards a
      // is free at v.
      path.clear();
      int node = v, c = a, d = b;
      bool right = true;
      for (;;) {
        const int f = right ? atR[node][c] : atL[node][c];
        if (f < 0) break;
        path.push_back(f);
        node = right ? L[f] : R[f];
        right = !right;
        std::swap(c, d);
      }
      for (int f : path) {
        atL[L[f]][col[f]] = -1;
        atR[R[f]][col[f]] = -1;
      }
      for (int f : path) {
        col[f] = static_cast<uint8_t>(col[f] == a ? b : a);
        atL[L[f]][col[f]] = static_cast<int16_t>(f);
        atR[R[f]][col[f]] = static_cast<int16_t>(f);
      }
      if (b + 1 > ncol) ncol = b + 1;
    }
    col[e] = static_cast<uint8_t>(a);
    atL[u][a] = static_cast<int16_t>(e);
    atR[v][a] = static_cast<int16_t>(e);
    if (a + 1 > ncol) ncol = a + 1;
  }
  return ncol;
}

// Builds the section of one tile into out (cleared); returns false on overflow.
bool build_tile(const uint32_t* bucket_sign, int T, std::vector<uint16_t>& out) {
  // rows per warp, in increasing row order
  std::vector<uint16_t> rows[CS_WARPS];
  for (int w = 0; w < CS_WARPS; ++w) rows[w].reserve(2 * T / CS_WARPS);
  for (int r = 0; r < T; ++r) {
    const uint32_t b = bucket_sign[r] & 0xFFFFu;
    rows[(b % CS_THREADS) / 32].push_back(static_cast<uint16_t>(r));
  }
  out.assign(64, 0);
  int total = 0;
  std::vector<uint8_t> L[2], R[2], C[2];
  std::vector<uint16_t> E[2];
  for (int w = 0; w < CS_WARPS; ++w) {
    for (int h = 0; h < 2; ++h) {
      L[h].clear();
      R[h].clear();
      E[h].clear();
    }
    for (uint16_t r : rows[w]) {
      const uint32_t e = bucket_sign[r];
      const uint32_t b = e & 0xFFFFu;
      const int lane = static_cast<int>(b % 32);
      const int h = lane >> 4;
      L[h].push_back(static_cast<uint8_t>(lane & 15));
      R[h].push_back(static_cast<uint8_t>(r & 15));
      const uint32_t slot = b / CS_THREADS;
      const uint32_t sg = ((e >> 16) & 1u) ^ 1u;  // 1 = negative
      E[h].push_back(static_cast<uint16_t>(r | (slot << 12) | (sg << 14) | (1u << 15)));
    }
    int iters = 0;
    for (int h = 0; h < 2; ++h) {
      C[h].assign(L[h].size(), 0);
      const int nc = color_half(static_cast<int>(L[h].size()), L[h].data(), R[h].data(), C[h].data());
      if (nc < 0) return false;
      iters = std::max(iters, nc);
    }
    out[static_cast<size_t>(w)] = static_cast<uint16_t>(total);
    const size_t base = out.size();
    out.resize(base + static_cast<size_t>(iters) * 32, 0);
    for (int h = 0; h < 2; ++h)
      for (size_t x = 0; x < E[h].size(); ++x) {
        const int lane = h * 16 + L[h][x];
        out[base + static_cast<size_t>(C[h][x]) * 32 + static_cast<size_t>(lane)] = E[h][x];
      }
    // Idle lanes still execute the shared loads: point each at a row whose bank
    // pair no active lane of its half-warp uses (entry without the valid bit).
    for (int k = 0; k < iters; ++k)
      for (int h = 0; h < 2; ++h) {
        uint16_t* it = out.data() + base + static_cast<size_t>(k) * 32 + 16 * h;
        uint32_t used = 0;
        for (int l = 0; l < 16; ++l)
          if (it[l] & 0x8000u) used |= 1u << (it[l] & 15u);
        int p = 0;
        for (int l = 0; l < 16; ++l)
          if (!(it[l] & 0x8000u)) {
            while (used & (1u << p)) ++p;
            it[l] = static_cast<uint16_t>(p);
            used |= 1u << p;
          }
      }
    total += iters;
    if (total > 0xFFFF) return false;
  }
  out[CS_WARPS] = static_cast<uint16_t>(total);
  return true;
}

}  // namespace

int cs_tile_rows() {
  const char* v = std::getenv("NSK_CS_T");
  if (v && std::atoi(v) == 3072) return 3072;
  return 4096;
}

int build_cs_schedule(const uint32_t* table, int64_t ntiles, int T, int64_t s, std::vector<uint8_t>& sec,
                      std::vector<uint64_t>& off, uint32_t& max_bytes) {
  if (s < 1 || s > 4 * CS_THREADS) return EINVAL_;
  if (T < 16 || T > CS_T_MAX || T % 16) return EINVAL_;
  std::vector<std::vector<uint16_t>> tiles(static_cast<size_t>(ntiles));
  unsigned nth = std::thread::hardware_concurrency();
  if (nth < 1) nth = 1;
  if (nth > 32) nth = 32;
  if (static_cast<int64_t>(nth) > ntiles) nth = static_cast<unsigned>(ntiles > 0 ? ntiles : 1);
  std::vector<char> ok(nth, 1);
  std::vector<std::thread> pool;
  for (unsigned q = 0; q < nth; ++q)
    pool.emplace_back([&, q]() {
      for (int64_t t = q; t < ntiles; t += nth)
        if (!build_tile(table + t * T, T, tiles[static_cast<size_t>(t)])) {
          ok[q] = 0;
          return;
        }
    });
  for (auto& th : pool) th.join();
  for (char c : ok)
    if (!c) return EINVAL_;
  off.assign(static_cast<size_t>(ntiles) + 1, 0);
  max_bytes = 0;
  for (int64_t t = 0; t < ntiles; ++t) {
    const uint64_t bytes = tiles[static_cast<size_t>(t)].size() * 2;  // 128 + 64 * total: 16-byte multiple
    off[static_cast<size_t>(t) + 1] = off[static_cast<size_t>(t)] + bytes;
    if (bytes > max_bytes) max_bytes = static_cast<uint32_t>(bytes);
  }
  sec.resize(off.back());
  for (int64_t t = 0; t < ntiles; ++t)
    std::memcpy(sec.data() + off[static_cast<size_t>(t)], tiles[static_cast<size_t>(t)].data(),
                tiles[static_cast<size_t>(t)].size() * 2);
  return OK;
}

}  // namespace nsk

// Test hook (not part of the public header): builds the schedule for a host
// table of ntiles * T entries (bits 0-15 bucket, bit 16 sign) into caller
// buffers.  Returns the section byte count, or -1 on failure / short buffers.
extern "C" long long nsk_internal_cs_schedule(const uint32_t* table, long long ntiles, int T, long long s,
                                              uint8_t* sec, long long sec_cap, unsigned long long* off) {
  std::vector<uint8_t> v;
  std::vector<uint64_t> o;
  uint32_t mx = 0;
  if (nsk::build_cs_schedule(table, ntiles, T, s, v, o, mx) != nsk::OK) return -1;
  if (sec && static_cast<long long>(v.size()) <= sec_cap) std::memcpy(sec, v.data(), v.size());
  if (off) std::memcpy(off, o.data(), o.size() * sizeof(uint64_t));
  return static_cast<long long>(v.size());
}
