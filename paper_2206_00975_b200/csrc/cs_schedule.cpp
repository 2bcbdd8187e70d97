// cs_schedule.cpp -- owner schedule for the CountSketch register-bin kernel.
//
// CountSketch has no reference implementation; the draw
// protocol is documented in countsketch.cu.  The schedule is a pure function
// of the operator's buckets h(i) and signs sigma(i), built once per operator:
//
//   * the kernel runs CS_THREADS threads per CTA and every thread OWNS the
//     buckets b with b % CS_THREADS == thread, holding their bins in registers
//     (slot j = b / CS_THREADS), so no two threads ever update the same bin;
//   * a T-row tile (T <= 4096) of a column pair is staged in shared memory; the
//     rows of warp w (rows whose bucket's owner lives in warp w) are processed
//     in "iterations": in each iteration a lane handles at most one of its rows;
//   * the rows of each half-warp form a bipartite multigraph (lane, r mod 16)
//     -- r mod 16 is the shared-memory bank pair of the staged double.  An
//     iteration gives every lane at most one row and every bank pair at most
//     two (a 2-way conflict costs one extra wavefront; demanding distinct bank
//     pairs would add ~10% iterations, each ~30 instructions).  Splitting each
//     bank pair into two vertices that take its rows alternately turns this
//     into bipartite edge colouring (Koenig: Delta colours, alternating-path
//     recolouring): iterations = max(lane degree, ceil(bank degree / 2)).
//
// Layout (read by the kernel straight from global memory / L2):
//   cnt[tile][warp]                         u8   iterations of the warp
//   ent[tile][warp][group][lane]            u64  iterations 4*group + j in bits 16j..16j+15,
//                                                group < CS_GMAX (fixed stride: no offsets)
//   entry = row | slot << 12 | valid << 14 | negative << 15; an idle lane's
//   entry has no valid bit and a row whose bank pair no active lane uses.
#include <algorithm>
#include <cstring>
#include <thread>
#include <vector>

#include "nsk_internal.hpp"

namespace nsk {

namespace {

constexpr int MAXC = 4 * CS_GMAX;  // iterations per warp and tile (Delta ~ 9 at 4 rows per lane)

// Edge-colours ne edges (L[e] in [0,16), R[e] in [0,32)); returns the colour
// count or -1 if more than MAXC would be needed.
int color_half(int ne, const uint8_t* L, const uint8_t* R, uint8_t* col) {
  int16_t atL[16][MAXC], atR[32][MAXC];
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

// Builds one tile: ent (CS_WARPS * CS_GMAX * 32 u64, zeroed) and cnt
// (CS_WARPS u8).  Returns false if a warp needs more than MAXC iterations.
bool build_tile(const uint32_t* bucket_sign, int T, uint64_t* ent, uint8_t* cnt) {
  std::vector<uint16_t> rows[CS_WARPS];  // rows per warp, in increasing row order
  for (int w = 0; w < CS_WARPS; ++w) rows[w].reserve(2 * T / CS_WARPS);
  for (int r = 0; r < T; ++r) {
    const uint32_t b = bucket_sign[r] & 0xFFFFu;
    rows[(b % CS_THREADS) / 32].push_back(static_cast<uint16_t>(r));
  }
  std::vector<uint8_t> L[2], R[2], C[2];
  std::vector<uint16_t> E[2];
  uint16_t grid[MAXC][32];
  for (int w = 0; w < CS_WARPS; ++w) {
    for (int h = 0; h < 2; ++h) {
      L[h].clear();
      R[h].clear();
      E[h].clear();
    }
    // Right vertices: the two copies of each bank pair (a bank pair may serve two
    // lanes of a half-warp per iteration: at most one extra wavefront), the
    // rows of a bank pair dealt to its copies alternately.
    uint8_t seen[2][16] = {};
    for (uint16_t r : rows[w]) {
      const uint32_t e = bucket_sign[r];
      const uint32_t b = e & 0xFFFFu;
      const int lane = static_cast<int>(b % 32);
      const int h = lane >> 4;
      L[h].push_back(static_cast<uint8_t>(lane & 15));
      R[h].push_back(static_cast<uint8_t>((r & 15) * 2 + (seen[h][r & 15]++ & 1)));
      const uint32_t slot = b / CS_THREADS;
      const uint32_t neg = ((e >> 16) & 1u) ^ 1u;
      E[h].push_back(static_cast<uint16_t>(r | (slot << 12) | (1u << 14) | (neg << 15)));
    }
    int iters = 0;
    for (int h = 0; h < 2; ++h) {
      C[h].assign(L[h].size(), 0);
      const int nc = color_half(static_cast<int>(L[h].size()), L[h].data(), R[h].data(), C[h].data());
      if (nc < 0) return false;
      iters = std::max(iters, nc);
    }
    std::memset(grid, 0, sizeof grid);
    for (int h = 0; h < 2; ++h)
      for (size_t x = 0; x < E[h].size(); ++x) grid[C[h][x]][h * 16 + L[h][x]] = E[h][x];
    // Idle lanes still execute the shared loads: point each at a row whose bank
    // pair no active lane of its half-warp uses (entry without the valid bit;
    // k active lanes leave at least 16 - k bank pairs free).
    for (int k = 0; k < iters; ++k)
      for (int h = 0; h < 2; ++h) {
        uint16_t* it = grid[k] + 16 * h;
        uint32_t used = 0;
        for (int l = 0; l < 16; ++l)
          if (it[l] & 0x4000u) used |= 1u << (it[l] & 15u);
        int p = 0;
        for (int l = 0; l < 16; ++l)
          if (!(it[l] & 0x4000u)) {
            while (used & (1u << p)) ++p;
            it[l] = static_cast<uint16_t>(p);
            used |= 1u << p;
          }
      }
    cnt[w] = static_cast<uint8_t>(iters);
    uint64_t* we = ent + static_cast<size_t>(w) * CS_GMAX * 32;
    for (int k = 0; k < iters; ++k)
      for (int l = 0; l < 32; ++l)
        we[(k >> 2) * 32 + l] |= static_cast<uint64_t>(grid[k][l]) << (16 * (k & 3));
  }
  return true;
}

}  // namespace

int build_cs_schedule(const uint32_t* table, int64_t ntiles, int T, int64_t s, std::vector<uint64_t>& ent,
                      std::vector<uint8_t>& cnt) {
  const size_t per_tile = static_cast<size_t>(CS_WARPS) * CS_GMAX * 32;
  ent.resize(static_cast<size_t>(ntiles) * per_tile);
  cnt.resize(static_cast<size_t>(ntiles) * CS_WARPS);
  return build_cs_schedule_into(table, ntiles, T, s, ent.data(), cnt.data());
}

// The same into caller buffers (ntiles * CS_WARPS * CS_GMAX * 32 u64, ntiles * CS_WARPS u8); every
// worker thread zeroes its own tiles, so a pinned buffer is filled without a serial memset.
int build_cs_schedule_into(const uint32_t* table, int64_t ntiles, int T, int64_t s, uint64_t* ent_out,
                           uint8_t* cnt_out) {
  if (s < 1 || s > 4 * CS_THREADS) return EINVAL_;
  if (T < 16 || T > CS_T_MAX || T % 16) return EINVAL_;
  const size_t per_tile = static_cast<size_t>(CS_WARPS) * CS_GMAX * 32;
  unsigned nth = std::thread::hardware_concurrency();
  if (nth < 1) nth = 1;
  if (nth > 32) nth = 32;
  if (static_cast<int64_t>(nth) > ntiles) nth = static_cast<unsigned>(ntiles > 0 ? ntiles : 1);
  std::vector<char> ok(nth, 1);
  std::vector<std::thread> pool;
  for (unsigned q = 0; q < nth; ++q)
    pool.emplace_back([&, q]() {
      for (int64_t t = q; t < ntiles; t += nth) {
        uint64_t* et = ent_out + static_cast<size_t>(t) * per_tile;
        uint8_t* ct = cnt_out + static_cast<size_t>(t) * CS_WARPS;
        std::memset(et, 0, per_tile * sizeof(uint64_t));
        std::memset(ct, 0, CS_WARPS);
        if (!build_tile(table + t * T, T, et, ct)) {
          ok[q] = 0;
          return;
        }
      }
    });
  for (auto& th : pool) th.join();
  for (char c : ok)
    if (!c) return EINVAL_;
  return OK;
}

}  // namespace nsk

// Test hook (not part of the public header): builds the schedule of a host
// table of ntiles * T entries (bits 0-15 bucket, bit 16 sign) into caller
// buffers ent (ntiles * 32 * CS_GMAX * 32 u64) and cnt (ntiles * 32 u8).
// Returns 0, or -1 when no schedule exists (the streaming kernel is used).
extern "C" int nsk_internal_cs_schedule(const uint32_t* table, long long ntiles, int T, long long s, uint64_t* ent,
                                        uint8_t* cnt) {
  std::vector<uint64_t> e;
  std::vector<uint8_t> c;
  if (nsk::build_cs_schedule(table, ntiles, T, s, e, c) != nsk::OK) return -1;
  if (ent) std::memcpy(ent, e.data(), e.size() * sizeof(uint64_t));
  if (cnt) std::memcpy(cnt, c.data(), c.size());
  return 0;
}

// Group capacity, for the test hook's callers.
extern "C" int nsk_internal_cs_gmax() { return nsk::CS_GMAX; }
