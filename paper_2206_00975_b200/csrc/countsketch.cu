// countsketch.cu -- K3: SA[h(i), :] += sigma(i) A[i, :]  (CountSketch).
//
// No reference implementation exists (SPEC.md:15,210 list CountSketch as a
// non-goal).  Draw protocol, defined on the reference's stream
// (rng.hpp:57,60-63): on stream (seed, 0) issue m x next_sign() then
// m x next_below(s); so sigma(i) = bit 0 of word i and h(i) = mulhi64 of the
// u64 (word m+2i+1 : word m+2i) with s.  Bit-exact against the compiled
// reference header (tests/test_oracle_pins.py, tests/test_capi_host.py).
//
// B200 design (HBM-bound streaming read of A, deterministic scatter-add):
//   * a per-operator row table (4 B/row, built once on the device) packs h(i),
//     sigma(i) and, inside each 512-row chain tile, whether row i is the first
//     of its bucket ("leader") and the offset of the next same-bucket row.
//   * a CTA owns NC columns and a contiguous range of 512-row tiles.  Thread 0
//     streams each tile's NC column segments (4 KiB each) and its 2 KiB of
//     table into a D-stage shared-memory ring with 1-D TMA bulk copies
//     (cp.async.bulk ... mbarrier::complete_tx), so ~D tiles are in flight.
//   * inside a tile the leaders' buckets are unique, so each leader sums its
//     chain (rows in increasing order) and adds it to shared-memory bins with
//     a plain read-modify-write; one barrier per tile orders the tiles.  No
//     float atomics anywhere: bit-identical re-runs.
//   * per-CTA bins are summed over row splits in fixed order by cs_reduce.
#include "nsk_internal.hpp"

namespace nsk {

namespace {
constexpr int CT = 512;        // chain tile (rows)
constexpr int THREADS = 256;   // 2 rows per thread per tile
constexpr int STAGES = 4;      // TMA ring depth

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
}  // namespace

// Row table entry: bits 0-15 bucket, bit 16 sign(+1), bit 17 leader,
// bits 18-26 offset of the next same-bucket row in the 512-row tile (0 = none).
// Rows [base, base + rows) (base a multiple of CT), entry of global row i at out[i - base].
__global__ void build_cs_table_kernel(PhiloxKey key, int64_t m, int64_t s, int64_t base, int64_t rows,
                                      uint32_t* __restrict__ out) {
  __shared__ uint32_t bucket[CT];
  const int64_t ntiles = (rows + CT - 1) / CT, end = base + rows;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    for (int r = threadIdx.x; r < CT; r += blockDim.x) {
      const int64_t i = base + tile * CT + r;
      uint32_t b = 0xFFFFFFFFu;
      if (i < end) {
        const uint64_t w = static_cast<uint64_t>(m) + 2u * static_cast<uint64_t>(i);
        const uint64_t u = (static_cast<uint64_t>(stream_word(key, w + 1)) << 32) | stream_word(key, w);
        b = static_cast<uint32_t>(mulhi64(u, static_cast<uint64_t>(s)));
      }
      bucket[r] = b;
    }
    __syncthreads();
    for (int r = threadIdx.x; r < CT; r += blockDim.x) {
      const int64_t i = base + tile * CT + r;
      if (i >= end) continue;
      const uint32_t b = bucket[r];
      bool leader = true;
      for (int q = 0; q < r; ++q)
        if (bucket[q] == b) {
          leader = false;
          break;
        }
      uint32_t next = 0;
      for (int q = r + 1; q < CT; ++q)
        if (bucket[q] == b) {
          next = static_cast<uint32_t>(q - r);
          break;
        }
      const uint32_t sg = stream_word(key, static_cast<uint64_t>(i)) & 1u;
      out[i - base] = (b & 0xFFFFu) | (sg << 16) | (static_cast<uint32_t>(leader) << 17) | (next << 18);
    }
    __syncthreads();
  }
}

int build_cs_table(PhiloxKey key, int64_t m, int64_t s, int64_t base, int64_t rows, uint32_t** out) {
  *out = nullptr;
  if (rows <= 0) return OK;
  NSK_CUDA_OK(cudaMalloc(out, sizeof(uint32_t) * rows));
  const int64_t ntiles = (rows + CT - 1) / CT;
  int64_t blocks = ntiles < 16L * sm_count() ? ntiles : 16L * sm_count();
  build_cs_table_kernel<<<static_cast<unsigned>(blocks), 256>>>(key, m, s, base, rows, *out);
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  NSK_CUDA_OK(cudaStreamSynchronize(0));  // the table kernels ran on the legacy stream (copies on other streams continue)
  return OK;
}

namespace {

__device__ __forceinline__ uint32_t cs_bucket(uint32_t e) { return e & 0xFFFFu; }
__device__ __forceinline__ double cs_sign(uint32_t e) { return ((e >> 16) & 1u) ? 1.0 : -1.0; }
__device__ __forceinline__ bool cs_leader(uint32_t e) { return (e >> 17) & 1u; }
__device__ __forceinline__ uint32_t cs_next(uint32_t e) { return (e >> 18) & 0x1FFu; }

struct CsParams {
  const double* A;
  int64_t lda;
  int64_t n;
  int64_t s;
  const uint32_t* table;  // indexed by global row
  int64_t row0;           // table row (window-relative) of local row 0 (multiple of CT)
  int64_t t0;             // first tile (local) handled by split 0
  int64_t ntiles;         // tiles handled by this launch
  int64_t per;            // tiles per split
  int64_t rows_last;      // valid rows in the last tile of this launch (CT for full tiles)
  int64_t split_base;     // first partial slot written by this launch
  double* P;              // partials [split][n][s]
  double* gbins;          // bins in global memory when they do not fit in shared memory
};

// Sums one tile (values in sv[c][r], table entries in se[r]) into bins.
template <int NC>
__device__ __forceinline__ void tile_add(const double* sv, const uint32_t* se, int rows, double* bins, int64_t s,
                                         int64_t c0, int64_t n) {
  for (int r = threadIdx.x; r < rows; r += THREADS) {
    const uint32_t e = se[r];
    if (!cs_leader(e)) continue;
    double acc[NC];
    const double sg = cs_sign(e);
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = sg * sv[c * CT + r];
    int q = r;
    uint32_t nx = cs_next(e);
    while (nx) {
      q += static_cast<int>(nx);
      if (q >= rows) break;
      const uint32_t eq = se[q];
      const double sq = cs_sign(eq);
#pragma unroll
      for (int c = 0; c < NC; ++c) acc[c] += sq * sv[c * CT + q];
      nx = cs_next(eq);
    }
    const uint32_t b = cs_bucket(e);
#pragma unroll
    for (int c = 0; c < NC; ++c)
      if (c0 + c < n) bins[c * s + b] += acc[c];
  }
}

// TMA-streamed kernel: full 512-row tiles, 16-byte aligned column segments.
template <int NC, bool GLOBAL_BINS>
__global__ void __launch_bounds__(THREADS, 2) countsketch_tma_kernel(CsParams p) {
  extern __shared__ __align__(128) unsigned char smraw[];
  __shared__ __align__(8) uint64_t bars[STAGES];
  const int64_t cg = blockIdx.x, split = blockIdx.y;
  const int64_t c0 = cg * NC;
  int ncol = static_cast<int>(p.n - c0 < NC ? p.n - c0 : NC);
  double* stage_v = reinterpret_cast<double*>(smraw);                                  // [STAGES][NC][CT]
  uint32_t* stage_e = reinterpret_cast<uint32_t*>(stage_v + STAGES * NC * CT);         // [STAGES][CT]
  double* bins = GLOBAL_BINS ? p.gbins + (split * gridDim.x + cg) * NC * p.s
                             : reinterpret_cast<double*>(stage_e + STAGES * CT);       // [NC][s]
  for (int64_t e = threadIdx.x; e < NC * p.s; e += THREADS) bins[e] = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STAGES; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  const int64_t tbeg = p.t0 + split * p.per;
  int64_t tend = tbeg + p.per;
  if (tend > p.t0 + p.ntiles) tend = p.t0 + p.ntiles;
  const uint32_t vbytes = CT * 8, ebytes = CT * 4;
  auto issue = [&](int64_t t, int st) {
    mbar_expect_tx(&bars[st], vbytes * ncol + ebytes);
    for (int c = 0; c < ncol; ++c)
      tma_load_1d(stage_v + (st * NC + c) * CT, p.A + t * CT + (c0 + c) * p.lda, vbytes, &bars[st]);
    tma_load_1d(stage_e + st * CT, p.table + p.row0 + t * CT, ebytes, &bars[st]);
  };
  if (threadIdx.x == 0)
    for (int i = 0; i < STAGES; ++i)
      if (tbeg + i < tend) issue(tbeg + i, i);

  for (int64_t t = tbeg; t < tend; ++t) {
    const int64_t k = t - tbeg;
    const int st = static_cast<int>(k % STAGES);
    mbar_wait(&bars[st], static_cast<uint32_t>((k / STAGES) & 1));
    tile_add<NC>(stage_v + st * NC * CT, stage_e + st * CT, CT, bins, p.s, c0, p.n);
    __syncthreads();  // tile done: bins ordered, stage free
    if (threadIdx.x == 0 && t + STAGES < tend) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      issue(t + STAGES, st);
    }
  }
  double* P = p.P + ((p.split_base + split) * p.n + c0) * p.s;
  for (int64_t x = threadIdx.x; x < ncol * p.s; x += THREADS) P[x] = bins[x];
}

// Register-streamed kernel (default): each thread owns rows 2t, 2t+1 of every
// tile and keeps DEPTH tiles of 16-byte vector loads in flight in registers,
// so A never passes through shared memory; only the values of chain members
// (non-leaders, ~10% of rows) are staged for their leader.  Shared-memory
// traffic is the bins' read-modify-write alone.
template <int NC, bool GLOBAL_BINS>
__global__ void __launch_bounds__(THREADS, 3) countsketch_stream_kernel(CsParams p) {
  constexpr int DEPTH = NC >= 4 ? 2 : 4;  // 16-byte loads in flight per thread: DEPTH * NC
  extern __shared__ __align__(128) unsigned char smraw[];
  const int64_t cg = blockIdx.x, split = blockIdx.y;
  const int64_t c0 = cg * NC;
  const int ncol = static_cast<int>(p.n - c0 < NC ? p.n - c0 : NC);
  double* stage = reinterpret_cast<double*>(smraw);                       // [2][NC][CT] member values
  uint16_t* snext = reinterpret_cast<uint16_t*>(stage + 2 * NC * CT);    // [2][CT] member chain links
  double* bins = GLOBAL_BINS ? p.gbins + (split * gridDim.x + cg) * NC * p.s
                             : reinterpret_cast<double*>(snext + 2 * CT);
  for (int64_t e = threadIdx.x; e < NC * p.s; e += THREADS) bins[e] = 0.0;

  const int64_t tbeg = p.t0 + split * p.per;
  int64_t tend = tbeg + p.per;
  if (tend > p.t0 + p.ntiles) tend = p.t0 + p.ntiles;
  const int r0 = 2 * threadIdx.x;
  double2 v[DEPTH][NC];
  uint2 e[DEPTH];
  auto fetch = [&](int64_t t, int u) {
    if (t < tend) {
      e[u] = __ldg(reinterpret_cast<const uint2*>(p.table + p.row0 + t * CT + r0));
#pragma unroll
      for (int c = 0; c < NC; ++c)
        v[u][c] = c < ncol ? __ldcs(reinterpret_cast<const double2*>(p.A + t * CT + r0 + (c0 + c) * p.lda))
                           : make_double2(0.0, 0.0);
    }
  };
#pragma unroll
  for (int u = 0; u < DEPTH; ++u) fetch(tbeg + u, u);

  for (int64_t t = tbeg; t < tend; t += DEPTH) {
#pragma unroll
    for (int u = 0; u < DEPTH; ++u) {
      const int64_t tt = t + u;
      if (tt >= tend) break;
      double* st = stage + (tt & 1) * NC * CT;
      uint16_t* sn = snext + (tt & 1) * CT;
      const uint32_t ee[2] = {e[u].x, e[u].y};
      double vv[2][NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        vv[0][c] = cs_sign(ee[0]) * v[u][c].x;
        vv[1][c] = cs_sign(ee[1]) * v[u][c].y;
      }
#pragma unroll
      for (int j = 0; j < 2; ++j)
        if (!cs_leader(ee[j])) {
          sn[r0 + j] = static_cast<uint16_t>(cs_next(ee[j]));
#pragma unroll
          for (int c = 0; c < NC; ++c) st[c * CT + r0 + j] = vv[j][c];
        }
      fetch(tt + DEPTH, u);  // refill this slot while the tile is summed
      __syncthreads();       // staged members visible; previous tile's bin updates done
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        if (!cs_leader(ee[j])) continue;
        double acc[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[c] = vv[j][c];
        int q = r0 + j;
        uint32_t nx = cs_next(ee[j]);
        while (nx) {  // chain members, in row order, from shared memory
          q += static_cast<int>(nx);
          nx = sn[q];
#pragma unroll
          for (int c = 0; c < NC; ++c) acc[c] += st[c * CT + q];
        }
        const uint32_t b = cs_bucket(ee[j]);
#pragma unroll
        for (int c = 0; c < NC; ++c)
          if (c < ncol) bins[c * p.s + b] += acc[c];
      }
    }
  }
  __syncthreads();
  double* P = p.P + ((p.split_base + split) * p.n + c0) * p.s;
  for (int64_t x = threadIdx.x; x < ncol * p.s; x += THREADS) P[x] = bins[x];
}

// Generic kernel (unaligned inputs, the last partial tile): plain loads.
template <int NC, bool GLOBAL_BINS>
__global__ void __launch_bounds__(THREADS) countsketch_generic_kernel(CsParams p) {
  extern __shared__ __align__(128) unsigned char smraw[];
  const int64_t cg = blockIdx.x, split = blockIdx.y;
  const int64_t c0 = cg * NC;
  const int ncol = static_cast<int>(p.n - c0 < NC ? p.n - c0 : NC);
  double* sv = reinterpret_cast<double*>(smraw);                  // [NC][CT]
  uint32_t* se = reinterpret_cast<uint32_t*>(sv + NC * CT);       // [CT]
  double* bins = GLOBAL_BINS ? p.gbins + (split * gridDim.x + cg) * NC * p.s : reinterpret_cast<double*>(se + CT);
  for (int64_t e = threadIdx.x; e < NC * p.s; e += THREADS) bins[e] = 0.0;
  const int64_t tbeg = p.t0 + split * p.per;
  int64_t tend = tbeg + p.per;
  if (tend > p.t0 + p.ntiles) tend = p.t0 + p.ntiles;
  for (int64_t t = tbeg; t < tend; ++t) {
    const int rows = (t == p.t0 + p.ntiles - 1) ? static_cast<int>(p.rows_last) : CT;
    __syncthreads();
    for (int r = threadIdx.x; r < CT; r += THREADS) {
      const bool ok = r < rows;
      se[r] = ok ? __ldg(p.table + p.row0 + t * CT + r) : 0u;
#pragma unroll
      for (int c = 0; c < NC; ++c) sv[c * CT + r] = (ok && c < ncol) ? p.A[t * CT + r + (c0 + c) * p.lda] : 0.0;
    }
    __syncthreads();
    tile_add<NC>(sv, se, rows, bins, p.s, c0, p.n);
  }
  __syncthreads();
  double* P = p.P + ((p.split_base + split) * p.n + c0) * p.s;
  for (int64_t x = threadIdx.x; x < ncol * p.s; x += THREADS) P[x] = bins[x];
}

// Owner kernel (default when the schedule exists, cs_schedule.cpp): one CTA of
// CS_THREADS threads per pair of columns and row split; thread t owns the
// bins of the buckets b = t + j * CS_THREADS (j < BPT) of both columns in
// registers.  One thread streams each tile's two column segments (2 x 32 KiB)
// into a STG-deep shared-memory ring with 1-D TMA; each warp walks its
// iterations -- entries read straight from the L2-resident schedule, one
// 8-byte group of four iterations per lane, prefetched a group and a tile
// ahead -- and in every iteration each lane adds at most one staged row (both
// columns) to one of its own bins, the 16 lanes of a half-warp reading 16
// distinct bank pairs.  No bin is shared: no shared-memory read-modify-write
// and no barrier per tile; the last warp to finish a stage refills it.
struct CsOwnerParams {
  const double* A;
  int64_t lda;
  int64_t n;
  int64_t s;
  const uint64_t* ent;  // schedule of global tile 0
  const uint8_t* cnt;
  int64_t g0;           // global tile of local tile 0
  int64_t ntiles;       // tiles handled by this launch
  int64_t per;          // tiles per split
  int64_t split_base;
  double* P;            // partials [split][n][s]
};

// One schedule entry (bits 0-15 of e): bin j of both columns += sigma * value,
// as an FMA with a multiplier that is sigma for the entry's slot and 0 for the
// other slots (ptxas if-converts predicated DADDs into DADD + 2 FSEL; the
// multiplier costs one SEL per slot for both columns).  x * 0 = +-0 leaves a
// bin unchanged for every finite x; a non-finite entry of A reaches all bins
// of its owner thread.
template <int BPT>
__device__ __forceinline__ void owner_step(uint32_t e, const unsigned char* base, double (&b0)[BPT],
                                           double (&b1)[BPT]) {
  const uint32_t off = (e & 0xFFFu) * 8u;
  const double v0 = *reinterpret_cast<const double*>(base + off);
  const double v1 = *reinterpret_cast<const double*>(base + CS_T * 8 + off);
  const uint32_t one_hi = 0x3FF00000u | ((e << 16) & 0x80000000u);  // +-1.0, high word
  const uint32_t sel = e & 0x7000u;                                   // valid | slot
#pragma unroll
  for (int j = 0; j < BPT; ++j) {
    const uint32_t hi = sel == (0x4000u | (static_cast<uint32_t>(j) << 12)) ? one_hi : 0u;
    const double mj = __hiloint2double(static_cast<int>(hi), 0);
    b0[j] = fma(v0, mj, b0[j]);
    b1[j] = fma(v1, mj, b1[j]);
  }
}

// Blocking wait with a suspend-time hint: the warp sleeps until the phase
// flips instead of re-issuing try_wait.
__device__ __forceinline__ void mbar_sleep_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <int BPT, int STG>
__global__ void __launch_bounds__(CS_THREADS, 1) countsketch_owner_kernel(CsOwnerParams p) {
  extern __shared__ __align__(128) unsigned char smraw[];  // [STG][2][CS_T] doubles
  __shared__ __align__(8) uint64_t full[STG];
  __shared__ uint32_t done[STG];  // warps finished with the stage's current tile
  constexpr uint32_t stage_bytes = 2 * CS_T * 8;
  constexpr int64_t TILE_ENT = static_cast<int64_t>(CS_WARPS) * CS_GMAX * 32;  // u64 per tile
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c0 = 2 * static_cast<int64_t>(blockIdx.x), split = blockIdx.y;
  const int ncol = p.n - c0 >= 2 ? 2 : 1;
  if (threadIdx.x == 0) {
    for (int i = 0; i < STG; ++i) {
      mbar_init(&full[i], 1);
      done[i] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int64_t tbeg = split * p.per;
  const int ntl = static_cast<int>((tbeg + p.per < p.ntiles ? tbeg + p.per : p.ntiles) - tbeg);
  const double* Acol = p.A + c0 * p.lda + tbeg * CS_T;
  auto issue = [&](int k, int st) {  // one thread: tile k into stage st
    unsigned char* base = smraw + static_cast<size_t>(st) * stage_bytes;
    mbar_expect_tx(&full[st], ncol * CS_T * 8);
    tma_load_1d(base, Acol + static_cast<int64_t>(k) * CS_T, CS_T * 8, &full[st]);
    if (ncol == 2) tma_load_1d(base + CS_T * 8, Acol + p.lda + static_cast<int64_t>(k) * CS_T, CS_T * 8, &full[st]);
  };
  if (threadIdx.x == 0)
    for (int k = 0; k < STG && k < ntl; ++k) issue(k, k);

  const uint64_t* ew = p.ent + (p.g0 + tbeg) * TILE_ENT + static_cast<int64_t>(w) * (CS_GMAX * 32) + lane;
  const uint8_t* cw = p.cnt + (p.g0 + tbeg) * CS_WARPS + w;
  int n_next = ntl > 0 ? __ldg(cw) : 0;
  uint64_t g_next = ntl > 0 ? __ldg(ew) : 0;
  double b0[BPT], b1[BPT];
#pragma unroll
  for (int j = 0; j < BPT; ++j) b0[j] = b1[j] = 0.0;
  int st = 0;
  uint32_t ph = 0;
  const unsigned char* base = smraw;
  for (int k = 0; k < ntl; ++k) {
    int left = n_next;
    uint64_t E = g_next;
    const uint64_t* ek = ew + static_cast<int64_t>(k) * TILE_ENT;
    if (k + 1 < ntl) {  // next tile's count and first group
      n_next = __ldg(cw + static_cast<int64_t>(k + 1) * CS_WARPS);
      g_next = __ldg(ek + TILE_ENT);
    }
    mbar_sleep_wait(&full[st], ph);
    for (; left > 4; left -= 4) {  // full groups that have a successor
      ek += 32;
      const uint64_t En = __ldg(ek);
      const uint32_t lo = static_cast<uint32_t>(E), hi = static_cast<uint32_t>(E >> 32);
      owner_step<BPT>(lo, base, b0, b1);
      owner_step<BPT>(lo >> 16, base, b0, b1);
      owner_step<BPT>(hi, base, b0, b1);
      owner_step<BPT>(hi >> 16, base, b0, b1);
      E = En;
    }
    {  // last group: 0..4 iterations (warp-uniform)
      const uint32_t lo = static_cast<uint32_t>(E), hi = static_cast<uint32_t>(E >> 32);
      if (left > 0) owner_step<BPT>(lo, base, b0, b1);
      if (left > 1) owner_step<BPT>(lo >> 16, base, b0, b1);
      if (left > 2) owner_step<BPT>(hi, base, b0, b1);
      if (left > 3) owner_step<BPT>(hi >> 16, base, b0, b1);
    }
    __syncwarp();
    if (lane == 0) {  // the last warp to finish the stage refills it
      __threadfence_block();
      if (atomicAdd(&done[st], 1u) == CS_WARPS - 1) {
        done[st] = 0;
        __threadfence_block();
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        if (k + STG < ntl) issue(k + STG, st);
      }
    }
    if (++st == STG) {
      st = 0;
      ph ^= 1u;
      base = smraw;
    } else {
      base += stage_bytes;
    }
  }
  double* P = p.P + ((p.split_base + split) * p.n + c0) * p.s;
#pragma unroll
  for (int j = 0; j < BPT; ++j) {
    const int64_t b = static_cast<int64_t>(j) * CS_THREADS + threadIdx.x;
    if (b < p.s) {
      P[b] = b0[j];
      if (ncol == 2) P[p.s + b] = b1[j];
    }
  }
}

__global__ void cs_reduce(const double* __restrict__ P, int64_t splits, int64_t s, int64_t n,
                          double* __restrict__ SA, int64_t ldsa) {
  const int64_t total = s * n;
  for (int64_t x = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; x < total;
       x += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double v = 0.0;
    for (int64_t z = 0; z < splits; ++z) v += P[z * total + x];
    SA[(x % s) + (x / s) * ldsa] = v;
  }
}

enum Mode { GENERIC = 0, TMA_RING = 1, STREAM = 2 };

template <int NC, bool GB, int MODE>
int launch_cs(const CsParams& p, int64_t groups, int64_t splits, cudaStream_t st, bool timed) {
  size_t smem = MODE == TMA_RING ? (sizeof(double) * STAGES * NC * CT + sizeof(uint32_t) * STAGES * CT)
              : MODE == STREAM   ? sizeof(double) * 2 * NC * CT + sizeof(uint16_t) * 2 * CT
                                 : (sizeof(double) * NC * CT + sizeof(uint32_t) * CT);
  if (!GB) smem += sizeof(double) * NC * p.s;
  auto kern = MODE == TMA_RING ? countsketch_tma_kernel<NC, GB>
            : MODE == STREAM   ? countsketch_stream_kernel<NC, GB>
                               : countsketch_generic_kernel<NC, GB>;
  NSK_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  KernelTimer tm(st, MODE == TMA_RING ? "countsketch_tma_kernel" : "countsketch_kernel", timed);
  kern<<<dim3(static_cast<unsigned>(groups), static_cast<unsigned>(splits)), THREADS, smem, st>>>(p);
  tm.stop();
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  return OK;
}

template <int MODE>
int launch_nc(int NC, bool gb, const CsParams& p, int64_t groups, int64_t splits, cudaStream_t st, bool timed) {
  if (gb) {
    return NC == 4 ? launch_cs<4, true, MODE>(p, groups, splits, st, timed)
         : NC == 2 ? launch_cs<2, true, MODE>(p, groups, splits, st, timed)
                   : launch_cs<1, true, MODE>(p, groups, splits, st, timed);
  }
  return NC == 4 ? launch_cs<4, false, MODE>(p, groups, splits, st, timed)
       : NC == 2 ? launch_cs<2, false, MODE>(p, groups, splits, st, timed)
                 : launch_cs<1, false, MODE>(p, groups, splits, st, timed);
}

template <int NC, bool GB>
int stream_occupancy(int64_t s) {
  const size_t smem = sizeof(double) * 2 * NC * CT + sizeof(uint16_t) * 2 * CT + (GB ? 0 : sizeof(double) * NC * s);
  auto kern = countsketch_stream_kernel<NC, GB>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess)
    return 1;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, THREADS, smem) != cudaSuccess || occ < 1) return 1;
  return occ;
}

int stream_occupancy(int NC, bool gb, int64_t s) {
  if (gb) return NC == 4 ? stream_occupancy<4, true>(s) : NC == 2 ? stream_occupancy<2, true>(s)
                                                                  : stream_occupancy<1, true>(s);
  return NC == 4 ? stream_occupancy<4, false>(s) : NC == 2 ? stream_occupancy<2, false>(s)
                                                           : stream_occupancy<1, false>(s);
}

// NSK_CS_MODE=tma selects the TMA-ring kernel (kept for A/B measurements).
bool use_tma_ring() {
  const char* v = std::getenv("NSK_CS_MODE");
  return v && std::string(v) == "tma";
}

constexpr int CS_OWNER_STAGES = 3;  // 3 x 64 KiB of the 227 KiB

template <int BPT>
int launch_owner(const CsOwnerParams& p, int64_t splits, cudaStream_t st) {
  const size_t smem = static_cast<size_t>(CS_OWNER_STAGES) * 2 * CS_T * 8;
  auto kern = countsketch_owner_kernel<BPT, CS_OWNER_STAGES>;
  NSK_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  KernelTimer tm(st, "countsketch_owner_kernel", true);
  kern<<<dim3(static_cast<unsigned>((p.n + 1) / 2), static_cast<unsigned>(splits)), CS_THREADS, smem, st>>>(p);
  tm.stop();
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  return OK;
}

}  // namespace

bool cs_owner_eligible(int64_t s, int64_t m) {
  const char* v = std::getenv("NSK_CS_MODE");
  if (v && (std::string(v) == "tma" || std::string(v) == "stream")) return false;
  return s >= CS_THREADS && s <= 4 * CS_THREADS && m >= CS_T;
}

int countsketch_apply(const Operator& op, const RowMap& rows, int64_t n, const double* A, int64_t lda, double* SA,
                      int64_t ldsa, cudaStream_t st) {
  const int64_t s = op.s, mloc = rows.mloc;
  if (n == 0) return OK;
  if (rows.rstep != 1 || rows.row0 % CT != 0)
    return fail(EINVAL_, "countsketch shard: rows must be contiguous and start at a multiple of 512");
  if (s > 65536) return fail(EINVAL_, "countsketch: this build supports s <= 65536");
  if (mloc == 0) {
    for (int64_t c = 0; c < n; ++c) NSK_CUDA_OK(cudaMemsetAsync(SA + c * ldsa, 0, sizeof(double) * s, st));
    return OK;
  }
  const DeviceTables* tb = op.tables(rows.row0, rows.row0 + mloc);  // this shard's row window
  if (!tb || !tb->cs_table) return ECUDA;
  const int64_t wrow0 = rows.row0 - tb->cs_base;  // local row 0 inside the window
  // Columns per CTA: up to 32 KiB of shared-memory bins (3+ CTAs per SM keep
  // enough independent tiles in flight to cover the per-tile barrier).
  int NC = static_cast<int>(32768 / (s * 8));
  NC = NC >= 4 ? 4 : (NC >= 2 ? 2 : 1);
  if (n < NC) NC = n >= 2 ? 2 : 1;
  const bool gb = s * 8 > 96 * 1024;
  const int64_t groups = (n + NC - 1) / NC;
  const bool aligned = (reinterpret_cast<uintptr_t>(A) & 15) == 0 && (lda % 2) == 0;
  // Owner kernel over the leading T-row tiles that have a schedule.
  const int T = CS_T;
  int64_t own_tiles = 0, splits_o = 0, per_o = 0;
  if (aligned && tb->cs_ent && wrow0 % T == 0) {
    const int64_t g0 = wrow0 / T;
    own_tiles = mloc / T;
    if (own_tiles > tb->cs_ntiles - g0) own_tiles = tb->cs_ntiles - g0 > 0 ? tb->cs_ntiles - g0 : 0;
  }
  if (own_tiles > 0) {
    // waves of one CTA per SM: column pairs * splits a multiple of the SM count
    const int64_t sms = sm_count(), pairs = (n + 1) / 2;
    int64_t g = pairs, q = sms;
    while (q) {
      const int64_t r = g % q;
      g = q;
      q = r;
    }
    splits_o = sms / g;
    while (pairs * splits_o < 2 * sms && splits_o * 2 <= own_tiles) splits_o *= 2;
    if (splits_o > own_tiles) splits_o = own_tiles;
    per_o = (own_tiles + splits_o - 1) / splits_o;
    splits_o = (own_tiles + per_o - 1) / per_o;
  }
  const int64_t own_rows = own_tiles * T;
  const double* Ar = A + own_rows;
  const RowMap rest_map{rows.row0 + own_rows, 1, mloc - own_rows};
  const int64_t full = aligned ? (mloc - own_rows) / CT : 0;  // tiles for the streaming kernel
  const int64_t rest_rows = (mloc - own_rows) - full * CT;
  const int64_t rest_tiles = (rest_rows + CT - 1) / CT;  // tiles for the generic kernel
  const int ctas_per_sm = use_tma_ring() ? 2 : stream_occupancy(NC, gb, s);
  int64_t splits_f = 0, per_f = 0;
  if (full > 0) {
    splits_f = (static_cast<int64_t>(ctas_per_sm) * sm_count()) / groups;
    if (splits_f < 1) splits_f = 1;
    if (splits_f > full) splits_f = full;
    per_f = (full + splits_f - 1) / splits_f;
    splits_f = (full + per_f - 1) / per_f;
  }
  int64_t splits_r = 0, per_r = 0;
  if (rest_tiles > 0) {
    splits_r = (static_cast<int64_t>(ctas_per_sm) * sm_count()) / groups;
    if (splits_r < 1) splits_r = 1;
    if (splits_r > rest_tiles) splits_r = rest_tiles;
    per_r = (rest_tiles + splits_r - 1) / splits_r;
    splits_r = (rest_tiles + per_r - 1) / per_r;
  }
  const int64_t splits = splits_o + splits_f + splits_r;
  Scratch part, gbins;
  NSK_CUDA_OK(part.alloc(sizeof(double) * splits * n * s, st));
  if (gb && splits_f + splits_r > 0)
    NSK_CUDA_OK(gbins.alloc(sizeof(double) * (splits_f + splits_r) * groups * NC * s, st));
  if (own_tiles > 0) {
    CsOwnerParams p{A, lda, n, s, tb->cs_ent, tb->cs_cnt, wrow0 / T, own_tiles, per_o, 0, part.as<double>()};
    const int bpt = static_cast<int>((s + CS_THREADS - 1) / CS_THREADS);
    const int rc = bpt == 1 ? launch_owner<1>(p, splits_o, st)
                 : bpt == 2 ? launch_owner<2>(p, splits_o, st)
                            : launch_owner<4>(p, splits_o, st);
    if (rc) return rc;
  }
  if (full > 0) {
    CsParams p{Ar, lda, n, s, tb->cs_table, rest_map.row0 - tb->cs_base, 0, full, per_f, CT, splits_o, part.as<double>(),
               gb ? gbins.as<double>() : nullptr};
    const bool timed = own_tiles == 0;  // one timed (dominant) kernel per apply
    const int rc = use_tma_ring() ? launch_nc<TMA_RING>(NC, gb, p, groups, splits_f, st, timed)
                                  : launch_nc<STREAM>(NC, gb, p, groups, splits_f, st, timed);
    if (rc) return rc;
  }
  if (rest_tiles > 0) {
    const int64_t last_rows = rest_rows - (rest_tiles - 1) * CT;
    CsParams p{Ar, lda, n, s, tb->cs_table, rest_map.row0 - tb->cs_base, full, rest_tiles, per_r, last_rows,
               splits_o + splits_f,
               part.as<double>(),
               gb ? gbins.as<double>() + splits_f * groups * NC * s : nullptr};
    if (int rc = launch_nc<GENERIC>(NC, gb, p, groups, splits_r, st, full == 0 && own_tiles == 0)) return rc;
  }
  int64_t blocks = (s * n + 255) / 256;
  if (blocks > 8L * sm_count()) blocks = 8L * sm_count();
  cs_reduce<<<static_cast<unsigned>(blocks), 256, 0, st>>>(part.as<double>(), splits, s, n, SA, ldsa);
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  return OK;
}

}  // namespace nsk
