// countsketch.cu -- K3: SA[h(i), :] += sigma(i) A[i, :]  (CountSketch).
//
// No reference implementation exists (SPEC.md:15,210 list CountSketch as a
// non-goal).  Draw protocol, defined on the reference's stream
// (rng.hpp:57,60-63): on stream (seed, 0) issue m x next_sign() then
// m x next_below(s); so sigma(i) = bit 0 of word i and h(i) = mulhi64 of the
// u64 (word m+2i+1 : word m+2i) with s.  Bit-exact against the compiled
// reference header (tests/test_draws.py).
//
// B200 design (HBM-bound streaming read of A, deterministic scatter-add):
//   * a per-operator row table (4 B/row, built once on the device) packs
//     h(i), sigma(i) and, inside each 256-row tile, whether row i is the
//     first of its bucket ("leader") and the offset of the next row of the
//     same bucket.  It is L2 resident (64 MiB at m = 2^24) and is re-read by
//     every column group of a row range, which the grid schedules together.
//   * a CTA owns NC columns and a contiguous range of row tiles; one thread
//     per row streams its NC values straight from HBM (coalesced 2 KiB
//     column segments) with a one-tile register prefetch.
//   * buckets inside a tile are unique among leaders, so leaders add their
//     chain's sum (rows in increasing order) into shared-memory bins with a
//     plain read-modify-write; one barrier per tile orders the tiles.  The
//     whole reduction order is fixed: bit-identical re-runs, no atomics.
//   * per-CTA bins are summed over row splits in fixed order by a second kernel.
#include "nsk_internal.hpp"

namespace nsk {

namespace {
constexpr int TILE = 256;  // rows per tile == threads per CTA
}

// Row table entry: bits 0-15 bucket, bit 16 sign(+1), bit 17 leader,
// bits 24-31 offset of the next same-bucket row in the tile (0 = none).
__global__ void build_cs_table_kernel(PhiloxKey key, int64_t m, int64_t s, uint32_t* __restrict__ out) {
  __shared__ uint32_t bucket[TILE];
  const int64_t ntiles = (m + TILE - 1) / TILE;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int r = threadIdx.x;
    const int64_t i = tile * TILE + r;
    uint32_t b = 0xFFFFFFFFu, sg = 0;
    if (i < m) {
      sg = stream_word(key, static_cast<uint64_t>(i)) & 1u;
      const uint64_t w = static_cast<uint64_t>(m) + 2u * static_cast<uint64_t>(i);
      const uint64_t u = (static_cast<uint64_t>(stream_word(key, w + 1)) << 32) | stream_word(key, w);
      b = static_cast<uint32_t>(mulhi64(u, static_cast<uint64_t>(s)));
    }
    bucket[r] = b;
    __syncthreads();
    if (i < m) {
      bool leader = true;
      for (int q = 0; q < r; ++q)
        if (bucket[q] == b) {
          leader = false;
          break;
        }
      uint32_t next = 0;
      for (int q = r + 1; q < TILE; ++q)
        if (bucket[q] == b) {
          next = static_cast<uint32_t>(q - r);
          break;
        }
      out[i] = (b & 0xFFFFu) | (sg << 16) | (static_cast<uint32_t>(leader) << 17) | (next << 24);
    }
    __syncthreads();
  }
}

int build_cs_table(PhiloxKey key, int64_t m, int64_t s, uint32_t** out) {
  *out = nullptr;
  NSK_CUDA_OK(cudaMalloc(out, sizeof(uint32_t) * m));
  const int64_t ntiles = (m + TILE - 1) / TILE;
  int64_t blocks = ntiles < 16L * sm_count() ? ntiles : 16L * sm_count();
  build_cs_table_kernel<<<static_cast<unsigned>(blocks), TILE>>>(key, m, s, *out);
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  NSK_CUDA_OK(cudaDeviceSynchronize());
  return OK;
}

namespace {

struct CsParams {
  const double* A;
  int64_t lda;
  int64_t mloc;
  int64_t row0;         // multiple of TILE
  int64_t n;
  int64_t s;
  const uint32_t* table;  // global rows
  int64_t tiles_per_split;
  int64_t ntiles;       // local tiles
  double* P;            // [split][n][s]
  double* gbins;        // global bins when they do not fit in shared memory
};

template <int NC, bool GLOBAL_BINS>
__global__ void __launch_bounds__(TILE, 2) countsketch_kernel(CsParams p) {
  extern __shared__ __align__(16) double sm[];
  const int64_t cg = blockIdx.x, split = blockIdx.y;
  const int64_t c0 = cg * NC;
  double* bins = GLOBAL_BINS ? p.gbins + (split * gridDim.x + cg) * NC * p.s : sm;
  double* stage = GLOBAL_BINS ? sm : sm + NC * p.s;  // [2][NC][TILE]
  for (int64_t e = threadIdx.x; e < NC * p.s; e += TILE) bins[e] = 0.0;

  const int r = threadIdx.x;
  int64_t t = split * p.tiles_per_split;
  int64_t tend = t + p.tiles_per_split;
  if (tend > p.ntiles) tend = p.ntiles;

  double v[NC], vn[NC];
  uint32_t e = 0, en = 0;
  auto fetch = [&](int64_t tile, double* dst, uint32_t& ent) {
    const int64_t i = tile * TILE + r;
    ent = 0;
#pragma unroll
    for (int c = 0; c < NC; ++c) dst[c] = 0.0;
    if (i < p.mloc) {
      ent = __ldg(p.table + p.row0 + i);
#pragma unroll
      for (int c = 0; c < NC; ++c)
        if (c0 + c < p.n) dst[c] = __ldcs(p.A + i + (c0 + c) * p.lda);
    }
  };
  if (t < tend) fetch(t, v, e);
  __syncthreads();
  int buf = 0;
  for (; t < tend; ++t) {
    if (t + 1 < tend) fetch(t + 1, vn, en);
    const bool leader = (e >> 17) & 1u;
    const double sg = ((e >> 16) & 1u) ? 1.0 : -1.0;
    double* st = stage + buf * NC * TILE;
    if (!leader) {  // rows past the shard stage zeros
#pragma unroll
      for (int c = 0; c < NC; ++c) st[c * TILE + r] = sg * v[c];
    }
    __syncthreads();  // stage visible; previous tile's bin updates complete
    if (leader) {
      const uint32_t b = e & 0xFFFFu;
      double acc[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) acc[c] = sg * v[c];
      int q = r;
      uint32_t nx = e >> 24;
      while (nx) {
        q += static_cast<int>(nx);
        const uint32_t eq = __ldg(p.table + p.row0 + t * TILE + q);
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[c] += st[c * TILE + q];
        nx = eq >> 24;
      }
#pragma unroll
      for (int c = 0; c < NC; ++c) bins[c * p.s + b] += acc[c];
    }
    buf ^= 1;
#pragma unroll
    for (int c = 0; c < NC; ++c) v[c] = vn[c];
    e = en;
  }
  __syncthreads();
  double* P = p.P + (split * p.n + c0) * p.s;
  for (int64_t x = threadIdx.x; x < NC * p.s; x += TILE) {
    const int64_t c = x / p.s;
    if (c0 + c < p.n) P[x] = bins[x];
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

template <int NC, bool GB>
int launch_cs(const CsParams& p, int64_t groups, int64_t splits, size_t smem, cudaStream_t st) {
  auto kern = countsketch_kernel<NC, GB>;
  NSK_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  KernelTimer tm(st);
  kern<<<dim3(static_cast<unsigned>(groups), static_cast<unsigned>(splits)), TILE, smem, st>>>(p);
  tm.stop();
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  return OK;
}

}  // namespace

int countsketch_apply(const Operator& op, const RowMap& rows, int64_t n, const double* A, int64_t lda,
                      double* SA, int64_t ldsa, cudaStream_t st) {
  const int64_t s = op.s, mloc = rows.mloc;
  if (n == 0) return OK;
  if (rows.rstep != 1 || rows.row0 % TILE != 0)
    return fail(EINVAL_, "countsketch shard: rows must be contiguous and start at a multiple of 256");
  if (s > 65536) return fail(EINVAL_, "countsketch: this build supports s <= 65536");
  const DeviceTables* tb = op.tables();
  if (!tb || !tb->cs_table) return ECUDA;
  // Columns per CTA: as many as fit next to 64 KiB of shared-memory bins.
  int NC = static_cast<int>(65536 / (s * 8));
  NC = NC >= 8 ? 8 : (NC >= 4 ? 4 : (NC >= 2 ? 2 : 1));
  const bool global_bins = s * 8 > 160 * 1024;
  if (n < NC) NC = n >= 4 ? 4 : (n >= 2 ? 2 : 1);
  const int64_t groups = (n + NC - 1) / NC;
  const int64_t ntiles = (mloc + TILE - 1) / TILE;
  int64_t splits = (2L * sm_count() + groups - 1) / groups;
  if (splits < 1) splits = 1;
  if (splits > ntiles) splits = ntiles > 0 ? ntiles : 1;
  const int64_t per = ntiles > 0 ? (ntiles + splits - 1) / splits : 0;
  if (per > 0) splits = (ntiles + per - 1) / per;
  Scratch part, gb;
  NSK_CUDA_OK(part.alloc(sizeof(double) * splits * n * s, st));
  if (global_bins) NSK_CUDA_OK(gb.alloc(sizeof(double) * splits * groups * NC * s, st));
  CsParams p{A, lda, mloc, rows.row0, n, s, tb->cs_table, per, ntiles, part.as<double>(),
             global_bins ? gb.as<double>() : nullptr};
  const size_t stage_bytes = sizeof(double) * 2 * NC * TILE;
  const size_t smem = (global_bins ? 0 : sizeof(double) * NC * s) + stage_bytes;
  int rc;
  if (global_bins) {
    rc = NC == 8 ? launch_cs<8, true>(p, groups, splits, smem, st)
                 : NC == 4 ? launch_cs<4, true>(p, groups, splits, smem, st)
                           : NC == 2 ? launch_cs<2, true>(p, groups, splits, smem, st)
                                     : launch_cs<1, true>(p, groups, splits, smem, st);
  } else {
    rc = NC == 8 ? launch_cs<8, false>(p, groups, splits, smem, st)
                 : NC == 4 ? launch_cs<4, false>(p, groups, splits, smem, st)
                           : NC == 2 ? launch_cs<2, false>(p, groups, splits, smem, st)
                                     : launch_cs<1, false>(p, groups, splits, smem, st);
  }
  if (rc != OK) return rc;
  int64_t blocks = (s * n + 255) / 256;
  if (blocks > 8L * sm_count()) blocks = 8L * sm_count();
  cs_reduce<<<static_cast<unsigned>(blocks), 256, 0, st>>>(part.as<double>(), splits, s, n, SA, ldsa);
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  return OK;
}

}  // namespace nsk
