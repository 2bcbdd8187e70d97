// gaussian_sketch.cu -- K1: SA = (1/sqrt s) G A with G regenerated on chip.
//
// Reference: apply(), gaussian branch (/root/reference/proj/src/sketch.cpp:195-205)
// multiplies the materialised s x m matrix gauss_ (filled column by column
// from stream (seed, 0), sketch.cpp:117-121) with A; complex A goes through
// two real products (real_times_complex, sketch.cpp:18-25).
//
// B200 design:
//   * G never touches HBM.  Entry G(i, j) is Gaussian #(j*s + i) of stream
//     (seed, 0) -- Philox block (j*s+i)>>1, cos for even, sin for odd -- so
//     each CTA regenerates the 64 x 32 tile it needs into shared memory.
//   * FP64 tensor cores: mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).  tcgen05 has
//     no f64 kind; on B200 DMMA and DFMA share the FP64 pipe (measured
//     36.9 TF/s DMMA-only), so Box-Muller work competes with the MMAs and the
//     n-tile is made as wide as the register file allows (G regenerated
//     ceil(n/BN) times).
//   * A tiles (32 rows x BN columns) stream in with cp.async double buffering.
//   * Split-K over m: every CTA writes a partial tile; a second kernel sums
//     the partials in fixed order (bit-identical re-runs).
#include "nsk_internal.hpp"

namespace nsk {
namespace {

constexpr int BM = 64;       // rows of G (sketch rows) per CTA
constexpr int BK = 32;       // rows of A per pipeline stage
constexpr int LDS_ = BK + 4; // padded leading dimension: conflict-free fragment loads
constexpr int THREADS = 256; // 8 warps: 2 along s x 4 along n

__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }

struct GaussParams {
  const double* A;
  int64_t lda;      // in scalars (complex elements for ncomp = 2)
  int64_t mloc;     // local rows
  int64_t row0;     // global row of local row 0
  int64_t s;
  int64_t nq;       // logical real columns = n * ncomp
  double* P;        // partials [split][nq][s]
  int64_t chunks_per_split;
  PhiloxKey key;
};

// Load the A tile for local rows [k0, k0 + BK) and logical columns
// [q0, q0 + BN) into sb[col][row].  Out-of-range entries are zero filled.
template <int BN, int NCOMP, bool VEC16>
__device__ __forceinline__ void load_a_tile(const GaussParams& p, double* sb, int64_t k0, int64_t q0) {
  if (NCOMP == 1 && VEC16) {
    constexpr int CHUNKS = BN * (BK / 2);  // 16-byte chunks
#pragma unroll
    for (int c = threadIdx.x; c < CHUNKS; c += THREADS) {
      const int col = c / (BK / 2), r2 = (c % (BK / 2)) * 2;
      const int64_t q = q0 + col, row = k0 + r2;
      int bytes = 0;
      const double* src = p.A;
      if (q < p.nq && row < p.mloc) {
        bytes = (row + 1 < p.mloc) ? 16 : 8;
        src = p.A + row + q * p.lda;
      }
      cp_async16(sb + col * LDS_ + r2, src, bytes);
    }
  } else {
    constexpr int ELEMS = BN * BK;
#pragma unroll 4
    for (int e = threadIdx.x; e < ELEMS; e += THREADS) {
      const int col = e / BK, r = e % BK;
      const int64_t q = q0 + col, row = k0 + r;
      int bytes = 0;
      const double* src = p.A;
      if (q < p.nq && row < p.mloc) {
        bytes = 8;
        if (NCOMP == 1)
          src = p.A + row + q * p.lda;
        else
          src = p.A + 2 * (row + (q >> 1) * p.lda) + (q & 1);
      }
      cp_async8(sb + col * LDS_ + r, src, bytes);
    }
  }
}

// Regenerate G rows [i0, i0 + BM) x A-rows [k0, k0 + BK) into sa[i][k].
__device__ __forceinline__ void gen_g_tile(const GaussParams& p, double* sa, int64_t i0, int64_t k0) {
  constexpr int PAIRS = (BM / 2) * BK;
#pragma unroll
  for (int t = threadIdx.x; t < PAIRS; t += THREADS) {
    const int k = t % BK, ii = (t / BK) * 2;
    const int64_t i = i0 + ii, row = k0 + k;
    double g0 = 0.0, g1 = 0.0;
    if (row < p.mloc) {
      const uint64_t L = static_cast<uint64_t>(p.row0 + row) * static_cast<uint64_t>(p.s) +
                         static_cast<uint64_t>(i);
      if ((L & 1u) == 0) {
        if (i < p.s) {
          const double2 g = gaussian_pair(p.key, L >> 1);
          g0 = g.x;
          g1 = (i + 1 < p.s) ? g.y : 0.0;
        }
      } else {  // odd s: the pair straddles two blocks
        if (i < p.s) g0 = gaussian_at(p.key, L);
        if (i + 1 < p.s) g1 = gaussian_at(p.key, L + 1);
      }
    }
    sa[ii * LDS_ + k] = g0;
    sa[(ii + 1) * LDS_ + k] = g1;
  }
}

template <int BN, int NCOMP, bool VEC16>
__global__ void __launch_bounds__(THREADS, (BN <= 128) ? 2 : 1)
    gaussian_sketch_kernel(GaussParams p) {
  constexpr int WN = BN / 4;   // columns per warp
  constexpr int TM = 32 / 8;   // 8-row MMA tiles per warp
  constexpr int TN = WN / 8;   // 8-col MMA tiles per warp
  extern __shared__ __align__(16) double smem[];
  double* sa = smem;                        // [2][BM][LDS_]
  double* sb = smem + 2 * BM * LDS_;        // [2][BN][LDS_]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp & 1, wn = warp >> 1;
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * BM;
  const int64_t q0 = static_cast<int64_t>(blockIdx.y) * BN;
  const int64_t split = blockIdx.z;
  const int64_t kbeg = split * p.chunks_per_split * BK;
  int64_t kend = kbeg + p.chunks_per_split * BK;
  if (kend > p.mloc) kend = p.mloc;

  double acc[TM][TN][2];
#pragma unroll
  for (int a = 0; a < TM; ++a)
#pragma unroll
    for (int b = 0; b < TN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  int buf = 0;
  if (kbeg < kend) {
    load_a_tile<BN, NCOMP, VEC16>(p, sb, kbeg, q0);
    cp_async_commit();
    gen_g_tile(p, sa, i0, kbeg);
  }
  for (int64_t k0 = kbeg; k0 < kend; k0 += BK) {
    const int64_t kn = k0 + BK;
    cp_async_wait_all();
    __syncthreads();  // stage `buf` complete and visible; stage buf^1 free
    if (kn < kend) {
      load_a_tile<BN, NCOMP, VEC16>(p, sb + (buf ^ 1) * BN * LDS_, kn, q0);
      cp_async_commit();
    }
    const double* A_ = sa + buf * BM * LDS_ + (wm * 32 + (lane >> 2)) * LDS_ + (lane & 3);
    const double* B_ = sb + buf * BN * LDS_ + (wn * WN + (lane >> 2)) * LDS_ + (lane & 3);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[TM], bf[TN];
#pragma unroll
      for (int a = 0; a < TM; ++a) af[a] = A_[a * 8 * LDS_ + kk];
#pragma unroll
      for (int b = 0; b < TN; ++b) bf[b] = B_[b * 8 * LDS_ + kk];
#pragma unroll
      for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < TN; ++b) dmma_884(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
    }
    if (kn < kend) gen_g_tile(p, sa + (buf ^ 1) * BM * LDS_, i0, kn);
    buf ^= 1;
  }

  // Partial tile -> P[split][q][i].  Fragment: row = lane/4, cols 2*(lane%4)+{0,1}.
  double* P = p.P + split * p.nq * p.s;
#pragma unroll
  for (int a = 0; a < TM; ++a) {
    const int64_t i = i0 + wm * 32 + a * 8 + (lane >> 2);
#pragma unroll
    for (int b = 0; b < TN; ++b) {
      const int64_t q = q0 + wn * WN + b * 8 + 2 * (lane & 3);
      if (i < p.s) {
        if (q < p.nq) P[q * p.s + i] = acc[a][b][0];
        if (q + 1 < p.nq) P[(q + 1) * p.s + i] = acc[a][b][1];
      }
    }
  }
}

// SA(i, q) = scale * sum_z P[z][q][i], z in increasing order.
template <int NCOMP>
__global__ void reduce_partials(const double* __restrict__ P, int64_t splits, int64_t s, int64_t nq,
                                double scale, double* __restrict__ SA, int64_t ldsa) {
  const int64_t total = s * nq;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t q = e / s, i = e % s;
    double v = 0.0;
    for (int64_t z = 0; z < splits; ++z) v += P[z * total + e];
    if (NCOMP == 1)
      SA[i + q * ldsa] = scale * v;
    else
      SA[2 * (i + (q >> 1) * ldsa) + (q & 1)] = scale * v;
  }
}

template <int BN, int NCOMP, bool VEC16>
int launch(const GaussParams& p0, int64_t n_tiles_q, int64_t s_tiles, int64_t splits, cudaStream_t st) {
  const size_t smem = sizeof(double) * 2 * (BM + BN) * LDS_;
  auto kern = gaussian_sketch_kernel<BN, NCOMP, VEC16>;
  NSK_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
  dim3 grid(static_cast<unsigned>(s_tiles), static_cast<unsigned>(n_tiles_q),
            static_cast<unsigned>(splits));
  KernelTimer tm(st);
  kern<<<grid, THREADS, smem, st>>>(p0);
  tm.stop();
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  return OK;
}

}  // namespace

int gaussian_apply(const Operator& op, int ncomp, const RowMap& rows, int64_t n, const double* A,
                   int64_t lda, double* SA, int64_t ldsa, cudaStream_t st) {
  if (rows.rstep != 1) return fail(EINVAL_, "gaussian shard: rows must be contiguous (rstep 1)");
  const int64_t s = op.s, nq = n * ncomp, mloc = rows.mloc;
  const double scale = 1.0 / std::sqrt(static_cast<double>(s));
  if (nq == 0) return OK;
  if (mloc == 0) {
    for (int64_t c = 0; c < n; ++c)
      NSK_CUDA_OK(cudaMemsetAsync(SA + c * ldsa * ncomp, 0, sizeof(double) * s * ncomp, st));
    return OK;
  }
  const int BN = nq <= 64 ? 64 : (nq <= 128 ? 128 : 256);
  const int64_t q_tiles = (nq + BN - 1) / BN;
  const int64_t s_tiles = (s + BM - 1) / BM;
  const int64_t chunks = (mloc + BK - 1) / BK;
  const int ctas_per_sm = BN <= 128 ? 2 : 1;
  const int64_t want = static_cast<int64_t>(sm_count()) * ctas_per_sm;
  int64_t splits = (want + s_tiles * q_tiles - 1) / (s_tiles * q_tiles);
  if (splits < 1) splits = 1;
  if (splits > chunks) splits = chunks;
  if (splits > 65535) splits = 65535;
  const int64_t per = (chunks + splits - 1) / splits;
  splits = (chunks + per - 1) / per;

  Scratch part;
  NSK_CUDA_OK(part.alloc(sizeof(double) * splits * nq * s, st));
  GaussParams p{A, lda, mloc, rows.row0, s, nq, part.as<double>(), per, op.key0};
  const bool vec16 = ncomp == 1 && (lda % 2 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
  int rc;
  if (ncomp == 2) {
    rc = BN == 64 ? launch<64, 2, false>(p, q_tiles, s_tiles, splits, st)
                  : (BN == 128 ? launch<128, 2, false>(p, q_tiles, s_tiles, splits, st)
                               : launch<256, 2, false>(p, q_tiles, s_tiles, splits, st));
  } else if (vec16) {
    rc = BN == 64 ? launch<64, 1, true>(p, q_tiles, s_tiles, splits, st)
                  : (BN == 128 ? launch<128, 1, true>(p, q_tiles, s_tiles, splits, st)
                               : launch<256, 1, true>(p, q_tiles, s_tiles, splits, st));
  } else {
    rc = BN == 64 ? launch<64, 1, false>(p, q_tiles, s_tiles, splits, st)
                  : (BN == 128 ? launch<128, 1, false>(p, q_tiles, s_tiles, splits, st)
                               : launch<256, 1, false>(p, q_tiles, s_tiles, splits, st));
  }
  if (rc != OK) return rc;
  const int64_t total = s * nq;
  const int threads = 256;
  int64_t blocks = (total + threads - 1) / threads;
  if (blocks > 4L * sm_count()) blocks = 4L * sm_count();
  if (ncomp == 1)
    reduce_partials<1><<<static_cast<unsigned>(blocks), threads, 0, st>>>(part.as<double>(), splits, s, nq,
                                                                           scale, SA, ldsa);
  else
    reduce_partials<2><<<static_cast<unsigned>(blocks), threads, 0, st>>>(part.as<double>(), splits, s, nq,
                                                                           scale, SA, ldsa);
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  return OK;
}

}  // namespace nsk
