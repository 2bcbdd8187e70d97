// gaussian_sketch.cu -- K1: SA = (1/sqrt s) G A with G regenerated on chip.
//
// Reference: apply(), gaussian branch (/root/reference/proj/src/sketch.cpp:195-205)
// multiplies the materialised s x m matrix gauss_ (filled column by column
// from stream (seed, 0), sketch.cpp:117-121) with A; complex A goes through
// two real products (real_times_complex, sketch.cpp:18-25).
//
// B200 design:
//   * G never touches HBM.  Entry G(i, j) is Gaussian #(j*s + i) of stream
//     (seed, 0) -- Philox block (j*s+i)>>1, cos for even, sin for odd.
//   * FP64 tensor cores: mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).  tcgen05 has
//     no f64 kind.  On B200 DMMA and DFMA share the FP64 pipe (measured
//     36.9 TF/s DMMA-only), so the Box-Muller work competes with the MMAs:
//     the CTA tile is as wide in n as the register file allows (BM x BN =
//     16384 accumulators: 128x128, 64x256 or 32x512; 32x384 when 256 < n <= 384
//     so fewer columns are padding) so each G entry is regenerated ceil(n / BN)
//     times.
//   * A tiles by TMA (one producer thread, 128-byte swizzled boxes, stage
//     mbarriers) for real A, contiguous [A | B] and complex A; cp.async otherwise.
//   * warp specialisation: producer warps regenerate the G tile into
//     shared memory (and stream the A tile in when TMA does not apply); 8 consumer warps
//     run the DMMAs (warp tile 32 x 64).  A 3-stage ring with named-barrier
//     full/empty handshakes overlaps generation, loads and MMAs.
//   * split-K over m: every CTA writes a partial tile; reduce_partials sums
//     them in fixed order (bit-identical re-runs).
#include <cuda.h>
#include <cstring>
#include <cudaTypedefs.h>

#include "nsk_internal.hpp"

namespace nsk {
namespace {

constexpr int CONSUMERS = 256;  // 8 MMA warps (warpgroups 0, 1)
#ifndef NSK_GAUSS_PRODUCERS
#define NSK_GAUSS_PRODUCERS 256
#endif
constexpr int PRODUCERS = NSK_GAUSS_PRODUCERS;  // generator / loader warps (warpgroups 2, 3)
constexpr int THREADS = CONSUMERS + PRODUCERS;
// With two producer warpgroups the register file is re-split with setmaxnreg:
// consumers hold 64 FP64 accumulators (128 registers) plus fragments,
// producers only Philox / Box-Muller state.
constexpr int REG_CONSUMER = 168, REG_PRODUCER = 88;

// Shared-memory tiles use a "k4-interleaved" layout: element (row x, k) of a
// tile with X rows sits at (k / 4) * (4 X) + 4 x + (k % 4).  An m8n8k4
// fragment load (x = lane / 4, k = lane % 4) then covers 32 consecutive
// doubles -- conflict-free without padding -- and a 16-byte cp.async of two
// consecutive A rows of one column stays contiguous.
template <int BN>
struct Tile {
  static constexpr int BM = BN == 384 ? 32 : 16384 / BN;              // 128, 64, 32, 32
  static constexpr int BK = BN == 128 ? 32 : 16;                       // A rows per stage
  static constexpr int STAGE = (BM + BN) * BK;                         // doubles per stage
  static constexpr int STAGES = BN == 512 ? 3 : (BN == 256 || BN == 384 ? 4 : 3);  // ring depth (<= 216 KiB)
  static constexpr int WGM = BM / 32;                                  // consumer warp grid rows
  static constexpr int TN = BN / (8 / WGM) / 8;                        // 8-column MMA tiles per warp (8 or 6)
};
// A tile by TMA: boxes {BK = 16 rows, <= 256 columns} with the 128-byte swizzle, i.e. column c's 16
// rows are one 128-byte line whose 16-byte pairs are XOR-permuted by c mod 8 (conflict-free m8n8k4
// fragment loads); the cp.async path keeps the k4 layout.
// Complex A: the column-major complex matrix as a 2-D array of doubles {2 mloc, columns}; two boxes of 8
// complex rows (128 bytes) x BN / 2 columns per tile, i.e. per half [col][8 rows][re/im] with the same
// 128-byte swizzle (complex row k of column c is 16-byte chunk (k % 8) ^ (c % 8) of c's line).  An MMA
// fragment's 8 logical columns are complex columns {0, 1, 4, 5} (+2 for odd fragments) of a group of 8,
// re and im, so its 16-byte chunks cover both halves of the bank space (2 wavefronts per load).
template <int BN, bool TMA> constexpr int box_w() { return TMA && BN > 256 ? (BN == 384 ? 192 : 256) : BN; }

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ int k4(int x, int k, int X) { return (k >> 2) * (4 * X) + 4 * x + (k & 3); }

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
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

struct GaussParams {
  const double* A;
  int64_t lda;      // in scalars (complex elements for ncomp = 2)
  const double* B;  // [A | B] in one pass (sketched TLS, tls.cpp:108-109): logical columns q >= nqa
  int64_t ldb;      //   come from B (column (q - nqa) / ncomp); B = A, nqa = nq without a second block
  int64_t nqa;
  int64_t mloc;     // local rows
  int64_t row0;     // global row of local row 0
  int64_t s;
  int64_t nq;       // logical real columns = n * ncomp
  double* P;        // partials [split][nq][s]
  int64_t chunks_per_split;
  PhiloxKey key;
  const uint32_t* zmask;  // zeroed rows (bit zoff + global row), or nullptr
  int64_t zoff;
};

// Address of [A | B](row, logical column q).
template <int NCOMP>
__device__ __forceinline__ const double* a_elem(const GaussParams& p, int64_t row, int64_t q) {
  if (q < p.nqa) return NCOMP == 1 ? p.A + row + q * p.lda : p.A + 2 * (row + (q >> 1) * p.lda) + (q & 1);
  const int64_t qb = q - p.nqa;
  return NCOMP == 1 ? p.B + row + qb * p.ldb : p.B + 2 * (row + (qb >> 1) * p.ldb) + (qb & 1);
}

// Producer: A rows [k0, k0 + BK) x logical columns [q0, q0 + BN) -> sb[col][row].
template <int BN, int NCOMP, bool VEC16>
__device__ __forceinline__ void load_a_tile(const GaussParams& p, double* sb, int64_t k0, int64_t q0, int pt) {
  using T = Tile<BN>;
  if (NCOMP == 1 && VEC16) {
    constexpr int CHUNKS = BN * (T::BK / 2);
#pragma unroll 4
    for (int c = pt; c < CHUNKS; c += PRODUCERS) {
      const int col = c / (T::BK / 2), r2 = (c % (T::BK / 2)) * 2;
      const int64_t q = q0 + col, row = k0 + r2;
      int bytes = 0;
      const double* src = p.A;
      if (q < p.nq && row < p.mloc) {
        bytes = (row + 1 < p.mloc) ? 16 : 8;
        src = a_elem<1>(p, row, q);
      }
      cp_async16(sb + k4(col, r2, BN), src, bytes);
    }
  } else {
    constexpr int ELEMS = BN * T::BK;
#pragma unroll 4
    for (int e = pt; e < ELEMS; e += PRODUCERS) {
      const int col = e / T::BK, r = e % T::BK;
      const int64_t q = q0 + col, row = k0 + r;
      int bytes = 0;
      const double* src = p.A;
      if (q < p.nq && row < p.mloc) {
        bytes = 8;
        src = a_elem<NCOMP>(p, row, q);
      }
      cp_async8(sb + k4(col, r, BN), src, bytes);
    }
  }
}

// Producer: G rows [i0, i0 + BM) x A rows [k0, k0 + BK) -> sa[i][k].
template <int BN>
__device__ __forceinline__ void gen_g_tile(const GaussParams& p, double* sa, int64_t i0, int64_t k0, int pt) {
  using T = Tile<BN>;
  constexpr int PAIRS = (T::BM / 2) * T::BK;
#pragma unroll 2
  for (int t = pt; t < PAIRS; t += PRODUCERS) {
    const int k = t % T::BK, ii = (t / T::BK) * 2;
    const int64_t i = i0 + ii, row = k0 + k;
    double g0 = 0.0, g1 = 0.0;
    bool live = row < p.mloc && i < p.s;
    if (live && p.zmask) {
      const uint64_t zb = static_cast<uint64_t>(p.zoff + p.row0 + row);
      live = ((__ldg(p.zmask + (zb >> 5)) >> (zb & 31)) & 1u) == 0;
    }
    if (live) {
      const uint64_t L = static_cast<uint64_t>(p.row0 + row) * static_cast<uint64_t>(p.s) + static_cast<uint64_t>(i);
      if ((L & 1u) == 0) {
        const double2 g = gaussian_pair(p.key, L >> 1);
        g0 = g.x;
        g1 = (i + 1 < p.s) ? g.y : 0.0;
      } else {  // odd s: the pair straddles two Philox blocks
        g0 = gaussian_at(p.key, L);
        if (i + 1 < p.s) g1 = gaussian_at(p.key, L + 1);
      }
    }
    sa[k4(ii, k, T::BM)] = g0;
    sa[k4(ii + 1, k, T::BM)] = g1;
  }
}

// TMA: the A tile of a stage comes in by cp.async.bulk.tensor (one producer thread, completion on the
// stage's mbarrier) instead of 16 cp.async per producer thread -- the producers keep their issue slots
// and registers for the Box-Muller work (real A without a second column block, mloc % 4 == 0).
template <int BN, int NCOMP, bool VEC16, bool TMA>
__global__ void __launch_bounds__(THREADS, 1) gaussian_sketch_kernel(GaussParams p,
                                                                     const __grid_constant__ CUtensorMap tmA) {
  using T = Tile<BN>;
  constexpr int BW = box_w<BN, TMA>();
  constexpr int TN = T::TN;   // 8-col MMA tiles per warp (a warp tile is 32 x 8 TN)
  constexpr int TM = 32 / 8;  // 8-row MMA tiles per warp
  extern __shared__ __align__(1024) double smem[];
  const int64_t i0 = static_cast<int64_t>(blockIdx.x) * T::BM;
  const int64_t q0 = static_cast<int64_t>(blockIdx.y) * BN;
  const int64_t split = blockIdx.z;
  const int64_t kbeg = split * p.chunks_per_split * T::BK;
  int64_t kend = kbeg + p.chunks_per_split * T::BK;
  if (kend > p.mloc) kend = p.mloc;
  const int64_t nchunks = kend > kbeg ? (kend - kbeg + T::BK - 1) / T::BK : 0;

  uint64_t* full_mb = reinterpret_cast<uint64_t*>(smem + T::STAGES * T::STAGE);  // [STAGES] (TMA)
  if (threadIdx.x >= CONSUMERS) {
    if (PRODUCERS == 256) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(REG_PRODUCER));
    if constexpr (TMA) {
      if (threadIdx.x == CONSUMERS) {
        for (int s2 = 0; s2 < T::STAGES; ++s2)
          asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_addr(full_mb + s2)));
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tmA) : "memory");
      }
      named_sync(15, PRODUCERS);  // barriers initialised before any producer waits on them
    }
    // ---------------- producers ----------------
    // Loads of LAG + 1 stages are in flight at once: stage c is issued (one
    // cp.async group) and its G tile generated while stages c-1 .. c-LAG are
    // still landing; stage c-LAG is published once its group has completed.
    constexpr int LAG = T::STAGES - 2;
    const int pt = threadIdx.x - CONSUMERS;
    // Real, 16-byte aligned A: this thread's cp.async slots are the same in
    // every chunk up to the row offset k0, so their source offsets and k4
    // destinations are computed once (the producers' register budget is the
    // consumers'): a full chunk then costs ~3 instructions per 16-byte copy.
    // Slot i of this thread is column colx0 + i * CSTEP at row offset r2 (PRODUCERS is a multiple of
    // BK / 2), so its k4 destination is soff0 + i * 4 * CSTEP; only the source addresses are kept
    // (the column may sit in A or in B).
    constexpr int PER = (BN * (T::BK / 2)) / PRODUCERS;
    constexpr int CSTEP = PRODUCERS / (T::BK / 2);
    static_assert(PRODUCERS % (T::BK / 2) == 0, "slot columns form a progression");
    const double* abase[PER];  // row-0 address of the slot's column ([A | B]), + r2
    uint32_t okmask = 0;
    const uint32_t soff0 = static_cast<uint32_t>(k4(pt / (T::BK / 2), (pt % (T::BK / 2)) * 2, BN));
    if (NCOMP == 1 && VEC16 && !TMA) {
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int cc = pt + PRODUCERS * i, colx = cc / (T::BK / 2), r2 = (cc % (T::BK / 2)) * 2;
        const int64_t q = q0 + colx;
        abase[i] = q < p.nq ? a_elem<1>(p, r2, q) : p.A;
        okmask |= (q < p.nq ? 1u : 0u) << i;
      }
    }
    for (int64_t c = 0; c < nchunks + LAG; ++c) {
      if (c < nchunks) {
        const int st = static_cast<int>(c % T::STAGES);
        if (c >= T::STAGES) named_sync(1 + T::STAGES + st, THREADS);  // consumers released stage
        double* sa = smem + st * T::STAGE;
        double* sb = sa + T::BM * T::BK;
        const int64_t k0 = kbeg + c * T::BK;
        if constexpr (TMA) {
          if (pt == 0) {  // the whole A tile: BN / BW boxes {16 rows, BW columns} (complex: one 3-D box)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_addr(full_mb + st)),
                         "r"(static_cast<uint32_t>(sizeof(double) * BN * T::BK))
                         : "memory");
            if constexpr (NCOMP == 2) {
#pragma unroll
              for (int hk = 0; hk < 2; ++hk)
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                    "[%4];\n" ::"r"(smem_addr(sb + hk * (BN / 2) * 16)),
                    "l"(&tmA), "r"(static_cast<int>(2 * k0 + 16 * hk)), "r"(static_cast<int>(q0 >> 1)),
                    "r"(smem_addr(full_mb + st))
                    : "memory");
            } else
#pragma unroll
            for (int h = 0; h < BN / BW; ++h)
              asm volatile(
                  "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
                  "[%4];\n" ::"r"(smem_addr(sb + h * BW * T::BK)),
                  "l"(&tmA), "r"(static_cast<int>(k0)), "r"(static_cast<int>(q0 + h * BW)),
                  "r"(smem_addr(full_mb + st))
                  : "memory");
          }
        } else if (NCOMP == 1 && VEC16 && k0 + T::BK <= p.mloc) {
#pragma unroll
          for (int i = 0; i < PER; ++i) {
            const bool ok = (okmask >> i) & 1u;
            cp_async16(sb + soff0 + i * 4 * CSTEP, ok ? abase[i] + k0 : p.A, ok ? 16 : 0);
          }
        } else {
          load_a_tile<BN, NCOMP, VEC16>(p, sb, k0, q0, pt);
        }
        if constexpr (!TMA) cp_async_commit();
        gen_g_tile<BN>(p, sa, i0, k0, pt);
      }
      if (c >= LAG) {
        if constexpr (TMA) {
          const int64_t cl = c - LAG;  // its A tile has landed (use cl / STAGES of that stage's barrier)
          mbar_wait(full_mb + cl % T::STAGES, static_cast<uint32_t>((cl / T::STAGES) & 1));
        } else if (c < nchunks) {
          cp_async_wait_group<LAG>();
        } else {
          cp_async_wait_all();
        }
        named_arrive(1 + static_cast<int>((c - LAG) % T::STAGES), THREADS);  // stage c-LAG full
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  if (PRODUCERS == 256) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(REG_CONSUMER));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm = warp % T::WGM, wn = warp / T::WGM;
  double acc[TM][TN][2];
#pragma unroll
  for (int a = 0; a < TM; ++a)
#pragma unroll
    for (int b = 0; b < TN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  for (int64_t c = 0; c < nchunks; ++c) {
    const int st = static_cast<int>(c % T::STAGES);
    named_sync(1 + st, THREADS);  // wait: stage full
    // k4 layout: fragment (x = lane/4, k = lane%4) of k-step kk at (kk/4)*4X + 4x + k.
    const double* A_ = smem + st * T::STAGE + 4 * (wm * 32) + lane;
    const double* B_ = smem + st * T::STAGE + T::BM * T::BK + 4 * (wn * TN * 8) + lane;
    // TMA layout: element (k, col) at col * 16 + (((k >> 1) ^ (col & 7)) << 1 | (k & 1)); a fragment's
    // column is wn * 8 TN + 8 b + lane / 4, so col & 7 = lane >> 2
    const double* Bt = smem + st * T::STAGE + T::BM * T::BK + 16 * (wn * TN * 8 + (lane >> 2));
    const double* Bc = smem + st * T::STAGE + T::BM * T::BK + 16 * (wn * TN * 4);  // complex TMA layout
#pragma unroll
    for (int kk = 0; kk < T::BK; kk += 4) {
      double af[TM];
#pragma unroll
      for (int a = 0; a < TM; ++a) af[a] = A_[kk * T::BM + a * 32];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double bf[TN / 2];
#pragma unroll
        for (int b = 0; b < TN / 2; ++b) {
          if constexpr (TMA && NCOMP == 2) {
            // fragment f = h TN / 2 + b of the warp: group g = f / 2 of 8 complex columns, complex column
            // c = wn 4 TN + 8 g + 2 (f & 1) + (j & 1) + 4 (j >> 1), j = lane / 8, re/im r = (lane / 4) & 1,
            // row k = kk + lane % 4: doubles (k / 8) (BN / 2) 16 + c 16 + 2 ((k % 8) ^ (c % 8)) + r
            const int f = h * (TN / 2) + b;
            const int j = lane >> 3;
            const int cx = 2 * (f & 1) + (j & 1) + 4 * (j >> 1);  // c % 8 (wn 4 TN + 8 g is a multiple of 8)
            const int off = (kk >> 3) * (BN / 2) * 16 + (8 * (f >> 1) + cx) * 16 +
                            ((((kk & 7) + (lane & 3)) ^ cx) << 1) + ((lane >> 2) & 1);
            bf[b] = Bc[off];
          } else if constexpr (TMA) {
            const int kx = (((kk >> 1) + ((lane >> 1) & 1)) ^ (lane >> 2)) << 1 | (lane & 1);
            bf[b] = Bt[(h * (TN / 2) + b) * 8 * 16 + kx];
          } else {
            bf[b] = B_[kk * BN + (h * (TN / 2) + b) * 32];
          }
        }
#pragma unroll
        for (int a = 0; a < TM; ++a)
#pragma unroll
          for (int b = 0; b < TN / 2; ++b)
            dmma_884(acc[a][h * (TN / 2) + b][0], acc[a][h * (TN / 2) + b][1], af[a], bf[b]);
      }
    }
    if (c + T::STAGES < nchunks) named_arrive(1 + T::STAGES + st, THREADS);  // stage free
  }

  // Partial tile -> P[split][q][i].  Fragment: row = lane/4, cols 2*(lane%4)+{0,1}.
  double* P = p.P + split * p.nq * p.s;
#pragma unroll
  for (int a = 0; a < TM; ++a) {
    const int64_t i = i0 + wm * 32 + a * 8 + (lane >> 2);
#pragma unroll
    for (int b = 0; b < TN; ++b) {
      // complex TMA: output column 2 (lane % 4) + e of fragment b is complex column
      // wn 4 TN + 8 (b / 2) + 2 (b & 1) + (j & 1) + 4 (j >> 1), j = lane % 4, re/im e
      const int jj = lane & 3;
      const int64_t q = (TMA && NCOMP == 2)
                            ? q0 + 2 * (wn * TN * 4 + 8 * (b >> 1) + 2 * (b & 1) + (jj & 1) + 4 * (jj >> 1))
                            : q0 + wn * TN * 8 + b * 8 + 2 * jj;
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

template <int BN, int NCOMP, bool VEC16, bool TMA>
int launch(const GaussParams& p0, const CUtensorMap& tm_a, int64_t n_tiles_q, int64_t s_tiles, int64_t splits,
           cudaStream_t st) {
  const size_t smem = sizeof(double) * Tile<BN>::STAGES * Tile<BN>::STAGE + sizeof(uint64_t) * Tile<BN>::STAGES;
  auto kern = gaussian_sketch_kernel<BN, NCOMP, VEC16, TMA>;
  NSK_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  dim3 grid(static_cast<unsigned>(s_tiles), static_cast<unsigned>(n_tiles_q), static_cast<unsigned>(splits));
  KernelTimer tm(st, "gaussian_sketch_kernel");
  kern<<<grid, THREADS, smem, st>>>(p0, tm_a);
  tm.stop();
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  return OK;
}

template <int NCOMP, bool VEC16, bool TMA = false>
int launch_bn(int BN, const GaussParams& p, const CUtensorMap& tm_a, int64_t q_tiles, int64_t s_tiles, int64_t splits,
              cudaStream_t st) {
  return BN == 128 ? launch<128, NCOMP, VEC16, TMA>(p, tm_a, q_tiles, s_tiles, splits, st)
       : BN == 256 ? launch<256, NCOMP, VEC16, TMA>(p, tm_a, q_tiles, s_tiles, splits, st)
       : BN == 384 ? launch<384, NCOMP, VEC16, TMA>(p, tm_a, q_tiles, s_tiles, splits, st)
                   : launch<512, NCOMP, VEC16, TMA>(p, tm_a, q_tiles, s_tiles, splits, st);
}

PFN_cuTensorMapEncodeTiled tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return static_cast<PFN_cuTensorMapEncodeTiled>(nullptr);
    }
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
  }();
  return encode;
}

// Complex A (mloc x nc complex columns, ld lda complex elements) as doubles {2 mloc, nc}: a box
// {16 doubles = 8 complex rows, BWc columns} lands as [col][8 rows][re/im] with the 128-byte swizzle.
bool encode_c_map(const double* A, int64_t lda, int64_t mloc, int64_t nc, int BWc, int BK, CUtensorMap* out) {
  PFN_cuTensorMapEncodeTiled encode = tensor_map_encoder();
  if (!encode || BWc > 256 || BK != 16) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(2 * mloc), static_cast<cuuint64_t>(nc)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(lda) * 2 * sizeof(double)};
  const cuuint32_t box[2] = {16, static_cast<cuuint32_t>(BWc)};
  const cuuint32_t estr[2] = {1, 1};
  return encode(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(A), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Tensor map of a real column-major A (mloc x nq, ld lda): a box {BK = 16 rows, BW columns} lands in
// shared memory as [col][16 rows] with the 128-byte swizzle.  false when the driver entry point is
// unavailable or the encode fails (the cp.async path runs instead).
bool encode_a_map(const double* A, int64_t lda, int64_t mloc, int64_t nq, int BW, int BK, CUtensorMap* out) {
  PFN_cuTensorMapEncodeTiled encode = tensor_map_encoder();
  if (!encode) return false;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(mloc), static_cast<cuuint64_t>(nq)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(lda) * sizeof(double)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(BK), static_cast<cuuint32_t>(BW)};
  const cuuint32_t estr[2] = {1, 1};
  return encode(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(A), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

int gaussian_apply(const Operator& op, int ncomp, const RowMap& rows, int64_t n, const double* A, int64_t lda,
                   double* SA, int64_t ldsa, cudaStream_t st) {
  const uint32_t* zmask = nullptr;
  if (int rc = op.zero_mask(&zmask)) return rc;
  return gaussian_apply_key(op.key0, op.s, zmask, 0, ncomp, rows, n, A, lda, SA, ldsa, st);
}

int gaussian_apply_key(PhiloxKey key, int64_t s, const uint32_t* zmask, int64_t zoff, int ncomp, const RowMap& rows,
                       int64_t n, const double* A, int64_t lda, double* SA, int64_t ldsa, cudaStream_t st) {
  return gaussian_apply_key2(key, s, zmask, zoff, ncomp, rows, n, A, lda, 0, nullptr, 0, SA, ldsa, st);
}

// S [A | B] in one pass: every G tile is generated once for the n + k columns (the reference forms the
// m x (n+k) copy hcat(A, B) first, tls.cpp:108); SA columns n .. n+k-1 hold S B.
int gaussian_apply_key2(PhiloxKey key, int64_t s, const uint32_t* zmask, int64_t zoff, int ncomp, const RowMap& rows,
                        int64_t n, const double* A, int64_t lda, int64_t kb, const double* B, int64_t ldb,
                        double* SA, int64_t ldsa, cudaStream_t st) {
  if (rows.rstep != 1) return fail(EINVAL_, "gaussian shard: rows must be contiguous (rstep 1)");
  if (kb == 0) B = nullptr;
  const int64_t nqa = n * ncomp;
  n += kb;
  const int64_t nq = n * ncomp, mloc = rows.mloc;
  const double scale = 1.0 / std::sqrt(static_cast<double>(s));
  if (nq == 0) return OK;
  if (mloc == 0) {
    for (int64_t c = 0; c < n; ++c)
      NSK_CUDA_OK(cudaMemsetAsync(SA + c * ldsa * ncomp, 0, sizeof(double) * s * ncomp, st));
    return OK;
  }
  // Widest n-tile that the problem fills (each G entry is regenerated once per n-tile).
  // (384: a 32 x 384 tile with 6-fragment warp tiles for 256 < nq <= 384, e.g. the 300 logical
  // columns of configs[4], 78% useful against 59% in a 512-wide tile)
  int BN = nq <= 128 ? 128 : (nq <= 256 ? 256 : (nq <= 384 ? 384 : 512));
  if (const char* e = std::getenv("NSK_GAUSS_BN")) {  // A/B override: 128, 256 or 512
    const int v = std::atoi(e);
    if (v == 128 || v == 256 || v == 384 || v == 512) BN = v;
  }
  // Must match Tile<BN>::BK: the kernel walks chunks of Tile<BN>::BK rows.
  const int BM = BN == 384 ? Tile<384>::BM : 16384 / BN, BK = BN == 128 ? Tile<128>::BK : 16;
  const int64_t q_tiles = (nq + BN - 1) / BN;
  const int64_t s_tiles = (s + BM - 1) / BM;
  const int64_t chunks = (mloc + BK - 1) / BK;
  // One CTA per SM; pick the split count so the grid is a whole number of waves.
  const int64_t sms = sm_count(), tiles = s_tiles * q_tiles;
  int64_t g = sms, t = tiles;
  while (t) {
    const int64_t r = g % t;
    g = t;
    t = r;
  }
  int64_t splits = sms / g;
  if (splits > chunks) splits = chunks;
  if (splits > 65535) splits = 65535;
  const int64_t per = (chunks + splits - 1) / splits;
  splits = (chunks + per - 1) / per;

  Scratch part;
  NSK_CUDA_OK(part.alloc(sizeof(double) * splits * nq * s, st));
  GaussParams p{A, lda, B ? B : A, B ? ldb : lda, B ? nqa : nq, mloc, rows.row0, s, nq, part.as<double>(), per, key,
                zmask, zoff};
  const bool vec16 = ncomp == 1 && (lda % 2 == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0) &&
                     (!B || ((ldb % 2 == 0) && ((reinterpret_cast<uintptr_t>(B) & 15) == 0)));
  // TMA A tiles: real A without a second column block, whole 4-row groups, lda even, 16-byte aligned
  CUtensorMap tm_a;
  std::memset(&tm_a, 0, sizeof(tm_a));
  const char* te = std::getenv("NSK_GAUSS_TMA");
  // [A | B] stored back to back with one leading dimension (the usual sketched-TLS caller: one m x (n+k)
  // buffer) is a single matrix to the tensor map
  const bool one_matrix = !B || (ldb == lda && B == A + nqa * lda);
  const bool tma_ok = one_matrix && BK == 16 && !(te && te[0] == '0');
  const int bw = BN > 256 ? (BN == 384 ? 192 : 256) : BN;
  const bool tma = vec16 && tma_ok && encode_a_map(A, lda, mloc, nq, bw, BK, &tm_a);
  const bool tma_c = ncomp == 2 && tma_ok && (reinterpret_cast<uintptr_t>(A) & 15) == 0 &&
                     encode_c_map(A, lda, mloc, nq / 2, BN / 2, BK, &tm_a);
  int rc = tma_c       ? launch_bn<2, false, true>(BN, p, tm_a, q_tiles, s_tiles, splits, st)
         : ncomp == 2 ? launch_bn<2, false>(BN, p, tm_a, q_tiles, s_tiles, splits, st)
         : tma       ? launch_bn<1, true, true>(BN, p, tm_a, q_tiles, s_tiles, splits, st)
         : vec16     ? launch_bn<1, true>(BN, p, tm_a, q_tiles, s_tiles, splits, st)
                     : launch_bn<1, false>(BN, p, tm_a, q_tiles, s_tiles, splits, st);
  if (rc != OK) return rc;
  const int64_t total = s * nq;
  const int threads = 256;
  int64_t blocks = (total + threads - 1) / threads;
  if (blocks > 4L * sm_count()) blocks = 4L * sm_count();
  if (ncomp == 1)
    reduce_partials<1><<<static_cast<unsigned>(blocks), threads, 0, st>>>(part.as<double>(), splits, s, nq, scale,
                                                                           SA, ldsa);
  else
    reduce_partials<2><<<static_cast<unsigned>(blocks), threads, 0, st>>>(part.as<double>(), splits, s, nq, scale,
                                                                           SA, ldsa);
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  return OK;
}

}  // namespace nsk
