// srht_sketch.cu -- K2b: SA = sqrt(m/s) R H D A, H the normalised Hadamard matrix.
//
// No reference implementation exists (SPEC.md:15,210 list H-RHT as a
// non-goal); the draw protocol is the reference's srdct one
// (sketch.cpp:122-126): D = sign of stream word i, R = sorted Fisher-Yates
// sample.  With H_m[r, j] = (-1)^popcount(r & j) / sqrt(m):
//     SA[r, c] = (1/sqrt s) * sum_j (-1)^popcount(idx_r & j) d_j A[j, c].
//
// B200 design (HBM-bound, one pass over A):
//   * split j = j_lo + 1024 j_hi and idx = r_lo + 1024 r_hi, so the sign
//     factorises: (-1)^popc(r_lo & j_lo) * (-1)^popc(r_hi & j_hi).
//   * one warp owns a (column, j_hi) block of 2048 contiguous rows (16 KiB;
//     1024 when the shard is not 2048-row aligned): coalesced loads, butterfly
//     stages in registers on the row bits held by the register index, a padded
//     shared-memory transpose, the remaining stages: a full length-2048 FWHT
//     with no block-wide barrier.  srht_kernel16 (A 16-byte aligned, lda even)
//     moves 16 bytes per access everywhere (LDG.128, STS.128 / LDS.128);
//     srht_kernel<NQ, LB> is the 8-byte form for every other case.
//   * the warp then gathers the s sampled rows r_lo from shared memory (the
//     output slots are pre-sorted by r_lo so the gather is nearly
//     sequential) and accumulates (-1)^popc(r_hi & j_hi) Z[r_lo] in registers.
//   * persistent warps walk a contiguous range of (column, j_hi) blocks; the
//     per-warp partial sums are reduced in fixed order by a second kernel.
//   * the sign diagonal is expanded once per operator into an m-bit mask laid
//     out so that lane l's 32 rows {l + 32 t} are the bits of one u32.
#include "nsk_internal.hpp"

namespace nsk {

// ---- sign mask (m/8 bytes), built once per operator and device ------------
// word[b*32 + l] bit t = (stream word (b*1024 + l + 32 t)) & 1.
__global__ void build_sign_mask_kernel(PhiloxKey key, int64_t nblocks, uint32_t* __restrict__ out) {
  const int64_t total = nblocks * 32;
  for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w < total;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = w >> 5;
    const int l = static_cast<int>(w & 31);
    uint32_t bits = 0;
#pragma unroll 4
    for (int t = 0; t < 32; ++t) {
      const uint64_t row = static_cast<uint64_t>(b) * 1024u + static_cast<uint64_t>(l + 32 * t);
      bits |= (stream_word(key, row) & 1u) << t;
    }
    out[w] = bits;
  }
}

int build_sign_mask(PhiloxKey key, int64_t m, uint32_t** out) {
  const int64_t nblocks = m / 1024;
  *out = nullptr;
  if (nblocks == 0) return OK;
  NSK_CUDA_OK(cudaMalloc(out, sizeof(uint32_t) * nblocks * 32));
  const int64_t total = nblocks * 32;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 8L * sm_count()) blocks = 8L * sm_count();
  build_sign_mask_kernel<<<static_cast<unsigned>(blocks), 256>>>(key, nblocks, *out);
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  NSK_CUDA_OK(cudaStreamSynchronize(0));  // the table kernels ran on the legacy stream (copies on other streams continue)
  return OK;
}

namespace {

constexpr int WARPS_PER_CTA = 4;
#ifndef SRHT_GATHER_BATCH
#define SRHT_GATHER_BATCH 8
#endif
constexpr int SRHT_HI_BITS = 20;  // r_hi and j_hi bits (host-checked: m / 2048 < 2^20)

struct SrhtParams {
  const double* A;
  int64_t lda;
  int64_t n;
  int64_t nb;          // 1024-row blocks per column (local)
  int64_t jhi0;        // global j_hi of local block 0
  int64_t total;       // n * nb work items
  int64_t per;         // items per warp
  const uint32_t* mask;  // sign mask, global block index
  const uint32_t* slot;  // s_pass slot values (idx), sorted by r_lo
  int nslots;
  double* P;           // partials [warp*2 + seg][NQ*32]
  int pf;              // blocks of look-ahead for the L2 bulk prefetch (0: off; NSK_SRHT_PF)
};

__device__ __forceinline__ void bfly(double& a, double& b) {
  const double x = a, y = b;
  a = x + y;
  b = x - y;
}

// LB = log2 of the per-warp block (10: 1024 rows, 32 values per lane;
// 11: 2048 rows, 64 values per lane, which halves the gather work per element
// at the price of occupancy).
template <int NQ, int LB>
__global__ void __launch_bounds__(WARPS_PER_CTA * 32, LB == 10 ? 3 : 2) srht_kernel(SrhtParams p) {
  constexpr int L = 1 << LB, T = L / 32, PAD = L + L / 32;
  extern __shared__ double zbuf[];  // [WARPS_PER_CTA][PAD]
  __shared__ uint32_t sslot[NQ * 32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  // Slots in shared memory, packed: the padded z offset r_lo + r_lo / 32
  // (< 2^12) in the low 12 bits, r_hi (< 2^20, host-checked) above, so the
  // gather is one AND for the offset and one AND + POPC for the parity.
  for (int t = threadIdx.x; t < NQ * 32; t += blockDim.x) {
    const uint32_t v = t < p.nslots ? p.slot[t] : 0u;
    const uint32_t rlo = v & (L - 1), rhi = v >> LB;
    sslot[t] = (rlo + (rlo >> 5)) | (rhi << 12);
  }
  __syncthreads();

  const int64_t warp = static_cast<int64_t>(blockIdx.x) * WARPS_PER_CTA + wib;
  int64_t it = warp * p.per;
  int64_t end = it + p.per;
  if (end > p.total) end = p.total;
  double* z = zbuf + wib * PAD;

  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
  int seg = 0;
  // (col, blk) of item it, advanced incrementally (no 64-bit divisions in the loop).
  int64_t col = it < end ? it / p.nb : -1, blk = it < end ? it - col * p.nb : 0;
  int64_t cur_col = col;
  // Lane holds rows lane + 32 t (coalesced 256 B per load), streamed once.  The
  // next block and its sign-mask words are issued into the same registers as
  // soon as the current one has been written to shared memory, so the loads
  // overlap the gather phase.
  double x[T];
  uint32_t smk[T / 32];
  if (it < end) {
    const double* a = p.A + col * p.lda + blk * L + lane;
#pragma unroll
    for (int t = 0; t < T; ++t) x[t] = __ldcs(a + 32 * t);
#pragma unroll
    for (int h = 0; h < T / 32; ++h) smk[h] = __ldg(p.mask + ((p.jhi0 + blk) * (T / 32) + h) * 32 + lane);
  }

  for (; it < end; ++it) {
    if (p.pf > 0 && lane == 0 && it + p.pf < end) {  // stage block it + pf in L2 (one bulk prefetch)
      int64_t c3 = col, b3 = blk + p.pf;
      while (b3 >= p.nb) {
        b3 -= p.nb;
        ++c3;
      }
      const double* a3 = p.A + c3 * p.lda + b3 * L;
      if ((reinterpret_cast<uintptr_t>(a3) & 15) == 0)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a3), "r"(static_cast<unsigned>(L * 8))
                     : "memory");
    }
    if (col != cur_col) {  // column boundary: flush segment 0
      double* P = p.P + (warp * 2 + seg) * (NQ * 32);
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        P[q * 32 + lane] = acc[q];
        acc[q] = 0.0;
      }
      seg = 1;
      cur_col = col;
    }
    const int64_t jhi = p.jhi0 + blk;  // global L-row block index
    // D: flip the sign where the stream bit is 0 (rng.hpp:57); masks are per 1024 rows.
#pragma unroll
    for (int h = 0; h < T / 32; ++h) {
      const uint32_t sm = smk[h];
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        const uint32_t flip = ((~sm) >> t) & 1u;
        double& v = x[h * 32 + t];
        v = __hiloint2double(__double2hiint(v) ^ static_cast<int>(flip << 31), __double2loint(v));
      }
    }
    // Stages on row bits 5 .. LB-1 (register index t).
#pragma unroll
    for (int h = 1; h < T; h <<= 1)
#pragma unroll
      for (int t = 0; t < T; ++t)
        if ((t & h) == 0) bfly(x[t], x[t + h]);
    // Transpose through shared memory: row j at j + j/32.
#pragma unroll
    for (int t = 0; t < T; ++t) z[lane + 33 * t] = x[t];
    __syncwarp();
    // Lane now holds rows u + 32 lane + 1024 w (u < 32, w < T/32) in x[w*32 + u].
#pragma unroll
    for (int w = 0; w < T / 32; ++w)
#pragma unroll
      for (int u = 0; u < 32; ++u) x[w * 32 + u] = z[u + 33 * lane + 1056 * w];
    // Stages on row bits 0..4.
#pragma unroll
    for (int w = 0; w < T / 32; ++w)
#pragma unroll
      for (int h = 1; h < 32; h <<= 1)
#pragma unroll
        for (int u = 0; u < 32; ++u)
          if ((u & h) == 0) bfly(x[w * 32 + u], x[w * 32 + u + h]);
    __syncwarp();
#pragma unroll
    for (int w = 0; w < T / 32; ++w)
#pragma unroll
      for (int u = 0; u < 32; ++u) z[u + 33 * lane + 1056 * w] = x[w * 32 + u];
    int64_t c2 = col, b2 = blk + 1;
    if (b2 == p.nb) {
      b2 = 0;
      ++c2;
    }
    if (it + 1 < end) {  // prefetch the next block into the now free registers
      const double* a2 = p.A + c2 * p.lda + b2 * L + lane;
#pragma unroll
      for (int t = 0; t < T; ++t) x[t] = __ldcs(a2 + 32 * t);
#pragma unroll
      for (int h = 0; h < T / 32; ++h) smk[h] = __ldg(p.mask + ((p.jhi0 + b2) * (T / 32) + h) * 32 + lane);
    }
    __syncwarp();
    // Sampled second stage: acc += (-1)^popc(r_hi & j_hi) Z[r_lo].
    const uint32_t jh12 = static_cast<uint32_t>(jhi) << 12;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const uint32_t v = sslot[q * 32 + lane];
      const double zz = z[v & 0xfffu];
      const int par = static_cast<int>(__popc(v & jh12) << 31);  // (-1)^popc(r_hi & j_hi) on the sign bit
      acc[q] += __hiloint2double(__double2hiint(zz) ^ par, __double2loint(zz));
    }
    __syncwarp();
    col = c2;
    blk = b2;
  }
  if (cur_col >= 0) {
    double* P = p.P + (warp * 2 + seg) * (NQ * 32);
#pragma unroll
    for (int q = 0; q < NQ; ++q) P[q * 32 + lane] = acc[q];
  }
}

// 16-byte variant of the 2048-row kernel (A 16-byte aligned, lda even): lane l
// holds rows 2l + b + 64 t (b < 2, t < 32) as x[2t + b], so a block is 32
// LDG.128 instead of 64 LDG.64, row bit 0 and bits 6-10 are register stages,
// and both shared-memory passes move double2: row r sits at r + 2 (r >> 6), the
// transposed read gives lane l the 64 contiguous rows [64 l, 64 l + 64) (lane
// stride 528 B: conflict-free quarter-warps), bits 1-5 are the second set of
// register stages.  Half the LSU / MIO instructions of srht_kernel<NQ, 11>.
template <int NQ>
__global__ void __launch_bounds__(WARPS_PER_CTA * 32, 2) srht_kernel16(SrhtParams p) {
  constexpr int L = 2048, PAD = L + 64;
  extern __shared__ __align__(16) double zbuf[];  // [WARPS_PER_CTA][PAD], then saddr [WARPS_PER_CTA][NQ * 16]
  // gpar[k][lane] bit q = bit k of r_hi of slot q * 32 + lane: the parity word of a block,
  // pb bit q = popc(r_hi & j_hi) & 1, is the XOR of gpar[k] over the set bits k of j_hi and is
  // carried from block to block (XOR over the bits of j_hi ^ previous j_hi, ~2 per step).
  __shared__ uint32_t gpar[SRHT_HI_BITS * 32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* z = zbuf + wib * PAD;
  double2* zv = reinterpret_cast<double2*>(z);
  // Per warp: the byte offset in z of each slot's row, two 16-bit offsets per word (slots 2h, 2h + 1).
  uint32_t* saddr = reinterpret_cast<uint32_t*>(zbuf + WARPS_PER_CTA * PAD) + wib * (NQ * 16);
  const uint32_t zb = static_cast<uint32_t>(__cvta_generic_to_shared(z));
  {
    uint32_t rh[NQ], off[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int t = q * 32 + lane;
      const uint32_t v = t < p.nslots ? p.slot[t] : 0u;
      const uint32_t rlo = v & (L - 1);
      rh[q] = v >> 11;
      off[q] = 8u * (rlo + 2 * (rlo >> 6));
    }
#pragma unroll
    for (int h = 0; h < NQ / 2; ++h) saddr[h * 32 + lane] = off[2 * h] | (off[2 * h + 1] << 16);
    for (int k = wib; k < SRHT_HI_BITS; k += WARPS_PER_CTA) {
      uint32_t w = 0;
#pragma unroll
      for (int q = 0; q < NQ; ++q) w |= ((rh[q] >> k) & 1u) << q;
      gpar[k * 32 + lane] = w;
    }
  }
  __syncthreads();

  const int64_t warp = static_cast<int64_t>(blockIdx.x) * WARPS_PER_CTA + wib;
  int64_t it = warp * p.per;
  int64_t end = it + p.per;
  if (end > p.total) end = p.total;

  double acc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) acc[q] = 0.0;
  int seg = 0;
  int64_t col = it < end ? it / p.nb : -1, blk = it < end ? it - col * p.nb : 0;
  int64_t cur_col = col;
  double x[64];
  uint32_t smk[4];  // [1024-row half][b]: word of mask lane (2 lane + b) % 32 (bit lane / 16 + 2 (t % 16))
  uint32_t pb = 0, jprev = 0;
  const int mlane0 = (2 * lane) & 31, msh = lane >> 4;
  if (it < end) {
    const double2* a = reinterpret_cast<const double2*>(p.A + col * p.lda + blk * L) + lane;
#pragma unroll
    for (int t = 0; t < 32; ++t) {
      const double2 v = __ldcs(a + 32 * t);
      x[2 * t] = v.x;
      x[2 * t + 1] = v.y;
    }
#pragma unroll
    for (int h = 0; h < 4; ++h)
      smk[h] = __ldg(p.mask + ((p.jhi0 + blk) * 2 + (h >> 1)) * 32 + mlane0 + (h & 1));
  }

  for (; it < end; ++it) {
    if (p.pf > 0 && lane == 0 && it + p.pf < end) {  // stage block it + pf in L2 (one bulk prefetch)
      int64_t c3 = col, b3 = blk + p.pf;
      while (b3 >= p.nb) {
        b3 -= p.nb;
        ++c3;
      }
      const double* a3 = p.A + c3 * p.lda + b3 * L;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a3), "r"(static_cast<unsigned>(L * 8))
                   : "memory");
    }
    if (col != cur_col) {  // column boundary: flush segment 0
      double* P = p.P + (warp * 2 + seg) * (NQ * 32);
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        P[q * 32 + lane] = acc[q];
        acc[q] = 0.0;
      }
      seg = 1;
      cur_col = col;
    }
    const int64_t jhi = p.jhi0 + blk;
    for (uint32_t d = static_cast<uint32_t>(jhi) ^ jprev; d; d &= d - 1) pb ^= gpar[(__ffs(d) - 1) * 32 + lane];
    jprev = static_cast<uint32_t>(jhi);
#pragma unroll
    for (int h = 0; h < 4; ++h) smk[h] = ~(smk[h] >> msh);  // a set bit now means flip (rng.hpp:57)
    // D: row 2l + b + 64 t is bit (l / 16) + 2 (t % 16) of mask word (t / 16, lane (2l + b) % 32).
#pragma unroll
    for (int t = 0; t < 32; ++t)
#pragma unroll
      for (int b = 0; b < 2; ++b) {
        const uint32_t flip = (smk[(t >> 4) * 2 + b] >> (2 * (t & 15))) & 1u;
        double& v = x[2 * t + b];
        v = __hiloint2double(__double2hiint(v) ^ static_cast<int>(flip << 31), __double2loint(v));
      }
    // Row bit 0, then bits 6..10 (register index t).
#pragma unroll
    for (int t = 0; t < 32; ++t) bfly(x[2 * t], x[2 * t + 1]);
#pragma unroll
    for (int h = 1; h < 32; h <<= 1)
#pragma unroll
      for (int t = 0; t < 32; ++t)
        if ((t & h) == 0) {
          bfly(x[2 * t], x[2 * (t + h)]);
          bfly(x[2 * t + 1], x[2 * (t + h) + 1]);
        }
#pragma unroll
    for (int t = 0; t < 32; ++t) zv[lane + 33 * t] = make_double2(x[2 * t], x[2 * t + 1]);
    __syncwarp();
    // Lane now holds rows 64 lane + j in x[j].
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const double2 v = zv[33 * lane + j];
      x[2 * j] = v.x;
      x[2 * j + 1] = v.y;
    }
    // Row bits 1..5.
#pragma unroll
    for (int h = 2; h < 64; h <<= 1)
#pragma unroll
      for (int j = 0; j < 64; ++j)
        if ((j & h) == 0) bfly(x[j], x[j + h]);
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 32; ++j) zv[33 * lane + j] = make_double2(x[2 * j], x[2 * j + 1]);
    int64_t c2 = col, b2 = blk + 1;
    if (b2 == p.nb) {
      b2 = 0;
      ++c2;
    }
    if (it + 1 < end) {  // prefetch the next block into the now free registers
      const double2* a2 = reinterpret_cast<const double2*>(p.A + c2 * p.lda + b2 * L) + lane;
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        const double2 v = __ldcs(a2 + 32 * t);
        x[2 * t] = v.x;
        x[2 * t + 1] = v.y;
      }
#pragma unroll
      for (int h = 0; h < 4; ++h)
        smk[h] = __ldg(p.mask + ((p.jhi0 + b2) * 2 + (h >> 1)) * 32 + mlane0 + (h & 1));
    }
    __syncwarp();
    // Sampled second stage: acc += (-1)^popc(r_hi & j_hi) Z[r_lo], the parity from pb.
    // Batches of GB slots: all addresses, then all rows, then the sums, so the two shared-memory
    // latencies are paid once per batch instead of once per slot.
    constexpr int GB = SRHT_GATHER_BATCH;
#pragma unroll
    for (int q0 = 0; q0 < NQ; q0 += GB) {
      uint32_t ad[GB];
      double zz[GB];
#pragma unroll
      for (int u = 0; u < GB; u += 2) {
        const uint32_t w2 = saddr[((q0 + u) >> 1) * 32 + lane];
        ad[u] = zb + (w2 & 0xffffu);
        ad[u + 1] = zb + (w2 >> 16);
      }
#pragma unroll
      for (int u = 0; u < GB; ++u) asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(zz[u]) : "r"(ad[u]) : "memory");
#pragma unroll
      for (int u = 0; u < GB; ++u) {
        const int par = static_cast<int>((pb << (31 - (q0 + u))) & 0x80000000u);
        acc[q0 + u] += __hiloint2double(__double2hiint(zz[u]) ^ par, __double2loint(zz[u]));
      }
    }
    __syncwarp();
    col = c2;
    blk = b2;
  }
  if (cur_col >= 0) {
    double* P = p.P + (warp * 2 + seg) * (NQ * 32);
#pragma unroll
    for (int q = 0; q < NQ; ++q) P[q * 32 + lane] = acc[q];
  }
}

// SA[row(t), c] = scale * sum over the warps that touched column c, in warp
// order.  One CTA per column: the warp range and segments are uniform, the
// threads walk the slots (coalesced partial reads, several sums in flight).
__global__ void __launch_bounds__(256) srht_reduce(const double* __restrict__ P, int64_t nb, int64_t per,
                                                   int nslots, int slot_stride,
                                                   const int32_t* __restrict__ row_of_slot, double scale,
                                                   double* __restrict__ SA, int64_t ldsa) {
  const int64_t c = blockIdx.x;
  const int64_t w0 = (c * nb) / per, w1 = ((c + 1) * nb - 1) / per;
  constexpr int U = 4;
  for (int t0 = threadIdx.x; t0 < nslots; t0 += 256 * U) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = 0.0;
    for (int64_t wb = w0; wb <= w1; wb += 4) {  // four warps' partials in flight, summed in warp order
      double t4[4][U];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t w = wb + j;
        const int seg = w * per >= c * nb ? 0 : 1;  // the warp's first item lies in column c
        const double* Pw = P + (w * 2 + seg) * slot_stride;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int t = t0 + 256 * u;
          t4[j][u] = (w <= w1 && t < nslots) ? __ldcg(Pw + t) : 0.0;
        }
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] += t4[j][u];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int t = t0 + 256 * u;
      if (t < nslots) SA[row_of_slot[t] + c * ldsa] = scale * v[u];
    }
  }
}

// Small or misaligned shards: direct evaluation, O(s * mloc) per column.
__global__ void srht_direct(const double* __restrict__ A, int64_t lda, int64_t mloc, int64_t row0,
                            int64_t n, const int64_t* __restrict__ idx, int64_t s, PhiloxKey key,
                            double scale, double* __restrict__ SA, int64_t ldsa) {
  const int64_t total = s * n;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / s, r = e % s;
    const uint64_t ir = static_cast<uint64_t>(idx[r]);
    double v = 0.0;
    for (int64_t j = 0; j < mloc; ++j) {
      const uint64_t g = static_cast<uint64_t>(row0 + j);
      double a = apply_sign(A[j + c * lda], stream_word(key, g));
      v += (__popcll(ir & g) & 1) ? -a : a;
    }
    SA[r + c * ldsa] = scale * v;
  }
}

template <int NQ, int LB>
int launch_srht_lb(SrhtParams p, int64_t warps, cudaStream_t st) {
  const int64_t ctas = (warps + WARPS_PER_CTA - 1) / WARPS_PER_CTA;
  const size_t smem = sizeof(double) * WARPS_PER_CTA * ((1 << LB) + (1 << LB) / 32);
  auto kern = srht_kernel<NQ, LB>;
  NSK_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  KernelTimer tm(st, "srht_kernel");
  kern<<<static_cast<unsigned>(ctas), WARPS_PER_CTA * 32, smem, st>>>(p);
  tm.stop();
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  return OK;
}

template <int NQ>
int launch_srht16(SrhtParams p, int64_t warps, cudaStream_t st) {
  const int64_t ctas = (warps + WARPS_PER_CTA - 1) / WARPS_PER_CTA;
  const size_t smem = sizeof(double) * WARPS_PER_CTA * (2048 + 64) + sizeof(uint32_t) * WARPS_PER_CTA * NQ * 16;
  auto kern = srht_kernel16<NQ>;
  NSK_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  KernelTimer tm(st, "srht_kernel16");
  kern<<<static_cast<unsigned>(ctas), WARPS_PER_CTA * 32, smem, st>>>(p);
  tm.stop();
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  return OK;
}

// lb: 10, 11, or 12 = the 16-byte variant of 11
template <int NQ>
int launch_srht(SrhtParams p, int64_t warps, int lb, cudaStream_t st) {
  return lb == 12 ? launch_srht16<NQ>(p, warps, st)
       : lb == 11 ? launch_srht_lb<NQ, 11>(p, warps, st)
                  : launch_srht_lb<NQ, 10>(p, warps, st);
}

}  // namespace

int srht_apply(const Operator& op, const RowMap& rows, int64_t n, const double* A, int64_t lda,
               double* SA, int64_t ldsa, cudaStream_t st) {
  const int64_t s = op.s, mloc = rows.mloc;
  const double scale = 1.0 / std::sqrt(static_cast<double>(s));
  if (n == 0) return OK;
  const DeviceTables* tb = op.tables();
  if (!tb) return ECUDA;
  if (rows.rstep != 1) return fail(EINVAL_, "srht shard: rows must be contiguous (rstep 1)");
  // Per-warp block of 2^lb rows: 2048 when the shard allows (NSK_SRHT_LB=10 forces 1024).
  const char* lbenv = std::getenv("NSK_SRHT_LB");
  int lb = (lbenv && lbenv[0] == '1' && lbenv[1] == '0') ? 10 : 11;
  if (!(op.m >= 2048 && mloc % 2048 == 0 && rows.row0 % 2048 == 0)) lb = 10;
  const int64_t L = int64_t(1) << lb;
  const bool blocked = op.m >= L && mloc >= L && (mloc % L) == 0 && (rows.row0 % L) == 0 &&
                       tb->sign_mask != nullptr && (op.m >> lb) < (int64_t(1) << 20);  // packed slot words
  if (!blocked) {
    int64_t blocks = (s * n + 127) / 128;
    if (blocks > 16L * sm_count()) blocks = 16L * sm_count();
    srht_direct<<<static_cast<unsigned>(blocks), 128, 0, st>>>(A, lda, mloc, rows.row0, n, tb->idx, s, op.key0,
                                                               scale, SA, ldsa);
    count_launch();
    NSK_CUDA_OK(cudaGetLastError());
    return OK;
  }
  const int64_t nb = mloc / L;
  const int64_t total = n * nb;
  const int64_t max_warps = static_cast<int64_t>(sm_count()) * (lb == 10 ? 3 : 2) * WARPS_PER_CTA;
  int64_t warps = total < max_warps ? total : max_warps;
  int64_t per = (total + warps - 1) / warps;
  if (per > nb) per = nb;  // a warp touches at most two columns
  warps = (total + per - 1) / per;
  // Outputs in passes of at most 1024 slots (one register accumulator each).
  for (int64_t base = 0; base < s; base += 1024) {
    const int ns = static_cast<int>((s - base) < 1024 ? (s - base) : 1024);
    const int nq = (ns + 31) / 32;
    const int NQ = nq <= 8 ? 8 : (nq <= 16 ? 16 : 32);
    Scratch part;
    NSK_CUDA_OK(part.alloc(sizeof(double) * warps * 2 * NQ * 32, st));
    const char* pfe = std::getenv("NSK_SRHT_PF");
    SrhtParams p{A, lda, n, nb, rows.row0 / L, total, per, tb->sign_mask, tb->srht_slot + base, ns,
                 part.as<double>(), pfe ? std::atoi(pfe) : 1};  // 1 vs 2 blocks ahead: 0.3727 vs 0.3744 ms at configs[1]
    // 2048-row blocks by 16-byte loads when every block start is 16-byte aligned (NSK_SRHT_V16=0: 8-byte kernel)
    const char* v16e = std::getenv("NSK_SRHT_V16");
    const bool v16 = lb == 11 && (reinterpret_cast<uintptr_t>(A) & 15) == 0 && (lda % 2 == 0) &&
                     !(v16e && v16e[0] == '0');
    const int lbk = v16 ? 12 : lb;
    int rc = NQ == 8 ? launch_srht<8>(p, warps, lbk, st)
                     : (NQ == 16 ? launch_srht<16>(p, warps, lbk, st) : launch_srht<32>(p, warps, lbk, st));
    if (rc != OK) return rc;
    srht_reduce<<<static_cast<unsigned>(n), 256, 0, st>>>(part.as<double>(), nb, per, ns, NQ * 32,
                                                          tb->srht_row + base, scale, SA, ldsa);
    count_launch();
    NSK_CUDA_OK(cudaGetLastError());
  }
  return OK;
}

}  // namespace nsk
