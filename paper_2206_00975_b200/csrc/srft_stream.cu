// srft_stream.cu -- sampled srft of a real A, register-streamed tiles.
//
// Reference: apply(), srft branch (/root/reference/proj/src/sketch.cpp:206-217)
// and idft_unitary_columns (transforms.cpp:17-36): SA = R F^* D A / sqrt(s) with
// the unnormalised kernel e^{+2 pi i f j / m}.  Same algebra as srtt_tile.cu
// (decimation in time, L = 1024, j = k1 + P k2, 16 real k1 columns per tile
// paired into 8 complex sequences); what changes is how a tile reaches the
// FP64 pipe:
//
//  * no shared-memory staging of A.  Warp v loads the rows k2 = a + 32 b with
//    a in [4v, 4v + 4) for all 8 sequences straight into registers (lane =
//    sequence i + 8 (a - 4v); one 16-byte load per b covers four whole
//    128-byte row segments), so the first 32-point DFT pass starts from
//    registers, and the next tile's loads are issued right after the second
//    pass and land while the sampled stage runs (the registers of the FFT are
//    free then).  An L2 prefetch runs one more tile ahead.
//  * the Rademacher signs come as one 64-bit negate mask per lane and tile
//    (operator table built once: bit 2b + e = row a + 32 b, column K + 2i + e),
//    applied by flipping the sign bit.
//  * the sampled stage evaluates sum_i st^{2i} Z_i[q] and sum_i st^{2i}
//    conj Z_i[-q] by Horner and unpacks the Hermitian pairs once per slot and
//    tile: 8 DFMA per slot and sequence instead of 20.
//  * persistent CTAs walk equal (column, tile range) items; the next tile may
//    belong to the next item, so the stream never drains between items.
#include "fft32.cuh"
#include "nsk_internal.hpp"

namespace nsk {

namespace {

using namespace fft;

constexpr int FL = 1024;          // FFT length
constexpr int FW = 8;             // warps = complex sequences per tile
constexpr int FT = 32 * FW;       // threads
constexpr int FROW = FW + 1;      // double2 per shared-memory row (odd: conflict-free)
constexpr int FNQ = 1024 / FT;    // output slots per thread
constexpr int FKT = 2 * FW;       // real k1 columns per tile
constexpr int FANCHOR = 16;       // exact twiddles every FANCHOR tiles of an item

struct StreamParams {
  const double* A;
  int64_t lda;
  int64_t m;
  int64_t P;        // m / FL
  int64_t tiles;    // tiles per column (P / FKT)
  int64_t per;      // tiles per item
  int64_t ranges;   // items per column
  int64_t items;    // n * ranges
  const uint64_t* sgn;   // [tile][a][i] negate masks
  const int64_t* freq;   // sample index of each slot (sorted by idx mod FL)
  int nslots;
  double2* part;    // [item][FNQ * FT]
  const double2* anc;    // [range][anchor point][FNQ * FT]: w_m^{f K} at tile t0 + FANCHOR j
  int64_t apoints;       // anchor points per range: ceil(per / FANCHOR)
};

__device__ __forceinline__ double flip(double v, uint32_t mask) {
  return __hiloint2double(__double2hiint(v) ^ static_cast<int>(mask), __double2loint(v));
}
__device__ __forceinline__ void prefetch_l2(const void* p) {  // the 128-byte line holding p
  asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p));
}

// Negate masks: word (T, a, i) bit 2b + e = 1 iff the Rademacher bit of row
// j = FKT T + 2 i + e + P (a + 32 b) is 0 (rng.hpp:57: bit 1 -> +1).
__global__ void build_srft_sgn_kernel(const uint32_t* __restrict__ bits, int64_t P, int64_t words,
                                      uint64_t* __restrict__ out) {
  for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w < words;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t T = w / 256, a = (w / 8) % 32, i = w % 8;
    uint64_t v = 0;
    for (int b = 0; b < 32; ++b) {
      const int64_t j = FKT * T + 2 * i + P * (a + 32 * b);  // even: j and j + 1 share a word
      const uint32_t wd = bits[j >> 5];
      v |= static_cast<uint64_t>((~wd >> (j & 31)) & 1u) << (2 * b);
      v |= static_cast<uint64_t>((~wd >> ((j + 1) & 31)) & 1u) << (2 * b + 1);
    }
    out[w] = v;
  }
}

// anc[r][j][o] = w_m^{f_o K}, K = FKT (r per + FANCHOR j): the exact twiddle of
// slot o at every anchor point of every range (exact integer phase, then sincospi).
__global__ void srft_anchor_kernel(const int64_t* __restrict__ freq, int nslots, int64_t m, int64_t ranges,
                                   int64_t per, int64_t apoints, double2* __restrict__ anc) {
  const int64_t total = ranges * apoints * (FNQ * FT);
  const double inv_m = 1.0 / static_cast<double>(m), two_m = 2.0 / static_cast<double>(m);
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int o = static_cast<int>(e % (FNQ * FT));
    const int64_t j = (e / (FNQ * FT)) % apoints, r = e / (FNQ * FT * apoints);
    const uint64_t f = o < nslots ? static_cast<uint64_t>(freq[o]) : 0;
    const uint64_t K = static_cast<uint64_t>(FKT * (r * per + FANCHOR * j));
    anc[e] = unit_phase(mulmod_fast(f, K % static_cast<uint64_t>(m), static_cast<uint64_t>(m), inv_m), two_m);
  }
}

// (Issuing the next tile's loads after the sampled stage instead, behind an L2
// prefetch, measured 1.13 ms instead of 0.88 ms at the configs[1] shape.)
template <int PF>  // PF: L2 prefetch of the tile after the next one (NSK_STREAM_PF=0: off, 0.98 ms vs 0.88 ms)
__global__ void __launch_bounds__(FT, 1) srft_stream_kernel(StreamParams p) {
  extern __shared__ __align__(16) double2 sm2[];
  double2* U = sm2;              // [FL][FROW]
  double2* tw = U + FL * FROW;   // w_1024^k
  double2* STP = tw + FL;        // [2][FNQ][FT]: per-slot w_m^f (one column) and w_m^{16 f} (one tile)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int li = lane & 7, a = 4 * warp + (lane >> 3);
  const uint64_t m = static_cast<uint64_t>(p.m);
  const int64_t P = p.P;

  const double two_m = 2.0 / static_cast<double>(m);
  for (int k = threadIdx.x; k < FL; k += FT) tw[k] = unit_phase(static_cast<uint64_t>(k), 2.0 / FL);

  auto freq_of = [&](int q) -> uint64_t {
    const int o = threadIdx.x + FT * q;
    return o < p.nslots ? static_cast<uint64_t>(__ldg(p.freq + o)) : 0;
  };
  double2 acc[FNQ], base[FNQ];
  int bins[FNQ];  // FFT bin q | mirror bin -q << 16 of each slot
#pragma unroll
  for (int q = 0; q < FNQ; ++q) {
    const uint64_t f = freq_of(q);
    const int qi = static_cast<int>(f & (FL - 1));
    bins[q] = qi | (((FL - qi) & (FL - 1)) << 16);
    double2 s1 = unit_phase(f, two_m);
    STP[FT * q + threadIdx.x] = s1;  // w_m^f: one k1 column
#pragma unroll
    for (int r = 0; r < 4; ++r) s1 = cmul(s1, s1);
    STP[FT * (FNQ + q) + threadIdx.x] = s1;  // w_m^{16 f}: one tile
    acc[q] = make_double2(0.0, 0.0);
  }

  int64_t item = blockIdx.x;
  if (item >= p.items) return;
  int64_t col = item / p.ranges, t0 = (item % p.ranges) * p.per;
  int64_t t1 = t0 + p.per < p.tiles ? t0 + p.per : p.tiles;
  int64_t t = t0;

  double2 x[32];
  uint64_t sw;
  auto issue = [&](int64_t c, int64_t tt) {  // registers <- tile tt of column c
    const double* src = p.A + c * p.lda + FKT * tt + 2 * li + P * a;
#pragma unroll
    for (int b = 0; b < 32; ++b) x[b] = __ldcs(reinterpret_cast<const double2*>(src + P * 32 * b));
    sw = __ldg(p.sgn + (tt * 32 + a) * 8 + li);
  };
  auto prefetch = [&](int64_t c, int64_t tt) {  // L2 <- tile tt of column c (4 rows per thread)
    if (!PF) return;
    const double* src = p.A + c * p.lda + FKT * tt;
#pragma unroll
    for (int r = 0; r < FL / FT; ++r) prefetch_l2(src + P * (threadIdx.x + FT * r));
  };
  issue(col, t);
  if (t + 1 < t1) prefetch(col, t + 1);
  __syncthreads();  // twiddle table

  while (true) {
    // ---- pass 1 (registers): signs, 32-point DFT over b, twiddle w_1024^{a k}
    {
      const uint32_t lo = static_cast<uint32_t>(sw), hi = static_cast<uint32_t>(sw >> 32);
#pragma unroll
      for (int b = 0; b < 32; ++b) {
        const uint32_t wd = b < 16 ? lo : hi;
        const int sh = 2 * (b & 15);
        x[b].x = flip(x[b].x, (wd << (31 - sh)) & 0x80000000u);
        x[b].y = flip(x[b].y, (wd << (30 - sh)) & 0x80000000u);
      }
    }
    dft32(x);
#pragma unroll
    for (int k = 1; k < 32; ++k) x[k] = cmul(x[k], tw[(a * k) & (FL - 1)]);
    __syncthreads();  // previous tile's sampled stage has read U
#pragma unroll
    for (int k = 0; k < 32; ++k) U[(32 * a + k) * FROW + li] = x[k];  // 8 lanes per a: conflict-free
    __syncthreads();
    // ---- pass 2: warp = sequence, lane = k; 32-point DFT over a, bins to rows
#pragma unroll
    for (int l = 0; l < 32; ++l) x[l] = U[(32 * l + lane) * FROW + warp];
    dft32(x);
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 32; ++k) U[(lane + 32 * k) * FROW + warp] = x[k];

    // ---- next tile: same item, or the first tile of this CTA's next item
    const int64_t tcur = t, t0cur = t0, itcur = item;
    bool more = true;
    if (t + 1 < t1) {
      ++t;
    } else {
      item += gridDim.x;
      more = item < p.items;
      if (more) {
        col = item / p.ranges;
        t0 = (item % p.ranges) * p.per;
        t1 = t0 + p.per < p.tiles ? t0 + p.per : p.tiles;
        t = t0;
      }
    }
    if (more) {
      issue(col, t);
      if (t + 1 < t1) prefetch(col, t + 1);
    }
    __syncthreads();  // all bins of the tile are in U

    // ---- sampled stage: acc += w^{fK} sum_i w^{2fi} (E_i - i w^f D_i)
    // exact twiddles w_m^{f K} at the anchor points (table: no sincospi in the loop)
    if (((tcur - t0cur) % FANCHOR) == 0) {
      const double2* an = p.anc + ((itcur % p.ranges) * p.apoints + (tcur - t0cur) / FANCHOR) * (FNQ * FT);
#pragma unroll
      for (int q = 0; q < FNQ; ++q) base[q] = __ldg(an + threadIdx.x + FT * q);
    }
#pragma unroll
    for (int q = 0; q < FNQ; ++q) {
      const double2 st = STP[FT * q + threadIdx.x];
      const double2 st2 = cmul(st, st);
      const int qi = bins[q] & 0xffff, qm = bins[q] >> 16;
      double2 hq = U[qi * FROW + FW - 1], hm = U[qm * FROW + FW - 1];
      hm.y = -hm.y;
#pragma unroll
      for (int i = FW - 2; i >= 0; --i) {
        const double2 zq = U[qi * FROW + i], zm = U[qm * FROW + i];
        hq = make_double2(fma(st2.x, hq.x, fma(-st2.y, hq.y, zq.x)), fma(st2.x, hq.y, fma(st2.y, hq.x, zq.y)));
        hm = make_double2(fma(st2.x, hm.x, fma(-st2.y, hm.y, zm.x)), fma(st2.x, hm.y, fma(st2.y, hm.x, -zm.y)));
      }
      const double2 e = cadd(hq, hm), d = csub(hq, hm);
      const double2 sd = cmul(st, d);
      const double2 term = make_double2(e.x + sd.y, e.y - sd.x);
      const double2 w = base[q];
      acc[q] = make_double2(fma(w.x, term.x, fma(-w.y, term.y, acc[q].x)),
                            fma(w.x, term.y, fma(w.y, term.x, acc[q].y)));
      base[q] = cmul(w, STP[FT * (FNQ + q) + threadIdx.x]);
    }
    if (itcur != item || !more) {  // item done: its partial sums out
      double2* part = p.part + itcur * (FNQ * FT);
#pragma unroll
      for (int q = 0; q < FNQ; ++q) {
        part[threadIdx.x + FT * q] = acc[q];
        acc[q] = make_double2(0.0, 0.0);
      }
    }
    if (!more) break;
  }
}

// SA(row, c) = scale * sum_r part[c * ranges + r][o], fixed order.
__global__ void srft_stream_reduce(const double2* __restrict__ part, int64_t ranges, int64_t n, int nslots,
                                   const int32_t* __restrict__ row_of_slot, double scale, double* __restrict__ SA,
                                   int64_t ldsa) {
  const int64_t total = n * nslots;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / nslots;
    const int o = static_cast<int>(e % nslots);
    double2 v = make_double2(0.0, 0.0);
    for (int64_t r = 0; r < ranges; ++r) {
      const double2 x = part[(c * ranges + r) * (FNQ * FT) + o];
      v.x += x.x;
      v.y += x.y;
    }
    const int64_t row = row_of_slot[o];
    SA[2 * (row + c * ldsa)] = scale * v.x;
    SA[2 * (row + c * ldsa) + 1] = scale * v.y;
  }
}

}  // namespace

int build_srft_sgn(const uint32_t* sign_bits, int64_t m, uint64_t** out) {
  *out = nullptr;
  if (m % (FL * FKT) != 0) return OK;  // the stream kernel does not apply
  const int64_t P = m / FL, words = (P / FKT) * 256;
  NSK_CUDA_OK(cudaMalloc(out, sizeof(uint64_t) * words));
  int64_t blocks = (words + 255) / 256;
  if (blocks > 8L * sm_count()) blocks = 8L * sm_count();
  build_srft_sgn_kernel<<<static_cast<unsigned>(blocks), 256>>>(sign_bits, P, words, *out);
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  NSK_CUDA_OK(cudaStreamSynchronize(0));  // the table kernels ran on the legacy stream (copies on other streams continue)
  return OK;
}

// NOTAPPLICABLE unless the whole column of a real A is applied, m is a
// multiple of 16 * 1024 and A is 16-byte aligned with an even lda.
int srft_stream_apply(const Operator& op, int ncomp, const RowMap& rows, int64_t n, const double* A, int64_t lda,
                      double* SA, int64_t ldsa, cudaStream_t st) {
  if (std::getenv("NSK_SRFT_NOSTREAM")) return NOTAPPLICABLE;
  const int64_t m = op.m, s = op.s;
  if (op.kind != SRFT || ncomp != 1 || n == 0) return NOTAPPLICABLE;
  if (!(rows.row0 == 0 && rows.rstep == 1 && rows.mloc == m)) return NOTAPPLICABLE;
  if (m % (FL * FKT) != 0 || (reinterpret_cast<uintptr_t>(A) & 15) != 0 || (lda & 1) != 0) return NOTAPPLICABLE;
  const DeviceTables* tb = op.tables();
  if (!tb || !tb->srft_sgn || !tb->srtt_freq || !tb->srtt_row) return ECUDA;
  const int64_t P = m / FL, tiles = P / FKT;
  // items (column, tile range): the range count among the divisors of `tiles`
  // that minimises the busiest SM's tile count (one CTA per SM)
  const int64_t G = sm_count();
  int64_t ranges = 1, best = INT64_MAX;
  for (int64_t r = 1; r <= tiles; r *= 2) {
    if (tiles % r) break;
    const int64_t waves = (n * r + G - 1) / G, cost = waves * (tiles / r);
    if (cost < best) {
      best = cost;
      ranges = r;
    }
  }
  const int64_t per = tiles / ranges, items = n * ranges;
  const size_t smem = sizeof(double2) * (FL * FROW + FL + 2 * FNQ * FT);
  const char* pfe = std::getenv("NSK_STREAM_PF");
  auto kern = pfe && !std::atoi(pfe) ? srft_stream_kernel<0> : srft_stream_kernel<1>;
  NSK_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const double scale = 0.5 / std::sqrt(static_cast<double>(s));  // unnormalised DFT / sqrt(s); pairs carry 2
  for (int64_t b = 0; b < s; b += FNQ * FT) {
    const int ns = static_cast<int>((s - b) < FNQ * FT ? (s - b) : FNQ * FT);
    Scratch part, anc;
    const int64_t apoints = (per + FANCHOR - 1) / FANCHOR;
    NSK_CUDA_OK(part.alloc(sizeof(double2) * items * FNQ * FT, st));
    NSK_CUDA_OK(anc.alloc(sizeof(double2) * ranges * apoints * FNQ * FT, st));
    {
      int64_t blocks = (ranges * apoints * FNQ * FT + 255) / 256;
      if (blocks > 8L * G) blocks = 8L * G;
      srft_anchor_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(tb->srtt_freq + b, ns, m, ranges, per,
                                                                        apoints, anc.as<double2>());
      count_launch();
      NSK_CUDA_OK(cudaGetLastError());
    }
    StreamParams p{A, lda, m, P, tiles, per, ranges, items, tb->srft_sgn, tb->srtt_freq + b, ns,
                   part.as<double2>(), anc.as<double2>(), apoints};
    const int64_t grid = items < G ? items : G;
    KernelTimer tm(st, "srft_stream_kernel");
    kern<<<static_cast<unsigned>(grid), FT, smem, st>>>(p);
    tm.stop();
    count_launch();
    NSK_CUDA_OK(cudaGetLastError());
    int64_t blocks = (n * ns + 255) / 256;
    if (blocks > 8L * sm_count()) blocks = 8L * sm_count();
    srft_stream_reduce<<<static_cast<unsigned>(blocks), 256, 0, st>>>(part.as<double2>(), ranges, n, ns,
                                                                      tb->srtt_row + b, scale, SA, ldsa);
    count_launch();
    NSK_CUDA_OK(cudaGetLastError());
  }
  return OK;
}

}  // namespace nsk
