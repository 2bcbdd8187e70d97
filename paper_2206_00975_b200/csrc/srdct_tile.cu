// srdct_tile.cu -- sampled srdct with half the FFT work of the zero-padded
// formulation in srtt_tile.cu: Makhoul's pairing of row k with row N - k.
//
// Reference: apply(), srdct branch (sketch.cpp:218-229) and the orthonormal
// DCT-III of transforms.cpp:38-64:  y_a = sum_k X_k cos(pi k (2a+1) / 2N),
// X_k = c_k d_k A[k] (c_0 = sqrt(1/N), c_k = sqrt(2/N)), SA = sqrt(N/s) y_idx.
//
// With omega = e^{i pi / 2N}, W = e^{2 pi i / N} and
//   G_k = (X_k - i X_{N-k}) omega^k / 2   (G_0 = X_0, X_N = 0),
// G is Hermitian (G_{N-k} = conj G_k), v_n = sum_k G_k W^{kn} is real, and
//   y_{2n} = v_n,   y_{2n+1} = v_{N-1-n}
// (the transpose of Makhoul's DCT-II; checked against scipy's DCT-III).
// Hermitian symmetry halves the sum: with k = k1 + P k2 (P = N / L, L = 1024),
// only the columns k1 in [0, P/2] are transformed and
//   v_n = sum_{k1 <= P/2} 2 Re( W^{n k1} F_{k1}[n mod L] ),  F_{k1} = DFT_L(e_{k1})
// where e_{k1}[k2] = G_{k1 + P k2} for 0 < k1 < P/2 (the mirror k1' = P - k1
// is conj), and the self-mirrored columns k1 = 0 and P/2 keep their lower
// half (k2 < L/2) with half weights at k2 = 0 and L/2 (column 0).  Each
// complex FFT now carries 2048 real inputs (srtt_tile's srdct: 1024).
//
// A CTA (8 warps) walks tiles of 8 consecutive k1 in [0, P/2) plus one tile
// holding column P/2.  Per tile it stages, for every k2, the 8 main elements
// (64 contiguous bytes) and the 9 mirror elements P - 8t - 8 .. P - 8t at row
// L - 1 - k2 (64 + 8 bytes), with their sign words, into one 144-byte row of
// shared memory; forms G in place (a thread owns rows k2 and L - 1 - k2, so
// each row's raw data is read before its G is written); one in-place
// 1024-point FFT per warp (the srtt_tile pattern); and accumulates the real
// sampled sums for 4 output slots per thread, slots sorted by n mod L.
#include "fft32.cuh"
#include "nsk_internal.hpp"

namespace nsk {

namespace {

using namespace fft;

constexpr int DL = 1024;      // FFT length
constexpr int DANCHOR = 16;   // exact twiddles every DANCHOR tiles

// W = k1 columns per tile = warps per CTA (8: one CTA per SM, the default; 4: two).
template <int W>
struct DTile {
  static constexpr int T = 32 * W;       // threads
  static constexpr int RS = 2 * W + 2;   // doubles per staged row: W main | W + 1 mirror | pad
  static constexpr int RS2 = RS / 2;     // ... in double2 (odd: 16-byte aligned, conflict-free columns)
  static constexpr int NQ = 1024 / T;    // output slots per thread (T * NQ = 1024 per pass)
  static constexpr size_t SMEM = sizeof(double) * DL * RS + sizeof(double2) * DL + sizeof(uint32_t) * 3 * DL;
};

struct DctParams {
  const double* A;
  int64_t lda;
  int64_t N;        // rows (transform length)
  int64_t n;        // columns
  int64_t P;        // N / DL
  int64_t tiles;    // tiles per column: P / (2 W) + 1
  int64_t per;      // tiles per work item
  int64_t ranges;   // work items per column
  const uint32_t* sign_bits;
  const int64_t* freq;  // slot -> n (output of v), sorted by n mod DL
  int nslots;
  double* part;     // [column][range][DNQ * DT]
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int bytes) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int bytes) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, int bytes) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(gmem), "r"(bytes));
}

// e^{2 pi i r / Q} for an exact integer r in [0, Q).
__device__ __forceinline__ double2 unitq(uint64_t r, uint64_t Q) {
  double sn, cs;
  sincospi(2.0 * static_cast<double>(r) / static_cast<double>(Q), &sn, &cs);
  return make_double2(cs, sn);
}
__device__ __forceinline__ double sgn(uint32_t bits, int pos, double v) {
  return ((bits >> pos) & 1u) ? v : -v;  // Rademacher bit 1 -> +1 (rng.hpp:57)
}

template <int W>
__global__ void __launch_bounds__(32 * W, W == 4 ? 2 : 1) srdct_tile_kernel(DctParams p) {
  using TT = DTile<W>;
  constexpr int DT = TT::T, RS = TT::RS, RS2 = TT::RS2, DNQ = TT::NQ;
  extern __shared__ __align__(16) double smd[];
  double* U = smd;                                        // [DL][RS]
  double2* U2 = reinterpret_cast<double2*>(U);            // [DL][RS2]
  double2* tw = U2 + DL * RS2;                            // e^{2 pi i k / DL}
  uint32_t* SBm = reinterpret_cast<uint32_t*>(tw + DL);   // main sign word per row
  uint32_t* SBr = SBm + DL;                               // mirror sign words per row (2)
  __shared__ double2 om1[W];                              // omega^{k1} of the tile's columns
  __shared__ double2 r4[4];                               // e^{2 pi i r / 4 DL}
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t N = static_cast<uint64_t>(p.N);
  const int64_t P = p.P, half_tiles = P / (2 * W);
  const double c0 = sqrt(1.0 / static_cast<double>(p.N)), c1 = sqrt(2.0 / static_cast<double>(p.N));
  const double rs2 = 0.70710678118654752440;

  for (int k = threadIdx.x; k < DL; k += DT) tw[k] = unitq(static_cast<uint64_t>(k), DL);
  if (threadIdx.x < 4) r4[threadIdx.x] = unitq(static_cast<uint64_t>(threadIdx.x), 4 * DL);
  // omega^{P k2} = e^{i pi k2 / 2L} = tw[k2 / 4] * r4[k2 % 4]
  auto wp = [&](int k2) { return cmul(tw[k2 >> 2], r4[k2 & 3]); };
  auto freq_of = [&](int q) -> uint64_t {
    const int o = threadIdx.x + DT * q;
    return o < p.nslots ? static_cast<uint64_t>(__ldg(p.freq + o)) : 0;
  };
  double2 step[DNQ];
#pragma unroll
  for (int q = 0; q < DNQ; ++q) step[q] = unitq(freq_of(q) % N, N);  // W^n
  __syncthreads();

  const int64_t items = p.n * p.ranges;
  for (int64_t item = blockIdx.x; item < items; item += gridDim.x) {
    const int64_t col = item / p.ranges, range = item % p.ranges;
    const int64_t t0 = range * p.per, t1 = t0 + p.per < p.tiles ? t0 + p.per : p.tiles;
    const double* Acol = p.A + col * p.lda;
    double acc[DNQ];
    double2 base[DNQ];
#pragma unroll
    for (int q = 0; q < DNQ; ++q) acc[q] = 0.0;

    for (int64_t t = t0; t < t1; ++t) {
      const bool last = t == half_tiles;  // the tile of column P/2 alone
      const int64_t K = last ? P / 2 : W * t;
      const int64_t B0 = P - W * t - W;   // mirror block start (main tiles): columns B0 .. B0 + W
      __syncthreads();                    // previous tile's reads of U are done
      // ---- stage: W main + W + 1 mirror elements per row, sign words
      for (int c = threadIdx.x; c < DL * (W / 2); c += DT) {
        const int k2 = c / (W / 2), ch = c % (W / 2);
        const int64_t j0 = K + P * k2 + 2 * ch;
        cp_async16(U + k2 * RS + 2 * ch, Acol + (last ? (ch == 0 ? j0 : 0) : j0), last && ch ? 0 : 16);
        if (!last) {
          const int64_t m0 = B0 + P * (DL - 1 - k2) + 2 * ch;  // mirror block of global row L - 1 - k2
          cp_async16(U + k2 * RS + W + 2 * ch, Acol + m0, 16);
        }
      }
      for (int k2 = threadIdx.x; k2 < DL; k2 += DT) {
        const uint64_t jm = static_cast<uint64_t>(K + P * k2);
        cp_async4(SBm + k2, p.sign_bits + (jm >> 5), 4);
        if (!last) {
          const uint64_t jr = static_cast<uint64_t>(B0 + P * (DL - 1 - k2));
          const uint64_t jW = jr + W;  // the (W+1)-th mirror element
          cp_async8(U + k2 * RS + 2 * W, Acol + (jW < N ? jW : 0), jW < N ? 8 : 0);
          cp_async4(SBr + 2 * k2, p.sign_bits + (jr >> 5), 4);
          const uint64_t w1 = jW >> 5;
          cp_async4(SBr + 2 * k2 + 1, p.sign_bits + (w1 < (N + 31) / 32 ? w1 : 0), 4);
        }
      }
      if (threadIdx.x < W) {
        double sn, cs;
        sincospi(static_cast<double>(K + threadIdx.x) / (2.0 * static_cast<double>(p.N)), &sn, &cs);
        om1[threadIdx.x] = make_double2(cs, sn);  // omega^{k1}
      }
      asm volatile("cp.async.wait_all;\n" ::: "memory");
      __syncthreads();

      // ---- column 0 of tile 0 (k1 = 0, self-mirrored by k2 <-> L - k2): computed first
      constexpr int E0 = DL / DT;
      double2 e0[E0];
      const bool col0 = t == 0;
      if (col0) {
#pragma unroll
        for (int i = 0; i < E0; ++i) {
          const int k2 = threadIdx.x + DT * i;
          double2 v = make_double2(0.0, 0.0);
          const double x = sgn(SBm[k2], static_cast<int>((P * k2) & 31), U[k2 * RS]);
          if (k2 == 0) {
            v = make_double2(0.5 * c0 * x, 0.0);
          } else if (k2 == DL / 2) {
            v = make_double2(0.5 * rs2 * c1 * x, 0.0);  // G_{N/2} / 2 = X_{N/2} / (2 sqrt 2)
          } else if (k2 < DL / 2) {
            const int k2m = DL - k2;  // N - P k2 = P (L - k2)
            const double xm = sgn(SBm[k2m], static_cast<int>((P * k2m) & 31), U[k2m * RS]);
            v = cmul(make_double2(0.5 * c1 * x, -0.5 * c1 * xm), wp(k2));  // (X_k - i X_{N-k}) omega^k / 2
          }
          e0[i] = v;
        }
      }
      __syncthreads();
      // ---- G in place: a thread owns the row pair (k2, L - 1 - k2)
      for (int k2 = threadIdx.x; k2 < DL / 2; k2 += DT) {
        const int k2b = DL - 1 - k2;
        double ma[W], mb[W], ra[W + 1], rb[W + 1];
#pragma unroll
        for (int j = 0; j < W; ++j) {
          ma[j] = U[k2 * RS + j];
          mb[j] = U[k2b * RS + j];
        }
        if (!last) {
#pragma unroll
          for (int i = 0; i <= W; ++i) {
            ra[i] = U[k2 * RS + W + i];   // mirror block of global row k2b: partners of main row k2
            rb[i] = U[k2b * RS + W + i];  // mirror block of global row k2: partners of main row k2b
          }
        }
        const uint32_t sma = SBm[k2], smb = SBm[k2b];
        const int sha = static_cast<int>((K + P * k2) & 31), shb = static_cast<int>((K + P * k2b) & 31);
        uint64_t sra = 0, srb = 0;
        int shra = 0, shrb = 0;
        if (!last) {
          sra = static_cast<uint64_t>(SBr[2 * k2]) | (static_cast<uint64_t>(SBr[2 * k2 + 1]) << 32);
          srb = static_cast<uint64_t>(SBr[2 * k2b]) | (static_cast<uint64_t>(SBr[2 * k2b + 1]) << 32);
          shra = static_cast<int>((B0 + P * k2b) & 31);
          shrb = static_cast<int>((B0 + P * k2) & 31);
        }
        const double2 wa = wp(k2), wb = wp(k2b);
#pragma unroll
        for (int j = 0; j < W; ++j) {
          if (col0 && j == 0) continue;  // column 0 written from e0 below
          double2 ga = make_double2(0.0, 0.0), gb = make_double2(0.0, 0.0);
          if (!last) {
            // mirror element W - j of a staged row is column P - K - j (the partner of column K + j)
            const double xa = c1 * sgn(sma, sha + j, ma[j]);
            const double xma = c1 * (((sra >> (shra + W - j)) & 1u) ? ra[W - j] : -ra[W - j]);
            const double xb = c1 * sgn(smb, shb + j, mb[j]);
            const double xmb = c1 * (((srb >> (shrb + W - j)) & 1u) ? rb[W - j] : -rb[W - j]);
            const double2 om = om1[j];
            ga = cmul(cmul(make_double2(0.5 * xa, -0.5 * xma), om), wa);
            gb = cmul(cmul(make_double2(0.5 * xb, -0.5 * xmb), om), wb);
          } else if (j == 0) {  // column P/2: pairs k2 <-> L - 1 - k2 within the column, lower half only
            const double xa = c1 * sgn(sma, sha, ma[0]);
            const double xb = c1 * sgn(smb, shb, mb[0]);
            ga = cmul(cmul(make_double2(0.5 * xa, -0.5 * xb), om1[0]), wa);
          }
          U2[k2 * RS2 + j] = ga;
          U2[k2b * RS2 + j] = gb;
        }
      }
      __syncthreads();
      if (col0) {
#pragma unroll
        for (int i = 0; i < E0; ++i) U2[(threadIdx.x + DT * i) * RS2] = e0[i];
      }
      __syncthreads();
      // ---- warp `warp`: in-place 1024-point FFT of column `warp`
      {
        double2 x[32];
#pragma unroll
        for (int tt = 0; tt < 32; ++tt) x[tt] = U2[(lane + 32 * tt) * RS2 + warp];
        dft32(x);
#pragma unroll
        for (int k = 1; k < 32; ++k) x[k] = cmul(x[k], tw[(lane * k) & (DL - 1)]);
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 32; ++k) U2[(32 * lane + ((k + lane) & 31)) * RS2 + warp] = x[k];
        __syncwarp();
#pragma unroll
        for (int l = 0; l < 32; ++l) x[l] = U2[(32 * l + ((lane + l) & 31)) * RS2 + warp];
        dft32(x);
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 32; ++k) U2[(lane + 32 * k) * RS2 + warp] = x[k];
      }
      __syncthreads();
      // ---- sampled sums: acc += Re sum_j W^{n (K + j)} F_j[n mod L]
      const bool anchor = ((t - t0) % DANCHOR) == 0 || last;
#pragma unroll
      for (int q = 0; q < DNQ; ++q) {
        const uint64_t f = freq_of(q);
        if (anchor)
          base[q] = unit_phase(mulmod_fast(f, static_cast<uint64_t>(K), N, 1.0 / static_cast<double>(N)),
                               2.0 / static_cast<double>(N));
        double2 w = base[q];
        const int qi = static_cast<int>(f & (DL - 1));
        const double2 st = step[q];
        double sacc = 0.0;
        const int jn = last ? 1 : W;
        for (int j = 0; j < jn; ++j) {
          const double2 F = U2[qi * RS2 + j];
          sacc = fma(w.x, F.x, fma(-w.y, F.y, sacc));
          w = cmul(w, st);
        }
        acc[q] += sacc;
        base[q] = w;  // W^{n (K + W)}
      }
    }
    double* part = p.part + (col * p.ranges + range) * 1024;
#pragma unroll
    for (int q = 0; q < DNQ; ++q) part[threadIdx.x + DT * q] = acc[q];
  }
}

// SA(row, c) = scale * sum_r part[c][r][o] in fixed order (scale carries the 2 of 2 Re).
__global__ void srdct_tile_reduce(const double* __restrict__ part, int64_t ranges, int64_t n, int nslots,
                                  int stride, const int32_t* __restrict__ row_of_slot, double scale,
                                  double* __restrict__ SA, int64_t ldsa) {
  const int64_t total = n * nslots;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / nslots;
    const int o = static_cast<int>(e % nslots);
    double v = 0.0;
    for (int64_t r = 0; r < ranges; ++r) v += part[(c * ranges + r) * stride + o];
    SA[row_of_slot[o] + c * ldsa] = scale * v;
  }
}

}  // namespace

// NOTAPPLICABLE unless the whole column is applied (no shard), N is a multiple
// of 16 * 1024, real input, and A is 16-byte aligned with an even lda.
int srdct_tile_apply(const Operator& op, const RowMap& rows, int64_t n, const double* A, int64_t lda, double* SA,
                     int64_t ldsa, cudaStream_t st) {
  if (std::getenv("NSK_SRDCT_NOMAKHOUL")) return NOTAPPLICABLE;
  const int64_t m = op.m, s = op.s;
  if (!(rows.row0 == 0 && rows.rstep == 1 && rows.mloc == m) || n == 0) return NOTAPPLICABLE;
  if (m % (16 * DL) != 0 || m > (int64_t(1) << 40)) return NOTAPPLICABLE;
  if ((reinterpret_cast<uintptr_t>(A) & 15) != 0 || (lda & 1) != 0) return NOTAPPLICABLE;
  const DeviceTables* tb = op.tables();
  if (!tb || !tb->sign_bits || !tb->dct_freq || !tb->dct_row) return ECUDA;
  // tile width: 8 columns, one CTA of 8 warps per SM (NSK_SRDCT_W=4: two CTAs of 4 warps,
  // measured 1.5x slower -- the per-tile sampled stage and barriers are paid twice as often)
  const char* we = std::getenv("NSK_SRDCT_W");
  const int W = we && std::atoi(we) == 4 ? 4 : 8;
  const int64_t P = m / DL, tiles = P / (2 * W) + 1;
  const int per_sm = W == 4 ? 2 : 1;
  // work items (column, tile range): about two waves of resident CTAs
  const int64_t slots = sm_count() * per_sm;
  int64_t ranges = (2 * slots + n - 1) / n;
  if (ranges > tiles) ranges = tiles;
  const int64_t per = (tiles + ranges - 1) / ranges;
  ranges = (tiles + per - 1) / per;
  const int64_t items = n * ranges;
  const size_t smem = W == 4 ? DTile<4>::SMEM : DTile<8>::SMEM;
  auto kern = W == 4 ? srdct_tile_kernel<4> : srdct_tile_kernel<8>;
  NSK_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  const double scale = 2.0 * std::sqrt(static_cast<double>(m) / static_cast<double>(s));
  for (int64_t b = 0; b < s; b += 1024) {
    const int ns = static_cast<int>((s - b) < 1024 ? (s - b) : 1024);
    Scratch part;
    NSK_CUDA_OK(part.alloc(sizeof(double) * items * 1024, st));
    DctParams p{A, lda, m, n, P, tiles, per, ranges, tb->sign_bits, tb->dct_freq + b, ns, part.as<double>()};
    const int64_t grid = items < slots ? items : slots;
    KernelTimer tm(st, "srdct_tile_kernel");
    kern<<<static_cast<unsigned>(grid), 32 * W, smem, st>>>(p);
    tm.stop();
    count_launch();
    NSK_CUDA_OK(cudaGetLastError());
    int64_t blocks = (n * ns + 255) / 256;
    if (blocks > 8L * sm_count()) blocks = 8L * sm_count();
    srdct_tile_reduce<<<static_cast<unsigned>(blocks), 256, 0, st>>>(part.as<double>(), ranges, n, ns, 1024,
                                                                     tb->dct_row + b, scale, SA, ldsa);
    count_launch();
    NSK_CUDA_OK(cudaGetLastError());
  }
  return OK;
}

}  // namespace nsk
