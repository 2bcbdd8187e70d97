// srtt_tile.cu -- K2 (default fast path): sampled srft / srdct with one
// coalesced pass over A.
//
// Both kinds are s samples of one DFT (kernel e^{+2 pi i/N}, the unitary
// inverse DFT of transforms.cpp:17-36):
//   srft : X[f] = sum_{j<m} u_j w_m^{f j},  u = d .* A,  SA[r] = X[idx_r] / sqrt(s)
//   srdct: the orthonormal DCT-III (transforms.cpp:38-64) is
//          y_a = Re Y[a],  Y[a] = sum_{k<m} c_k x_k w_{4m}^{(2a+1) k},  x = d .* A,
//          c_0 = sqrt(1/m), c_k = sqrt(2/m); SA[r] = sqrt(m/s) y_{idx_r}
//          (a length-2m DFT of a zero-padded, pre-twiddled real sequence).
// Decimation in time with an FFT length L = 1024: index j = k1 + P k2
// (P = m / L for srft, P = 2m / L for srdct where only k2 < L/2 is non-zero):
//   X[f] = sum_{k1<P} w^{f k1} F_{k1}[f mod L],  F_{k1} = DFT_L(u[k1 + P k2]).
// Viewed as the row-major L x P matrix M[k2][k1], a tile of 8 consecutive k1
// is L (or L/2) contiguous 64-byte row segments: a CTA streams whole tiles
// with cp.async (no re-reads of A), pairs the 8 real columns into 4 complex
// sequences (z = u_e + i u_o; complex input: 4 columns as is), runs one
// 1024-point FFT per warp in place in shared memory (two register DFT32
// passes, a skewed conflict-free transpose), unpacks the pairs with the
// Hermitian mirror (F_e = (Z[q] + conj Z[-q]) / 2, F_o = (Z[q] - conj Z[-q]) / 2i;
// srdct mirrors at L - 1 - q) and accumulates the sampled outputs in
// registers with incremental twiddles re-anchored exactly every 16 tiles.
// Per-(column, range) partials are summed in fixed order.
#include "fft32.cuh"
#include "nsk_internal.hpp"

namespace nsk {

namespace {

using namespace fft;

constexpr int TL = 1024;        // FFT length
constexpr int TW = 8;           // complex sequences per tile (one warp each)
constexpr int TT = 32 * TW;     // threads per CTA
constexpr int TROW = TW + 1;    // complex slots per shared-memory row (padded: conflict-free columns)
constexpr int TNQ = 1024 / TT;  // output slots per thread (TT * TNQ = 1024 per pass)
constexpr int TANCHOR = 16;     // exact twiddles every TANCHOR tiles

struct TileParams {
  const double* A;
  int64_t lda;
  int64_t m;
  int64_t n;
  int64_t P;       // k1 count: m / TL (srft), 2m / TL (srdct)
  int64_t tiles;   // tiles per column
  int64_t ranges;  // CTAs per column
  int64_t per;     // tiles per CTA
  const uint32_t* sign_bits;
  const int64_t* freq;  // srft: DFT frequency of the slot; srdct: DCT index a
  int nslots;
  double* part;    // [column][range][TNQ * TT] complex
};

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}

// w_N^r = e^{2 pi i r / N} for an exact integer r in [0, N).
__device__ __forceinline__ double2 unit(uint64_t r, uint64_t N) {
  double sn, cs;
  sincospi(2.0 * static_cast<double>(r) / static_cast<double>(N), &sn, &cs);
  return make_double2(cs, sn);
}


// KIND 0 srft, 1 srdct; NCIN 1 real input (pairs), 2 complex input.
template <int KIND, int NCIN>
__global__ void __launch_bounds__(TT, TW == 8 ? 1 : 2) srtt_tile_kernel(TileParams p) {
  extern __shared__ __align__(16) double2 sm2[];
  double2* U = sm2;                 // [TL][TROW]
  double2* tw = U + TL * TROW;      // w_1024^k, k < 1024
  double2* tw2 = tw + TL;           // srdct: w_2048^k, k < 512
  uint32_t* SB = reinterpret_cast<uint32_t*>(tw2 + TL / 2);  // [ROWS] sign words of the tile
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t col = blockIdx.x / p.ranges, range = blockIdx.x % p.ranges;
  const int64_t t0 = range * p.per;
  const int64_t t1 = t0 + p.per < p.tiles ? t0 + p.per : p.tiles;
  const double* Acol = p.A + col * p.lda * NCIN;
  const uint64_t m = static_cast<uint64_t>(p.m);
  constexpr int KT = NCIN == 1 ? 2 * TW : TW;        // k1 columns per tile
  constexpr int ROWS = KIND == 1 ? TL / 2 : TL;      // non-zero k2 rows
  const uint64_t N = KIND == 1 ? 4 * m : m;          // twiddle modulus (w_N)

  for (int k = threadIdx.x; k < TL; k += TT) tw[k] = unit(static_cast<uint64_t>(k), TL);
  if (KIND == 1)
    for (int k = threadIdx.x; k < TL / 2; k += TT) tw2[k] = unit(static_cast<uint64_t>(k), 2 * TL);

  // Output slots of this thread: g = frequency (srft f, srdct 2a+1) in w_N.
  // Only the accumulators and the two twiddles stay in registers; the slot's
  // frequency is re-read (L1) when it is needed (register budget of the FFT).
  auto freq_of = [&](int q) -> uint64_t {
    const int o = threadIdx.x + TT * q;
    return o < p.nslots ? static_cast<uint64_t>(__ldg(p.freq + o)) : 0;
  };
  double2 acc[TNQ], step[TNQ], base[TNQ];
#pragma unroll
  for (int q = 0; q < TNQ; ++q) {
    const uint64_t f = freq_of(q);
    acc[q] = make_double2(0.0, 0.0);
    step[q] = unit((KIND == 1 ? 2 * f + 1 : f) % N, N);  // w_N^g: one k1 column
  }
  const double c0 = sqrt(1.0 / static_cast<double>(p.m)), c1 = sqrt(2.0 / static_cast<double>(p.m));

  for (int64_t t = t0; t < t1; ++t) {
    const int64_t K = t * KT;  // first k1 of the tile
    __syncthreads();           // previous tile's reads of U are done
    // ---- stage rows k2 < ROWS: 16 TW contiguous bytes each (TW x 16 B)
    for (int c = threadIdx.x; c < ROWS * TW; c += TT) {
      const int k2 = c / TW, ch = c % TW;
      cp_async16(U + k2 * TROW + ch, Acol + (K + p.P * k2) * NCIN + 2 * ch);
    }
    for (int k2 = threadIdx.x; k2 < ROWS; k2 += TT)  // sign word of each row (bits K .. K + KT - 1)
      cp_async4(SB + k2, p.sign_bits + ((static_cast<uint64_t>(K) + static_cast<uint64_t>(p.P) * k2) >> 5));
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    // ---- warp `warp`: in-place 1024-point FFT of sequence `warp` (column of U)
    {
      double2 x[32];
#pragma unroll
      for (int tt = 0; tt < 32; ++tt) {
        const int k2 = lane + 32 * tt;
        if (KIND == 1 && k2 >= ROWS) {
          x[tt] = make_double2(0.0, 0.0);
          continue;
        }
        double2 v = U[k2 * TROW + warp];
        if (NCIN == 1) {  // v = (u_e, u_o) of columns K + 2 warp, K + 2 warp + 1
          const uint64_t j = static_cast<uint64_t>(K + 2 * warp) + static_cast<uint64_t>(p.P) * k2;
          const uint32_t bits = SB[k2] >> (j & 31);
          if (!(bits & 1u)) v.x = -v.x;
          if (!(bits & 2u)) v.y = -v.y;
          if (KIND == 1) {
            v.x *= (j == 0 ? c0 : c1);
            v.y *= c1;
            v = cmul(v, tw2[k2]);  // w_{2L}^{k2}
          }
        } else {
          const uint64_t j = static_cast<uint64_t>(K + warp) + static_cast<uint64_t>(p.P) * k2;
          if (!((SB[k2] >> (j & 31)) & 1u)) v = make_double2(-v.x, -v.y);
        }
        x[tt] = v;
      }
      dft32(x);  // over tt: lane l holds Y[l][k2'] in x[k2']
#pragma unroll
      for (int k = 1; k < 32; ++k) x[k] = cmul(x[k], tw[(lane * k) & (TL - 1)]);
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 32; ++k) U[(32 * lane + ((k + lane) & 31)) * TROW + warp] = x[k];
      __syncwarp();
#pragma unroll
      for (int l = 0; l < 32; ++l) x[l] = U[(32 * l + ((lane + l) & 31)) * TROW + warp];
      dft32(x);  // over l: lane k2' holds X[k2' + 32 k1'] in x[k1']
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 32; ++k) U[(lane + 32 * k) * TROW + warp] = x[k];
    }
    __syncthreads();
    // ---- sampled second stage
    const bool anchor = ((t - t0) % TANCHOR) == 0;
#pragma unroll
    for (int q = 0; q < TNQ; ++q) {
      const uint64_t f = freq_of(q);
      if (anchor)
        base[q] = unit_phase(mulmod_fast(KIND == 1 ? 2 * f + 1 : f, static_cast<uint64_t>(K), N, 1.0 / static_cast<double>(N)),
                             2.0 / static_cast<double>(N));
      double2 w = base[q];  // w_N^{g K}
      const int qi = static_cast<int>(f & (TL - 1));
      if (NCIN == 1) {
        const int qm = KIND == 1 ? TL - 1 - qi : (TL - qi) & (TL - 1);
        const double2 st = step[q], st2 = cmul(st, st);
        double2 a2 = make_double2(0.0, 0.0);
#pragma unroll
        for (int i = 0; i < TW; ++i) {
          const double2 zq = U[qi * TROW + i], zm = U[qm * TROW + i];
          const double2 e = make_double2(zq.x + zm.x, zq.y - zm.y);  // Z[q] + conj Z[-q] = 2 F_e
          const double2 d = make_double2(zq.x - zm.x, zq.y + zm.y);  // Z[q] - conj Z[-q] = 2i F_o
          const double2 sd = cmul(st, d);
          const double2 term = make_double2(e.x + sd.y, e.y - sd.x);  // E - i w^g D = 2 (F_e + w^g F_o)
          a2 = cadd(a2, cmul(w, term));
          w = cmul(w, st2);
        }
        acc[q] = cadd(acc[q], a2);
      } else {
        const double2 st = step[q];
#pragma unroll
        for (int i = 0; i < TW; ++i) {
          acc[q] = cadd(acc[q], cmul(w, U[qi * TROW + i]));
          w = cmul(w, st);
        }
      }
      base[q] = w;  // w_N^{g (K + KT)}
    }
  }
  double2* part = reinterpret_cast<double2*>(p.part) + (col * p.ranges + range) * (TNQ * TT);
#pragma unroll
  for (int q = 0; q < TNQ; ++q) part[threadIdx.x + TT * q] = acc[q];
}

// SA(row, c) = scale * sum_r part[c][r][o] in fixed order; srft complex out,
// srdct the real part (the pair unpacking's factor 1/2 folded into scale).
template <int KIND>
__global__ void srtt_tile_reduce(const double2* __restrict__ part, int64_t ranges, int64_t n, int nslots, int stride,
                                 const int32_t* __restrict__ row_of_slot, double scale, double* __restrict__ SA,
                                 int64_t ldsa) {
  const int64_t total = n * nslots;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / nslots;
    const int o = static_cast<int>(e % nslots);
    double2 v = make_double2(0.0, 0.0);
    for (int64_t r = 0; r < ranges; ++r) {
      const double2 x = part[(c * ranges + r) * stride + o];
      v.x += x.x;
      v.y += x.y;
    }
    const int64_t row = row_of_slot[o];
    if (KIND == 0) {
      SA[2 * (row + c * ldsa)] = scale * v.x;
      SA[2 * (row + c * ldsa) + 1] = scale * v.y;
    } else {
      SA[row + c * ldsa] = scale * v.x;
    }
  }
}

template <int KIND, int NCIN>
int launch_tile(const TileParams& p, int64_t ctas, cudaStream_t st) {
  const size_t smem = sizeof(double2) * (TL * TROW + TL + TL / 2) + sizeof(uint32_t) * TL;
  auto kern = srtt_tile_kernel<KIND, NCIN>;
  NSK_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  KernelTimer tm(st, "srtt_tile_kernel");
  kern<<<static_cast<unsigned>(ctas), TT, smem, st>>>(p);
  tm.stop();
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  return OK;
}

}  // namespace

// Returns NOTAPPLICABLE when the shapes or the layout do not fit the tiling
// (the caller falls back to the strided FFT or the direct evaluator).
int srtt_tile_apply(const Operator& op, int ncomp, const RowMap& rows, int64_t n, const double* A, int64_t lda,
                    double* SA, int64_t ldsa, cudaStream_t st) {
  if (std::getenv("NSK_SRTT_NOTILE")) return NOTAPPLICABLE;
  const int64_t m = op.m, s = op.s;
  const bool full = rows.row0 == 0 && rows.rstep == 1 && rows.mloc == m;
  const int kind = op.kind == SRFT ? 0 : 1;
  if (!full || n == 0) return NOTAPPLICABLE;
  const int64_t P = kind == 0 ? m / TL : 2 * m / TL;
  const int64_t KT = ncomp == 1 ? 2 * TW : TW;
  if ((kind == 0 && m % (TL * KT) != 0) || (kind == 1 && (2 * m) % (TL * KT) != 0)) return NOTAPPLICABLE;
  if ((reinterpret_cast<uintptr_t>(A) & 15) != 0 || (ncomp == 1 && (lda & 1) != 0)) return NOTAPPLICABLE;
  const DeviceTables* tb = op.tables();
  if (!tb || !tb->sign_bits) return ECUDA;
  // Slots sorted by their FFT bin (idx mod TL, operator tables): the threads
  // of a warp then gather neighbouring rows of the tile (conflict-free in the
  // padded layout); the reduce scatters slot t to output row srtt_row[t].
  if (!tb->srtt_freq || !tb->srtt_row) return ECUDA;
  const int64_t tiles = P / KT;
  const int64_t target = 2L * sm_count();
  int64_t ranges = (target + n - 1) / n;
  if (ranges > tiles) ranges = tiles;
  const int64_t per = (tiles + ranges - 1) / ranges;
  ranges = (tiles + per - 1) / per;
  // srft: unnormalised DFT / sqrt(s); srdct: sqrt(m/s) * Re Y; real pairs carry a factor 2.
  double scale = kind == 0 ? 1.0 / std::sqrt(static_cast<double>(s))
                           : std::sqrt(static_cast<double>(m) / static_cast<double>(s));
  if (ncomp == 1) scale *= 0.5;
  for (int64_t base = 0; base < s; base += TNQ * TT) {
    const int ns = static_cast<int>((s - base) < TNQ * TT ? (s - base) : TNQ * TT);
    Scratch part;
    NSK_CUDA_OK(part.alloc(sizeof(double2) * n * ranges * TNQ * TT, st));
    TileParams p{A, lda, m, n, P, tiles, ranges, per, tb->sign_bits, tb->srtt_freq + base, ns,
                 part.as<double>()};
    const int64_t ctas = n * ranges;
    int rc = kind == 0 ? (ncomp == 1 ? launch_tile<0, 1>(p, ctas, st) : launch_tile<0, 2>(p, ctas, st))
                       : launch_tile<1, 1>(p, ctas, st);
    if (rc != OK) return rc;
    int64_t blocks = (n * ns + 255) / 256;
    if (blocks > 8L * sm_count()) blocks = 8L * sm_count();
    if (kind == 0)
      srtt_tile_reduce<0><<<static_cast<unsigned>(blocks), 256, 0, st>>>(
          reinterpret_cast<const double2*>(part.p), ranges, n, ns, TNQ * TT, tb->srtt_row + base, scale, SA, ldsa);
    else
      srtt_tile_reduce<1><<<static_cast<unsigned>(blocks), 256, 0, st>>>(
          reinterpret_cast<const double2*>(part.p), ranges, n, ns, TNQ * TT, tb->srtt_row + base, scale, SA, ldsa);
    count_launch();
    NSK_CUDA_OK(cudaGetLastError());
  }
  return OK;
}

}  // namespace nsk
