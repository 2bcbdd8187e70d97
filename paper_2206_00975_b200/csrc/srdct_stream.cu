// srdct_stream.cu -- sampled srdct, register-streamed Makhoul tiles.
//
// Reference: apply(), srdct branch (/root/reference/proj/src/sketch.cpp:218-229)
// and dct3_unitary_columns (transforms.cpp:38-64):
//   y_a = sum_k X_k cos(pi k (2a+1) / 2N),  X_k = c_k d_k A[k],  SA = sqrt(N/s) y_idx.
// Makhoul: G_k = (X_k - i X_{N-k}) w^k / 2 with w = e^{i pi / 2N} is Hermitian,
// v_n = sum_k G_k W^{kn} is real, y_{2n} = v_n, y_{2n+1} = v_{N-1-n}; with
// k = k1 + P k2, L = 1024, only k1 in [0, P/2] is transformed and
// v_n = sum_{k1} 2 Re(W^{n k1} F_{k1}[n mod L]).  Organised for the FP64 pipe
// (register-streamed tiles, no shared-memory staging of A):
//
//  * the factor w^{k1} of a column is constant over k2, so it moves out of the
//    FFT into the sampled stage: the per-column step becomes
//    W_{4N}^{4n+1} = W^n w.  The remaining pre-twiddle w^{P k2} = W_{4L}^{k2}
//    with k2 = a + 32 b splits into W_128^b (a compile-time constant of the
//    register holding row b) and W_4096^a, which merges with the inter-pass
//    twiddle into W_4096^{a (4k + 1)} (a [k][a] shared table of 1024 entries);
//  * a lane (sequence i, row class a) loads its main elements
//    A[K + i + P (a + 32 b)] and mirror elements A[N - (K + i + P k2)] straight
//    into the FFT registers (two 8-byte loads per b, 64-byte row segments; the
//    mirror set [P-K-7, P-K] straddles two aligned blocks, so lane 0 reads the
//    aligned block's first element P-K-8 for the next tile and takes its own
//    P-K from a shared-memory carry written one tile earlier),
//    the next tile's loads land during the sampled stage, an L2 prefetch runs
//    one tile further ahead; signs come as one 64-bit negate mask per lane;
//  * the sampled stage is one complex Horner chain per slot (v is real:
//    Re(base * sum_i st^i F_i[q]), 4 DFMA per slot and sequence);
//  * tile 0 of a column holds the two self-mirrored columns k1 = 0 (rows
//    k2 <= L/2, weight 1/sqrt2 at k2 = 0 for c_0 / c_1 and 1/2 at L/2) and
//    k1 = P/2 (rows k2 < L/2); tiles 1 .. P/16 hold k1 = 8 (T - 1) + i;
//  * each CTA walks a contiguous chunk of the (column, tile) sequence (within
//    one tile of perfect balance); partial sums per (CTA, column piece) are
//    reduced in a fixed order.
#include "fft32.cuh"
#include "nsk_internal.hpp"

namespace nsk {

namespace {

using namespace fft;

constexpr int SL = 1024;       // FFT length
constexpr int SW = 8;          // warps = sequences per tile
constexpr int ST = 32 * SW;    // threads
constexpr int SNQ = 1024 / ST; // output slots per thread
constexpr int SANCH = 16;      // exact twiddles every SANCH tiles
constexpr int STW = 1024;      // [k][a] table of W_4096^{a (4k+1)}
static_assert(SNQ == 4, "the next tile loads in SNQ parts of 8 rows");

struct DStreamParams {
  const double* A;
  int64_t lda;
  int64_t N;
  int64_t P;         // N / SL
  int64_t tiles;     // per column: P / 16 + 1
  int64_t total;     // n * tiles
  int64_t chunk;     // tiles per CTA
  int64_t jmax;      // column pieces per CTA
  const uint64_t* sgn;   // [tile][a][i] negate masks: bits b main, 32 + b mirror
  const int64_t* freq;   // v index n of each slot, sorted by n mod SL
  int nslots;
  const double2* anc;    // [tile][SNQ * ST]: W_4N^{(4n+1) K(tile)}
  double* part;          // [cta][jmax][SNQ * ST]
};

// cos(pi b / 64), b = 0 .. 32 (W_128^b = C[b] + i C[32 - b])
__device__ __forceinline__ double2 pre128(double2 v, int b) {
  constexpr double C[33] = {1.0,
                            0.998795456205172392714771604759,
                            0.995184726672196886244836953109,
                            0.989176509964780973451673738016,
                            0.980785280403230449126182236134,
                            0.970031253194543992603984207286,
                            0.95694033573220886493579788698,
                            0.9415440651830207784125094026,
                            0.923879532511286756128183189397,
                            0.903989293123443331586200297231,
                            0.88192126434835502971275686366,
                            0.857728610000272069902269984285,
                            0.831469612302545237078788377618,
                            0.803207531480644909806676512963,
                            0.773010453362736960810906609758,
                            0.740951125354959091175616897495,
                            0.707106781186547524400844362105,
                            0.671558954847018400625376850427,
                            0.634393284163645498215171613225,
                            0.59569930449243334346703652883,
                            0.555570233019602224742830813949,
                            0.514102744193221726593693838969,
                            0.471396736825997648556387625905,
                            0.427555093430282094320966856889,
                            0.38268343236508977172845998403,
                            0.336889853392220050689253212619,
                            0.290284677254462367636192375817,
                            0.242980179903263889948274162077,
                            0.195090322016128267848284868477,
                            0.146730474455361751658850129647,
                            0.0980171403295606019941955638886,
                            0.0490676743274180142549549769427,
                            0.0};
  if (b == 0) return v;
  const double c = C[b], s = C[32 - b];
  return make_double2(fma(v.x, c, -v.y * s), fma(v.x, s, v.y * c));
}

__device__ __forceinline__ double flipd(double v, uint32_t mask) {
  return __hiloint2double(__double2hiint(v) ^ static_cast<int>(mask), __double2loint(v));
}
__device__ __forceinline__ void prefetch_l2(const void* p) {  // the 128-byte line holding p
  asm volatile("prefetch.global.L2 [%0];\n" ::"l"(p));
}

// Rows of A behind lane (i, a), element b of tile T: main row jm and mirror
// row jr (N - jm), with validity.  Tile 0: lane 0 = column 0 (mirror row
// N - P k2, none at k2 = 0), lane 1 = column P/2 (mirror P/2 + P (L-1-k2)).
__device__ __forceinline__ void tile_rows(int64_t T, int i, int a, int b, int64_t N, int64_t P, int64_t& jm,
                                          int64_t& jr, bool& vm, bool& vr) {
  const int64_t k2 = a + 32 * b;
  if (T == 0) {
    vm = i < 2;
    jm = i == 0 ? P * k2 : P / 2 + P * k2;
    vr = i == 1 || (i == 0 && k2 > 0);
    jr = i == 0 ? N - P * k2 : P / 2 + P * (SL - 1 - k2);
  } else {
    jm = 8 * (T - 1) + i + P * k2;
    vm = true;
    jr = N - jm;
    vr = jm > 0;
  }
}

// Negate masks: bit b = main element negated (Rademacher bit 0, rng.hpp:57),
// bit 32 + b = mirror element negated, i.e. G's imaginary part -x_r d_r is
// stored as x_r with the sign bit flipped when d_r = +1.
__global__ void build_srdct_sgn_kernel(const uint32_t* __restrict__ bits, int64_t N, int64_t P, int64_t words,
                                       uint64_t* __restrict__ out) {
  for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w < words;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t T = w / 256;
    const int a = static_cast<int>((w / 8) % 32), i = static_cast<int>(w % 8);
    uint64_t v = 0;
    for (int b = 0; b < 32; ++b) {
      int64_t jm, jr;
      bool vm, vr;
      tile_rows(T, i, a, b, N, P, jm, jr, vm, vr);
      if (vm && !((bits[jm >> 5] >> (jm & 31)) & 1u)) v |= uint64_t(1) << b;
      if (vr && ((bits[jr >> 5] >> (jr & 31)) & 1u)) v |= uint64_t(1) << (32 + b);
    }
    out[w] = v;
  }
}

// anc[T][o] = W_4N^{(4n_o + 1) K(T)}, K(0) = P/2 (column P/2 of tile 0), K(T) = 8 (T - 1).
__global__ void srdct_anchor_kernel(const int64_t* __restrict__ freq, int nslots, int64_t N, int64_t P,
                                    int64_t tiles, double2* __restrict__ anc) {
  const int64_t total = tiles * (SNQ * ST);
  const uint64_t N4 = 4 * static_cast<uint64_t>(N);
  const double inv = 1.0 / static_cast<double>(N4), two = 2.0 / static_cast<double>(N4);
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int o = static_cast<int>(e % (SNQ * ST));
    const int64_t T = e / (SNQ * ST);
    const uint64_t n = o < nslots ? static_cast<uint64_t>(freq[o]) : 0;
    const uint64_t K = T == 0 ? static_cast<uint64_t>(P / 2) : static_cast<uint64_t>(8 * (T - 1));
    anc[e] = unit_phase(mulmod_fast(4 * n + 1, K, N4, inv), two);
  }
}

// PF: L2 prefetch of the tile after the next one (NSK_STREAM_PF=0 turns it off:
// 1.31 ms instead of 1.09 ms at the configs[1] shape).  Interleaving the next
// tile's loads with the sampled stage measured slower (1.25 ms).
template <int PF>
__global__ void __launch_bounds__(ST, 1) srdct_stream_kernel(DStreamParams p) {
  extern __shared__ __align__(16) double2 sm2[];
  double2* U = sm2;              // [SL][SW], sequence i of row r at column i ^ (r & 7)
  double2* tw = U + SL * SW;     // [k][a]: W_4096^{a (4k+1)} (a warp's 4 row classes: one wavefront)
  double2* STP = tw + STW;       // [2][SNQ][ST]: W_4N^{4n+1} (one column), its 8th power (one tile)
  double* CARRY = reinterpret_cast<double*>(STP + 2 * SNQ * ST);  // [b][a]: sequence-0 mirror carried one tile
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int li = lane & 7, a = 4 * warp + (lane >> 3);
  const int64_t N = p.N, P = p.P;
  const uint64_t N4 = 4 * static_cast<uint64_t>(N);

  for (int e = threadIdx.x; e < STW; e += ST)
    tw[e] = unit_phase(static_cast<uint64_t>((e & 31) * (4 * (e >> 5) + 1)), 2.0 / 4096);
  double acc[SNQ];
  double2 base[SNQ];
  int bin[SNQ];
#pragma unroll
  for (int q = 0; q < SNQ; ++q) {
    const int o = threadIdx.x + ST * q;
    const uint64_t n = o < p.nslots ? static_cast<uint64_t>(__ldg(p.freq + o)) : 0;
    bin[q] = static_cast<int>(n & (SL - 1));
    double2 s1 = unit_phase(4 * n + 1, 2.0 / static_cast<double>(N4));
    STP[ST * q + threadIdx.x] = s1;
#pragma unroll
    for (int r = 0; r < 3; ++r) s1 = cmul(s1, s1);
    STP[ST * (SNQ + q) + threadIdx.x] = s1;
    acc[q] = 0.0;
    base[q] = make_double2(1.0, 0.0);
  }

  const int64_t u0 = blockIdx.x * p.chunk;
  const int64_t u1 = u0 + p.chunk < p.total ? u0 + p.chunk : p.total;
  if (u0 >= u1) return;
  int64_t u = u0, c = u0 / p.tiles, T = u0 % p.tiles;
  int64_t piece = 0;

  double2 x[32];
  uint64_t sw;
  // registers <- tile TT of column cc (regular tiles: setup + four parts of
  // eight rows b); main and mirror loads are aligned 64-byte blocks (normal
  // L2 priority: the other half of each 128-byte line is the neighbouring
  // tile's), sequence 0's mirror is carried one tile through CARRY.
  const double* mp = nullptr;
  const double* rp = nullptr;
  int64_t rs = 0;
  auto issue_special = [&](int64_t cc) {
    const double* col = p.A + cc * p.lda;
#pragma unroll
    for (int b = 0; b < 32; ++b) {
      int64_t jm, jr;
      bool vm, vr;
      tile_rows(0, li, a, b, N, P, jm, jr, vm, vr);
      x[b] = make_double2(vm ? __ldcs(col + jm) : 0.0, vr ? __ldcg(col + jr) : 0.0);
    }
    sw = __ldg(p.sgn + a * 8 + li);
  };
  auto setup = [&](int64_t cc, int64_t TT) {
    const double* col = p.A + cc * p.lda;
    const int64_t jm0 = 8 * (TT - 1) + li + P * a;
    mp = col + jm0;
    // mirror of element b: N - jm0 - 32 P b.  Lane 0 reads N - jm0 - 8 - 32 P b instead, the
    // first element of the 64-byte-aligned block [P-K-8, P-K) of the row, which is the NEXT
    // tile's sequence-0 mirror; its own arrives through CARRY from the previous tile's block.
    // Every mirror block is then read once, aligned (was 1.22x the algorithmic DRAM bytes).
    rp = col + (N - jm0 - (li == 0 ? 8 : 0));
    rs = 32 * P;
    sw = __ldg(p.sgn + (TT * 32 + a) * 8 + li);
  };
  auto issue_part = [&](int part) {
#pragma unroll
    for (int b = 8 * part; b < 8 * part + 8; ++b) x[b] = make_double2(__ldcg(mp + 32 * P * b), __ldcg(rp - rs * b));
  };
  auto prefetch = [&](int64_t cc, int64_t TT) {  // L2 <- main and mirror row segments of a regular tile
    if (!PF || TT == 0) return;
    const double* col = p.A + cc * p.lda;
    const int64_t K = 8 * (TT - 1);
#pragma unroll
    for (int r = 0; r < SL / ST; ++r) {
      const int64_t k2 = threadIdx.x + ST * r;
      prefetch_l2(col + K + P * k2);
      prefetch_l2(col + (P - K - 8) + P * (SL - 1 - k2));  // mirror block [P-K-8, P-K) of row L-1-k2
    }
  };
  auto advance = [&](int64_t& cc, int64_t& TT) {
    if (++TT == p.tiles) {
      TT = 0;
      ++cc;
    }
  };
  if (T >= 2 && li == 0) {  // chunk starts inside a column: the first tile's carry is read directly
    const double* col = p.A + c * p.lda;
    const int64_t jm0 = 8 * (T - 1) + P * a;
#pragma unroll 8
    for (int b = 0; b < 32; ++b) CARRY[32 * b + a] = __ldcg(col + (N - jm0 - 32 * P * b));
  }
  if (T == 0) {
    issue_special(c);
  } else {
    setup(c, T);
#pragma unroll
    for (int part = 0; part < 4; ++part) issue_part(part);
  }
  if (u + 1 < u1) {
    int64_t c2 = c, T2 = T;
    advance(c2, T2);
    prefetch(c2, T2);
  }
  __syncthreads();  // tables

  while (true) {
    const bool special = T == 0;
    // ---- pass 1: signs, weights, pre-twiddle W_128^b, 32-point DFT over b, twiddle W_4096^{a(4k+1)}
    {
      if (!special && li == 0) {  // sequence 0: swap the carried mirror in, keep the next tile's
        if (T == 1) {
#pragma unroll
          for (int b = 0; b < 32; ++b) CARRY[32 * b + a] = x[b].y;
        } else {
#pragma unroll
          for (int b = 0; b < 32; ++b) {
            const double t = CARRY[32 * b + a];
            CARRY[32 * b + a] = x[b].y;
            x[b].y = t;
          }
        }
      }
      const uint32_t lo = static_cast<uint32_t>(sw), hi = static_cast<uint32_t>(sw >> 32);
#pragma unroll
      for (int b = 0; b < 32; ++b) {
        x[b].x = flipd(x[b].x, (lo << (31 - b)) & 0x80000000u);
        x[b].y = flipd(x[b].y, (hi << (31 - b)) & 0x80000000u);
      }
      if (special) {  // column 0: k2 <= L/2, 1/sqrt2 at 0 (c_0 / c_1), 1/2 at L/2; column P/2: k2 < L/2
#pragma unroll
        for (int b = 0; b < 32; ++b) {
          const int k2 = a + 32 * b;
          double wgt = 0.0;
          if (li == 0) wgt = k2 == 0 ? 0.70710678118654752440 : (k2 < SL / 2 ? 1.0 : (k2 == SL / 2 ? 0.5 : 0.0));
          if (li == 1) wgt = k2 < SL / 2 ? 1.0 : 0.0;
          x[b] = make_double2(x[b].x * wgt, x[b].y * wgt);
        }
      } else if (T == 1 && li == 0) {  // column 0 lives in tile 0
#pragma unroll
        for (int b = 0; b < 32; ++b) x[b] = make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int b = 1; b < 32; ++b) x[b] = pre128(x[b], b);
    }
    dft32f(x);
#pragma unroll
    for (int k = 0; k < 32; ++k) x[k] = cmul(x[k], tw[32 * k + a]);
    __syncthreads();  // previous tile's sampled stage has read U
#pragma unroll
    for (int k = 0; k < 32; ++k) U[(32 * a + k) * SW + (li ^ (k & 7))] = x[k];
    __syncthreads();
    // ---- pass 2: warp = sequence, lane = k; 32-point DFT over a, bins to rows
    const int sc = warp ^ (lane & 7);
#pragma unroll
    for (int l = 0; l < 32; ++l) x[l] = U[(32 * l + lane) * SW + sc];
    dft32f(x);
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 32; ++k) U[(lane + 32 * k) * SW + sc] = x[k];

    // ---- next tile
    const int64_t ucur = u, Tcur = T;
    const bool more = u + 1 < u1;
    bool next_regular = false;
    if (more) {
      ++u;
      advance(c, T);
      if (T == 0) {
        issue_special(c);
      } else {
        setup(c, T);
        next_regular = true;
#pragma unroll
        for (int part = 0; part < 4; ++part) issue_part(part);
      }
      if (u + 1 < u1) {
        int64_t c2 = c, T2 = T;
        advance(c2, T2);
        prefetch(c2, T2);
      }
    }
    __syncthreads();  // all bins of the tile are in U

    // ---- sampled stage
    if (special) {  // v_n += 2 Re F_0[q] + 2 Re(W_4N^{(4n+1) P/2} F_1[q])  (the 2 is in the scale)
#pragma unroll
      for (int q = 0; q < SNQ; ++q) {
        const double2 w = __ldg(p.anc + threadIdx.x + ST * q);
        const int r = bin[q];
        const double2 f0 = U[r * SW + (r & 7)], f1 = U[r * SW + (1 ^ (r & 7))];
        acc[q] += f0.x + fma(w.x, f1.x, -w.y * f1.y);
      }
    } else {
      if ((Tcur % SANCH) == 1 || ucur == u0) {
#pragma unroll
        for (int q = 0; q < SNQ; ++q) base[q] = __ldg(p.anc + Tcur * (SNQ * ST) + threadIdx.x + ST * q);
      }
#pragma unroll
      for (int q = 0; q < SNQ; ++q) {
        const double2 st = STP[ST * q + threadIdx.x];
        const int r = bin[q], rx = r & 7;
        double2 h = U[r * SW + (7 ^ rx)];
#pragma unroll
        for (int i = SW - 2; i >= 0; --i) {
          const double2 z = U[r * SW + (i ^ rx)];
          h = make_double2(fma(st.x, h.x, fma(-st.y, h.y, z.x)), fma(st.x, h.y, fma(st.y, h.x, z.y)));
        }
        const double2 w = base[q];
        acc[q] += fma(w.x, h.x, -w.y * h.y);
        base[q] = cmul(w, STP[ST * (SNQ + q) + threadIdx.x]);
      }
    }
    if (!more || T == 0) {  // column piece done (the next tile starts a new column, or the chunk ends)
      double* part = p.part + (blockIdx.x * p.jmax + piece) * (SNQ * ST);
#pragma unroll
      for (int q = 0; q < SNQ; ++q) {
        part[threadIdx.x + ST * q] = acc[q];
        acc[q] = 0.0;
      }
      ++piece;
    }
    if (!more) break;
  }
}

// SA(row, c) = scale * sum over the CTAs covering column c of their piece for c (fixed order).
__global__ void srdct_stream_reduce(const double* __restrict__ part, int64_t tiles, int64_t chunk, int64_t jmax,
                                    int64_t n, int nslots, const int32_t* __restrict__ row_of_slot, double scale,
                                    double* __restrict__ SA, int64_t ldsa) {
  const int64_t total = n * nslots;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / nslots;
    const int o = static_cast<int>(e % nslots);
    const int64_t g0 = (c * tiles) / chunk, g1 = ((c + 1) * tiles - 1) / chunk;
    double v = 0.0;
    for (int64_t g = g0; g <= g1; ++g) {
      const int64_t j = c - (g * chunk) / tiles;
      v += part[(g * jmax + j) * (SNQ * ST) + o];
    }
    SA[row_of_slot[o] + c * ldsa] = scale * v;
  }
}

}  // namespace

int build_srdct_sgn(const uint32_t* sign_bits, int64_t m, uint64_t** out) {
  *out = nullptr;
  if (m % (SL * 16) != 0) return OK;  // the stream kernel does not apply
  const int64_t P = m / SL, tiles = P / 16 + 1, words = tiles * 256;
  NSK_CUDA_OK(cudaMalloc(out, sizeof(uint64_t) * words));
  int64_t blocks = (words + 255) / 256;
  if (blocks > 8L * sm_count()) blocks = 8L * sm_count();
  build_srdct_sgn_kernel<<<static_cast<unsigned>(blocks), 256>>>(sign_bits, m, P, words, *out);
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  NSK_CUDA_OK(cudaStreamSynchronize(0));  // the table kernels ran on the legacy stream (copies on other streams continue)
  return OK;
}

// NOTAPPLICABLE unless the whole column of a real A is applied and m is a
// multiple of 16 * 1024.
int srdct_stream_apply(const Operator& op, const RowMap& rows, int64_t n, const double* A, int64_t lda, double* SA,
                       int64_t ldsa, cudaStream_t st) {
  if (std::getenv("NSK_SRDCT_NOSTREAM")) return NOTAPPLICABLE;
  const int64_t N = op.m, s = op.s;
  if (!(rows.row0 == 0 && rows.rstep == 1 && rows.mloc == N) || n == 0) return NOTAPPLICABLE;
  if (N % (SL * 16) != 0 || N > (int64_t(1) << 40)) return NOTAPPLICABLE;
  const DeviceTables* tb = op.tables();
  if (!tb || !tb->srdct_sgn || !tb->dct_freq || !tb->dct_row) return ECUDA;
  const int64_t P = N / SL, tiles = P / 16 + 1, total = n * tiles;
  int64_t G = sm_count();
  if (G > total) G = total;
  const int64_t chunk = (total + G - 1) / G;
  G = (total + chunk - 1) / chunk;
  const int64_t jmax = chunk / tiles + 2;
  const size_t smem = sizeof(double2) * (SL * SW + STW + 2 * SNQ * ST) + sizeof(double) * 32 * 32;
  const char* pfe = std::getenv("NSK_STREAM_PF");
  auto kern = pfe && !std::atoi(pfe) ? srdct_stream_kernel<0> : srdct_stream_kernel<1>;
  NSK_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  // SA = sqrt(N/s) v, v = c_1 sum Re(...) (the pairs' 2 and G's 1/2 cancel): sqrt(N/s) sqrt(2/N)
  const double scale = std::sqrt(2.0 / static_cast<double>(s));
  for (int64_t b = 0; b < s; b += SNQ * ST) {
    const int ns = static_cast<int>((s - b) < SNQ * ST ? (s - b) : SNQ * ST);
    Scratch part, anc;
    NSK_CUDA_OK(part.alloc(sizeof(double) * G * jmax * SNQ * ST, st));
    NSK_CUDA_OK(anc.alloc(sizeof(double2) * tiles * SNQ * ST, st));
    {
      int64_t blocks = (tiles * SNQ * ST + 255) / 256;
      if (blocks > 8L * sm_count()) blocks = 8L * sm_count();
      srdct_anchor_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(tb->dct_freq + b, ns, N, P, tiles,
                                                                         anc.as<double2>());
      count_launch();
      NSK_CUDA_OK(cudaGetLastError());
    }
    DStreamParams p{A, lda, N, P, tiles, total, chunk, jmax, tb->srdct_sgn, tb->dct_freq + b, ns,
                    anc.as<double2>(), part.as<double>()};
    KernelTimer tm(st, "srdct_stream_kernel");
    kern<<<static_cast<unsigned>(G), ST, smem, st>>>(p);
    tm.stop();
    count_launch();
    NSK_CUDA_OK(cudaGetLastError());
    int64_t blocks = (n * ns + 255) / 256;
    if (blocks > 8L * sm_count()) blocks = 8L * sm_count();
    srdct_stream_reduce<<<static_cast<unsigned>(blocks), 256, 0, st>>>(part.as<double>(), tiles, chunk, jmax, n, ns,
                                                                       tb->dct_row + b, scale, SA, ldsa);
    count_launch();
    NSK_CUDA_OK(cudaGetLastError());
  }
  return OK;
}

}  // namespace nsk
