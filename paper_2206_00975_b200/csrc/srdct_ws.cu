// srdct_ws.cu -- sampled srdct: warp-specialised Makhoul tiles (FFT warps +
// sampler warps), the srdct counterpart of srft_ws.cu.
//
// Reference: apply(), srdct branch (/root/reference/proj/src/sketch.cpp:218-229)
// and dct3_unitary_columns (transforms.cpp:38-64).  Algebra as in
// srdct_stream.cu (Makhoul pairing of column k1 with P - k1 at row L-1-k2,
// w^{k1} moved into the sampled-stage step W_4N^{4n+1}, pre-twiddle
// W_128^b, inter-pass twiddle W_4096^{a(4k+1)}, tile 0 = the self-mirrored
// columns 0 and P/2), with tiles of 4 columns and the srft_ws.cu roles:
//
//  * sampler warps stage tile u+1 with 8-byte cp.async (main element
//    A[K+i+P k2] and its mirror A[N-K-i-P k2] side by side per row and
//    column) into the other of two tile buffers, completion on that buffer's
//    mbarrier, then run the sampled stage of tile u from V (one complex Horner
//    chain over 4 columns per slot, 8 slots per thread);
//  * FFT warps read (main, mirror) pairs with one 16-byte shared load per
//    row, form G, run both DFT32 passes with the transpose in place, and
//    write the 1024 bins to V.  The inter-pass twiddles W_4096^{a(4k+1)} of
//    the 32 row classes x 32 outputs sit in a 1024-entry table (a lane's a is
//    fixed).
#include "fft32.cuh"
#include "nsk_internal.hpp"

namespace nsk {

namespace {

using namespace fft;

constexpr int YL = 1024;       // FFT length
constexpr int YS = 4;          // columns (sequences) per regular tile
constexpr int YT = 256;        // threads: 128 FFT + 128 sampler
constexpr int YNQ = 8;         // output slots per sampler thread
constexpr int YANCH = 16;      // exact twiddles every YANCH tiles
constexpr int YBAR_FFT = 1, YBAR_V_FULL = 3, YBAR_V_FREE = 4;

struct DwsParams {
  const double* A;
  int64_t lda;
  int64_t N;
  int64_t P;         // N / YL
  int64_t tiles;     // per column: P / 8 + 1 (tile 0: columns 0 and P/2)
  int64_t total;     // n * tiles
  int64_t chunk;     // tiles per CTA
  int64_t jmax;      // column pieces per CTA
  const uint64_t* sgn;   // srdct_sgn: [8-column tile][a][8] negate masks (main bit b, mirror bit 32 + b)
  const int64_t* freq;   // v index n of each slot, sorted by n mod YL
  int nslots;
  const double2* anc;    // [tile][YNQ * 128]: W_4N^{(4n+1) K(tile)}, K(0) = P/2, K(T) = 4 (T - 1)
  double* part;          // [cta][jmax][YNQ * 128]
};

__device__ __forceinline__ uint32_t ysu32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void ynamed_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void ynamed_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void ymbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(ysu32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ double yflip(double v, uint32_t mask) {
  return __hiloint2double(__double2hiint(v) ^ static_cast<int>(mask), __double2loint(v));
}
__device__ __forceinline__ void cp8(void* dst, const double* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(ysu32(dst)), "l"(src), "r"(valid ? 8 : 0));
}
// v * W_128^b for a compile-time b < 32
__device__ __forceinline__ double2 ypre128(double2 v, int b) {
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

// Shared layouts (16-byte units): tile buffer / transpose element (row r,
// column i) at r * 4 + (i ^ ((r >> 1) & 3)) for the transpose and V, and at
// r * 4 + i for the staged pairs (already 4 wavefronts per warp).
__device__ __forceinline__ int yidx(int r, int i) { return r * 4 + (i ^ ((r >> 1) & 3)); }

__global__ void __launch_bounds__(YT, 1) srdct_ws_kernel(DwsParams p) {
  extern __shared__ __align__(16) double2 smy[];
  double2* BUF = smy;              // 2 x [YL][4]: staged (main, mirror) pairs, then the transpose
  double2* V = BUF + 2 * YL * YS;  // [YL][4] bins
  double2* TW = V + YL * YS;       // [k][a]: W_4096^{a (4k + 1)} (a warp's 8 row classes: one wavefront)
  double2* ST4 = TW + YL;          // [YNQ][128]: slot steps W_4N^{4 (4n+1)} (one tile)
  uint64_t* full = reinterpret_cast<uint64_t*>(ST4 + YNQ * 128);  // [2]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t N = p.N, P = p.P;
  const uint64_t N4 = 4 * static_cast<uint64_t>(N);

  for (int e = threadIdx.x; e < YL; e += YT) {
    const int k = e >> 5, a = e & 31;
    TW[e] = unit_phase(static_cast<uint64_t>(a * (4 * k + 1)), 2.0 / 4096.0);
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(ysu32(full)), "r"(128));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(ysu32(full + 1)), "r"(128));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int64_t u0 = blockIdx.x * p.chunk;
  const int64_t u1 = u0 + p.chunk < p.total ? u0 + p.chunk : p.total;
  if (u0 >= u1) return;

  if (warp < 4) {
    // ------------------------------------------------------------ FFT warps
    const int li = lane & 3, a = 8 * warp + (lane >> 2);
    int64_t T = u0 % p.tiles;
    uint32_t ph = 0;
    double2 x[32];
    for (int64_t u = u0; u < u1; ++u) {
      // negate masks: tile T >= 1 is half (T - 1) & 1 of 8-column tile (T - 1) / 2 + 1; tile 0 is tile 0
      const int64_t T8 = T == 0 ? 0 : (T - 1) / 2 + 1;
      const int i8 = T == 0 ? li : 4 * static_cast<int>((T - 1) & 1) + li;
      const uint64_t sw = __ldg(p.sgn + (T8 * 32 + a) * 8 + i8);
      const int bf = static_cast<int>((u - u0) & 1);
      double2* B = BUF + bf * (YL * YS);
      ymbar_wait(full + bf, (ph >> bf) & 1u);
      ph ^= 1u << bf;
#pragma unroll
      for (int b = 0; b < 32; ++b) x[b] = B[(a + 32 * b) * YS + li];
      {
        const uint32_t lo = static_cast<uint32_t>(sw), hi = static_cast<uint32_t>(sw >> 32);
#pragma unroll
        for (int b = 0; b < 32; ++b) {
          x[b].x = yflip(x[b].x, (lo << (31 - b)) & 0x80000000u);
          x[b].y = yflip(x[b].y, (hi << (31 - b)) & 0x80000000u);
        }
      }
      if (T == 0) {  // column 0: k2 <= L/2, 1/sqrt2 at 0 (c_0 / c_1), 1/2 at L/2; column P/2: k2 < L/2
#pragma unroll
        for (int b = 0; b < 32; ++b) {
          const int k2 = a + 32 * b;
          double wgt = 0.0;
          if (li == 0) wgt = k2 == 0 ? 0.70710678118654752440 : (k2 < YL / 2 ? 1.0 : (k2 == YL / 2 ? 0.5 : 0.0));
          if (li == 1) wgt = k2 < YL / 2 ? 1.0 : 0.0;
          x[b] = make_double2(x[b].x * wgt, x[b].y * wgt);
        }
      } else if (T == 1 && li == 0) {  // column 0 lives in tile 0
#pragma unroll
        for (int b = 0; b < 32; ++b) x[b] = make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int b = 1; b < 32; ++b) x[b] = ypre128(x[b], b);
      dft32(x);
#pragma unroll
      {  // W_4096^{a(4k+1)} = W_4096^a (W_1024^a)^k by recurrence: no shared loads on the critical path
        const double2 t1 = TW[32 + a], t0 = TW[a];  // W_4096^{5a}, W_4096^a
        const double2 r = cmul(t1, make_double2(t0.x, -t0.y));  // W_1024^a
        double2 t = t0;
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          x[k] = cmul(x[k], t);
          t = cmul(t, r);
        }
      }
      ynamed_sync(YBAR_FFT, 128);  // every warp has read the staged tile
#pragma unroll
      for (int k = 0; k < 32; ++k) B[yidx(32 * a + (k ^ (a & 1)), li)] = x[k];
      ynamed_sync(YBAR_FFT, 128);
#pragma unroll
      for (int l = 0; l < 32; ++l) x[l] = B[yidx(32 * l + (lane ^ (l & 1)), warp)];
      dft32(x);
      if (u > u0) ynamed_sync(YBAR_V_FREE, 256);
#pragma unroll
      for (int k = 0; k < 32; ++k) V[yidx(lane + 32 * k, warp)] = x[k];
      ynamed_arrive(YBAR_V_FULL, 256);
      if (++T == p.tiles) T = 0;
    }
    ynamed_sync(YBAR_V_FREE, 256);  // pair the samplers' last arrival
    return;
  }

  // -------------------------------------------------------------- samplers
  const int ts = threadIdx.x - 128;
  double acc[YNQ];
  double2 base[YNQ], step[YNQ];
  int bins[YNQ];
#pragma unroll
  for (int q = 0; q < YNQ; ++q) {
    const int o = ts + 128 * q;
    const uint64_t n = o < p.nslots ? static_cast<uint64_t>(__ldg(p.freq + o)) : 0;
    bins[q] = static_cast<int>(n & (YL - 1));
    double2 s1 = unit_phase(4 * n + 1, 2.0 / static_cast<double>(N4));
    step[q] = s1;
    s1 = cmul(s1, s1);
    ST4[128 * q + ts] = cmul(s1, s1);
    acc[q] = 0.0;
    base[q] = make_double2(1.0, 0.0);
  }
  // stage tile (cc, TT): element ch = ts + 128 j is row ch / 4, column ch % 4 (main and mirror)
  auto stage = [&](int64_t cc, int64_t TT, int bf) {
    const double* col = p.A + cc * p.lda;
    double2* B = BUF + bf * (YL * YS);
    if (TT == 0) {
#pragma unroll 4
      for (int j = 0; j < 32; ++j) {
        const int ch = ts + 128 * j, row = ch >> 2, i = ch & 3;
        const int64_t jm = i == 0 ? P * row : P / 2 + P * row;
        const int64_t jr = i == 0 ? N - P * row : P / 2 + P * (YL - 1 - row);
        const bool vm = i < 2, vr = i == 1 || (i == 0 && row > 0);
        double* d = reinterpret_cast<double*>(B + row * YS + i);
        cp8(d, vm ? col + jm : col, vm);
        cp8(d + 1, vr ? col + jr : col, vr);
      }
    } else {
      const int64_t K = 4 * (TT - 1);
#pragma unroll 8
      for (int j = 0; j < 32; ++j) {
        const int ch = ts + 128 * j, row = ch >> 2, i = ch & 3;
        const int64_t jm = K + i + P * row;
        double* d = reinterpret_cast<double*>(B + row * YS + i);
        cp8(d, col + jm, true);
        cp8(d + 1, jm > 0 ? col + (N - jm) : col, jm > 0);
      }
    }
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(ysu32(full + bf)) : "memory");
  };
  auto prefetch = [&](int64_t cc, int64_t TT) {  // L2 <- main and mirror row segments of a regular tile
    if (TT == 0) return;
    const double* col = p.A + cc * p.lda;
    const int64_t K = 4 * (TT - 1);
#pragma unroll
    for (int r = 0; r < YL / 128; ++r) {
      const int64_t k2 = ts + 128 * r;
      asm volatile("prefetch.global.L2 [%0];\n" ::"l"(col + K + P * k2));
      asm volatile("prefetch.global.L2 [%0];\n" ::"l"(col + (P - K - 3) + P * (YL - 1 - k2)));
    }
  };
  int64_t c = u0 / p.tiles, T = u0 % p.tiles, piece = 0;
  stage(c, T, 0);
  for (int64_t u = u0; u < u1; ++u) {
    const int64_t Tcur = T;
    int64_t cn = c, Tn = T;
    if (++Tn == p.tiles) {
      Tn = 0;
      ++cn;
    }
    if (u + 1 < u1) {  // tile u+1 into the buffer of tile u-1 (its V_FULL was seen)
      stage(cn, Tn, static_cast<int>((u + 1 - u0) & 1));
      if (u + 2 < u1) {
        int64_t c2 = cn, T2 = Tn;
        if (++T2 == p.tiles) {
          T2 = 0;
          ++c2;
        }
        prefetch(c2, T2);
      }
    }
    double2 wsp[YNQ];
    if (Tcur == 0) {
#pragma unroll
      for (int q = 0; q < YNQ; ++q) wsp[q] = __ldg(p.anc + ts + 128 * q);
    } else if ((Tcur % YANCH) == 1 || u == u0) {
#pragma unroll
      for (int q = 0; q < YNQ; ++q) base[q] = __ldg(p.anc + Tcur * (YNQ * 128) + ts + 128 * q);
    }
    ynamed_sync(YBAR_V_FULL, 256);
    if (Tcur == 0) {  // v_n += 2 Re F_0[q] + 2 Re(W_4N^{(4n+1) P/2} F_1[q])  (the 2 is in the scale)
#pragma unroll
      for (int q = 0; q < YNQ; ++q) {
        const int r = bins[q];
        const double2 f0 = V[yidx(r, 0)], f1 = V[yidx(r, 1)];
        acc[q] += f0.x + fma(wsp[q].x, f1.x, -wsp[q].y * f1.y);
      }
    } else {
#pragma unroll
      for (int q = 0; q < YNQ; ++q) {
        const double2 st = step[q];
        const int r = bins[q];
        double2 h = V[yidx(r, YS - 1)];
#pragma unroll
        for (int i = YS - 2; i >= 0; --i) {
          const double2 z = V[yidx(r, i)];
          h = make_double2(fma(st.x, h.x, fma(-st.y, h.y, z.x)), fma(st.x, h.y, fma(st.y, h.x, z.y)));
        }
        const double2 w = base[q];
        acc[q] += fma(w.x, h.x, -w.y * h.y);
        base[q] = cmul(w, ST4[128 * q + ts]);
      }
    }
    ynamed_arrive(YBAR_V_FREE, 256);
    if (u + 1 == u1 || Tn == 0) {  // column piece done
      double* part = p.part + (blockIdx.x * p.jmax + piece) * (YNQ * 128);
#pragma unroll
      for (int q = 0; q < YNQ; ++q) {
        part[ts + 128 * q] = acc[q];
        acc[q] = 0.0;
      }
      ++piece;
    }
    c = cn;
    T = Tn;
  }
}

// anc[T][o] = W_4N^{(4n_o + 1) K(T)}, K(0) = P/2, K(T) = 4 (T - 1).
__global__ void srdct_ws_anchor_kernel(const int64_t* __restrict__ freq, int nslots, int64_t N, int64_t P,
                                       int64_t tiles, double2* __restrict__ anc) {
  const int64_t total = tiles * (YNQ * 128);
  const uint64_t N4 = 4 * static_cast<uint64_t>(N);
  const double inv = 1.0 / static_cast<double>(N4), two = 2.0 / static_cast<double>(N4);
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int o = static_cast<int>(e % (YNQ * 128));
    const int64_t T = e / (YNQ * 128);
    const uint64_t n = o < nslots ? static_cast<uint64_t>(freq[o]) : 0;
    const uint64_t K = T == 0 ? static_cast<uint64_t>(P / 2) : static_cast<uint64_t>(4 * (T - 1));
    anc[e] = unit_phase(mulmod_fast(4 * n + 1, K, N4, inv), two);
  }
}

__global__ void srdct_ws_reduce(const double* __restrict__ part, int64_t tiles, int64_t chunk, int64_t jmax,
                                int64_t n, int nslots, const int32_t* __restrict__ row_of_slot, double scale,
                                double* __restrict__ SA, int64_t ldsa) {
  const int64_t total = n * nslots;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / nslots;
    const int o = static_cast<int>(e % nslots);
    const int64_t g0 = (c * tiles) / chunk, g1 = ((c + 1) * tiles - 1) / chunk;
    double v = 0.0;
    for (int64_t g = g0; g <= g1; ++g) v += part[(g * jmax + (c - (g * chunk) / tiles)) * (YNQ * 128) + o];
    SA[row_of_slot[o] + c * ldsa] = scale * v;
  }
}

}  // namespace

// Opt-in (NSK_SRDCT_WS=1): measured 1.21 ms against 1.07 ms for the single-role
// stream kernel at the configs[1] shape -- the staging needs 64 eight-byte
// cp.async per sampler thread and tile (a row's mirror block is not 16-byte
// aligned), and the FFT warps carry the Makhoul pre-twiddles.  NOTAPPLICABLE
// unless the whole column of a real A is applied and m is a multiple of 16 * 1024.
int srdct_ws_apply(const Operator& op, const RowMap& rows, int64_t n, const double* A, int64_t lda, double* SA,
                   int64_t ldsa, cudaStream_t st) {
  const char* e = std::getenv("NSK_SRDCT_WS");
  if (!e || !std::atoi(e)) return NOTAPPLICABLE;
  if (std::getenv("NSK_SRDCT_NOSTREAM")) return NOTAPPLICABLE;
  const int64_t N = op.m, s = op.s;
  if (!(rows.row0 == 0 && rows.rstep == 1 && rows.mloc == N) || n == 0) return NOTAPPLICABLE;
  if (N % (YL * 16) != 0 || N > (int64_t(1) << 40)) return NOTAPPLICABLE;
  const DeviceTables* tb = op.tables();
  if (!tb || !tb->srdct_sgn || !tb->dct_freq || !tb->dct_row) return ECUDA;
  const int64_t P = N / YL, tiles = P / 8 + 1, total = n * tiles;
  int64_t G = sm_count();
  if (G > total) G = total;
  const int64_t chunk = (total + G - 1) / G;
  G = (total + chunk - 1) / chunk;
  const int64_t jmax = chunk / tiles + 2;
  const size_t smem = sizeof(double2) * (3 * YL * YS + YL + YNQ * 128) + 16;
  NSK_CUDA_OK(cudaFuncSetAttribute(srdct_ws_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
  const double scale = std::sqrt(2.0 / static_cast<double>(s));  // sqrt(N/s) c_1, as srdct_stream.cu
  for (int64_t b = 0; b < s; b += YNQ * 128) {
    const int ns = static_cast<int>((s - b) < YNQ * 128 ? (s - b) : YNQ * 128);
    Scratch part, anc;
    NSK_CUDA_OK(part.alloc(sizeof(double) * G * jmax * YNQ * 128, st));
    NSK_CUDA_OK(anc.alloc(sizeof(double2) * tiles * YNQ * 128, st));
    {
      int64_t blocks = (tiles * YNQ * 128 + 255) / 256;
      if (blocks > 8L * sm_count()) blocks = 8L * sm_count();
      srdct_ws_anchor_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(tb->dct_freq + b, ns, N, P, tiles,
                                                                            anc.as<double2>());
      count_launch();
      NSK_CUDA_OK(cudaGetLastError());
    }
    DwsParams p{A, lda, N, P, tiles, total, chunk, jmax, tb->srdct_sgn, tb->dct_freq + b, ns, anc.as<double2>(),
                part.as<double>()};
    KernelTimer tm(st);
    srdct_ws_kernel<<<static_cast<unsigned>(G), YT, smem, st>>>(p);
    tm.stop();
    count_launch();
    NSK_CUDA_OK(cudaGetLastError());
    int64_t blocks = (n * ns + 255) / 256;
    if (blocks > 8L * sm_count()) blocks = 8L * sm_count();
    srdct_ws_reduce<<<static_cast<unsigned>(blocks), 256, 0, st>>>(part.as<double>(), tiles, chunk, jmax, n, ns,
                                                                   tb->dct_row + b, scale, SA, ldsa);
    count_launch();
    NSK_CUDA_OK(cudaGetLastError());
  }
  return OK;
}

}  // namespace nsk
