// srft_ws.cu -- sampled srft of a real A: warp-specialised tiles (FFT warps +
// sampler warps) so the sampled stage of one tile overlaps the FFT of the next.
//
// Reference: apply(), srft branch (/root/reference/proj/src/sketch.cpp:206-217)
// and idft_unitary_columns (transforms.cpp:17-36).  srft as s samples of one
// length-m DFT by decimation in time, L = 1024, j = k1 + P k2: the real k1
// sequences of a column are paired into complex sequences z = u_e + i u_o
// (u_k1 = d_j A[j]), each z gets a 1024-point DFT (two register DFT32 passes
// with an in-place transpose), and the sampled stage forms
// sum_k1 w_m^{f k1} U_k1[f mod L] with the Hermitian unpacking of each pair
// (Z[q], conj Z[-q]); tiles of 8 real k1 columns (4 sequences), two roles in
// one CTA of 8 warps:
//
//  * FFT warps 0-3: a lane (sequence i, row class a, 8 row classes per warp)
//    reads its 32 rows of the staged tile from shared memory, flips signs,
//    runs the first DFT32 (over b, k2 = a + 32 b) and the inter-pass twiddle,
//    transposes in place through the same buffer (128-thread named barriers,
//    no CTA barrier), runs the second DFT32 (warp = sequence) and writes all
//    1024 bins to V;
//  * sampler warps 4-7: stage tile u+1 with cp.async into the other of two
//    tile buffers (completion tracked by that buffer's mbarrier, no thread
//    waits on it) while the FFT warps work on tile u, then run the sampled
//    stage of tile u from V (8 slots per thread, Horner over 4 sequences).
//
// Hand-offs: V_FULL / V_FREE are producer-arrive, consumer-sync named
// barriers (256 threads; each producer's next arrival depends on the
// consumer's previous sync, so no phase can be lapped); a tile buffer is
// restaged only after the samplers have seen V_FULL of the tile that last
// used it.  Shared memory: two tile buffers and V (64 KiB each, swizzled so
// every access is 4 wavefronts per warp) and the w_1024 twiddles.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>
#include <mutex>
#include "fft32.cuh"
#include "nsk_internal.hpp"

namespace nsk {

namespace {

using namespace fft;

constexpr int XL = 1024;       // FFT length
constexpr int XS = 4;          // sequences per tile
constexpr int XKT = 2 * XS;    // real columns per tile
constexpr int XT = 256;        // threads: 128 FFT + 128 sampler
constexpr int XNQ = 8;         // output slots per sampler thread (128 x 8 = 1024)
constexpr int XANCH = 16;      // exact twiddles every XANCH tiles
constexpr int BAR_FFT = 1, BAR_V_FULL = 3, BAR_V_FREE = 4;

struct WsParams {
  const double* A;
  int64_t lda;
  int64_t m;
  int64_t P;         // m / XL
  int64_t tiles;     // per column: P / XKT
  int64_t total;     // n * tiles
  int64_t chunk;     // tiles per CTA
  int64_t jmax;      // column pieces per CTA
  const uint64_t* sgn;  // srft_sgn: [16-column tile][a][8] negate masks, bits 2b + e
  const int64_t* freq;  // sample index of each slot (sorted by idx mod XL)
  int nslots;
  const double2* anc;   // [tile][XNQ * 128]: w_m^{f K}, K = XKT tile
  double2* part;        // [cta][jmax][XNQ * 128]
};

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void named_sync(int id, int count) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_arrive(int id, int count) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(su32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ double flipx(double v, uint32_t mask) {
  return __hiloint2double(__double2hiint(v) ^ static_cast<int>(mask), __double2loint(v));
}

// U: element (row r, sequence i) at r * 4 + (i ^ ((r >> 1) & 3)); the pass-1
// output (a, k) lives in row 32 a + (k ^ (a & 1)).  V: bin q, sequence i at
// q * 4 + (i ^ ((q >> 1) & 3)).
__device__ __forceinline__ int uidx(int r, int i) { return r * 4 + (i ^ ((r >> 1) & 3)); }

// Negate masks (16-k1 tiles of 8 sequence pairs): word (T, a, i) bit 2b + e = 1 iff the Rademacher
// bit of row j = 16 T + 2 i + e + P (a + 32 b) is 0 (rng.hpp:57: bit 1 -> +1).  srft_ws_kernel reads
// the masks of two 8-column tiles from one 16-column word set.
__global__ void build_srft_sgn_kernel(const uint32_t* __restrict__ bits, int64_t P, int64_t words,
                                      uint64_t* __restrict__ out) {
  for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w < words;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t T = w / 256, a = (w / 8) % 32, i = w % 8;
    uint64_t v = 0;
    for (int b = 0; b < 32; ++b) {
      const int64_t j = 16 * T + 2 * i + P * (a + 32 * b);  // even: j and j + 1 share a word
      const uint32_t wd = bits[j >> 5];
      v |= static_cast<uint64_t>((~wd >> (j & 31)) & 1u) << (2 * b);
      v |= static_cast<uint64_t>((~wd >> ((j + 1) & 31)) & 1u) << (2 * b + 1);
    }
    out[w] = v;
  }
}

// TMA: the tile is staged by four 3-D tensor boxes {8 doubles, 256 rows, 1 column} issued by one
// sampler thread (no LSU work: the cp.async form costs 32 instructions per sampler thread and tile and
// twice the ideal shared-memory wavefronts, one per 64-byte row segment).
template <bool TMA>
__global__ void __launch_bounds__(XT, 1) srft_ws_kernel(WsParams p, const __grid_constant__ CUtensorMap tmA) {
  extern __shared__ __align__(128) double2 smx[];
  double2* BUF = smx;             // 2 x [XL][4]: staged tile (row k2, sequence i), then its transpose
  double2* V = BUF + 2 * XL * XS; // [XL][4] bins
  double2* tw = V + XL * XS;      // [k][a]: w_1024^{a k} (a warp's 8 row classes: one wavefront)
  double2* ST8 = tw + XL;         // [XNQ][128]: sampler slot steps w_m^{8 f} (one tile)
  uint64_t* full = reinterpret_cast<uint64_t*>(ST8 + XNQ * 128);  // [2] per tile buffer
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t m = static_cast<uint64_t>(p.m);
  const int64_t P = p.P;

  for (int e = threadIdx.x; e < XL; e += XT)
    tw[e] = unit_phase(static_cast<uint64_t>((e >> 5) * (e & 31)), 2.0 / XL);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(full)), "r"(TMA ? 1 : 128));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(full + 1)), "r"(TMA ? 1 : 128));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int64_t u0 = blockIdx.x * p.chunk;
  const int64_t u1 = u0 + p.chunk < p.total ? u0 + p.chunk : p.total;
  if (u0 >= u1) return;

  if (warp < 4) {
    // ------------------------------------------------------------ FFT warps
    const int li = lane & 3, a = 8 * warp + (lane >> 2);
    int64_t c = u0 / p.tiles, T = u0 % p.tiles;
    uint32_t ph = 0;  // bit j: phase of buffer j
    double2 x[32];
    auto sgn_of = [&](int64_t TT) { return __ldg(p.sgn + ((TT >> 1) * 32 + a) * 8 + 4 * (TT & 1) + li); };
    uint64_t sw_next = sgn_of(T);
    for (int64_t u = u0; u < u1; ++u) {
      const uint64_t sw = sw_next;  // loaded one tile ahead (an L2 round trip off the critical path)
      if (u + 1 < u1) sw_next = sgn_of(T + 1 == p.tiles ? 0 : T + 1);
      const int bf = static_cast<int>((u - u0) & 1);
      double2* RAW = BUF + bf * (XL * XS);
      double2* U = RAW;  // the transpose reuses the tile's buffer
      mbar_wait_parity(full + bf, (ph >> bf) & 1u);
      ph ^= 1u << bf;
#pragma unroll
      for (int b = 0; b < 32; ++b) x[b] = RAW[(a + 32 * b) * XS + li];
      {
        const uint32_t lo = static_cast<uint32_t>(sw), hi = static_cast<uint32_t>(sw >> 32);
#pragma unroll
        for (int b = 0; b < 32; ++b) {
          const uint32_t wd = b < 16 ? lo : hi;
          const int sh = 2 * (b & 15);
          x[b].x = flipx(x[b].x, (wd << (31 - sh)) & 0x80000000u);
          x[b].y = flipx(x[b].y, (wd << (30 - sh)) & 0x80000000u);
        }
      }
      dft32(x);
#pragma unroll
      for (int k = 1; k < 32; ++k) x[k] = cmul(x[k], tw[k * 32 + a]);
      named_sync(BAR_FFT, 128);  // every warp has read the staged tile
#pragma unroll
      for (int k = 0; k < 32; ++k) U[uidx(32 * a + (k ^ (a & 1)), li)] = x[k];
      named_sync(BAR_FFT, 128);
#pragma unroll
      for (int l = 0; l < 32; ++l) x[l] = U[uidx(32 * l + (lane ^ (l & 1)), warp)];
      dft32(x);
      if (u > u0) named_sync(BAR_V_FREE, 256);  // samplers are done with the previous tile's V
#pragma unroll
      for (int k = 0; k < 32; ++k) V[uidx(lane + 32 * k, warp)] = x[k];
      named_arrive(BAR_V_FULL, 256);
      if (++T == p.tiles) {
        T = 0;
        ++c;
      }
    }
    named_sync(BAR_V_FREE, 256);  // pair the samplers' last arrival
    return;
  }

  // -------------------------------------------------------------- samplers
  const int ts = threadIdx.x - 128;
  const double two_m = 2.0 / static_cast<double>(m);
  double2 acc[XNQ], base[XNQ], step[XNQ];
  int bins[XNQ];
#pragma unroll
  for (int q = 0; q < XNQ; ++q) {
    const int o = ts + 128 * q;
    const uint64_t f = o < p.nslots ? static_cast<uint64_t>(__ldg(p.freq + o)) : 0;
    const int qi = static_cast<int>(f & (XL - 1));
    bins[q] = qi | (((XL - qi) & (XL - 1)) << 16);
    double2 s1 = unit_phase(f, two_m);
    step[q] = s1;
#pragma unroll
    for (int r = 0; r < 3; ++r) s1 = cmul(s1, s1);
    ST8[128 * q + ts] = s1;  // w_m^{8 f}: one tile
    acc[q] = make_double2(0.0, 0.0);
    base[q] = make_double2(1.0, 0.0);
  }
  // stage tile (cc, TT): chunk ch = ts + 128 j is row ch / 4, sequence ch % 4
  auto stage = [&](int64_t cc, int64_t TT, int bf) {
    double2* RAW = BUF + bf * (XL * XS);
    uint64_t* bar = full + bf;
    if constexpr (TMA) {
      if (ts == 0) {
        // the buffer's last generic-proxy accesses (the previous tile's transpose) precede the async writes
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(bar)),
                     "r"(static_cast<uint32_t>(sizeof(double2) * XL * XS))
                     : "memory");
#pragma unroll
        for (int h = 0; h < XL / 256; ++h)
          asm volatile(
              "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
              "[%5];\n" ::"r"(su32(RAW + h * 256 * XS)),
              "l"(&tmA), "r"(static_cast<int>(XKT * TT)), "r"(256 * h), "r"(static_cast<int>(cc)), "r"(su32(bar))
              : "memory");
      }
      return;
    }
    const double* src = p.A + cc * p.lda + XKT * TT;
#pragma unroll 8
    for (int j = 0; j < 32; ++j) {
      const int ch = ts + 128 * j, row = ch >> 2, i = ch & 3;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(su32(RAW + row * XS + i)),
                   "l"(src + 2 * i + P * row));
    }
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(su32(bar)) : "memory");
  };
  auto prefetch = [&](int64_t cc, int64_t TT) {  // L2 <- 8 of the tile's 64-byte rows per thread
    const double* src = p.A + cc * p.lda + XKT * TT;
#pragma unroll
    for (int r = 0; r < XL / 128; ++r)
      asm volatile("prefetch.global.L2 [%0];\n" ::"l"(src + P * (ts + 128 * r)));
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
    if (u + 1 < u1) {  // tile u+1 into the buffer of tile u-1 (its V_FULL was seen: transposed and read)
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
    if ((Tcur % XANCH) == 0 || u == u0) {
#pragma unroll
      for (int q = 0; q < XNQ; ++q) base[q] = __ldg(p.anc + Tcur * (XNQ * 128) + ts + 128 * q);
    }
    named_sync(BAR_V_FULL, 256);
    // acc += w^{fK} sum_i w^{2fi} (E_i - i w^f D_i), E/D from Z[q] and conj Z[-q] by Horner
#pragma unroll
    for (int q = 0; q < XNQ; ++q) {
      const double2 st = step[q];
      const double2 st2 = cmul(st, st);
      const int qi = bins[q] & 0xffff, qm = bins[q] >> 16;
      double2 hq = V[uidx(qi, XS - 1)], hm = V[uidx(qm, XS - 1)];
      hm.y = -hm.y;
#pragma unroll
      for (int i = XS - 2; i >= 0; --i) {
        const double2 zq = V[uidx(qi, i)], zm = V[uidx(qm, i)];
        hq = make_double2(fma(st2.x, hq.x, fma(-st2.y, hq.y, zq.x)), fma(st2.x, hq.y, fma(st2.y, hq.x, zq.y)));
        hm = make_double2(fma(st2.x, hm.x, fma(-st2.y, hm.y, zm.x)), fma(st2.x, hm.y, fma(st2.y, hm.x, -zm.y)));
      }
      const double2 e = cadd(hq, hm), d = csub(hq, hm);
      const double2 sd = cmul(st, d);
      const double2 term = make_double2(e.x + sd.y, e.y - sd.x);
      const double2 w = base[q];
      acc[q] = make_double2(fma(w.x, term.x, fma(-w.y, term.y, acc[q].x)),
                            fma(w.x, term.y, fma(w.y, term.x, acc[q].y)));
      base[q] = cmul(w, ST8[128 * q + ts]);
    }
    named_arrive(BAR_V_FREE, 256);
    if (u + 1 == u1 || Tn == 0) {  // column piece done
      double2* part = p.part + (blockIdx.x * p.jmax + piece) * (XNQ * 128);
#pragma unroll
      for (int q = 0; q < XNQ; ++q) {
        part[ts + 128 * q] = acc[q];
        acc[q] = make_double2(0.0, 0.0);
      }
      ++piece;
    }
    c = cn;
    T = Tn;
  }
}

// anc[T][o] = w_m^{f_o K}, K = XKT T.
__global__ void srft_ws_anchor_kernel(const int64_t* __restrict__ freq, int nslots, int64_t m, int64_t tiles,
                                      double2* __restrict__ anc) {
  const int64_t total = tiles * (XNQ * 128);
  const double inv_m = 1.0 / static_cast<double>(m), two_m = 2.0 / static_cast<double>(m);
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int o = static_cast<int>(e % (XNQ * 128));
    const int64_t T = e / (XNQ * 128);
    const uint64_t f = o < nslots ? static_cast<uint64_t>(freq[o]) : 0;
    const uint64_t K = static_cast<uint64_t>(XKT * T) % static_cast<uint64_t>(m);
    anc[e] = unit_phase(mulmod_fast(f, K, static_cast<uint64_t>(m), inv_m), two_m);
  }
}

// SA(row, c) = scale * sum over the CTAs covering column c of their piece for c (fixed order).
__global__ void srft_ws_reduce(const double2* __restrict__ part, int64_t tiles, int64_t chunk, int64_t jmax,
                               int64_t n, int nslots, const int32_t* __restrict__ row_of_slot, double scale,
                               const double2* __restrict__ post, double* __restrict__ SA, int64_t ldsa) {
  const int64_t total = n * nslots;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / nslots;
    const int o = static_cast<int>(e % nslots);
    const int64_t g0 = (c * tiles) / chunk, g1 = ((c + 1) * tiles - 1) / chunk;
    double2 v = make_double2(0.0, 0.0);
    for (int64_t g = g0; g <= g1; ++g) {
      const double2 x = part[(g * jmax + (c - (g * chunk) / tiles)) * (XNQ * 128) + o];
      v.x += x.x;
      v.y += x.y;
    }
    const int64_t row = row_of_slot[o];
    if (post) {  // cyclic shard: w_m^{a g} of this output row
      const double2 w = post[row];
      v = make_double2(w.x * v.x - w.y * v.y, w.x * v.y + w.y * v.x);
    }
    SA[2 * (row + c * ldsa)] = scale * v.x;
    SA[2 * (row + c * ldsa) + 1] = scale * v.y;
  }
}

// Sign bits of a cyclic shard: bit l of the result = bit (g + P l) of the operator's sign bits.
__global__ void gather_shard_bits(const uint32_t* __restrict__ bits, int64_t g, int64_t P, int64_t N,
                                  uint32_t* __restrict__ out) {
  const int64_t words = (N + 31) / 32;
  for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w < words;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint32_t v = 0;
    for (int b = 0; b < 32; ++b) {
      const int64_t l = 32 * w + b;
      if (l >= N) break;
      const int64_t j = g + P * l;
      v |= ((bits[j >> 5] >> (j & 31)) & 1u) << b;
    }
    out[w] = v;
  }
}

}  // namespace

int build_srft_sgn(const uint32_t* sign_bits, int64_t m, uint64_t** out) {
  *out = nullptr;
  if (m % (XL * 16) != 0) return OK;  // the tile kernel does not apply
  const int64_t P = m / XL, words = (P / 16) * 256;
  NSK_CUDA_OK(cudaMalloc(out, sizeof(uint64_t) * words));
  int64_t blocks = (words + 255) / 256;
  if (blocks > 8L * sm_count()) blocks = 8L * sm_count();
  build_srft_sgn_kernel<<<static_cast<unsigned>(blocks), 256>>>(sign_bits, P, words, *out);
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  NSK_CUDA_OK(cudaStreamSynchronize(0));  // the table kernels ran on the legacy stream (copies on other streams continue)
  return OK;
}

namespace {

bool encode_tile_map(const double* A, int64_t lda, int64_t P, int64_t n, CUtensorMap* out) {
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
  if (!encode || P > 0xffffffffLL || n > 0x7fffffffLL) return false;
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(P), static_cast<cuuint64_t>(XL), static_cast<cuuint64_t>(n)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(P) * sizeof(double),
                                 static_cast<cuuint64_t>(lda) * sizeof(double)};
  const cuuint32_t box[3] = {XKT, 256, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return encode(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(A), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The warp-specialised apply over one length-m sequence per column (the whole operator, or a cyclic
// shard with its own tables and the shard twiddle `post`).
int srft_ws_run(int64_t m, int64_t s, int64_t n, const double* A, int64_t lda, const uint64_t* sgn,
                const int64_t* freq, const int32_t* row, const double2* post, double* SA, int64_t ldsa,
                cudaStream_t st) {
  const int64_t P = m / XL, tiles = P / XKT, total = n * tiles;
  int64_t G = sm_count();
  if (G > total) G = total;
  const int64_t chunk = (total + G - 1) / G;
  G = (total + chunk - 1) / chunk;
  const int64_t jmax = chunk / tiles + 2;
  // two tile buffers, V, twiddles, slot steps, 2 mbarriers
  const size_t smem = sizeof(double2) * (3 * XL * XS + XL + XNQ * 128) + 16;
  NSK_CUDA_OK(cudaFuncSetAttribute(srft_ws_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
  NSK_CUDA_OK(cudaFuncSetAttribute(srft_ws_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
  // A as {k1 (P, contiguous), k2 (1024, stride P), column (n, stride lda)}: tile T of column c is the
  // boxes {8, 256, 1} at (8 T, 256 h, c).  NSK_SRFT_TMA=0 or a failed encode: cp.async staging.
  CUtensorMap tm_a;
  std::memset(&tm_a, 0, sizeof(tm_a));
  const char* te = std::getenv("NSK_SRFT_TMA");
  const bool tma = !(te && te[0] == '0') && encode_tile_map(A, lda, P, n, &tm_a);
  const double scale = 0.5 / std::sqrt(static_cast<double>(s));  // unnormalised DFT / sqrt(s); pairs carry 2
  for (int64_t b = 0; b < s; b += XNQ * 128) {
    const int ns = static_cast<int>((s - b) < XNQ * 128 ? (s - b) : XNQ * 128);
    Scratch part, anc;
    NSK_CUDA_OK(part.alloc(sizeof(double2) * G * jmax * XNQ * 128, st));
    NSK_CUDA_OK(anc.alloc(sizeof(double2) * tiles * XNQ * 128, st));
    {
      int64_t blocks = (tiles * XNQ * 128 + 255) / 256;
      if (blocks > 8L * sm_count()) blocks = 8L * sm_count();
      srft_ws_anchor_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(freq + b, ns, m, tiles,
                                                                           anc.as<double2>());
      count_launch();
      NSK_CUDA_OK(cudaGetLastError());
    }
    WsParams p{A, lda, m, P, tiles, total, chunk, jmax, sgn, freq + b, ns, anc.as<double2>(), part.as<double2>()};
    KernelTimer tm(st, "srft_ws_kernel");
    if (tma)
      srft_ws_kernel<true><<<static_cast<unsigned>(G), XT, smem, st>>>(p, tm_a);
    else
      srft_ws_kernel<false><<<static_cast<unsigned>(G), XT, smem, st>>>(p, tm_a);
    tm.stop();
    count_launch();
    NSK_CUDA_OK(cudaGetLastError());
    int64_t blocks = (n * ns + 255) / 256;
    if (blocks > 8L * sm_count()) blocks = 8L * sm_count();
    srft_ws_reduce<<<static_cast<unsigned>(blocks), 256, 0, st>>>(part.as<double2>(), tiles, chunk, jmax, n, ns,
                                                                  row + b, scale, post, SA, ldsa);
    count_launch();
    NSK_CUDA_OK(cudaGetLastError());
  }
  return OK;
}

}  // namespace

// NOTAPPLICABLE unless the whole column of a real A is applied, m is a multiple of 16 * 1024 and A
// is 16-byte aligned with an even lda.
int srft_ws_apply(const Operator& op, int ncomp, const RowMap& rows, int64_t n, const double* A, int64_t lda,
                  double* SA, int64_t ldsa, cudaStream_t st) {
  const char* e = std::getenv("NSK_SRFT_WS");
  if (e && !std::atoi(e)) return NOTAPPLICABLE;
  const int64_t m = op.m;
  if (op.kind != SRFT || ncomp != 1 || n == 0) return NOTAPPLICABLE;
  if (!(rows.row0 == 0 && rows.rstep == 1 && rows.mloc == m)) return NOTAPPLICABLE;
  if (m % (XL * 16) != 0 || (reinterpret_cast<uintptr_t>(A) & 15) != 0 || (lda & 1) != 0) return NOTAPPLICABLE;
  const DeviceTables* tb = op.tables();
  if (!tb || !tb->srft_sgn || !tb->srtt_freq || !tb->srtt_row) return ECUDA;
  return srft_ws_run(m, op.s, n, A, lda, tb->srft_sgn, tb->srtt_freq, tb->srtt_row, nullptr, SA, ldsa, st);
}

// Cyclic shard g of P (local rows g + P l, N = m / P a multiple of 16 * 1024): the same kernel on the
// local sequence with the shard's own signs and frequencies a mod N, then the twiddle w_m^{a g}
// (decimation in time, srtt_general.cu header).  Tables are built once per (operator, device, g, P).
int srft_ws_shard(const Operator& op, int ncomp, const RowMap& rows, int64_t n, const double* A, int64_t lda,
                  double* SA, int64_t ldsa, cudaStream_t st) {
  const char* e = std::getenv("NSK_SRFT_WS");
  if (e && !std::atoi(e)) return NOTAPPLICABLE;
  const int64_t m = op.m, s = op.s, P = rows.rstep, g = rows.row0, N = rows.mloc;
  if (op.kind != SRFT || ncomp != 1 || n == 0 || P < 2 || g < 0 || g >= P || m % P != 0 || N != m / P)
    return NOTAPPLICABLE;
  if (N % (XL * 16) != 0 || (reinterpret_cast<uintptr_t>(A) & 15) != 0 || (lda & 1) != 0) return NOTAPPLICABLE;
  const DeviceTables* tb = op.tables();
  if (!tb || !tb->sign_bits) return ECUDA;
  int devno = 0;
  NSK_CUDA_OK(cudaGetDevice(&devno));
  const Operator::ShardTables* sh = nullptr;
  {
    std::lock_guard<std::mutex> lock(op.mu);
    for (auto& t : op.shard_tabs)
      if (t.device == devno && t.g == g && t.P == P) sh = &t;
    if (!sh) {
      Operator::ShardTables t;
      t.device = devno;
      t.g = g;
      t.P = P;
      auto bail = [&t](cudaError_t err, const char* what) {
        void* ptrs[] = {t.bits, t.sgn, t.freq, t.row, t.post};
        for (void* q : ptrs)
          if (q) cudaFree(q);
        return cuda_fail(err, what);
      };
      const int64_t words = (N + 31) / 32;
      if (cudaError_t err = cudaMalloc(&t.bits, sizeof(uint32_t) * words)) return bail(err, "shard sign bits");
      int64_t blocks = (words + 255) / 256;
      if (blocks > 8L * sm_count()) blocks = 8L * sm_count();
      gather_shard_bits<<<static_cast<unsigned>(blocks), 256>>>(tb->sign_bits, g, P, N, t.bits);
      count_launch();
      if (cudaError_t err = cudaStreamSynchronize(0)) return bail(err, "shard sign bits");
      if (build_srft_sgn(t.bits, N, &t.sgn) != OK || !t.sgn) return bail(cudaErrorUnknown, "shard negate masks");
      // slots sorted by bin (a mod N) mod 1024, output row = original slot, twiddle w_m^{a g}
      std::vector<int32_t> order(static_cast<size_t>(s));
      for (int64_t r = 0; r < s; ++r) order[r] = static_cast<int32_t>(r);
      std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) {
        return ((op.idx[x] % N) & (XL - 1)) < ((op.idx[y] % N) & (XL - 1));
      });
      std::vector<int64_t> freq(static_cast<size_t>(s));
      std::vector<double2> post(static_cast<size_t>(s));
      for (int64_t r = 0; r < s; ++r) {
        freq[r] = op.idx[order[r]] % N;
        const uint64_t e2 = static_cast<uint64_t>((static_cast<unsigned __int128>(op.idx[r]) * static_cast<uint64_t>(g)) %
                                                  static_cast<uint64_t>(m));
        const double ang = 2.0 * M_PI * static_cast<double>(e2) / static_cast<double>(m);
        post[r] = make_double2(std::cos(ang), std::sin(ang));
      }
      if (cudaError_t err = cudaMalloc(&t.freq, sizeof(int64_t) * s)) return bail(err, "shard slots");
      if (cudaError_t err = cudaMalloc(&t.row, sizeof(int32_t) * s)) return bail(err, "shard slots");
      if (cudaError_t err = cudaMalloc(&t.post, sizeof(double2) * s)) return bail(err, "shard slots");
      if (cudaError_t err = cudaMemcpy(t.freq, freq.data(), sizeof(int64_t) * s, cudaMemcpyHostToDevice))
        return bail(err, "shard slots");
      if (cudaError_t err = cudaMemcpy(t.row, order.data(), sizeof(int32_t) * s, cudaMemcpyHostToDevice))
        return bail(err, "shard slots");
      if (cudaError_t err = cudaMemcpy(t.post, post.data(), sizeof(double2) * s, cudaMemcpyHostToDevice))
        return bail(err, "shard slots");
      op.shard_tabs.push_back(t);
      sh = &op.shard_tabs.back();
    }
  }
  return srft_ws_run(N, s, n, A, lda, sh->sgn, sh->freq, sh->row, sh->post, SA, ldsa, st);
}

}  // namespace nsk
