// srtt_fast.cu -- K2 fast path: sampled srft / srdct in O(m n log m).
//
// Both kinds reduce to s sampled outputs of one length-m DFT with kernel
// e^{+2 pi i jk/m} (the unitary inverse DFT of transforms.cpp:17-36):
//   srft : u_j = d_j A[j]                          X[a] = sum_j u_j w^{aj}
//          SA[r] = (1/sqrt s) X[idx_r]
//   srdct: Makhoul's DCT-III via a Hermitian DFT (transforms.cpp:38-64 computes
//          the same orthonormal DCT-III with FFTW REDFT01):
//          X_0 = 2 c_0 d_0 A[0], X_k = c_k d_k A[k],  V_k = e^{i pi k/2m}(X_k - i X_{m-k})
//          v_p = sum_k V_k w^{kp} (real),  y_a = v_p / 2 with p = a/2 (a even),
//          p = m-1-(a-1)/2 (a odd);  SA[r] = sqrt(m/s) y_{idx_r}.
// Decimation in time with stride P = m/1024: X[a] = sum_{k1<P} w_m^{a k1} F_{k1}[a mod 1024],
// F_{k1} = DFT_1024(u[k1 + P k2]).  Only the s sampled outputs of the second
// stage are formed, so no intermediate of A's size is ever written.
//
// Kernel: a CTA owns one column and a contiguous range of 4-wide k1 blocks.
// Per block it stages the 4 x 1024 strided sequences in shared memory
// (coalesced 32-64 B row segments), each warp runs one 1024-point FFT as
// 32 x 32 (register radix-2 DFT32, twiddle, padded shared-memory transpose,
// DFT32), and every thread accumulates its output slots
// acc += w_m^{a (k1)} F_{k1}[a mod 1024] in registers.  Per-CTA partials
// are reduced in fixed order.  Requires m % 4096 == 0; other sizes use the
// direct evaluator.
#include <cstdlib>

#include "fft32.cuh"
#include "nsk_internal.hpp"

namespace nsk {

int srtt_direct_apply(const Operator& op, int ncomp, const RowMap& rows, int64_t n, const double* A,
                      int64_t lda, double* SA, int64_t ldsa, cudaStream_t st);
int srtt_general_apply(const Operator& op, int ncomp, const RowMap& rows, int64_t n, const double* A,
                       int64_t lda, double* SA, int64_t ldsa, cudaStream_t st);
int srft_ws_shard(const Operator& op, int ncomp, const RowMap& rows, int64_t n, const double* A, int64_t lda,
                  double* SA, int64_t ldsa, cudaStream_t st);

// ---- plain sign bitmask for srft/srdct (m/8 bytes) -------------------------
__global__ void build_sign_bits_kernel(PhiloxKey key, int64_t m, uint32_t* __restrict__ out) {
  const int64_t words = (m + 31) / 32;
  for (int64_t w = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; w < words;
       w += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint32_t bits = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const uint4 blk = philox4x32_10(key, static_cast<uint64_t>(w) * 8u + b);
      bits |= (blk.x & 1u) << (4 * b) | (blk.y & 1u) << (4 * b + 1) | (blk.z & 1u) << (4 * b + 2) |
              (blk.w & 1u) << (4 * b + 3);
    }
    out[w] = bits;  // rows beyond m carry bits that are never read
  }
}

int build_sign_bits(PhiloxKey key, int64_t m, uint32_t** out) {
  *out = nullptr;
  const int64_t words = (m + 31) / 32;
  NSK_CUDA_OK(cudaMalloc(out, sizeof(uint32_t) * words));
  int64_t blocks = (words + 255) / 256;
  if (blocks > 8L * sm_count()) blocks = 8L * sm_count();
  build_sign_bits_kernel<<<static_cast<unsigned>(blocks), 256>>>(key, m, *out);
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  NSK_CUDA_OK(cudaStreamSynchronize(0));  // the table kernels ran on the legacy stream (copies on other streams continue)
  return OK;
}

namespace {

constexpr int L = 1024;         // local DFT length
constexpr int W = 4;            // k1 values per block (one warp each)
constexpr int T = 32 * W;       // threads per CTA
constexpr int UPAD = 32 * 33;   // per-warp buffer: 1024 values or a padded 32 x 33 transpose
constexpr int REANCHOR = 32;    // exact twiddle every REANCHOR blocks

using namespace fft;

struct SrttParams {
  const double* A;
  int64_t lda;
  int64_t m;
  int64_t n;
  int64_t P;               // m / L
  int64_t blocks_per_col;  // P / W
  int64_t ranges;          // CTA ranges per column
  int64_t per;             // blocks per range
  const uint32_t* sign_bits;
  const int64_t* freq;     // DFT frequency of each output slot (s_pass)
  int nslots;
  double* part;            // [column][range][slot] complex
  int64_t g, rstep;        // global row of local row k: g + rstep k (cyclic shard; 0, 1 unsharded)
  double c0, c1;           // KIND 2: orthonormal DCT-III weights of the GLOBAL length
};

__device__ __forceinline__ double row_sign(const uint32_t* bits, int64_t j) {
  return ((bits[j >> 5] >> (j & 31)) & 1u) ? 1.0 : -1.0;
}

template <int KIND, int NCIN, int NQ>
__global__ void __launch_bounds__(T, 2) srtt_fft_kernel(SrttParams p) {
  extern __shared__ __align__(16) double2 sm2[];
  double2* U = sm2;                 // [W][UPAD]
  double2* tw = U + W * UPAD;       // [L] w_1024^k
  double2* q32 = tw + L;            // [64]: e^{i pi a/64} (a<32), e^{i pi b/2048} (b<32)  (srdct)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t col = blockIdx.x / p.ranges, range = blockIdx.x % p.ranges;
  const int64_t b0 = range * p.per;
  int64_t b1 = b0 + p.per;
  if (b1 > p.blocks_per_col) b1 = p.blocks_per_col;
  const double* Acol = p.A + col * p.lda * NCIN;
  const int64_t m = p.m, P = p.P;

  for (int k = threadIdx.x; k < L; k += T) {
    double sn, cs;
    sincospi(static_cast<double>(k) / (L / 2), &sn, &cs);
    tw[k] = make_double2(cs, sn);
  }
  if (KIND != 0)
    for (int k = threadIdx.x; k < 64; k += T) {
      double sn, cs;
      sincospi(k < 32 ? static_cast<double>(k) / 64.0 : static_cast<double>(k - 32) / 2048.0, &sn, &cs);
      q32[k] = make_double2(cs, sn);
    }

  // Output slots owned by this thread.
  int64_t fq[NQ];
  double2 acc[NQ], wa[NQ], base[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int o = threadIdx.x + T * q;
    fq[q] = o < p.nslots ? p.freq[o] : 0;
    acc[q] = make_double2(0.0, 0.0);
    double sn, cs;
    sincospi(2.0 * static_cast<double>(fq[q]) / static_cast<double>(m), &sn, &cs);
    wa[q] = make_double2(cs, sn);  // w_m^{a}
  }
  const double c0 = sqrt(1.0 / static_cast<double>(m)), c1 = sqrt(2.0 / static_cast<double>(m));

  for (int64_t blk = b0; blk < b1; ++blk) {
    const int64_t K = blk * W;
    __syncthreads();  // previous block's gather done
    // ---- stage the W strided sequences u[k1 + P k2], k1 = K + w (w is fixed per thread)
    const int w_me = threadIdx.x % W;
    double2 ph_w = make_double2(1.0, 0.0);
    if (KIND != 0) {  // e^{i pi (K + w) / 2m}
      double sn, cs;
      sincospi(static_cast<double>(K + w_me) / (2.0 * static_cast<double>(m)), &sn, &cs);
      ph_w = make_double2(cs, sn);
    }
#pragma unroll 8
    for (int i = threadIdx.x; i < W * L; i += T) {
      const int k2 = i / W;
      const int64_t k = K + w_me + P * k2;
      double2 u;
      if (KIND == 0) {
        const double sg = row_sign(p.sign_bits, p.g + p.rstep * k);
        u = NCIN == 1 ? make_double2(sg * Acol[k], 0.0) : make_double2(sg * Acol[2 * k], sg * Acol[2 * k + 1]);
      } else if (KIND == 2) {  // srdct of a cyclic shard: c_j d_j x_k w_{4N}^k (srtt_general.cu derivation)
        const int64_t j = p.g + p.rstep * k;
        const double xk = (j == 0 ? p.c0 : p.c1) * row_sign(p.sign_bits, j) * Acol[k];
        const double2 ph = cmul(ph_w, cmul(q32[k2 >> 5], q32[32 + (k2 & 31)]));
        u = make_double2(ph.x * xk, ph.y * xk);
      } else {
        const double xk = (k == 0 ? 2.0 * c0 : c1) * row_sign(p.sign_bits, k) * Acol[k];
        const double xm = k == 0 ? 0.0 : c1 * row_sign(p.sign_bits, m - k) * Acol[m - k];
        // e^{i pi k / 2m} = e^{i pi (K + w) / 2m} * e^{i pi k2 / 2048}, k2 = 32 a + b
        const double2 ph = cmul(ph_w, cmul(q32[k2 >> 5], q32[32 + (k2 & 31)]));
        u = cmul(ph, make_double2(xk, -xm));
      }
      U[w_me * UPAD + k2] = u;
    }
    __syncthreads();
    // ---- warp w: 1024-point DFT of U[w] as 32 x 32 (n = l + 32 t, f = k2' + 32 k1')
    {
      double2* Uw = U + warp * UPAD;
      double2 x[32];
#pragma unroll
      for (int t = 0; t < 32; ++t) x[t] = Uw[lane + 32 * t];
      dft32(x);  // over t: Y[l][k2']
#pragma unroll
      for (int k2 = 1; k2 < 32; ++k2) x[k2] = cmul(x[k2], tw[(lane * k2) & (L - 1)]);
      __syncwarp();
#pragma unroll
      for (int k2 = 0; k2 < 32; ++k2) Uw[k2 * 33 + lane] = x[k2];
      __syncwarp();
#pragma unroll
      for (int l = 0; l < 32; ++l) x[l] = Uw[lane * 33 + l];
      dft32(x);  // over l: lane k2' holds X[k2' + 32 k1']
      __syncwarp();
#pragma unroll
      for (int k1 = 0; k1 < 32; ++k1) Uw[lane + 32 * k1] = x[k1];
    }
    __syncthreads();
    // ---- sampled second stage: acc += w_m^{a (K + w)} F_{K+w}[a mod L]
    const bool anchor = ((blk - b0) % REANCHOR) == 0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      if (anchor) {
        const uint64_t r = static_cast<uint64_t>(
            (static_cast<unsigned __int128>(fq[q]) * static_cast<uint64_t>(K)) % static_cast<uint64_t>(m));
        double sn, cs;
        sincospi(2.0 * static_cast<double>(r) / static_cast<double>(m), &sn, &cs);
        base[q] = make_double2(cs, sn);
      }
      const int bq = static_cast<int>(fq[q] & (L - 1));
      double2 t = base[q];
#pragma unroll
      for (int w = 0; w < W; ++w) {
        const double2 f = U[w * UPAD + bq];
        acc[q].x = fma(t.x, f.x, fma(-t.y, f.y, acc[q].x));
        acc[q].y = fma(t.x, f.y, fma(t.y, f.x, acc[q].y));
        t = cmul(t, wa[q]);
      }
      base[q] = t;  // w_m^{a (K + W)}
    }
  }
  double2* part = reinterpret_cast<double2*>(p.part) + (col * p.ranges + range) * (NQ * T);
#pragma unroll
  for (int q = 0; q < NQ; ++q) part[threadIdx.x + T * q] = acc[q];
}

template <int KIND>
__global__ void srtt_reduce(const double2* __restrict__ part, int64_t ranges, int64_t n, int nslots, int stride,
                            int slot_base, double scale, double* __restrict__ SA, int64_t ldsa) {
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
    const int64_t row = slot_base + o;
    if (KIND == 0) {
      SA[2 * (row + c * ldsa)] = scale * v.x;
      SA[2 * (row + c * ldsa) + 1] = scale * v.y;
    } else {
      SA[row + c * ldsa] = scale * 0.5 * v.x;
    }
  }
}

template <int KIND, int NCIN, int NQ>
int launch_fft(const SrttParams& p, int64_t ctas, cudaStream_t st) {
  const size_t smem = sizeof(double2) * (W * UPAD + L + 64);
  auto kern = srtt_fft_kernel<KIND, NCIN, NQ>;
  NSK_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  KernelTimer tm(st, "srtt_fft_kernel");
  kern<<<static_cast<unsigned>(ctas), T, smem, st>>>(p);
  tm.stop();
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  return OK;
}

template <int KIND, int NCIN>
int launch_nq(int nq, const SrttParams& p, int64_t ctas, cudaStream_t st) {
  return nq <= 2 ? launch_fft<KIND, NCIN, 2>(p, ctas, st)
       : nq <= 4 ? launch_fft<KIND, NCIN, 4>(p, ctas, st)
                 : launch_fft<KIND, NCIN, 8>(p, ctas, st);
}

// Cyclic shard g of P (local length N = m / P, a multiple of 4096): the same strided DFT32 x 32
// kernel over the local rows with the signs of the global rows; srft samples W[a mod N], srdct
// takes the complex formulation (KIND 2, srtt_general.cu header); the reduce applies the shard
// twiddle, the conjugation and the scale.
int srtt_fast_shard(const Operator& op, int ncomp, const RowMap& rows, int64_t n, const double* A, int64_t lda,
                    double* SA, int64_t ldsa, cudaStream_t st) {
  const DeviceTables* tb = op.tables();
  if (!tb || !tb->sign_bits) return ECUDA;
  const int64_t m = op.m, s = op.s, N = rows.mloc;
  const int kind = op.kind == SRFT ? 0 : 1;
  Scratch tab;
  int64_t* dfreq = nullptr;
  double2* dpost = nullptr;
  uint8_t* dconj = nullptr;
  if (int rc = shard_slot_tables(op, rows.row0, N, tab, &dfreq, &dpost, &dconj, st)) return rc;
  const int64_t P = N / L, bpc = P / W;
  const int64_t target = 2L * sm_count();
  int64_t ranges = (target + n - 1) / n;
  if (ranges > bpc) ranges = bpc;
  const int64_t per = (bpc + ranges - 1) / ranges;
  ranges = (bpc + per - 1) / per;
  const double scale = kind == 0 ? 1.0 / std::sqrt(static_cast<double>(s))
                                 : std::sqrt(static_cast<double>(m) / static_cast<double>(s));
  for (int64_t base = 0; base < s; base += 8 * T) {
    const int ns = static_cast<int>((s - base) < 8 * T ? (s - base) : 8 * T);
    const int nq = (ns + T - 1) / T;
    const int NQ = nq <= 2 ? 2 : (nq <= 4 ? 4 : 8);
    Scratch part;
    NSK_CUDA_OK(part.alloc(sizeof(double2) * n * ranges * NQ * T, st));
    SrttParams p{A, lda, N, n, P, bpc, ranges, per, tb->sign_bits, dfreq + base, ns, part.as<double>(),
                 rows.row0, rows.rstep, std::sqrt(1.0 / static_cast<double>(m)), std::sqrt(2.0 / static_cast<double>(m))};
    const int64_t ctas = n * ranges;
    int rc = kind == 0 ? (ncomp == 1 ? launch_nq<0, 1>(NQ, p, ctas, st) : launch_nq<0, 2>(NQ, p, ctas, st))
                       : launch_nq<2, 1>(NQ, p, ctas, st);
    if (rc != OK) return rc;
    // partials are [column][range][slot]
    if (int rc2 = srtt_post_reduce(kind, reinterpret_cast<const double2*>(part.p), NQ * T, ranges * NQ * T, ranges,
                                   n, ns, static_cast<int>(base), dpost, dconj, scale, SA, ldsa, st))
      return rc2;
  }
  return OK;
}

}  // namespace

int srtt_fast_apply(const Operator& op, int ncomp, const RowMap& rows, int64_t n, const double* A, int64_t lda,
                    double* SA, int64_t ldsa, cudaStream_t st) {
  const int64_t m = op.m, s = op.s;
  const bool full = rows.row0 == 0 && rows.rstep == 1 && rows.mloc == m;
  if (!full && n > 0 && rows.mloc % (L * W) == 0 && srtt_general_eligible(op, rows) &&
      !std::getenv("NSK_SRTT_DIRECT") && !(op.kind == SRDCT && ncomp != 1)) {
    // srft of a real A on a shard of 16 * 1024 multiples: the warp-specialised tiles (srft_ws.cu)
    const int rw = srft_ws_shard(op, ncomp, rows, n, A, lda, SA, ldsa, st);
    if (rw != NOTAPPLICABLE) return rw;
    return srtt_fast_shard(op, ncomp, rows, n, A, lda, SA, ldsa, st);
  }
  if (!full || m % (L * W) != 0 || n == 0) {
    // any other length, and the cyclic shards: the mixed-radix engine (srtt_general.cu); the direct
    // O(s m n) evaluator only for contiguous partial shards (or NSK_SRTT_DIRECT=1)
    if (!std::getenv("NSK_SRTT_DIRECT")) {
      const int rg = srtt_general_apply(op, ncomp, rows, n, A, lda, SA, ldsa, st);
      if (rg != NOTAPPLICABLE) return rg;
    }
    return srtt_direct_apply(op, ncomp, rows, n, A, lda, SA, ldsa, st);
  }
  const DeviceTables* tb = op.tables();
  if (!tb || !tb->sign_bits) return ECUDA;
  const int kind = op.kind == SRFT ? 0 : 1;
  // DFT frequency of every output row (srdct: Makhoul's index map).
  std::vector<int64_t> freq(static_cast<size_t>(s));
  for (int64_t r = 0; r < s; ++r) {
    const int64_t a = op.idx[static_cast<size_t>(r)];
    freq[static_cast<size_t>(r)] = kind == 0 ? a : ((a % 2 == 0) ? a / 2 : m - 1 - (a - 1) / 2);
  }
  Scratch dfreq;
  NSK_CUDA_OK(dfreq.alloc(sizeof(int64_t) * s, st));
  NSK_CUDA_OK(cudaMemcpyAsync(dfreq.p, freq.data(), sizeof(int64_t) * s, cudaMemcpyHostToDevice, st));
  const int64_t P = m / L, bpc = P / W;
  const int64_t target = 2L * sm_count();
  int64_t ranges = (target + n - 1) / n;
  if (ranges > bpc) ranges = bpc;
  const int64_t per = (bpc + ranges - 1) / ranges;
  ranges = (bpc + per - 1) / per;
  const double scale = kind == 0 ? 1.0 / std::sqrt(static_cast<double>(s))
                                 : std::sqrt(static_cast<double>(m) / static_cast<double>(s));
  for (int64_t base = 0; base < s; base += 8 * T) {
    const int ns = static_cast<int>((s - base) < 8 * T ? (s - base) : 8 * T);
    const int nq = (ns + T - 1) / T;
    const int NQ = nq <= 2 ? 2 : (nq <= 4 ? 4 : 8);
    Scratch part;
    NSK_CUDA_OK(part.alloc(sizeof(double2) * n * ranges * NQ * T, st));
    SrttParams p{A, lda, m, n, P, bpc, ranges, per, tb->sign_bits, dfreq.as<int64_t>() + base, ns, part.as<double>(),
                 0, 1, 0.0, 0.0};
    const int64_t ctas = n * ranges;
    int rc = kind == 0 ? (ncomp == 1 ? launch_nq<0, 1>(NQ, p, ctas, st) : launch_nq<0, 2>(NQ, p, ctas, st))
                       : launch_nq<1, 1>(NQ, p, ctas, st);
    if (rc != OK) return rc;
    int64_t blocks = (n * ns + 255) / 256;
    if (blocks > 8L * sm_count()) blocks = 8L * sm_count();
    if (kind == 0)
      srtt_reduce<0><<<static_cast<unsigned>(blocks), 256, 0, st>>>(reinterpret_cast<const double2*>(part.p), ranges, n,
                                                                   ns, NQ * T, static_cast<int>(base), scale, SA, ldsa);
    else
      srtt_reduce<1><<<static_cast<unsigned>(blocks), 256, 0, st>>>(reinterpret_cast<const double2*>(part.p), ranges, n,
                                                                   ns, NQ * T, static_cast<int>(base), scale, SA, ldsa);
    count_launch();
    NSK_CUDA_OK(cudaGetLastError());
  }
  return OK;
}

}  // namespace nsk
