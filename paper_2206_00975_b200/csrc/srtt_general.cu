// srtt_general.cu -- srft / srdct of ANY length m, and of cyclic row shards.
//
// Reference: apply(), srft and srdct branches (/root/reference/proj/src/
// sketch.cpp:206-229) over FFTW's exact-length transforms (transforms.cpp:
// 17-64; no padding, sketch.hpp:34-35).  The tuned tile / stream kernels need
// m % 16384 == 0 (or % 4096); this engine takes every other shape -- m =
// 20000, 100000, 99850 (= 2 5^2 1997), ... -- and the cyclic shards of the
// multi-GPU path (rank g of P holds global rows g, g + P, ...), in
// O(N log Q + s N / Q) per column instead of the O(s N) direct sum.
//
// Both kinds become s samples of one unnormalised inverse DFT of a local
// sequence u of length N = m / P (P = row stride, g = first global row):
//   srft : u_l = d_j x_l (j = g + P l),   W = DFT_N(u),
//          SA[i] = (1/sqrt s) w_m^{a_i g} W[a_i mod N]
//   srdct: u_l = c_j d_j x_l w_{4N}^l (c_0 = sqrt(1/m), c_j = sqrt(2/m)),
//          q = (2 a_i + 1) mod 4N, b = (q - 1) / 2,
//          Z = W[b / 2] (b even)  or  conj(W[(-(b - 1) / 2 - 1) mod N]) (b odd),
//          SA[i] = sqrt(m/s) Re(w_{4m}^{(2 a_i + 1) g} Z)
// since cos(pi (2a+1) j / 2m) = Re w_{4m}^{(2a+1) j} and (2a+1) P l / 4m =
// (2a+1) l / 4N; for real u the odd-b half is the conjugate mirror of W.
// (w_K = e^{+2 pi i / K}; summing the partials of the P shards gives the full
// SA, and P = 1, g = 0 is the unsharded apply.)
//
// W at the sampled frequencies by decimation in time, N = Q P2 with Q the
// largest 2,3,5,7-smooth divisor of N up to 512 (1024 with NSK_GEN_QMAX):
//   W[f] = sum_{k1 < P2} w_N^{f k1} F_{k1}[f mod Q],  F_{k1} = DFT_Q(u[k1 + P2 k2]).
// A CTA owns one column and a range of k1; it stages G = 4 consecutive k1
// sequences at a time (32-byte row segments), runs a self-sorting mixed-radix
// (4, 2, 3, 5, 7) Stockham FFT on all four in shared memory with an exact
// twiddle table, and every thread accumulates its output slots in registers
// with exact outer twiddles (integer argument reduction + sincospi).  Per-CTA
// partials are reduced in fixed order, which also applies the shard twiddle,
// the conjugation and the scale.  N with a large prime factor leaves a small
// Q and a long outer sum (N = 99850: Q = 50, P2 = 1997); still s N / Q, not s N.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "nsk_internal.hpp"

namespace nsk {

int srtt_direct_apply(const Operator& op, int ncomp, const RowMap& rows, int64_t n, const double* A,
                      int64_t lda, double* SA, int64_t ldsa, cudaStream_t st);

namespace {

constexpr int GT = 256;     // threads per CTA
constexpr int GG_MAX = 4;   // sequences (consecutive k1) per batch: 4, or 2 when Q > 704 (shared memory)
constexpr int QMAX = 1024;  // inner DFT length bound (shared memory: 2 G Q + 2 Q complex)
constexpr int MAXPASS = 12;

struct GenParams {
  const double* A;
  int64_t lda;
  int64_t n;
  int64_t N;       // local length
  int64_t Q, P2;   // N = Q P2
  int64_t per;     // k1 values per CTA range
  int64_t ranges;
  int64_t g, P;    // global row of local row l: g + P l
  double c0, c1;   // srdct weights: c_0 (global row 0) and c_j, j > 0
  const uint32_t* sign_bits;
  const int64_t* freq;  // [ns] DFT frequency in [0, N)
  int ns;               // output slots of this launch
  int npass;
  int radix[MAXPASS];
  double2* part;        // [ranges][n][NQ * GT]
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// Exact w_K^e for an integer exponent e (reduced mod K first).
__device__ __forceinline__ double2 root(int64_t e, int64_t K) {
  e %= K;
  if (e < 0) e += K;
  double sn, cs;
  sincospi(2.0 * static_cast<double>(e) / static_cast<double>(K), &sn, &cs);
  return make_double2(cs, sn);
}

// In-register DFT of length R (kernel w_R^{+rp}); R in {2, 3, 4, 5, 7}.
template <int R>
__device__ __forceinline__ void small_dft(double2 (&v)[R]) {
  if (R == 2) {
    const double2 a = v[0], b = v[1];
    v[0] = make_double2(a.x + b.x, a.y + b.y);
    v[1] = make_double2(a.x - b.x, a.y - b.y);
  } else if (R == 4) {
    const double2 a = v[0], b = v[1], c = v[2], d = v[3];
    const double2 s0 = make_double2(a.x + c.x, a.y + c.y), d0 = make_double2(a.x - c.x, a.y - c.y);
    const double2 s1 = make_double2(b.x + d.x, b.y + d.y), d1 = make_double2(b.x - d.x, b.y - d.y);
    v[0] = make_double2(s0.x + s1.x, s0.y + s1.y);
    v[2] = make_double2(s0.x - s1.x, s0.y - s1.y);
    v[1] = make_double2(d0.x - d1.y, d0.y + d1.x);  // d0 + i d1
    v[3] = make_double2(d0.x + d1.y, d0.y - d1.x);  // d0 - i d1
  } else {
    // cos / sin (2 pi t / R), t < R, as literals (R = 3, 5, 7)
    constexpr double C3[3] = {1.0, -0.5, -0.5};
    constexpr double S3[3] = {0.0, 0.86602540378443864676, -0.86602540378443864676};
    constexpr double C5[5] = {1.0, 0.30901699437494742410, -0.80901699437494742410, -0.80901699437494742410,
                              0.30901699437494742410};
    constexpr double S5[5] = {0.0, 0.95105651629515357212, 0.58778525229247312917, -0.58778525229247312917,
                              -0.95105651629515357212};
    constexpr double C7[7] = {1.0, 0.62348980185873353053, -0.22252093395631440429, -0.90096886790241912624,
                              -0.90096886790241912624, -0.22252093395631440429, 0.62348980185873353053};
    constexpr double S7[7] = {0.0, 0.78183148246802980871, 0.97492791218182360702, 0.43388373911755812048,
                              -0.43388373911755812048, -0.97492791218182360702, -0.78183148246802980871};
    double2 out[R];
#pragma unroll
    for (int p = 0; p < R; ++p) {
      double2 acc = v[0];
#pragma unroll
      for (int r = 1; r < R; ++r) {
        const int t = (r * p) % R;
        const double cs = R == 3 ? C3[t] : R == 5 ? C5[t] : C7[t];
        const double sn = R == 3 ? S3[t] : R == 5 ? S5[t] : S7[t];
        acc.x = fma(v[r].x, cs, fma(-v[r].y, sn, acc.x));
        acc.y = fma(v[r].x, sn, fma(v[r].y, cs, acc.y));
      }
      out[p] = acc;
    }
#pragma unroll
    for (int p = 0; p < R; ++p) v[p] = out[p];
  }
}

// One Stockham pass over G sequences (each Q long, stored back to back).
template <int R>
__device__ void stockham_pass(const double2* __restrict__ in, double2* __restrict__ out, const double2* tw, int Q,
                              int Ns, int G) {
  const int nb = Q / R;
  const int tstep = Q / (Ns * R);  // w_{Ns R}^{r k} = w_Q^{r k tstep}
  for (int e = threadIdx.x; e < G * nb; e += GT) {
    const int gq = e / nb, j = e - gq * nb;
    const double2* src = in + gq * Q;
    double2* dst = out + gq * Q;
    const int k = j % Ns;
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = src[j + r * nb];
    if (Ns > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) v[r] = cmul(v[r], tw[r * k * tstep]);  // r k tstep < Q
    }
    small_dft<R>(v);
    const int base = (j / Ns) * Ns * R + k;
#pragma unroll
    for (int r = 0; r < R; ++r) dst[base + r * Ns] = v[r];
  }
}

template <int KIND, int NCIN, int NQ, int GG>  // KIND 0 srft, 1 srdct; GG sequences per batch
__global__ void __launch_bounds__(GT, 2) srtt_gen_kernel(GenParams p) {  // two CTAs (16 warps) per SM
  extern __shared__ __align__(16) double2 smem[];
  const int Q = static_cast<int>(p.Q);
  double2* buf0 = smem;               // [G][Q]
  double2* buf1 = smem + GG * Q;      // [G][Q]
  double2* tw = smem + 2 * GG * Q;    // w_Q^t
  double2* pre = tw + Q;              // srdct: w_{4Q}^{k2}
  for (int t = threadIdx.x; t < Q; t += GT) {
    tw[t] = root(t, Q);
    if (KIND == 1) pre[t] = root(t, 4 * static_cast<int64_t>(Q));
  }
  const int64_t c = blockIdx.y;
  const int64_t k1lo = static_cast<int64_t>(blockIdx.x) * p.per;
  const int64_t k1hi = p.P2 < k1lo + p.per ? p.P2 : k1lo + p.per;
  const double* Acol = p.A + c * p.lda * NCIN;
  double2 acc[NQ], step[NQ];
  int64_t fr[NQ];
#pragma unroll
  for (int t = 0; t < NQ; ++t) {
    acc[t] = make_double2(0.0, 0.0);
    const int i = threadIdx.x + GT * t;
    fr[t] = i < p.ns ? p.freq[i] : 0;
    step[t] = root(fr[t], p.N);  // w_N^{f}: the outer twiddle's step from k1 to k1 + 1
  }
  __syncthreads();
  __shared__ double2 seqtw[GG];  // srdct: w_{4N}^{k1} of the batch's sequences
  for (int64_t kb = k1lo; kb < k1hi; kb += GG) {
    const int G = static_cast<int>(k1hi - kb < GG ? k1hi - kb : GG);
    if (KIND == 1 && threadIdx.x < G) seqtw[threadIdx.x] = root(kb + threadIdx.x, 4 * p.N);
    if (KIND == 1) __syncthreads();
    // ---- stage u[k1 + P2 k2] for the G sequences (G consecutive local rows per k2)
    for (int e = threadIdx.x; e < GG * Q; e += GT) {
      const int k2 = e / GG, gq = e % GG;
      if (gq >= G) continue;
      const int64_t l = kb + gq + p.P2 * k2;
      const int64_t j = p.g + p.P * l;  // global row
      const bool pos = (__ldg(p.sign_bits + (j >> 5)) >> (j & 31)) & 1u;
      double2 x;
      if (NCIN == 1) {
        x = make_double2(__ldg(Acol + l), 0.0);
      } else {
        x = make_double2(__ldg(Acol + 2 * l), __ldg(Acol + 2 * l + 1));
      }
      if (!pos) x = make_double2(-x.x, -x.y);
      if (KIND == 1) {  // c_j x w_{4N}^{l},  w_{4N}^{k1 + P2 k2} = w_{4N}^{k1} w_{4Q}^{k2}
        const double cw = j == 0 ? p.c0 : p.c1;
        x = cmul(make_double2(cw * x.x, cw * x.y), cmul(seqtw[gq], pre[k2]));
      }
      buf0[gq * Q + k2] = x;
    }
    __syncthreads();
    // ---- Stockham passes (self-sorting), ping-pong between the two buffers
    double2* in = buf0;
    double2* out = buf1;
    int Ns = 1;
    for (int ps = 0; ps < p.npass; ++ps) {
      const int R = p.radix[ps];
      if (R == 4) stockham_pass<4>(in, out, tw, Q, Ns, G);
      else if (R == 2) stockham_pass<2>(in, out, tw, Q, Ns, G);
      else if (R == 3) stockham_pass<3>(in, out, tw, Q, Ns, G);
      else if (R == 5) stockham_pass<5>(in, out, tw, Q, Ns, G);
      else stockham_pass<7>(in, out, tw, Q, Ns, G);
      __syncthreads();
      double2* t = in;
      in = out;
      out = t;
      Ns *= R;
    }
    // ---- sampled outer stage: acc_i += w_N^{f_i k1} F_{k1}[f_i mod Q]
#pragma unroll
    for (int t = 0; t < NQ; ++t) {
      const int i = threadIdx.x + GT * t;
      if (i < p.ns) {
        const int fq = static_cast<int>(fr[t] % Q);
        // exact anchor w_N^{f kb} once per batch, then G - 1 steps (f kb < N P2 <= 2^62 for N < 2^31)
        double2 w = root(static_cast<int64_t>((static_cast<uint64_t>(fr[t]) * static_cast<uint64_t>(kb)) %
                                              static_cast<uint64_t>(p.N)), p.N);
        for (int gq = 0; gq < G; ++gq) {
          const double2 f = in[gq * Q + fq];
          acc[t].x = fma(w.x, f.x, fma(-w.y, f.y, acc[t].x));
          acc[t].y = fma(w.x, f.y, fma(w.y, f.x, acc[t].y));
          w = cmul(w, step[t]);
        }
      }
    }
    __syncthreads();
  }
  double2* out = p.part + (static_cast<int64_t>(blockIdx.x) * p.n + c) * (NQ * GT);
#pragma unroll
  for (int t = 0; t < NQ; ++t) out[threadIdx.x + GT * t] = acc[t];
}

// SA[i, c] = scale * post_i * (conj_i ? conj : id)(sum over ranges) -- srft complex, srdct real part.
template <int KIND>
__global__ void srtt_gen_reduce(const double2* __restrict__ part, int64_t rstride, int64_t cstride, int64_t ranges,
                                int64_t n, int ns, int base, const double2* __restrict__ post,
                                const uint8_t* __restrict__ conj, double scale, double* __restrict__ SA, int64_t ldsa) {
  const int64_t total = n * ns;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t c = e / ns;
    const int i = static_cast<int>(e - c * ns);
    double2 z = make_double2(0.0, 0.0);
    for (int64_t r = 0; r < ranges; ++r) {
      const double2 v = part[r * rstride + c * cstride + i];
      z.x += v.x;
      z.y += v.y;
    }
    if (conj[base + i]) z.y = -z.y;
    z = cmul(post[base + i], z);
    const int64_t row = base + i;
    if (KIND == 0) {
      SA[2 * (row + c * ldsa)] = scale * z.x;
      SA[2 * (row + c * ldsa) + 1] = scale * z.y;
    } else {
      SA[row + c * ldsa] = scale * z.x;
    }
  }
}

// Largest 2,3,5,7-smooth divisor of N not above QMAX, and its radix sequence (4s first).
int64_t plan_q(int64_t N, std::vector<int>& radix) {
  // Q <= 512 by default (NSK_GEN_QMAX up to 1024): four sequences per batch and two CTAs per SM fit; at
  // m = 10^6 this measured 5.75 ms against 6.57 ms for Q = 1000 (a longer outer sum, better occupancy)
  int64_t qmax = 512;
  if (const char* e = std::getenv("NSK_GEN_QMAX")) {
    const int64_t v = std::atoll(e);
    if (v >= 2 && v <= QMAX) qmax = v;  // QMAX = 1024: the shared-memory bound
  }
  int64_t best = 1;
  for (int64_t a = 1; a <= qmax; a *= 2)
    for (int64_t b = a; b <= qmax; b *= 3)
      for (int64_t c5 = b; c5 <= qmax; c5 *= 5)
        for (int64_t d = c5; d <= qmax; d *= 7)
          if (N % d == 0 && d > best) best = d;
  radix.clear();
  int64_t t = best;
  while (t % 4 == 0) {
    radix.push_back(4);
    t /= 4;
  }
  for (int r : {2, 3, 5, 7})
    while (t % r == 0) {
      radix.push_back(r);
      t /= r;
    }
  return best;
}

template <int KIND, int NCIN, int GG>
int launch_gen_g(int nq, const GenParams& p, dim3 grid, size_t smem, cudaStream_t st) {
  auto go = [&](auto kern) -> int {
    NSK_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    KernelTimer tm(st, "srtt_gen_kernel");
    kern<<<grid, GT, smem, st>>>(p);
    tm.stop();
    count_launch();
    NSK_CUDA_OK(cudaGetLastError());
    return OK;
  };
  if (nq <= 1) return go(srtt_gen_kernel<KIND, NCIN, 1, GG>);
  if (nq <= 2) return go(srtt_gen_kernel<KIND, NCIN, 2, GG>);
  if (nq <= 4) return go(srtt_gen_kernel<KIND, NCIN, 4, GG>);
  return go(srtt_gen_kernel<KIND, NCIN, 8, GG>);
}

template <int KIND, int NCIN>
int launch_gen(int gg, int nq, const GenParams& p, dim3 grid, size_t smem, cudaStream_t st) {
  return gg == 4 ? launch_gen_g<KIND, NCIN, 4>(nq, p, grid, smem, st) : launch_gen_g<KIND, NCIN, 2>(nq, p, grid, smem, st);
}

}  // namespace

// Partial layout part[r * rstride + c * cstride + i] (ranges r, columns c, slots i < ns of the chunk at
// `base`): SA[base + i, c] = scale * Re / complex (post_i * conj_i(sum_r)).  kind 0 srft (complex SA), 1 srdct.
int srtt_post_reduce(int kind, const double2* part, int64_t rstride, int64_t cstride, int64_t ranges, int64_t n,
                     int ns, int base, const double2* post, const uint8_t* conj, double scale, double* SA,
                     int64_t ldsa, cudaStream_t st) {
  int64_t blocks = (n * ns + 255) / 256;
  if (blocks > 8L * sm_count()) blocks = 8L * sm_count();
  if (blocks < 1) return OK;
  if (kind == 0)
    srtt_gen_reduce<0><<<static_cast<unsigned>(blocks), 256, 0, st>>>(part, rstride, cstride, ranges, n, ns, base,
                                                                     post, conj, scale, SA, ldsa);
  else
    srtt_gen_reduce<1><<<static_cast<unsigned>(blocks), 256, 0, st>>>(part, rstride, cstride, ranges, n, ns, base,
                                                                     post, conj, scale, SA, ldsa);
  count_launch();
  NSK_CUDA_OK(cudaGetLastError());
  return OK;
}

// Slot tables of a cyclic shard (first global row g, local length N = m / P; g = 0, N = m unsharded):
// DFT frequency in [0, N), conjugation flag and shard twiddle per output row (header comment).
int shard_slot_tables(const Operator& op, int64_t g, int64_t N, Scratch& tab, int64_t** dfreq, double2** dpost,
                      uint8_t** dconj, cudaStream_t st) {
  const int kind = op.kind == SRFT ? 0 : 1;
  const int64_t m = op.m, s = op.s;
  // slot tables: frequency, conjugation, shard twiddle
  std::vector<int64_t> freq(static_cast<size_t>(s));
  std::vector<uint8_t> conj(static_cast<size_t>(s), 0);
  std::vector<double2> post(static_cast<size_t>(s));
  for (int64_t i = 0; i < s; ++i) {
    const int64_t a = op.idx[static_cast<size_t>(i)];
    int64_t e, K;
    if (kind == 0) {
      freq[i] = a % N;
      e = static_cast<int64_t>((static_cast<unsigned __int128>(a) * static_cast<uint64_t>(g)) % static_cast<uint64_t>(m));
      K = m;
    } else {
      const int64_t q = (2 * a + 1) % (4 * N), b = (q - 1) / 2;
      if (b % 2 == 0) {
        freq[i] = b / 2;
      } else {
        freq[i] = ((-(b - 1) / 2 - 1) % N + N) % N;
        conj[i] = 1;
      }
      K = 4 * m;
      e = static_cast<int64_t>((static_cast<unsigned __int128>(2 * a + 1) * static_cast<uint64_t>(g)) %
                               static_cast<uint64_t>(K));
    }
    const double ang = 2.0 * M_PI * static_cast<double>(e) / static_cast<double>(K);
    post[i] = make_double2(std::cos(ang), std::sin(ang));
  }
  const size_t bytes = sizeof(int64_t) * s + sizeof(double2) * s + s;
  NSK_CUDA_OK(tab.alloc(bytes, st));
  *dpost = tab.as<double2>();  // 16-byte entries first: every table stays aligned for any s
  *dfreq = reinterpret_cast<int64_t*>(*dpost + s);
  *dconj = reinterpret_cast<uint8_t*>(*dfreq + s);
  NSK_CUDA_OK(cudaMemcpyAsync(*dfreq, freq.data(), sizeof(int64_t) * s, cudaMemcpyHostToDevice, st));
  NSK_CUDA_OK(cudaMemcpyAsync(*dpost, post.data(), sizeof(double2) * s, cudaMemcpyHostToDevice, st));
  NSK_CUDA_OK(cudaMemcpyAsync(*dconj, conj.data(), s, cudaMemcpyHostToDevice, st));
  return OK;
}

// Whether the engine takes this row map: the full matrix, or a cyclic shard
// (row0 = g < P = rstep, P divides m, mloc = m / P).
bool srtt_general_eligible(const Operator& op, const RowMap& rows) {
  if (rows.rstep < 1 || rows.row0 < 0 || rows.row0 >= rows.rstep) return false;
  if (op.m % rows.rstep != 0 || rows.mloc != op.m / rows.rstep) return false;
  return true;
}

int srtt_general_apply(const Operator& op, int ncomp, const RowMap& rows, int64_t n, const double* A, int64_t lda,
                       double* SA, int64_t ldsa, cudaStream_t st) {
  if (!srtt_general_eligible(op, rows) || n == 0 || rows.mloc >= (int64_t(1) << 31)) return NOTAPPLICABLE;
  const int kind = op.kind == SRFT ? 0 : 1;
  if (kind == 1 && ncomp != 1) return NOTAPPLICABLE;
  const DeviceTables* tb = op.tables();
  if (!tb || !tb->sign_bits) return ECUDA;
  const int64_t m = op.m, s = op.s, P = rows.rstep, g = rows.row0, N = rows.mloc;
  std::vector<int> radix;
  const int64_t Q = plan_q(N, radix);
  if (static_cast<int>(radix.size()) > MAXPASS) return NOTAPPLICABLE;
  const int64_t P2 = N / Q;
  Scratch dtab;
  int64_t* dfreq = nullptr;
  double2* dpost = nullptr;
  uint8_t* dconj = nullptr;
  if (int rc = shard_slot_tables(op, g, N, dtab, &dfreq, &dpost, &dconj, st)) return rc;
  // two CTAs per SM: (2 GG + 2) Q complex doubles <= ~113 KiB
  const int GG = (2 * GG_MAX + 2) * Q * 16 <= 113 * 1024 ? GG_MAX : 2;
  // CTA ranges of k1: about four CTAs per SM over all columns, each range a multiple of G
  const int64_t target = 4L * sm_count();
  int64_t ranges = std::max<int64_t>(1, std::min<int64_t>((target + n - 1) / n, (P2 + GG - 1) / GG));
  int64_t per = (P2 + ranges - 1) / ranges;
  per = (per + GG - 1) / GG * GG;
  ranges = (P2 + per - 1) / per;
  if (ranges > 65535) return NOTAPPLICABLE;
  const size_t smem = sizeof(double2) * (2 * GG * Q + 2 * Q);
  const double scale = kind == 0 ? 1.0 / std::sqrt(static_cast<double>(s))
                                 : std::sqrt(static_cast<double>(m) / static_cast<double>(s));
  for (int64_t base = 0; base < s; base += 8 * GT) {
    const int ns = static_cast<int>(std::min<int64_t>(s - base, 8 * GT));
    const int nq = (ns + GT - 1) / GT;
    const int NQ = nq <= 1 ? 1 : nq <= 2 ? 2 : nq <= 4 ? 4 : 8;
    Scratch part;
    NSK_CUDA_OK(part.alloc(sizeof(double2) * ranges * n * NQ * GT, st));
    GenParams p{};
    p.A = A;
    p.lda = lda;
    p.n = n;
    p.N = N;
    p.Q = Q;
    p.P2 = P2;
    p.per = per;
    p.ranges = ranges;
    p.g = g;
    p.P = P;
    p.c0 = std::sqrt(1.0 / static_cast<double>(m));
    p.c1 = std::sqrt(2.0 / static_cast<double>(m));
    p.sign_bits = tb->sign_bits;
    p.freq = dfreq + base;
    p.ns = ns;
    p.npass = static_cast<int>(radix.size());
    for (size_t r = 0; r < radix.size(); ++r) p.radix[r] = radix[r];
    p.part = part.as<double2>();
    const dim3 grid(static_cast<unsigned>(ranges), static_cast<unsigned>(n));
    int rc = kind == 0 ? (ncomp == 1 ? launch_gen<0, 1>(GG, nq, p, grid, smem, st)
                                     : launch_gen<0, 2>(GG, nq, p, grid, smem, st))
                       : launch_gen<1, 1>(GG, nq, p, grid, smem, st);
    if (rc != OK) return rc;
    if (int rc2 = srtt_post_reduce(kind, part.as<double2>(), n * NQ * GT, NQ * GT, ranges, n, ns, static_cast<int>(base),
                                   dpost, dconj, scale, SA, ldsa, st))
      return rc2;
  }
  return OK;
}

}  // namespace nsk
