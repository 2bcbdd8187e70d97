// cluster_jacobi.cu -- block one-sided Jacobi on [R; I] inside ONE
// thread-block cluster, the working matrix resident in distributed shared
// memory.
//
// Same rotations and stopping rule as the kernels in jacobi_svd.cu
// (reference: from_sketch_svd, nullspace.cpp:10-19, BDCSVD, kernels.cpp:14-22);
// what changes is where the columns live and how rounds synchronise.  A
// cooperative grid barrier costs several microseconds and the global-memory
// block kernel pays one per block round plus an L2 round trip of the block
// pair; measured on this part: barrier.cluster ~0.45k cycles, DSMEM load
// ~0.24k cycles, __syncthreads ~0.05k.  So:
//
//   * a cluster of C <= 16 CTAs holds the npad = 2 C b columns of [R; I]
//     (zero columns pad n; they never rotate) as 2C blocks of b columns, two
//     blocks per CTA ("top" and "bottom" slot) plus two inbox buffers;
//   * inner sweep: in the first outer round of a sweep the CTA pairs all its
//     2b local columns (round-robin, 2b - 1 rounds of b pairs), afterwards
//     only the b^2 pairs across its two blocks (b rounds): every pair once per
//     sweep; one warp per pair, shuffle reductions, one __syncthreads a round;
//   * outer round: blocks advance by the circle method (top[0] fixed, top row
//     right, bottom row left, wrap at both ends); a block crossing a CTA
//     boundary is copied straight into the neighbour's inbox with
//     st.shared::cluster, moves inside a CTA are renames; one cluster barrier
//     per outer round plus a split arrive/wait that keeps the neighbours'
//     renames ahead of the next copy.  2C - 1 outer rounds per sweep.
//
// Deterministic: fixed reduction orders, no atomics on data.
#include <cooperative_groups.h>

#include <cstdlib>

#include "jacobi_pair.cuh"
#include "nsk_internal.hpp"

namespace cg = cooperative_groups;

namespace nsk {
namespace {

constexpr int CJ_MAX_SWEEPS = 40;

struct CJParams {
  double* X;  // 2n x n (x NC), ld 2n: rows [0, n) = R part, [n, 2n) = V part
  int n;
  int b;      // columns per block
  double tol;
  int* counter;  // [CJ_MAX_SWEEPS] rotations per sweep (CTA 0 writes), [CJ_MAX_SWEEPS] = sweeps
};

__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() {
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__device__ __forceinline__ void round_robin(int N, int r, int i, int& p, int& q) {  // pair i of round r, N even
  const int M = N - 1;
  if (i == 0) {
    p = M;
    q = r;
  } else {
    p = (r + i) % M;
    q = (r - i + M) % M;
  }
  if (p > q) {
    const int t = p;
    p = q;
    q = t;
  }
}

template <int NC>
__global__ void __launch_bounds__(512) cluster_jacobi_kernel(CJParams p) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double buf[];  // [4 block buffers][b][colsz]
  __shared__ int slotbuf[2];                     // block buffer of the top / bottom slot
  __shared__ int inbox[2];                       // [0] filled by the left CTA, [1] by the right CTA
  __shared__ int blockid[4];                     // block held by each buffer
  __shared__ int rotated;                        // any rotation in this CTA and sweep
  __shared__ int sweep_rot[16];                  // CTA 0: per-CTA flags of the finished sweep
  __shared__ unsigned char ptab[31 * 16][2];     // inner round-robin pairs (2b <= 32)
  const int c = static_cast<int>(cluster.block_rank()), C = static_cast<int>(cluster.num_blocks());
  const int n = p.n, ld = 2 * n, colsz = ld * NC, b = p.b, twob = 2 * b;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nthr = blockDim.x;
  const int blksz = b * colsz;
  const double tol2 = p.tol * p.tol;

  for (int e = threadIdx.x; e < (twob - 1) * b; e += nthr) {
    int lp, lq;
    round_robin(twob, e / b, e % b, lp, lq);
    ptab[e][0] = static_cast<unsigned char>(lp);
    ptab[e][1] = static_cast<unsigned char>(lq);
  }
  if (threadIdx.x == 0) {  // initial: CTA c holds blocks 2c (top) and 2c + 1 (bottom)
    slotbuf[0] = 0;
    slotbuf[1] = 1;
    inbox[0] = 2;
    inbox[1] = 3;
    blockid[0] = 2 * c;
    blockid[1] = 2 * c + 1;
    blockid[2] = blockid[3] = -1;
    rotated = 0;
  }
  __syncthreads();
  for (int s = 0; s < 2; ++s) {
    const int64_t g0 = static_cast<int64_t>(2 * c + s) * b;  // first global column of the block
    double* dst = buf + s * blksz;
    for (int e = threadIdx.x; e < blksz; e += nthr) {
      const int64_t col = g0 + e / colsz;
      dst[e] = col < n ? __ldcg(p.X + g0 * colsz + e) : 0.0;
    }
  }
  __syncthreads();
  cluster.sync();
  cluster_arrive();  // opens the split barrier closed before the first copy

  int sweep = 0;
  const int outer = 2 * C - 1;
  for (; sweep < CJ_MAX_SWEEPS; ++sweep) {
    for (int r = 0; r < outer; ++r) {
      // ---- inner sweep over the 2b local columns
      // First outer round of a sweep: every block meets its partner for the
      // first time and its own columns are still to be paired -- full
      // round-robin over the 2b columns.  Later outer rounds: only the b^2
      // cross pairs (b rounds of b disjoint pairs).  A sweep thus visits every
      // column pair exactly once.
      double* const cols[2] = {buf + slotbuf[0] * blksz, buf + slotbuf[1] * blksz};
      const int inner = r == 0 ? twob - 1 : b;
      for (int t = 0; t < inner; ++t) {
        if (warp < b) {
          const int lp = r == 0 ? ptab[t * b + warp][0] : warp;
          const int lq = r == 0 ? ptab[t * b + warp][1] : b + (warp + t) % b;
          double* xp = cols[lp / b] + (lp % b) * colsz;
          double* xq = cols[lq / b] + (lq % b) * colsz;
          if (jacobi_pair<NC>(xp, xq, n, ld, lane, tol2) && lane == 0) rotated = 1;
        }
        __syncthreads();
      }
      if (C == 1) continue;  // a single block pair: nothing moves
      // ---- outer move (circle method on blocks): copy the blocks crossing a CTA boundary
      cluster_wait();  // neighbours renamed after the previous move
      if (c + 1 < C) {  // right: CTA 0 sends its bottom block (-> top[1]), the others their top block
        const int sb = slotbuf[c == 0 ? 1 : 0];
        const int db = cluster.map_shared_rank(inbox, c + 1)[0];
        const double2* s2 = reinterpret_cast<const double2*>(buf + sb * blksz);
        double2* d2 = reinterpret_cast<double2*>(cluster.map_shared_rank(buf, c + 1) + db * blksz);
        for (int e = threadIdx.x; e < blksz / 2; e += nthr) d2[e] = s2[e];
        if (threadIdx.x == 0) cluster.map_shared_rank(blockid, c + 1)[db] = blockid[sb];
      }
      if (c > 0) {  // left: bottom block -> bottom slot of CTA c - 1
        const int sb = slotbuf[1];
        const int db = cluster.map_shared_rank(inbox, c - 1)[1];
        const double2* s2 = reinterpret_cast<const double2*>(buf + sb * blksz);
        double2* d2 = reinterpret_cast<double2*>(cluster.map_shared_rank(buf, c - 1) + db * blksz);
        for (int e = threadIdx.x; e < blksz / 2; e += nthr) d2[e] = s2[e];
        if (threadIdx.x == 0) cluster.map_shared_rank(blockid, c - 1)[db] = blockid[sb];
      }
      cluster_arrive();
      cluster_wait();  // every copy of this move has landed
      if (threadIdx.x == 0) {  // rename; the freed buffers become the inboxes
        const int ot = slotbuf[0], ob = slotbuf[1], i0 = inbox[0], i1 = inbox[1];
        if (c == 0) {  // top fixed, bottom from the right; freed: old bottom (sent), unused inbox[0]
          slotbuf[1] = i1;
          inbox[0] = ob;
          inbox[1] = i0;
        } else if (c == C - 1) {  // top from the left, old top -> bottom; freed: old bottom, inbox[1]
          slotbuf[0] = i0;
          slotbuf[1] = ot;
          inbox[0] = ob;
          inbox[1] = i1;
        } else {  // both from the neighbours; freed: both old blocks (sent)
          slotbuf[0] = i0;
          slotbuf[1] = i1;
          inbox[0] = ot;
          inbox[1] = ob;
        }
      }
      __syncthreads();
      cluster_arrive();  // split barrier: closed by the next move's copy phase
    }
    // ---- sweep end: did any CTA rotate?
    if (threadIdx.x == 0) cluster.map_shared_rank(sweep_rot, 0)[c] = rotated;
    if (C > 1) cluster_wait();  // close the pending split barrier
    cluster.sync();             // flags visible
    int tot = 0;
    const int* f0 = cluster.map_shared_rank(sweep_rot, 0);
    for (int k = 0; k < C; ++k) tot += f0[k];
    if (c == 0 && threadIdx.x == 0) p.counter[sweep] = tot;
    __syncthreads();
    if (threadIdx.x == 0) rotated = 0;
    cluster.sync();  // everyone has read the flags before they are overwritten
    if (C > 1) cluster_arrive();
    if (tot == 0) break;
  }
  if (C > 1) cluster_wait();
  // ---- write back the two live blocks by their global block index
  for (int s = 0; s < 2; ++s) {
    const int bi = blockid[slotbuf[s]];
    const int64_t g0 = static_cast<int64_t>(bi) * b;
    const double* src = buf + slotbuf[s] * blksz;
    for (int e = threadIdx.x; e < blksz; e += nthr)
      if (g0 + e / colsz < n) p.X[g0 * colsz + e] = src[e];
  }
  if (c == 0 && threadIdx.x == 0) p.counter[CJ_MAX_SWEEPS] = sweep;
}

}  // namespace

// Returns OK after running, or NOTAPPLICABLE when [R; I] does not fit one
// cluster (the caller then uses the global-memory block kernel).
int cluster_jacobi(int ncomp, double* X, int64_t n, double tol, int* counter, cudaStream_t st) {
  if (std::getenv("NSK_SVD_NOCLUSTER")) return NOTAPPLICABLE;
  if (n < 2 || n > 4096) return NOTAPPLICABLE;
  int C = static_cast<int>((n + 3) / 4);  // >= 2 columns per block
  if (C > 16) C = 16;
  if (C < 1) C = 1;
  const int b = static_cast<int>((n + 2 * C - 1) / (2 * C));
  if (b > 16) return NOTAPPLICABLE;
  const size_t smem = sizeof(double) * static_cast<size_t>(4 * b) * 2 * n * ncomp;
  if (smem > 220 * 1024) return NOTAPPLICABLE;
  const int threads = 32 * (b < 1 ? 1 : b);
  CJParams prm{X, static_cast<int>(n), b, tol, counter};
  auto kern = ncomp == 1 ? cluster_jacobi_kernel<1> : cluster_jacobi_kernel<2>;
  NSK_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  if (C > 8) NSK_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(C));
  cfg.blockDim = dim3(static_cast<unsigned>(threads));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(C);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) != cudaSuccess || ncl < 1) {
    cudaGetLastError();
    return NOTAPPLICABLE;
  }
  NSK_CUDA_OK(cudaLaunchKernelEx(&cfg, kern, prm));
  count_launch();
  return OK;
}

}  // namespace nsk
