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

#include <cstdio>
#include <cstdlib>

#include "jacobi_pair.cuh"
#include <map>
#include <mutex>
#include <tuple>
#include "nsk_internal.hpp"

namespace cg = cooperative_groups;

namespace nsk {
namespace {

constexpr int CJ_MAX_SWEEPS = 80;  // == MAX_SWEEPS (jacobi_svd.cu): one counter layout

struct CJParams {
  double* X;  // 2n x n (x NC), ld 2n: rows [0, n) = R part, [n, 2n) = V part
  int n;
  int b;      // columns per block
  double tol;
  int* counter;  // [CJ_MAX_SWEEPS] rotations per sweep (CTA 0 writes), [CJ_MAX_SWEEPS] = sweeps
  int early;     // stop after a sweep of small rotations only (NSK_SVD_FULLCHECK=1: 0)
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

// Shared-memory bookkeeping of the block circle (one copy per CTA).
struct Circle {
  int slotbuf[2];                  // block buffer of the top / bottom slot
  int inbox[2];                    // [0] filled by the left CTA, [1] by the right CTA (nb = 3: [0] = free buffer)
  int nb;                          // block buffers per CTA: 4 (two inboxes) or 3 (one free buffer, two-phase moves)
  int sentA;                       // nb = 3: buffer sent right in phase A of the current move
  int blockid[4];                  // block held by each buffer
  int rotated;                     // rotations in this CTA and sweep
  int big;                         // a rotation with |cos| > sqrt(eps) / 2 in this CTA and sweep
  int sweep_big[16];               // CTA 0: per-CTA big flags of the finished sweep
  int sweep_rot[16];               // CTA 0: per-CTA rotation counts of the finished sweep
  unsigned char ptab[31 * 16][2];  // inner round-robin pairs (2b <= 32)
};

// Initial state: CTA c holds blocks 2c (top, buffer 0) and 2c + 1 (bottom, buffer 1).
__device__ void circle_init(Circle& cc, int c, int b, int nb = 4) {
  const int twob = 2 * b;
  for (int e = threadIdx.x; e < (twob - 1) * b; e += blockDim.x) {
    int lp, lq;
    round_robin(twob, e / b, e % b, lp, lq);
    cc.ptab[e][0] = static_cast<unsigned char>(lp);
    cc.ptab[e][1] = static_cast<unsigned char>(lq);
  }
  if (threadIdx.x == 0) {
    cc.slotbuf[0] = 0;
    cc.slotbuf[1] = 1;
    cc.inbox[0] = 2;
    cc.inbox[1] = nb == 4 ? 3 : -1;
    cc.nb = nb;
    cc.sentA = -1;
    cc.blockid[0] = 2 * c;
    cc.blockid[1] = 2 * c + 1;
    cc.blockid[2] = cc.blockid[3] = -1;
    cc.rotated = 0;
    cc.big = 0;
  }
}

// Block one-sided Jacobi sweeps over the 2 C b resident columns (colsz doubles
// each, inner products over rows [0, n), rotations over rows [0, ld)) until a
// sweep rotates nothing.  Entered and left with the cluster synchronised.
// Returns the number of sweeps (CTA 0 also records per-sweep counts).
template <int NC, int RPL>
__device__ int circle_sweeps(cg::cluster_group& cluster, double* buf, Circle& cc, int n, int ld, int b, double tol2,
                             int* counter, bool early, unsigned long long* prof = nullptr) {
  long long t_inner = 0, t_move = 0, t0 = 0, t1 = 0;
  const int c = static_cast<int>(cluster.block_rank()), C = static_cast<int>(cluster.num_blocks());
  // blksz: buffer stride, rounded up to an even count so every block buffer is 16-byte aligned for
  // the double2 block moves (b * n is odd for odd n and b in the real svd kernel)
  const int colsz = ld * NC, twob = 2 * b, blksz = (b * colsz + 1) & ~1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nthr = blockDim.x;
  if (C > 1) cluster_arrive();  // opens the split barrier closed before the first copy
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
      if (prof) t0 = clock64();
      double* const cols[2] = {buf + cc.slotbuf[0] * blksz, buf + cc.slotbuf[1] * blksz};
      // complex with 16 rows per lane would exceed the register budget of a
      // 512-thread CTA: that case keeps the shared-memory step
      constexpr bool REG = !(NC == 2 && RPL > 8);
      if (r == 0 || !REG) {
        const int inner = r == 0 ? twob - 1 : b;
        for (int t = 0; t < inner; ++t) {
          if (warp < b) {
            const int lp = r == 0 ? cc.ptab[t * b + warp][0] : warp;
            const int lq = r == 0 ? cc.ptab[t * b + warp][1] : b + (warp + t) % b;
            double* xp = cols[lp / b] + (lp % b) * colsz;
            double* xq = cols[lq / b] + (lq % b) * colsz;
            const int rot = REG ? jacobi_pair_reg<NC, RPL>(xp, xq, n, ld, lane, tol2)
                                : jacobi_pair<NC>(xp, xq, n, ld, lane, tol2);
            if (rot && lane == 0) atomicAdd(&cc.rotated, 1);
            if (rot == 2 && lane == 0) cc.big = 1;
          }
          __syncthreads();
        }
      } else if (warp < b) {
        // cross rounds: warp w keeps top column w in registers for all b
        // rounds; only the bottom columns pass through shared memory
        double* xp = cols[0] + warp * colsz;
        double pr[RPL], pim[RPL];
        load_col<NC, RPL>(xp, n, lane, pr, pim);
        int nrot = 0, big = 0;
        for (int t = 0; t < b; ++t) {
          double* xq = cols[1] + ((warp + t) % b) * colsz;
          const int rot = jacobi_step_preg<NC, RPL>(pr, pim, xp, xq, n, ld, lane, tol2);
          nrot += rot ? 1 : 0;
          big |= rot == 2;
          __syncthreads();
        }
        if (nrot) {
          store_col<NC, RPL>(xp, n, lane, pr, pim);
          if (lane == 0) atomicAdd(&cc.rotated, nrot);
          if (big && lane == 0) cc.big = 1;
        }
        __syncwarp();
        __syncthreads();  // p columns visible before the move copies them
      } else {
        for (int t = 0; t <= b; ++t) __syncthreads();  // idle warps keep the barrier count
      }
      if (prof) {
        t1 = clock64();
        t_inner += t1 - t0;
      }
      if (C == 1) continue;  // a single block pair: nothing moves
      // ---- outer move (circle method on blocks): copy the blocks crossing a CTA boundary
      cluster_wait();  // neighbours renamed after the previous move
      if (cc.nb == 3) {
        // Three buffers per CTA (two live blocks + one free): the move runs in
        // two phases.  A: every CTA but the last sends its right-going block
        // (CTA 0: bottom, others: top) into the right neighbour's free buffer.
        // B: every CTA but the first sends its bottom block into the buffer its
        // left neighbour emptied in phase A.
        if (c + 1 < C) {
          const int sb = cc.slotbuf[c == 0 ? 1 : 0];
          Circle* rc = cluster.map_shared_rank(&cc, c + 1);
          const int db = rc->inbox[0];
          const double2* s2 = reinterpret_cast<const double2*>(buf + sb * blksz);
          double2* d2 = reinterpret_cast<double2*>(cluster.map_shared_rank(buf, c + 1) + db * blksz);
          for (int e = threadIdx.x; e < blksz / 2; e += nthr) d2[e] = s2[e];
          if (threadIdx.x == 0) {
            rc->blockid[db] = cc.blockid[sb];
            cc.sentA = sb;
          }
        }
        cluster_arrive();
        cluster_wait();  // phase A landed, sentA published
        if (c > 0) {
          const int sb = cc.slotbuf[1];
          Circle* lc = cluster.map_shared_rank(&cc, c - 1);
          const int db = lc->sentA;
          const double2* s2 = reinterpret_cast<const double2*>(buf + sb * blksz);
          double2* d2 = reinterpret_cast<double2*>(cluster.map_shared_rank(buf, c - 1) + db * blksz);
          for (int e = threadIdx.x; e < blksz / 2; e += nthr) d2[e] = s2[e];
          if (threadIdx.x == 0) lc->blockid[db] = cc.blockid[sb];
        }
        cluster_arrive();
        cluster_wait();  // phase B landed
        if (threadIdx.x == 0) {
          const int ot = cc.slotbuf[0], ob = cc.slotbuf[1], fr = cc.inbox[0];
          if (c == 0) {
            // bottom sent in A, refilled from the right in B (same buffer): nothing renames
          } else if (c == C - 1) {  // top from the left (free buffer), old top -> bottom, old bottom sent
            cc.slotbuf[0] = fr;
            cc.slotbuf[1] = ot;
            cc.inbox[0] = ob;
          } else {  // top from the left (free buffer), bottom from the right (into the old top), old bottom sent
            cc.slotbuf[0] = fr;
            cc.slotbuf[1] = ot;
            cc.inbox[0] = ob;
          }
        }
      } else {
      if (c + 1 < C) {  // right: CTA 0 sends its bottom block (-> top[1]), the others their top block
        const int sb = cc.slotbuf[c == 0 ? 1 : 0];
        Circle* rc = cluster.map_shared_rank(&cc, c + 1);
        const int db = rc->inbox[0];
        const double2* s2 = reinterpret_cast<const double2*>(buf + sb * blksz);
        double2* d2 = reinterpret_cast<double2*>(cluster.map_shared_rank(buf, c + 1) + db * blksz);
        for (int e = threadIdx.x; e < blksz / 2; e += nthr) d2[e] = s2[e];
        if (threadIdx.x == 0) rc->blockid[db] = cc.blockid[sb];
      }
      if (c > 0) {  // left: bottom block -> bottom slot of CTA c - 1
        const int sb = cc.slotbuf[1];
        Circle* lc = cluster.map_shared_rank(&cc, c - 1);
        const int db = lc->inbox[1];
        const double2* s2 = reinterpret_cast<const double2*>(buf + sb * blksz);
        double2* d2 = reinterpret_cast<double2*>(cluster.map_shared_rank(buf, c - 1) + db * blksz);
        for (int e = threadIdx.x; e < blksz / 2; e += nthr) d2[e] = s2[e];
        if (threadIdx.x == 0) lc->blockid[db] = cc.blockid[sb];
      }
      cluster_arrive();
      cluster_wait();  // every copy of this move has landed
      if (threadIdx.x == 0) {  // rename; the freed buffers become the inboxes
        const int ot = cc.slotbuf[0], ob = cc.slotbuf[1], i0 = cc.inbox[0], i1 = cc.inbox[1];
        if (c == 0) {  // top fixed, bottom from the right; freed: old bottom (sent), unused inbox[0]
          cc.slotbuf[1] = i1;
          cc.inbox[0] = ob;
          cc.inbox[1] = i0;
        } else if (c == C - 1) {  // top from the left, old top -> bottom; freed: old bottom, inbox[1]
          cc.slotbuf[0] = i0;
          cc.slotbuf[1] = ot;
          cc.inbox[0] = ob;
          cc.inbox[1] = i1;
        } else {  // both from the neighbours; freed: both old blocks (sent)
          cc.slotbuf[0] = i0;
          cc.slotbuf[1] = i1;
          cc.inbox[0] = ot;
          cc.inbox[1] = ob;
        }
      }
      }
      __syncthreads();
      cluster_arrive();  // split barrier: closed by the next move's copy phase
      if (prof) t_move += clock64() - t1;
    }
    // ---- sweep end: did any CTA rotate, and was any rotation big?
    if (threadIdx.x == 0) {
      cluster.map_shared_rank(&cc, 0)->sweep_rot[c] = cc.rotated;
      cluster.map_shared_rank(&cc, 0)->sweep_big[c] = cc.big;
    }
    if (C > 1) cluster_wait();  // close the pending split barrier
    cluster.sync();             // flags visible
    int tot = 0, big = 0;
    const Circle* c0 = cluster.map_shared_rank(&cc, 0);
    for (int k = 0; k < C; ++k) {
      tot += c0->sweep_rot[k];
      big |= c0->sweep_big[k];
    }
    if (c == 0 && threadIdx.x == 0) counter[sweep] = tot;
    __syncthreads();
    if (threadIdx.x == 0) cc.rotated = cc.big = 0;
    cluster.sync();  // everyone has read the flags before they are overwritten
    if (C > 1) cluster_arrive();
    if (tot == 0) break;
    // Every rotation of this sweep was small (|cos| <= sqrt(eps)/2): by quadratic convergence the
    // next sweep would rotate nothing (it would only re-check), so stop here (JACOBI_BIG2).
    if (early && !big) {
      ++sweep;
      break;
    }
  }
  if (C > 1) cluster_wait();
  if (c == 0 && threadIdx.x == 0) {
    counter[CJ_MAX_SWEEPS] = sweep;
    if (prof) {
      prof[0] = static_cast<unsigned long long>(t_inner);
      prof[1] = static_cast<unsigned long long>(t_move);
    }
  }
  return sweep;
}

template <int NC, int RPL>
__global__ void __launch_bounds__(512) cluster_jacobi_kernel(CJParams p) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double buf[];  // [4 block buffers][b][colsz]
  __shared__ Circle cc;
  const int c = static_cast<int>(cluster.block_rank());
  const int n = p.n, ld = 2 * n, colsz = ld * NC, b = p.b;
  const int nthr = blockDim.x;
  const int blksz = b * colsz;

  circle_init(cc, c, b);
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
  circle_sweeps<NC, RPL>(cluster, buf, cc, n, ld, b, p.tol * p.tol, p.counter, p.early != 0);
  // ---- write back the two live blocks by their global block index
  for (int s = 0; s < 2; ++s) {
    const int bi = cc.blockid[cc.slotbuf[s]];
    const int64_t g0 = static_cast<int64_t>(bi) * b;
    const double* src = buf + cc.slotbuf[s] * blksz;
    for (int e = threadIdx.x; e < blksz; e += nthr)
      if (g0 + e / colsz < n) p.X[g0 * colsz + e] = src[e];
  }
}

// ---------------------------------------------------------------- preconditioned path
// Drmac-Veselic preconditioning (the structure of LAPACK dgejsv): the
// right singular vectors of R come from one-sided Jacobi on the TRANSPOSE of
// a column-pivoted R:
//
//   R P = Q1 R'           (QRCP of the n x n triangle, Householder, pivot = the
//                          largest remaining column norm, ties -> lowest index)
//   R'^H J = W = What Sigma   (one-sided Jacobi on X = R'^H, no V accumulation)
//   R = (Q1 J) Sigma (P What)^H,   so V_R = P What.
//
// Row pivoting makes R'^H strongly graded column-wise, and one-sided Jacobi
// on such a matrix converges in about half the sweeps of Jacobi on R for the
// graded spectra of the sketch-and-solve problems (numpy model: 16 -> 7
// sweeps at n = 64, 17 -> 8 at n = 128, unchanged on random spectra), with
// half the columns' length (no identity block).  Everything stays in the
// cluster's shared memory:
//
//   * QRCP without swaps: slot g (= input column g) carries lg[g], the step
//     at which it was chosen; each step every CTA proposes its largest
//     remaining norm to every CTA (remote stores), a cluster barrier, every
//     CTA picks the same winner, the owner forms the reflector and pushes it
//     to every CTA, a second barrier, every CTA applies it to its remaining
//     columns and recomputes their trailing norms exactly (no downdating);
//   * transpose: slot g gathers row lg[g] of R' from the owners of the later
//     pivots (DSMEM loads) into the spare buffers;
//   * the same block circle sweeps as cluster_jacobi_kernel, ld = n;
//   * output in the [R; I] layout norms_kernel / order_kernel read: rows
//     [0, n) = W column, rows n + phys[r] = What[r] / ||W column||.
// A W column of norm ~0 (an exactly singular R) leaves What undefined: the
// kernel raises *degenerate and the caller reruns the unpreconditioned path.
struct CSParams {
  double* X;  // in: rows [0, n) = R (ld 2n); out: [W; P What] in the same layout
  int n;
  int b;
  double tol;
  int* counter;
  int* degenerate;
  unsigned long long* stamps;  // debug: phase timestamps (ns) of CTA 0, or null
  int early;                   // as CJParams::early
};

__device__ __forceinline__ void stamp(unsigned long long* st, int i) {
  if (st && threadIdx.x == 0 && cg::this_cluster().block_rank() == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    st[i] = t;
  }
}

// Each warp's best remaining slot -> every CTA's candidate buffer.
__device__ __forceinline__ void push_candidate(cg::cluster_group& cluster, double (*cand_val)[256],
                                               int (*cand_idx)[256], int bufi, int entry, int C, int lane,
                                               double v, int idx) {
  if (lane < C) {
    cluster.map_shared_rank(&cand_val[bufi][0], lane)[entry] = v;
    cluster.map_shared_rank(&cand_idx[bufi][0], lane)[entry] = idx;
  }
}

// RPL = rows per lane of the register-resident QRCP step (n <= 32 RPL);
// NB = block buffers per CTA (4, or 3 when four do not fit: two-phase moves).
// Up to 16 warps (b <= 16) per CTA; the complex RPL = 8 kernel holds 162 registers and is capped at
// 12 warps (cluster_svd_max_b).
template <int NC, int RPL, int NB>
__global__ void __launch_bounds__(NC == 2 && RPL == 8 ? 384 : 512, 1) cluster_svd_kernel(CSParams p) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double buf[];  // [NB block buffers][b][n * NC], phys[n]
  __shared__ Circle cc;
  __shared__ double cand_val[2][256];  // [step parity][CTA * b + warp]: remaining squared norm
  __shared__ int cand_idx[2][256];     //                                 and its global slot
  __shared__ int lg[32];               // pivot step of each slot: -1 not yet, -2 padding
  const int c = static_cast<int>(cluster.block_rank()), C = static_cast<int>(cluster.num_blocks());
  const int n = p.n, colsz = n * NC, b = p.b, twob = 2 * b, blksz = (b * colsz + 1) & ~1;  // even stride
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nthr = blockDim.x;
  int* phys = reinterpret_cast<int*>(buf + NB * blksz);
  const int gbase = c * twob;  // global slot of local slot 0
  auto slot = [&](int li) { return buf + (li / b) * blksz + (li % b) * colsz; };
  auto stage = [&](int g) { return p.X + static_cast<int64_t>(g) * 2 * colsz + colsz; };  // V rows of column g

  stamp(p.stamps, 0);
  circle_init(cc, c, b, NB);
  for (int e = threadIdx.x; e < twob * colsz; e += nthr) {  // R columns (rows [0, n) of X)
    const int li = e / colsz, g = gbase + li;
    slot(li)[e % colsz] = g < n ? __ldcg(p.X + static_cast<int64_t>(g) * 2 * colsz + e % colsz) : 0.0;
  }
  __syncthreads();

  // ---- 1. QRCP of R (n steps, one cluster barrier each).  Warp w owns slots
  // w and w + b; their rows j + lane + 32 k live in registers during a step.
  // Every warp reduces the same candidate list, so all agree on the pivot
  // without a broadcast.  Each warp also stages the column it proposes in
  // global memory (the unused V rows of X), and every warp reads the winner
  // from there (L2): DSMEM serves only ~20 B/cycle per SM, far too little
  // for 16 x b warps reading one owner's column every step.  A pivoted
  // column is never proposed again, so its staged copy is stable while read.  The reflector needs only x_j and ||x[j:]||^2 (the
  // candidate value, exact):  beta = -phase(x_j) nrm,  v = x[j:] - beta e_1,
  // tau = 2 / ||v||^2 = 1 / (nrm (|x_j| + nrm)).  The pivot column keeps v
  // below the diagonal (never read again); its diagonal beta is written after
  // the next barrier, when no CTA reads the column any more.
  const int lis[2] = {warp, warp + b};
  bool act[2];
  double nr[2];
  for (int s2 = 0; s2 < 2; ++s2) {
    const double* x = slot(lis[s2]);
    double a = 0.0;
    for (int r = lane; r < colsz; r += 32) a = fma(x[r], x[r], a);
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    act[s2] = gbase + lis[s2] < n;
    nr[s2] = a;
    if (lane == 0) lg[lis[s2]] = act[s2] ? -1 : -2;
  }
  auto best_of_mine = [&](double& v, int& idx) {
    v = -1.0;
    idx = 0x7fffffff;
    for (int s2 = 0; s2 < 2; ++s2)
      if (act[s2]) {
        const double u = nr[s2] >= 0.0 ? nr[s2] : INFINITY;  // NaN: pick it, the NaN reaches sigma
        if (u > v) {
          v = u;
          idx = gbase + lis[s2];
        }
      }
  };
  {
    double v;
    int idx;
    best_of_mine(v, idx);
    if (idx < n) {
      const double* x = slot(idx - gbase);
      double* sg = stage(idx);
      for (int r = lane; r < colsz; r += 32) sg[r] = x[r];
    }
    push_candidate(cluster, cand_val, cand_idx, 0, c * b + warp, C, lane, v, idx);
  }
  int pend_li = -1;
  double pend_r = 0.0, pend_i = 0.0;
  const int ncand = C * b;
  cluster.sync();
  for (int j = 0; j < n; ++j) {
    if (pend_li >= 0 && lane == 0) {  // diagonal of the previous pivot
      double* x = slot(pend_li);
      x[(j - 1) * NC] = pend_r;
      if (NC == 2) x[(j - 1) * NC + 1] = pend_i;
    }
    pend_li = -1;
    // pivot: largest remaining norm, ties -> lowest slot
    double bv = -2.0;
    int bi = 0x7fffffff;
    for (int e = lane; e < ncand; e += 32) {
      const double v = cand_val[j & 1][e];
      const int i = cand_idx[j & 1][e];
      if (v > bv || (v == bv && i < bi)) {
        bv = v;
        bi = i;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    const int pv = bi;
    if (warp == 0 && lane == 0) phys[j] = pv;
    // pivot column (staged in L2) and my two columns, rows j + lane + 32 k
    const double* pc = stage(pv);
    double vr[RPL], vi[RPL], xr[2][RPL], xi[2][RPL];
#pragma unroll
    for (int k = 0; k < RPL; ++k) {
      const int r = j + lane + 32 * k;
      vr[k] = vi[k] = 0.0;
      if (r < n) {
        if (NC == 1) {
          vr[k] = __ldcg(pc + r);
        } else {
          const double2 t = __ldcg(reinterpret_cast<const double2*>(pc) + r);
          vr[k] = t.x;
          vi[k] = t.y;
        }
      }
    }
#pragma unroll
    for (int s2 = 0; s2 < 2; ++s2) {
      const double* x = slot(lis[s2]);
      const bool live = act[s2] && gbase + lis[s2] != pv;
#pragma unroll
      for (int k = 0; k < RPL; ++k) {
        const int r = j + lane + 32 * k;
        xr[s2][k] = xi[s2][k] = 0.0;
        if (live && r < n) {
          if (NC == 1) {
            xr[s2][k] = x[r];
          } else {
            const double2 t = reinterpret_cast<const double2*>(x)[r];
            xr[s2][k] = t.x;
            xi[s2][k] = t.y;
          }
        }
      }
    }
    // reflector scalars (identical in every warp)
    const double xjr = __shfl_sync(0xffffffffu, vr[0], 0), xji = NC == 2 ? __shfl_sync(0xffffffffu, vi[0], 0) : 0.0;
    const double ax = NC == 2 ? hypot(xjr, xji) : fabs(xjr);
    const double nrm = sqrt(bv);
    const double phr = ax > 0.0 ? xjr / ax : 1.0, phi = ax > 0.0 ? xji / ax : 0.0;
    const double d = ax + nrm;
    const double tau = nrm > 0.0 ? 1.0 / (nrm * d) : 0.0;
    if (lane == 0) {
      vr[0] = phr * d;
      vi[0] = phi * d;
    }
#pragma unroll
    for (int s2 = 0; s2 < 2; ++s2)
      if (gbase + lis[s2] == pv) {
        act[s2] = false;
        pend_li = lis[s2];
        pend_r = -phr * nrm;
        pend_i = -phi * nrm;
        if (lane == 0) lg[lis[s2]] = j;
      }
    // w = tau v^H x for both columns
    double wr[2] = {0.0, 0.0}, wi[2] = {0.0, 0.0};
#pragma unroll
    for (int s2 = 0; s2 < 2; ++s2)
#pragma unroll
      for (int k = 0; k < RPL; ++k) {
        wr[s2] = fma(vr[k], xr[s2][k], wr[s2]);
        if (NC == 2) {
          wr[s2] = fma(vi[k], xi[s2][k], wr[s2]);
          wi[s2] = fma(vr[k], xi[s2][k], wi[s2]);
          wi[s2] = fma(-vi[k], xr[s2][k], wi[s2]);
        }
      }
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
      for (int s2 = 0; s2 < 2; ++s2) {
        wr[s2] += __shfl_xor_sync(0xffffffffu, wr[s2], o);
        if (NC == 2) wi[s2] += __shfl_xor_sync(0xffffffffu, wi[s2], o);
      }
    }
    // x -= v w, trailing norms over rows > j
    double a[2] = {0.0, 0.0};
#pragma unroll
    for (int s2 = 0; s2 < 2; ++s2) {
      const double tr = tau * wr[s2], ti = tau * wi[s2];
      double* x = slot(lis[s2]);
      const bool live = act[s2];
#pragma unroll
      for (int k = 0; k < RPL; ++k) {
        const int r = j + lane + 32 * k;
        const double yr = xr[s2][k] - (vr[k] * tr - vi[k] * ti);
        const double yi = NC == 2 ? xi[s2][k] - (vr[k] * ti + vi[k] * tr) : 0.0;
        xr[s2][k] = yr;
        xi[s2][k] = yi;
        if (live && r < n) {
          if (NC == 1) {
            x[r] = yr;
          } else {
            reinterpret_cast<double2*>(x)[r] = make_double2(yr, yi);
          }
          if (r > j) a[s2] = fma(yr, yr, fma(yi, yi, a[s2]));
        }
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      a[0] += __shfl_xor_sync(0xffffffffu, a[0], o);
      a[1] += __shfl_xor_sync(0xffffffffu, a[1], o);
    }
    nr[0] = a[0];
    nr[1] = a[1];
    {
      double v;
      int idx;
      best_of_mine(v, idx);
      if (idx < n) {  // stage the proposed column, rows > j
        double* sg = stage(idx);
#pragma unroll
        for (int s2 = 0; s2 < 2; ++s2)
          if (gbase + lis[s2] == idx) {
#pragma unroll
            for (int k = 0; k < RPL; ++k) {
              const int r = j + lane + 32 * k;
              if (r > j && r < n) {
                if (NC == 1)
                  sg[r] = xr[s2][k];
                else
                  reinterpret_cast<double2*>(sg)[r] = make_double2(xr[s2][k], xi[s2][k]);
              }
            }
          }
      }
      push_candidate(cluster, cand_val, cand_idx, (j + 1) & 1, c * b + warp, C, lane, v, idx);
    }
    cluster.sync();  // release: candidates (DSMEM) and staged columns (global) visible
  }
  if (pend_li >= 0 && lane == 0) {
    double* x = slot(pend_li);
    x[(n - 1) * NC] = pend_r;
    if (NC == 2) x[(n - 1) * NC + 1] = pend_i;
  }
  cluster.sync();  // R' complete in every CTA
  stamp(p.stamps, 1);

  // ---- 2. X = R'^H: R' goes out to the R rows of the global X (the V rows
  // held the pivot staging, no longer needed), then slot li gathers conj(row
  // lg[li] of R') from L2 into its own buffer -- no DSMEM reads, and the
  // slot buffers are reused in place (three buffers suffice).
  for (int e = threadIdx.x; e < twob * colsz; e += nthr) {
    const int li = e / colsz, g = gbase + li;
    if (g < n) p.X[static_cast<int64_t>(g) * 2 * colsz + e % colsz] = slot(li)[e % colsz];
  }
  cluster.sync();  // R' in global memory, visible to the whole cluster
  for (int e = threadIdx.x; e < twob * n; e += nthr) {
    const int li = e / n, r = e % n, i = lg[li];
    double vr = 0.0, vi = 0.0;
    if (i >= 0 && r >= i) {
      const double* src = p.X + static_cast<int64_t>(phys[r]) * 2 * colsz + i * NC;
      vr = __ldcg(src);
      if (NC == 2) vi = -__ldcg(src + 1);
    }
    double* y = slot(li) + r * NC;
    y[0] = vr;
    if (NC == 2) y[1] = vi;
  }
  __syncthreads();
  cluster.sync();

  // ---- 3. one-sided Jacobi on X (no V accumulation)
  stamp(p.stamps, 2);
  circle_sweeps<NC, RPL>(cluster, buf, cc, n, n, b, p.tol * p.tol, p.counter, p.early != 0,
                         p.stamps ? p.stamps + 4 : nullptr);
  stamp(p.stamps, 3);

  // ---- 4. [W; P What] in the [R; I] layout
  for (int s = 0; s < 2; ++s) {
    const int bi = cc.blockid[cc.slotbuf[s]];
    const double* src = buf + cc.slotbuf[s] * blksz;
    for (int jj = warp; jj < b; jj += nthr / 32) {
      const int g = bi * b + jj;
      if (g >= n) continue;
      const double* w = src + jj * colsz;
      double a = 0.0;
      for (int r = lane; r < colsz; r += 32) a = fma(w[r], w[r], a);
      for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      const double nw = sqrt(a);
      if (lane == 0 && !(nw > 1e-290) && nw == nw) atomicExch(p.degenerate, 1);
      const double inv = nw > 0.0 ? 1.0 / nw : 0.0;
      double* out = p.X + static_cast<int64_t>(g) * 2 * colsz;
      for (int r = lane; r < n; r += 32) {
        const int pr = phys[r];
        for (int q = 0; q < NC; ++q) {
          out[r * NC + q] = w[r * NC + q];
          out[(n + pr) * NC + q] = w[r * NC + q] * inv;
        }
      }
    }
  }
}

}  // namespace

// Function attributes once per (kernel, device) at the largest shared memory seen: re-setting them
// while another launch of the same kernel runs (the concurrent stages of jacobi_trailing_pair) is
// avoided.
template <class K>
int set_attrs_once(K kern, size_t smem, bool nonportable) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  size_t& have = done[std::make_pair(reinterpret_cast<const void*>(kern), dev)];
  if (have >= smem && have > 0) return OK;
  NSK_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  if (nonportable) NSK_CUDA_OK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  have = smem;
  return OK;
}

// cudaOccupancyMaxActiveClusters once per (kernel, device, shared memory, cluster size): the query
// is not needed per call, and the concurrent SVD stages (jacobi_trailing_pair) must not wait on it.
template <class K>
int max_clusters_cached(K kern, const cudaLaunchConfig_t& cfg) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, size_t, unsigned>, int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(reinterpret_cast<const void*>(kern), dev, cfg.dynamicSmemBytes, cfg.gridDim.x);
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
  }
  int ncl = 0;
  if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) != cudaSuccess) {
    cudaGetLastError();
    ncl = 0;
  }
  std::lock_guard<std::mutex> lock(mu);
  cache[key] = ncl;
  return ncl;
}

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
  CJParams prm{X, static_cast<int>(n), b, tol, counter, std::getenv("NSK_SVD_FULLCHECK") ? 0 : 1};
  const int rpl = n <= 128 ? 4 : n <= 256 ? 8 : 16;
  auto kern = ncomp == 1 ? (rpl == 4 ? cluster_jacobi_kernel<1, 4> : rpl == 8 ? cluster_jacobi_kernel<1, 8>
                                                                              : cluster_jacobi_kernel<1, 16>)
                         : (rpl == 4 ? cluster_jacobi_kernel<2, 4> : rpl == 8 ? cluster_jacobi_kernel<2, 8>
                                                                              : cluster_jacobi_kernel<2, 16>);
  if (int rc = set_attrs_once(kern, smem, C > 8)) return rc;
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
  const int ncl = max_clusters_cached(kern, cfg);
  if (ncl < 1) return NOTAPPLICABLE;
  NSK_CUDA_OK(cudaLaunchKernelEx(&cfg, kern, prm));
  count_launch();
  return OK;
}

// Preconditioned SVD of R (QRCP + Jacobi on R'^H) in one cluster.  Returns OK
// after launching, NOTAPPLICABLE when it does not fit (or NSK_SVD_NORT is
// set); *degenerate (device) is raised when the caller must rerun without it.
int cluster_svd_rt(int ncomp, double* X, int64_t n, double tol, int* counter, int* degenerate, cudaStream_t st) {
  if (std::getenv("NSK_SVD_NORT") || std::getenv("NSK_SVD_NOCLUSTER")) return NOTAPPLICABLE;
  if (n < 2 || n > 4096) return NOTAPPLICABLE;
  // Cluster width: a sweep is 2Cb - 1 pair rounds (npad = 2Cb padded columns) plus 2C - 1 block
  // moves.  A round costs more as b warps share one SM, a move (DSMEM copy + cluster barriers)
  // ~3.5-4.5k cycles; measured on B200 (tools/svd_small.py, cycle stamps): real rounds ~700 + 65 b
  // cycles, complex ~1270 + 100 b.  Pick the C in [Cmin, 16] with the smallest modelled sweep (n = 64:
  // C = 4, n = 100: 5, n = 256 and 512: 16).  NSK_SVD_C overrides (A/B).
  const int rpl_ = n <= 128 ? 4 : n <= 256 ? 8 : 16;
  const int bmax = ncomp == 2 && rpl_ == 8 ? 12 : 16;
  const double l0 = ncomp == 2 ? 1270.0 : 700.0, lb = ncomp == 2 ? 100.0 : 65.0, mv = ncomp == 2 ? 4200.0 : 3500.0;
  int C = 16;
  double best = 1e300;
  for (int c = static_cast<int>((n + 2 * bmax - 1) / (2 * bmax)); c <= 16; ++c) {
    const int bb = static_cast<int>((n + 2 * c - 1) / (2 * c));
    const double cost = (2.0 * c * bb - 1.0) * (l0 + lb * bb) + (2.0 * c - 1.0) * mv;
    if (cost < best) {
      best = cost;
      C = c;
    }
  }
  if (const char* e = std::getenv("NSK_SVD_C")) {
    const int v = std::atoi(e);
    if (v >= 1 && v <= 16) C = v;
  }
  if (C > 16) C = 16;
  int b = 0, nbuf = 4;
  size_t smem = 0;
  for (;; ++C) {  // narrower blocks (more CTAs) until the block buffers fit
    if (C > 16) return NOTAPPLICABLE;
    b = static_cast<int>((n + 2 * C - 1) / (2 * C));
    if (b > bmax) continue;
    // four block buffers when they fit, else three (two-phase block moves)
    const size_t bstride = (static_cast<size_t>(b) * n * ncomp + 1) & ~static_cast<size_t>(1);  // as blksz
    nbuf = 4;
    smem = sizeof(double) * 4 * bstride + sizeof(int) * n;
    if (smem > 200 * 1024) {
      nbuf = 3;
      smem = sizeof(double) * 3 * bstride + sizeof(int) * n;
    }
    if (smem <= 210 * 1024 && (nbuf == 4 || rpl_ == 16)) break;  // three-buffer kernels: RPL = 16 only
  }
  if (n > 512) return NOTAPPLICABLE;
  const int threads = 32 * b;
  const bool dbg = std::getenv("NSK_SVD_DEBUG") != nullptr;
  unsigned long long* stamps = nullptr;
  if (dbg) NSK_CUDA_OK(cudaMallocAsync(&stamps, 6 * sizeof(unsigned long long), st));
  CSParams prm{X, static_cast<int>(n), b, tol, counter, degenerate, stamps, std::getenv("NSK_SVD_FULLCHECK") ? 0 : 1};
  const int rpl = n <= 128 ? 4 : n <= 256 ? 8 : 16;
  // (three buffers are only needed for n > 256: b = 16, RPL = 16)
  auto kern = ncomp == 1
                  ? (rpl == 4 ? cluster_svd_kernel<1, 4, 4>
                              : rpl == 8 ? cluster_svd_kernel<1, 8, 4>
                                         : (nbuf == 4 ? cluster_svd_kernel<1, 16, 4> : cluster_svd_kernel<1, 16, 3>))
                  : (rpl == 4 ? cluster_svd_kernel<2, 4, 4>
                              : rpl == 8 ? cluster_svd_kernel<2, 8, 4>
                                         : (nbuf == 4 ? cluster_svd_kernel<2, 16, 4> : cluster_svd_kernel<2, 16, 3>));
  if (int rc = set_attrs_once(kern, smem, C > 8)) return rc;
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
  const int ncl = max_clusters_cached(kern, cfg);
  if (ncl < 1) return NOTAPPLICABLE;
  NSK_CUDA_OK(cudaLaunchKernelEx(&cfg, kern, prm));
  count_launch();
  if (dbg) {
    unsigned long long h[6];
    NSK_CUDA_OK(cudaMemcpyAsync(h, stamps, sizeof(h), cudaMemcpyDeviceToHost, st));
    NSK_CUDA_OK(cudaStreamSynchronize(st));
    std::fprintf(stderr,
                 "nsk svd_rt: n=%lld C=%d b=%d max clusters %d qrcp %.3f ms transpose %.3f ms sweeps %.3f ms "
                 "(cycles inner %llu move %llu; globaltimer %llu .. %llu us)\n",
                 static_cast<long long>(n), C, b, ncl, (h[1] - h[0]) * 1e-6, (h[2] - h[1]) * 1e-6,
                 (h[3] - h[2]) * 1e-6, h[4], h[5], h[0] / 1000 % 100000000ull, h[3] / 1000 % 100000000ull);
    NSK_CUDA_OK(cudaFreeAsync(stamps, st));
  }
  return OK;
}

}  // namespace nsk
