// nccl_shard.cpp -- the multi-GPU entry points of the C ABI (one process per GPU).
//
// SA = sum_g S[:, rows_g] A_g: every rank sketches the rows it
// holds -- the operator regenerates S for the GLOBAL row indices, so nothing
// moves before the reduce -- and one ncclAllReduce (sum, FP64) of the s x n
// partials over NVLink / NVSwitch gives every rank the same SA, bit for bit
// (NCCL's reduction order is fixed for a fixed communicator).  solve_k then runs
// the on-device SVD on every rank (identical inputs give identical W and
// sigma, so no broadcast is needed).  Reference call sites this serves: solve_k
// (nullspace.cpp:23-32) and apply (sketch.cpp:184-232) with A row-sharded.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2: the one torch loaded,
// the system's, or NSK_NCCL_LIB), so the library has no link-time NCCL
// dependency and single-GPU users never load it.  Communicators are the
// caller's ncclComm_t; nsk_nccl_unique_id / nsk_nccl_comm_init wrap
// ncclGetUniqueId / ncclCommInitRank for callers without one.
#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include <nccl.h>

#include "../../include/nullsketch_b200.h"
#include "nsk_internal.hpp"

namespace nsk {
int dispatch_apply_c(const Operator& op, int ncomp, const RowMap& rows, int64_t n, const double* A, int64_t lda,
                     double* SA, int64_t ldsa, cudaStream_t st);
int host_sketch_shard(const Operator& op, int nc_in, int64_t row0, int64_t mloc, int64_t n, const void* A,
                      int64_t lda, double* SA, cudaStream_t st);
}

namespace {

struct NcclApi {
  bool ok = false;
  std::string err;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  decltype(&ncclGetUniqueId) unique_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclCommCount) count = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {std::getenv("NSK_NCCL_LIB"), "libnccl.so.2", "libnccl.so",
#ifdef NSK_NCCL_PATH
                           NSK_NCCL_PATH,
#endif
                           nullptr};
    void* h = nullptr;
    for (const char* nm : names) {
      if (!nm) continue;
      h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) {
      api.err = "NCCL not found (libnccl.so.2; set NSK_NCCL_LIB)";
      return;
    }
    api.all_reduce = reinterpret_cast<decltype(&ncclAllReduce)>(dlsym(h, "ncclAllReduce"));
    api.error_string = reinterpret_cast<decltype(&ncclGetErrorString)>(dlsym(h, "ncclGetErrorString"));
    api.unique_id = reinterpret_cast<decltype(&ncclGetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    api.init_rank = reinterpret_cast<decltype(&ncclCommInitRank)>(dlsym(h, "ncclCommInitRank"));
    api.destroy = reinterpret_cast<decltype(&ncclCommDestroy)>(dlsym(h, "ncclCommDestroy"));
    api.count = reinterpret_cast<decltype(&ncclCommCount)>(dlsym(h, "ncclCommCount"));
    api.ok = api.all_reduce && api.error_string && api.unique_id && api.init_rank && api.destroy && api.count;
    if (!api.ok) api.err = "NCCL library lacks a required symbol";
  });
  return api;
}

int nccl_fail(ncclResult_t r, const char* what) {
  return nsk::fail(nsk::ECUDA, std::string("NCCL error in ") + what + ": " + nccl().error_string(r));
}

int check_comm(void* comm) {
  if (!comm) return nsk::fail(nsk::EINVAL_, "null NCCL communicator");
  if (!nccl().ok) return nsk::fail(nsk::ECUDA, nccl().err);
  return nsk::OK;
}

int out_nc(const nsk::Operator& op, int scalar) { return op.kind == nsk::SRFT || scalar == NSK_COMPLEX ? 2 : 1; }

// Partial of this rank's rows into a contiguous s x n buffer, then the all-reduce in place.
int sharded_sketch(const nsk::Operator& op, int scalar, int64_t row0, int64_t rstep, int64_t mloc, int64_t n,
                   const void* A, int64_t lda, double* buf, void* comm, cudaStream_t st) {
  if (scalar != NSK_REAL && scalar != NSK_COMPLEX) return nsk::fail(nsk::EINVAL_, "unknown scalar kind");
  if (n < 0 || mloc < 0) return nsk::fail(nsk::EINVAL_, "sketch apply: negative dimension");
  if (rstep < 1 || row0 < 0) return nsk::fail(nsk::EINVAL_, "apply_shard: bad row map");
  if (mloc > 0 && row0 + rstep * (mloc - 1) >= op.m)
    return nsk::fail(nsk::ERANGE_, "apply_shard: rows beyond the operator's m");
  if (mloc > 0 && n > 0 && lda < mloc) return nsk::fail(nsk::EINVAL_, "sketch apply: lda < rows");
  if (op.appended > 0) return nsk::fail(nsk::EINVAL_, "apply_shard: operators with row updates are not sharded");
  nsk::RowMap rows{row0, rstep, mloc};
  if (mloc > 0) {
    if (int rc = nsk::dispatch_apply_c(op, scalar == NSK_COMPLEX ? 2 : 1, rows, n, static_cast<const double*>(A), lda,
                                       buf, op.s, st))
      return rc;
  } else {
    NSK_CUDA_OK(cudaMemsetAsync(buf, 0, sizeof(double) * op.s * n * out_nc(op, scalar), st));
  }
  const size_t count = static_cast<size_t>(op.s) * static_cast<size_t>(n) * out_nc(op, scalar);
  if (ncclResult_t r = nccl().all_reduce(buf, buf, count, ncclDouble, ncclSum, static_cast<ncclComm_t>(comm), st))
    return nccl_fail(r, "ncclAllReduce");
  return nsk::OK;
}

}  // namespace

extern "C" {

int nsk_nccl_unique_id(char* id_out) {
  if (!id_out) return nsk::fail(nsk::EINVAL_, "null unique-id buffer");
  if (!nccl().ok) return nsk::fail(nsk::ECUDA, nccl().err);
  ncclUniqueId id;
  if (ncclResult_t r = nccl().unique_id(&id)) return nccl_fail(r, "ncclGetUniqueId");
  static_assert(sizeof(ncclUniqueId) == NSK_NCCL_UNIQUE_ID_BYTES, "unique id size");
  std::memcpy(id_out, &id, sizeof(id));
  return nsk::OK;
}

int nsk_nccl_comm_init(int nranks, const char* id, int rank, void** comm_out) {
  if (!id || !comm_out || nranks < 1 || rank < 0 || rank >= nranks)
    return nsk::fail(nsk::EINVAL_, "nccl_comm_init: bad arguments");
  if (!nccl().ok) return nsk::fail(nsk::ECUDA, nccl().err);
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  if (ncclResult_t r = nccl().init_rank(&c, nranks, uid, rank)) return nccl_fail(r, "ncclCommInitRank");
  *comm_out = c;
  return nsk::OK;
}

int nsk_nccl_comm_destroy(void* comm) {
  if (!comm) return nsk::OK;
  if (!nccl().ok) return nsk::fail(nsk::ECUDA, nccl().err);
  if (ncclResult_t r = nccl().destroy(static_cast<ncclComm_t>(comm))) return nccl_fail(r, "ncclCommDestroy");
  return nsk::OK;
}

int nsk_apply_allreduce(const nsk_operator* h, int scalar, int64_t row0, int64_t rstep, int64_t mloc, int64_t n,
                        const void* A_local, int64_t lda, void* SA, int64_t ldsa, void* comm, void* stream) {
  if (!h) return nsk::fail(nsk::EINVAL_, "null sketch operator");
  if (int rc = check_comm(comm)) return rc;
  const nsk::Operator& op = *reinterpret_cast<const nsk::Operator*>(h);
  if (ldsa < op.s) return nsk::fail(nsk::EINVAL_, "sketch apply: ldsa < s");
  if (n > 0 && !SA) return nsk::fail(nsk::EINVAL_, "sketch apply: null SA");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n == 0) return nsk::OK;
  const int nc = out_nc(op, scalar);
  if (ldsa == op.s) return sharded_sketch(op, scalar, row0, rstep, mloc, n, A_local, lda, static_cast<double*>(SA), comm, st);
  nsk::Scratch buf;
  NSK_CUDA_OK(buf.alloc(sizeof(double) * op.s * n * nc, st));
  if (int rc = sharded_sketch(op, scalar, row0, rstep, mloc, n, A_local, lda, buf.as<double>(), comm, st)) return rc;
  NSK_CUDA_OK(cudaMemcpy2DAsync(SA, sizeof(double) * nc * ldsa, buf.p, sizeof(double) * nc * op.s,
                                sizeof(double) * nc * op.s, n, cudaMemcpyDeviceToDevice, st));
  return nsk::OK;
}

int nsk_solve_k_sharded(const nsk_operator* h, int scalar, int64_t row0, int64_t rstep, int64_t mloc, int64_t n,
                        const void* A_local, int64_t lda, int64_t k, void* W, int64_t ldw, double* sigma, void* comm,
                        void* stream) {
  if (!h) return nsk::fail(nsk::EINVAL_, "null sketch operator");
  if (int rc = check_comm(comm)) return rc;
  const nsk::Operator& op = *reinterpret_cast<const nsk::Operator*>(h);
  if (n < 1) return nsk::fail(nsk::EINVAL_, "nullspace: matrix has no columns");
  if (k < 0 || k >= n)
    return nsk::fail(nsk::EINVAL_, "nullspace: k must satisfy 0 <= k < n, got k = " + std::to_string(k) +
                                       ", n = " + std::to_string(n));
  if (op.s < n)
    return nsk::fail(nsk::EINVAL_, "nullspace: sketch size s = " + std::to_string(op.s) +
                                       " is smaller than n = " + std::to_string(n));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nc = out_nc(op, scalar);
  nsk::Scratch sa;
  NSK_CUDA_OK(sa.alloc(sizeof(double) * op.s * n * nc, st));
  if (int rc = sharded_sketch(op, scalar, row0, rstep, mloc, n, A_local, lda, sa.as<double>(), comm, st)) return rc;
  return nsk::jacobi_trailing(nc, op.s, n, sa.as<double>(), op.s, k, static_cast<double*>(W), ldw, sigma, st);
}

int nsk_solve_k_sharded_host(const nsk_operator* h, int scalar, int64_t row0, int64_t rstep, int64_t mloc, int64_t n,
                             const void* A_local, int64_t lda, int64_t k, void* W, int64_t ldw, double* sigma,
                             void* comm) {
  if (!h) return nsk::fail(nsk::EINVAL_, "null sketch operator");
  if (int rc = check_comm(comm)) return rc;
  const nsk::Operator& op = *reinterpret_cast<const nsk::Operator*>(h);
  if (scalar != NSK_REAL && scalar != NSK_COMPLEX) return nsk::fail(nsk::EINVAL_, "unknown scalar kind");
  if (n < 1 || k < 0 || k >= n) return nsk::fail(nsk::EINVAL_, "nullspace: k must satisfy 0 <= k < n");
  if (mloc > 0 && (lda < mloc || !A_local)) return nsk::fail(nsk::EINVAL_, "sketch apply: lda < rows");
  if ((k > 0 && (!W || ldw < n)) || !sigma) return nsk::fail(nsk::EINVAL_, "solve_k: bad outputs");
  cudaStream_t st = nsk::thread_stream();  // this thread's compute stream (h2d_rows copies on another)
  if (!st) return nsk::fail(nsk::ECUDA, "solve_k_sharded_host: no compute stream");
  const int nc_in = scalar == NSK_COMPLEX ? 2 : 1, nc = out_nc(op, scalar);
  nsk::Scratch a, w, sg;
  NSK_CUDA_OK(w.alloc(sizeof(double) * nc * n * (k > 0 ? k : 1), st));
  NSK_CUDA_OK(sg.alloc(sizeof(double) * n, st));
  if (rstep == 1 && mloc > 0 && op.appended == 0) {
    // contiguous shard: the single-GPU host pipeline (row chunks sketched as they land, the
    // operator's tables for this shard's rows built during the copy), then reduce + SVD
    if (row0 < 0 || row0 + mloc > op.m) return nsk::fail(nsk::ERANGE_, "apply_shard: rows beyond the operator's m");
    if (op.s < n)
      return nsk::fail(nsk::EINVAL_, "nullspace: sketch size s = " + std::to_string(op.s) +
                                         " is smaller than n = " + std::to_string(n));
    if (scalar == NSK_COMPLEX && (op.kind == nsk::SRDCT || op.kind == nsk::SRHT || op.kind == nsk::COUNTSKETCH))
      return nsk::fail(nsk::EINVAL_, "sketch apply: complex input needs a gaussian or srft operator");
    nsk::Scratch sa;
    NSK_CUDA_OK(sa.alloc(sizeof(double) * op.s * n * nc, st));
    if (int rc = nsk::host_sketch_shard(op, nc_in, row0, mloc, n, A_local, lda, sa.as<double>(), st)) return rc;
    const size_t count = static_cast<size_t>(op.s) * static_cast<size_t>(n) * nc;
    if (ncclResult_t r = nccl().all_reduce(sa.p, sa.p, count, ncclDouble, ncclSum, static_cast<ncclComm_t>(comm), st))
      return nccl_fail(r, "ncclAllReduce");
    if (int rc = nsk::jacobi_trailing(nc, op.s, n, sa.as<double>(), op.s, k, static_cast<double*>(w.p), n,
                                      sg.as<double>(), st))
      return rc;
  } else {
    NSK_CUDA_OK(a.alloc(sizeof(double) * nc_in * (mloc > 0 ? mloc : 1) * n, st));
    if (int rc = nsk::h2d_rows(A_local, mloc, n, lda, sizeof(double) * nc_in, a.p, mloc, st, nullptr)) return rc;
    if (int rc = nsk_solve_k_sharded(h, scalar, row0, rstep, mloc, n, a.p, mloc > 0 ? mloc : 1, k, w.p, n,
                                     sg.as<double>(), comm, st))
      return rc;
  }
  if (k > 0)
    NSK_CUDA_OK(cudaMemcpy2DAsync(W, sizeof(double) * nc * ldw, w.p, sizeof(double) * nc * n, sizeof(double) * nc * n,
                                  k, cudaMemcpyDeviceToHost, st));
  NSK_CUDA_OK(cudaMemcpyAsync(sigma, sg.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  NSK_CUDA_OK(cudaStreamSynchronize(st));
  return nsk::OK;
}

}  // extern "C"
