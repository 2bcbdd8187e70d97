// capi.cpp -- the extern "C" boundary (include/nullsketch_b200.h).
//
// Argument validation and error texts follow the reference
// (/root/reference/proj/src/sketch.cpp:103-107,184-188,219-221;
//  nullspace.cpp:10-53; kernels.cpp:54-57): std::invalid_argument becomes
// NSK_EINVAL, SvdConvergenceError NSK_ENOCONV, with nsk_last_error() holding
// the message.  No CPU fallback exists: every compute entry point launches
// the CUDA kernels of this library or fails.
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <algorithm>
#include <cstdlib>
#include <vector>
#include <chrono>
#include <future>

#include "../../include/nullsketch_b200.h"
#include "nsk_internal.hpp"

using nsk::Operator;

namespace nsk {
const char* last_error();
}

namespace {

inline Operator* OP(nsk_operator* h) { return reinterpret_cast<Operator*>(h); }
inline const Operator* OP(const nsk_operator* h) { return reinterpret_cast<const Operator*>(h); }
inline cudaStream_t ST(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int check_op(const nsk_operator* h) {
  if (!h) return nsk::fail(nsk::EINVAL_, "null sketch operator");
  return nsk::OK;
}

// Output scalar kind of apply(): srft -> complex, gaussian keeps the input kind,
// the rest are real-only (sketch.hpp:86-88).
int out_ncomp(const Operator& op, int in_ncomp) {
  if (op.kind == nsk::SRFT) return 2;
  return in_ncomp;
}

int validate_apply(const Operator& op, int scalar, int64_t m, int64_t n, const void* A, int64_t lda,
                   const void* SA, int64_t ldsa, bool shard) {
  if (scalar != NSK_REAL && scalar != NSK_COMPLEX) return nsk::fail(nsk::EINVAL_, "unknown scalar kind");
  if (!shard && m != op.m_eff())
    return nsk::fail(nsk::EINVAL_, "sketch apply: matrix has " + std::to_string(m) + " rows, operator expects " +
                                       std::to_string(op.m_eff()));
  if (n < 0 || m < 0) return nsk::fail(nsk::EINVAL_, "sketch apply: negative dimension");
  if (scalar == NSK_COMPLEX && op.kind == nsk::SRDCT)
    return nsk::fail(nsk::EINVAL_, "srdct sketch is defined for real matrices only");
  if (scalar == NSK_COMPLEX && op.kind == nsk::SRHT)
    return nsk::fail(nsk::EINVAL_, "srht sketch is defined for real matrices only");
  if (scalar == NSK_COMPLEX && op.kind == nsk::COUNTSKETCH)
    return nsk::fail(nsk::EINVAL_, "countsketch is defined for real matrices only");
  if (lda < (m > 1 ? m : 1)) return nsk::fail(nsk::EINVAL_, "sketch apply: lda < rows");
  if (ldsa < op.s) return nsk::fail(nsk::EINVAL_, "sketch apply: ldsa < s");
  if (n > 0 && m > 0 && !A) return nsk::fail(nsk::EINVAL_, "sketch apply: null A");
  if (n > 0 && !SA) return nsk::fail(nsk::EINVAL_, "sketch apply: null SA");
  return nsk::OK;
}

int dispatch_main(const Operator& op, int ncomp, const nsk::RowMap& rows, int64_t n, const double* A, int64_t lda,
                  double* SA, int64_t ldsa, cudaStream_t st) {
  switch (op.kind) {
    case nsk::GAUSSIAN: return nsk::gaussian_apply(op, ncomp, rows, n, A, lda, SA, ldsa, st);
    case nsk::SRFT:
    case nsk::SRDCT: return nsk::srtt_apply(op, ncomp, rows, n, A, lda, SA, ldsa, st);
    case nsk::SRHT: return nsk::srht_apply(op, rows, n, A, lda, SA, ldsa, st);
    case nsk::COUNTSKETCH: return nsk::countsketch_apply(op, rows, n, A, lda, SA, ldsa, st);
  }
  return nsk::fail(nsk::EINVAL_, "unknown sketch kind");
}

// Full apply of an operator with p appended rows (sketch.cpp:195-229): the first
// m rows go through the kind's kernel, the appended rows through the Gaussian
// kernel on stream (seed, 1) (appended column c = Gaussians #(c*s + i)), added in.
int dispatch_apply(const Operator& op, int ncomp, const nsk::RowMap& rows, int64_t n, const double* A, int64_t lda,
                   double* SA, int64_t ldsa, cudaStream_t st) {
  const bool full = rows.row0 == 0 && rows.rstep == 1 && rows.mloc == op.m_eff();
  if (op.appended == 0 || !full) {
    if (op.appended > 0) return nsk::fail(nsk::EINVAL_, "apply_shard: operators with row updates are not sharded");
    return dispatch_main(op, ncomp, rows, n, A, lda, SA, ldsa, st);
  }
  nsk::RowMap top{0, 1, op.m};
  if (int rc = dispatch_main(op, ncomp, top, n, A, lda, SA, ldsa, st)) return rc;
  const int nc_out = op.kind == nsk::SRFT ? 2 : ncomp;
  nsk::Scratch t;
  NSK_CUDA_OK(t.alloc(sizeof(double) * op.s * (n > 0 ? n : 1) * ncomp, st));
  nsk::RowMap app{0, 1, op.appended};
  const uint32_t* zmask = nullptr;
  if (int rc = op.zero_mask(&zmask)) return rc;
  if (int rc = nsk::gaussian_apply_key(op.key1, op.s, zmask, op.m, ncomp, app, n, A + op.m * ncomp, lda,
                                       t.as<double>(), op.s, st))
    return rc;
  return nsk::accumulate(SA, ldsa, nc_out, t.as<double>(), op.s, n, ncomp, st);
}

// S [A | B] into adjacent column blocks of SA (B: kb columns).  Gaussian: one pass, every G tile
// generated once for all n + kb columns (gaussian_apply_key2); the per-column kinds regenerate
// nothing across columns, so they run the two blocks one after the other.
int dispatch_main2(const Operator& op, int ncomp, const nsk::RowMap& rows, int64_t n, const double* A, int64_t lda,
                   int64_t kb, const double* B, int64_t ldb, double* SA, int64_t ldsa, cudaStream_t st) {
  if (kb > 0 && op.kind == nsk::GAUSSIAN) {
    const uint32_t* zmask = nullptr;
    if (int rc = op.zero_mask(&zmask)) return rc;
    return nsk::gaussian_apply_key2(op.key0, op.s, zmask, 0, ncomp, rows, n, A, lda, kb, B, ldb, SA, ldsa, st);
  }
  if (int rc = dispatch_main(op, ncomp, rows, n, A, lda, SA, ldsa, st)) return rc;
  if (kb == 0) return nsk::OK;
  return dispatch_main(op, ncomp, rows, kb, B, ldb, SA + ldsa * n * out_ncomp(op, ncomp), ldsa, st);
}

int dispatch_apply2(const Operator& op, int ncomp, const nsk::RowMap& rows, int64_t n, const double* A, int64_t lda,
                    int64_t kb, const double* B, int64_t ldb, double* SA, int64_t ldsa, cudaStream_t st) {
  if (op.appended == 0) return dispatch_main2(op, ncomp, rows, n, A, lda, kb, B, ldb, SA, ldsa, st);
  if (int rc = dispatch_apply(op, ncomp, rows, n, A, lda, SA, ldsa, st)) return rc;
  if (kb == 0) return nsk::OK;
  return dispatch_apply(op, ncomp, rows, kb, B, ldb, SA + ldsa * n * out_ncomp(op, ncomp), ldsa, st);
}

// Minimal JSON field readers for the descriptor (flat object, known keys).
bool json_find(const std::string& js, const std::string& key, size_t& pos) {
  const std::string pat = "\"" + key + "\"";
  size_t p = js.find(pat);
  if (p == std::string::npos) return false;
  p = js.find(':', p + pat.size());
  if (p == std::string::npos) return false;
  ++p;
  while (p < js.size() && (js[p] == ' ' || js[p] == '\t' || js[p] == '\n' || js[p] == '\r')) ++p;
  pos = p;
  return p < js.size();
}
bool json_u64(const std::string& js, const std::string& key, uint64_t& out, bool& neg) {
  size_t p;
  if (!json_find(js, key, p)) return false;
  neg = false;
  if (js[p] == '-') {
    neg = true;
    ++p;
  }
  if (p >= js.size() || js[p] < '0' || js[p] > '9') return false;
  uint64_t v = 0;
  while (p < js.size() && js[p] >= '0' && js[p] <= '9') v = v * 10 + static_cast<uint64_t>(js[p++] - '0');
  out = v;
  return true;
}
bool json_str(const std::string& js, const std::string& key, std::string& out) {
  size_t p;
  if (!json_find(js, key, p) || js[p] != '"') return false;
  size_t e = js.find('"', p + 1);
  if (e == std::string::npos) return false;
  out = js.substr(p + 1, e - p - 1);
  return true;
}

int kind_from_name(const std::string& k) {
  for (int i = 0; i <= nsk::COUNTSKETCH; ++i)
    if (k == nsk::kind_name(i)) return i;
  return -1;
}

// A per-thread non-blocking stream for the host-buffer entry points.
cudaStream_t host_stream() { return nsk::thread_stream(); }

int copy_in(const void* host, int64_t rows, int64_t cols, int64_t ld, int ncomp, double** dev, nsk::Scratch& s,
            cudaStream_t st) {
  const size_t elem = sizeof(double) * ncomp;
  NSK_CUDA_OK(s.alloc(elem * (rows > 0 ? rows : 1) * (cols > 0 ? cols : 1), st));
  *dev = s.as<double>();
  return nsk::h2d_rows(host, rows, cols, ld, elem, *dev, rows, st, nullptr);
}

// Host A (m x n, lda) -> SA (device, s x n, ld s).  Large inputs of the
// row-sharded kinds (gaussian, srht, countsketch) are copied in row chunks on
// a copy stream and each chunk is sketched (a row-shard apply) as soon as it
// has landed, so the PCIe transfer overlaps the sketch; the chunk partials
// are summed in chunk order (deterministic).  Everything else: copy, then
// apply.  a_buf receives the device copy of A.
int host_sketch(const Operator& op, int nc_in, int64_t m, int64_t n, const void* A, int64_t lda, nsk::Scratch& a_buf,
                double* SA, cudaStream_t st, int64_t kb = 0, const void* B = nullptr, int64_t ldb = 0,
                nsk::Scratch* b_buf = nullptr, int64_t row0 = 0) {
  // row0: global row of A's first row (a contiguous multi-GPU shard of m rows; 0 for the whole matrix)
  const int nc_out = out_ncomp(op, nc_in);
  const size_t elem = sizeof(double) * nc_in;
  // [A | B] (sketched TLS): B (a few columns) is copied whole first, then A streams in chunks and
  // every chunk is sketched together with the same rows of B (dispatch_main2)
  double* dB = nullptr;
  if (kb > 0)
    if (int rc = copy_in(B, m, kb, ldb, nc_in, &dB, *b_buf, st)) return rc;
  const int64_t ntot = n + kb;
  const int64_t align = op.kind == nsk::GAUSSIAN ? 16 : op.kind == nsk::SRHT ? 2048 : op.kind == nsk::COUNTSKETCH ? 12288 : 0;
  constexpr int64_t CHUNKS = 8;
  const int64_t chunk = align ? ((m + CHUNKS - 1) / CHUNKS + align - 1) / align * align : 0;
  const bool big = static_cast<double>(m) * static_cast<double>(n) * static_cast<double>(elem) >= 256.0 * (1 << 20);
  const bool pipelined = align && big && chunk < m && op.appended == 0 && op.zeroed.empty() &&
                         (op.kind != nsk::SRHT || m % 2048 == 0) && !std::getenv("NSK_NO_PIPELINE");
  double* dA = nullptr;
  if (!pipelined) {
    if (int rc = copy_in(A, m, n, lda, nc_in, &dA, a_buf, st)) return rc;
    nsk::RowMap rows{row0, 1, m};
    return dispatch_apply2(op, nc_in, rows, n, dA, m, kb, dB, m, SA, op.s, st);
  }
  // each row chunk lands as one rows x (n + kb) block: A's rows, then (copied on the device) the same
  // rows of B, so the chunk apply sees a single matrix [A | B] (the Gaussian kernel's TMA path)
  NSK_CUDA_OK(a_buf.alloc(elem * m * ntot, st));
  dA = a_buf.as<double>();
  const int64_t nchunks = (m + chunk - 1) / chunk;
  nsk::Scratch parts;
  const int64_t psz = op.s * ntot * nc_out;
  NSK_CUDA_OK(parts.alloc(sizeof(double) * psz * nchunks, st));
  // The operator's device tables (one window for all chunks; CountSketch's owner schedule takes
  // ~0.2 s of host work at m = 2^24) are built on a helper thread while the copy engine moves A.
  int devno = 0;
  NSK_CUDA_OK(cudaGetDevice(&devno));
  std::future<const nsk::DeviceTables*> tab = std::async(std::launch::async, [&op, m, row0, devno]() {
    cudaSetDevice(devno);
    return op.tables(row0, row0 + m);
  });
  bool have_tables = false;
  struct Pending {
    int64_t r0, rows;
    cudaEvent_t landed;
  };
  std::vector<Pending> pending;  // chunks that landed before the tables existed
  // chunk apply: st waits for exactly this chunk's copy, then the row-shard apply into its own partial
  auto run_chunk = [&](const Pending& c) {
    cudaError_t e = cudaStreamWaitEvent(st, c.landed, 0);
    cudaEventDestroy(c.landed);
    if (e != cudaSuccess) return nsk::cuda_fail(e, "chunk wait");
    nsk::RowMap shard{row0 + c.r0, 1, c.rows};  // chunk-major device copy: this chunk's block, ld = its rows
    double* blk = dA + c.r0 * ntot * nc_in;
    if (kb > 0) {
      if (cudaError_t e2 = cudaMemcpy2DAsync(blk + c.rows * n * nc_in, elem * c.rows, dB + c.r0 * nc_in, elem * m,
                                             elem * c.rows, kb, cudaMemcpyDeviceToDevice, st))
        return nsk::cuda_fail(e2, "chunk of B");
    }
    return dispatch_main2(op, nc_in, shard, ntot, blk, c.rows, 0, nullptr, m, parts.as<double>() + (c.r0 / chunk) * psz,
                          op.s, st);
  };
  auto flush = [&]() {
    have_tables = true;
    int rc = tab.get() ? static_cast<int>(nsk::OK) : static_cast<int>(nsk::ECUDA);
    for (auto& c : pending) {
      if (rc == nsk::OK)
        rc = run_chunk(c);
      else
        cudaEventDestroy(c.landed);
    }
    pending.clear();
    return rc;
  };
  // each row chunk is sketched as soon as it has landed (or, while the tables are still being built,
  // right after they exist -- each apply waits on its own chunk's event either way)
  auto sketch_chunk = [&](int64_t r0, int64_t rows, cudaEvent_t landed) {
    const Pending c{r0, rows, landed};
    if (!have_tables) {
      if (tab.wait_for(std::chrono::seconds(0)) != std::future_status::ready) {
        pending.push_back(c);
        return static_cast<int>(nsk::OK);
      }
      if (int rc = flush()) {
        cudaEventDestroy(landed);
        return rc;
      }
    }
    return run_chunk(c);
  };
  int rc = nsk::h2d_rows(A, m, n, lda, elem, dA, chunk, st, sketch_chunk, ntot);
  if (!have_tables) {
    const int rf = flush();  // also joins the helper thread on the error path
    if (rc == nsk::OK) rc = rf;
  }
  if (rc) return rc;
  NSK_CUDA_OK(cudaMemcpyAsync(SA, parts.as<double>(), sizeof(double) * psz, cudaMemcpyDeviceToDevice, st));
  for (int64_t c = 1; c < nchunks; ++c)
    if (int rc = nsk::accumulate(SA, op.s, nc_out, parts.as<double>() + c * psz, op.s, ntot, nc_out, st)) return rc;
  return nsk::OK;
}

int copy_out(void* host, int64_t ld, const double* dev, int64_t rows, int64_t cols, int ncomp, cudaStream_t st) {
  const size_t elem = sizeof(double) * ncomp;
  if (rows > 0 && cols > 0)
    NSK_CUDA_OK(cudaMemcpy2DAsync(host, elem * ld, dev, elem * rows, elem * rows, cols, cudaMemcpyDeviceToHost, st));
  return nsk::OK;
}

}  // namespace

namespace nsk {
// The pipelined host-buffer sketch of a contiguous row shard (nccl_shard.cpp's host entry point).
int host_sketch_shard(const Operator& op, int nc_in, int64_t row0, int64_t mloc, int64_t n, const void* A,
                      int64_t lda, double* SA, cudaStream_t st) {
  Scratch a;
  return host_sketch(op, nc_in, mloc, n, A, lda, a, SA, st, 0, nullptr, 0, nullptr, row0);
}
// dispatch_apply for the multi-GPU entry points (nccl_shard.cpp)
int dispatch_apply_c(const Operator& op, int ncomp, const RowMap& rows, int64_t n, const double* A, int64_t lda,
                     double* SA, int64_t ldsa, cudaStream_t st) {
  return dispatch_apply(op, ncomp, rows, n, A, lda, SA, ldsa, st);
}
}  // namespace nsk

extern "C" {

const char* nsk_last_error(void) { return nsk::last_error(); }

const char* nsk_version(void) { return "nullsketch-b200 0.1 (sm_100a, FP64 DMMA + CUDA cores)"; }

int nsk_op_draw(int kind, int64_t s, int64_t m, uint64_t seed, nsk_operator** out) {
  Operator* op = nullptr;
  int rc = nsk::draw_operator(kind, s, m, seed, &op);
  if (out) *out = reinterpret_cast<nsk_operator*>(op);
  return rc;
}

void nsk_op_destroy(nsk_operator* op) { delete OP(op); }

int nsk_op_info(const nsk_operator* h, int* kind, int64_t* s, int64_t* m, uint64_t* seed, uint64_t* id) {
  if (int rc = check_op(h)) return rc;
  const Operator& op = *OP(h);
  if (kind) *kind = op.kind;
  if (s) *s = op.s;
  if (m) *m = op.m;
  if (seed) *seed = op.seed;
  if (id) *id = op.id;
  return nsk::OK;
}

int nsk_op_sample_indices(const nsk_operator* h, int64_t* idx_host) {
  if (int rc = check_op(h)) return rc;
  const Operator& op = *OP(h);
  if (op.idx.empty()) return nsk::fail(nsk::EINVAL_, "sample indices exist for srft/srdct/srht only");
  if (!idx_host) return nsk::fail(nsk::EINVAL_, "null output");
  std::memcpy(idx_host, op.idx.data(), op.idx.size() * sizeof(int64_t));
  return nsk::OK;
}

// nlohmann::json::dump() order (keys sorted) as in sketch.cpp:303-313.
int nsk_op_descriptor(const nsk_operator* h, char* buf, size_t cap, size_t* len) {
  if (int rc = check_op(h)) return rc;
  const Operator& op = *OP(h);
  std::string js = "{\"appended\":" + std::to_string(op.appended) + ",\"format\":1,\"kind\":\"" +
                   nsk::kind_name(op.kind) + "\",\"m\":" + std::to_string(op.m) + ",\"s\":" + std::to_string(op.s) +
                   ",\"seed\":" + std::to_string(op.seed) + ",\"zeroed_rows\":[";
  for (size_t i = 0; i < op.zeroed.size(); ++i) js += (i ? "," : "") + std::to_string(op.zeroed[i]);
  js += "]}";
  if (len) *len = js.size();
  if (!buf || cap < js.size() + 1)
    return nsk::fail(nsk::ERANGE_, "descriptor: buffer too small (" + std::to_string(js.size() + 1) + " bytes needed)");
  std::memcpy(buf, js.c_str(), js.size() + 1);
  return nsk::OK;
}

// SketchOperator::from_descriptor (sketch.cpp:315-337): redraw, replay the
// appended-column count (their Gaussians are regenerated from stream (seed, 1)
// on use) and the zeroed rows, validating each like the reference.
int nsk_op_from_descriptor(const char* json, nsk_operator** out) {
  if (out) *out = nullptr;
  if (!json) return nsk::fail(nsk::EINVAL_, "sketch descriptor: null text");
  const std::string js(json);
  uint64_t fmt = 0, s = 0, m = 0, seed = 0, app = 0;
  bool neg = false;
  if (!json_u64(js, "format", fmt, neg) || neg || fmt != 1)
    return nsk::fail(nsk::EINVAL_, "sketch descriptor: unsupported format");
  std::string kind;
  if (!json_str(js, "kind", kind)) return nsk::fail(nsk::EINVAL_, "sketch descriptor: missing kind");
  const int k = kind_from_name(kind);
  if (k < 0) return nsk::fail(nsk::EINVAL_, "unknown sketch kind: " + kind);
  bool n1 = false, n2 = false, n3 = false;
  if (!json_u64(js, "s", s, n1) || !json_u64(js, "m", m, n2) || !json_u64(js, "seed", seed, n3) || n1 || n2 || n3)
    return nsk::fail(nsk::EINVAL_, "sketch descriptor: missing or negative s/m/seed");
  if (!json_u64(js, "appended", app, neg)) return nsk::fail(nsk::EINVAL_, "sketch descriptor: missing appended");
  if (neg) return nsk::fail(nsk::EINVAL_, "sketch descriptor: bad appended count");
  size_t p;
  if (!json_find(js, "zeroed_rows", p) || js[p] != '[')
    return nsk::fail(nsk::EINVAL_, "sketch descriptor: missing zeroed_rows");
  const size_t q = js.find(']', p);
  if (q == std::string::npos) return nsk::fail(nsk::EINVAL_, "sketch descriptor: malformed zeroed_rows");
  std::vector<int64_t> rows;
  for (size_t i = p + 1; i < q;) {
    while (i < q && (js[i] == ' ' || js[i] == ',' || js[i] == '\n' || js[i] == '\t' || js[i] == '\r')) ++i;
    if (i >= q) break;
    char* endp = nullptr;
    const long long z = std::strtoll(js.c_str() + i, &endp, 10);
    if (endp == js.c_str() + i) return nsk::fail(nsk::EINVAL_, "sketch descriptor: malformed zeroed_rows");
    rows.push_back(z);
    i = static_cast<size_t>(endp - js.c_str());
  }
  Operator* op = nullptr;
  int rc = nsk::draw_operator(k, static_cast<int64_t>(s), static_cast<int64_t>(m), seed, &op);
  if (rc) return rc;
  op->appended = static_cast<int64_t>(app);
  for (long long z : rows) {
    if (z < 0 || z >= op->m_eff() || op->is_zeroed(z)) {
      delete op;
      return nsk::fail(nsk::EINVAL_, "sketch descriptor: bad zeroed row " + std::to_string(z));
    }
    op->zeroed.insert(std::lower_bound(op->zeroed.begin(), op->zeroed.end(), static_cast<int64_t>(z)), z);
  }
  ++op->state_version;
  if (out) *out = reinterpret_cast<nsk_operator*>(op);
  return nsk::OK;
}

int nsk_apply(const nsk_operator* h, int scalar, int64_t m, int64_t n, const void* A, int64_t lda, void* SA,
              int64_t ldsa, void* stream) {
  if (int rc = check_op(h)) return rc;
  const Operator& op = *OP(h);
  if (int rc = validate_apply(op, scalar, m, n, A, lda, SA, ldsa, false)) return rc;
  nsk::RowMap rows{0, 1, m};
  return dispatch_apply(op, scalar == NSK_COMPLEX ? 2 : 1, rows, n, static_cast<const double*>(A), lda,
                        static_cast<double*>(SA), ldsa, ST(stream));
}

int nsk_apply_shard(const nsk_operator* h, int scalar, int64_t row0, int64_t rstep, int64_t mloc, int64_t n,
                    const void* A, int64_t lda, void* SA, int64_t ldsa, void* stream) {
  if (int rc = check_op(h)) return rc;
  const Operator& op = *OP(h);
  if (int rc = validate_apply(op, scalar, mloc, n, A, lda, SA, ldsa, true)) return rc;
  if (rstep < 1 || row0 < 0) return nsk::fail(nsk::EINVAL_, "apply_shard: bad row map");
  if (mloc > 0 && row0 + rstep * (mloc - 1) >= op.m)
    return nsk::fail(nsk::ERANGE_, "apply_shard: rows beyond the operator's m");
  nsk::RowMap rows{row0, rstep, mloc};
  return dispatch_apply(op, scalar == NSK_COMPLEX ? 2 : 1, rows, n, static_cast<const double*>(A), lda,
                        static_cast<double*>(SA), ldsa, ST(stream));
}

int nsk_svd_trailing(int scalar, int64_t s, int64_t n, const void* SA, int64_t ldsa, int64_t k, void* W,
                     int64_t ldw, double* sigma, void* stream) {
  if (scalar != NSK_REAL && scalar != NSK_COMPLEX) return nsk::fail(nsk::EINVAL_, "unknown scalar kind");
  if (s < 1 || n < 1) return nsk::fail(nsk::EINVAL_, "svd: matrix is empty");
  if (k < 0 || k >= n)
    return nsk::fail(nsk::EINVAL_, "nullspace: k must satisfy 0 <= k < n, got k = " + std::to_string(k) +
                                       ", n = " + std::to_string(n));
  if (s < n) return nsk::fail(nsk::EINVAL_, "svd_trailing: needs s >= n");
  if (ldsa < s || (k > 0 && ldw < n)) return nsk::fail(nsk::EINVAL_, "svd_trailing: bad leading dimension");
  if (!SA || !sigma || (k > 0 && !W)) return nsk::fail(nsk::EINVAL_, "svd_trailing: null pointer");
  return nsk::jacobi_trailing(scalar == NSK_COMPLEX ? 2 : 1, s, n, static_cast<const double*>(SA), ldsa, k,
                              static_cast<double*>(W), ldw, sigma, ST(stream));
}

static int solve_common(const Operator& op, int scalar, int64_t m, int64_t n, const void* A, int64_t lda,
                        nsk::Scratch& sa_buf, int& nc_out, cudaStream_t st) {
  if (m != op.m_eff()) return nsk::fail(nsk::EINVAL_, "nullspace: matrix rows do not match the sketch operator");
  if (op.s < n)
    return nsk::fail(nsk::EINVAL_, "nullspace: sketch size s = " + std::to_string(op.s) + " is smaller than n = " +
                                       std::to_string(n));
  if (int rc = validate_apply(op, scalar, m, n, A, lda, reinterpret_cast<const void*>(1), op.s, false)) return rc;
  const int nc_in = scalar == NSK_COMPLEX ? 2 : 1;
  nc_out = out_ncomp(op, nc_in);
  NSK_CUDA_OK(sa_buf.alloc(sizeof(double) * op.s * n * nc_out, st));
  nsk::RowMap rows{0, 1, m};
  return dispatch_apply(op, nc_in, rows, n, static_cast<const double*>(A), lda, sa_buf.as<double>(), op.s, st);
}

int nsk_solve_k(const nsk_operator* h, int scalar, int64_t m, int64_t n, const void* A, int64_t lda, int64_t k,
                void* W, int64_t ldw, double* sigma, void* stream) {
  if (int rc = check_op(h)) return rc;
  const Operator& op = *OP(h);
  if (n < 1) return nsk::fail(nsk::EINVAL_, "nullspace: matrix has no columns");
  if (k < 0 || k >= n)
    return nsk::fail(nsk::EINVAL_, "nullspace: k must satisfy 0 <= k < n, got k = " + std::to_string(k) +
                                       ", n = " + std::to_string(n));
  cudaStream_t st = ST(stream);
  nsk::Scratch sa;
  int nc = 1;
  if (int rc = solve_common(op, scalar, m, n, A, lda, sa, nc, st)) return rc;
  return nsk::jacobi_trailing(nc, op.s, n, sa.as<double>(), op.s, k, static_cast<double*>(W), ldw, sigma, st);
}

int nsk_solve_tol(const nsk_operator* h, int scalar, int64_t m, int64_t n, const void* A, int64_t lda, double eps,
                  int64_t* k_out, void* W, int64_t ldw, double* sigma, void* stream) {
  if (int rc = check_op(h)) return rc;
  const Operator& op = *OP(h);
  if (!(eps >= 0.0)) return nsk::fail(nsk::EINVAL_, "nullspace: eps must be non-negative");
  if (n < 1) return nsk::fail(nsk::EINVAL_, "nullspace: matrix has no columns");
  cudaStream_t st = ST(stream);
  nsk::Scratch sa, wf;
  int nc = 1;
  if (int rc = solve_common(op, scalar, m, n, A, lda, sa, nc, st)) return rc;
  const int64_t kf = n - 1;
  NSK_CUDA_OK(wf.alloc(sizeof(double) * n * (kf > 0 ? kf : 1) * nc, st));
  if (int rc = nsk::jacobi_trailing(nc, op.s, n, sa.as<double>(), op.s, kf, wf.as<double>(), n, sigma, st)) return rc;
  std::vector<double> sv(static_cast<size_t>(n));
  NSK_CUDA_OK(cudaMemcpyAsync(sv.data(), sigma, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  NSK_CUDA_OK(cudaStreamSynchronize(st));
  int64_t k = 0;
  while (k < n && sv[static_cast<size_t>(n - 1 - k)] < eps) ++k;
  if (k == n)
    return nsk::fail(nsk::EINVAL_,
                     "nullspace: eps selects every singular value; the trailing subspace would be the whole space");
  if (k_out) *k_out = k;
  if (k > 0) {
    const size_t elem = sizeof(double) * nc;
    NSK_CUDA_OK(cudaMemcpy2DAsync(W, elem * ldw, wf.as<double>() + (kf - k) * n * nc, elem * n, elem * n, k,
                                  cudaMemcpyDeviceToDevice, st));
  }
  return nsk::OK;
}

int nsk_residual_fro(int scalar, int64_t m, int64_t n, const void* A, int64_t lda, int64_t k, const void* W,
                     int64_t ldw, double* out, void* stream) {
  if (scalar != NSK_REAL && scalar != NSK_COMPLEX) return nsk::fail(nsk::EINVAL_, "unknown scalar kind");
  if (!out) return nsk::fail(nsk::EINVAL_, "residual_certificate: null output");
  if (m < 0 || n < 0 || k < 0 || lda < m || (k > 0 && ldw < n))
    return nsk::fail(nsk::EINVAL_, "residual_certificate: bad dimensions");
  return nsk::residual_fro(scalar == NSK_COMPLEX ? 2 : 1, m, n, static_cast<const double*>(A), lda, k,
                           static_cast<const double*>(W), ldw, out, ST(stream));
}

int nsk_apply_host(const nsk_operator* h, int scalar, int64_t m, int64_t n, const void* A, int64_t lda, void* SA,
                   int64_t ldsa) {
  if (int rc = check_op(h)) return rc;
  const Operator& op = *OP(h);
  if (int rc = validate_apply(op, scalar, m, n, A, lda, SA, ldsa, false)) return rc;
  cudaStream_t st = host_stream();
  const int nc_in = scalar == NSK_COMPLEX ? 2 : 1, nc_out = out_ncomp(op, nc_in);
  nsk::Scratch a, sa;
  NSK_CUDA_OK(sa.alloc(sizeof(double) * op.s * (n > 0 ? n : 1) * nc_out, st));
  if (int rc = host_sketch(op, nc_in, m, n, A, lda, a, sa.as<double>(), st)) return rc;
  if (int rc = copy_out(SA, ldsa, sa.as<double>(), op.s, n, nc_out, st)) return rc;
  NSK_CUDA_OK(cudaStreamSynchronize(st));
  return nsk::OK;
}

int nsk_solve_k_host(const nsk_operator* h, int scalar, int64_t m, int64_t n, const void* A, int64_t lda, int64_t k,
                     void* W, int64_t ldw, double* sigma) {
  if (int rc = check_op(h)) return rc;
  const Operator& op = *OP(h);
  if (lda < m) return nsk::fail(nsk::EINVAL_, "solve_k: lda < rows");
  if (k < 0 || k >= n)
    return nsk::fail(nsk::EINVAL_, "nullspace: k must satisfy 0 <= k < n, got k = " + std::to_string(k) +
                                       ", n = " + std::to_string(n));
  cudaStream_t st = host_stream();
  const int nc_in = scalar == NSK_COMPLEX ? 2 : 1, nc_out = out_ncomp(op, nc_in);
  if (n < 1) return nsk::fail(nsk::EINVAL_, "nullspace: matrix has no columns");
  if (m != op.m_eff()) return nsk::fail(nsk::EINVAL_, "nullspace: matrix rows do not match the sketch operator");
  if (op.s < n)
    return nsk::fail(nsk::EINVAL_, "nullspace: sketch size s = " + std::to_string(op.s) + " is smaller than n = " +
                                       std::to_string(n));
  if (int rc = validate_apply(op, scalar, m, n, A, lda, reinterpret_cast<const void*>(1), op.s, false)) return rc;
  nsk::Scratch a, sa, w, sg;
  NSK_CUDA_OK(sa.alloc(sizeof(double) * op.s * n * nc_out, st));
  if (int rc = host_sketch(op, nc_in, m, n, A, lda, a, sa.as<double>(), st)) return rc;
  NSK_CUDA_OK(w.alloc(sizeof(double) * n * (k > 0 ? k : 1) * nc_out, st));
  NSK_CUDA_OK(sg.alloc(sizeof(double) * n, st));
  if (int rc = nsk::jacobi_trailing(nc_out, op.s, n, sa.as<double>(), op.s, k, w.as<double>(), n, sg.as<double>(), st))
    return rc;
  if (int rc = copy_out(W, ldw, w.as<double>(), n, k, nc_out, st)) return rc;
  NSK_CUDA_OK(cudaMemcpyAsync(sigma, sg.as<double>(), sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  NSK_CUDA_OK(cudaStreamSynchronize(st));
  return nsk::OK;
}

int nsk_solve_tol_host(const nsk_operator* h, int scalar, int64_t m, int64_t n, const void* A, int64_t lda, double eps,
                       int64_t* k_out, void* W, int64_t ldw, double* sigma) {
  if (int rc = check_op(h)) return rc;
  const Operator& op = *OP(h);
  if (lda < m) return nsk::fail(nsk::EINVAL_, "solve_tol: lda < rows");
  if (n < 1) return nsk::fail(nsk::EINVAL_, "nullspace: matrix has no columns");
  cudaStream_t st = host_stream();
  const int nc_in = scalar == NSK_COMPLEX ? 2 : 1, nc_out = out_ncomp(op, nc_in);
  nsk::Scratch a, w, sg;
  double* dA = nullptr;
  if (int rc = copy_in(A, m, n, lda, nc_in, &dA, a, st)) return rc;
  NSK_CUDA_OK(w.alloc(sizeof(double) * n * n * nc_out, st));
  NSK_CUDA_OK(sg.alloc(sizeof(double) * n, st));
  int64_t k = 0;
  if (int rc = nsk_solve_tol(h, scalar, m, n, dA, m, eps, &k, w.as<double>(), n, sg.as<double>(), st)) return rc;
  if (int rc = copy_out(W, ldw, w.as<double>(), n, k, nc_out, st)) return rc;
  NSK_CUDA_OK(cudaMemcpyAsync(sigma, sg.as<double>(), sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  NSK_CUDA_OK(cudaStreamSynchronize(st));
  if (k_out) *k_out = k;
  return nsk::OK;
}

int nsk_residual_fro_host(int scalar, int64_t m, int64_t n, const void* A, int64_t lda, int64_t k, const void* W,
                          int64_t ldw, double* out) {
  if (scalar != NSK_REAL && scalar != NSK_COMPLEX) return nsk::fail(nsk::EINVAL_, "unknown scalar kind");
  if (m < 0 || n < 0 || k < 0 || lda < m || (k > 0 && ldw < n))
    return nsk::fail(nsk::EINVAL_, "residual_certificate: bad dimensions");
  cudaStream_t st = host_stream();
  const int nc = scalar == NSK_COMPLEX ? 2 : 1;
  nsk::Scratch a, w;
  double *dA = nullptr, *dW = nullptr;
  if (int rc = copy_in(A, m, n, lda, nc, &dA, a, st)) return rc;
  if (int rc = copy_in(W, n, k, ldw, nc, &dW, w, st)) return rc;
  return nsk::residual_fro(nc, m, n, dA, m > 0 ? m : 1, k, dW, n > 0 ? n : 1, out, st);
}

// ---- incremental maintenance (sketch.hpp:90-109) ----------------------------

int nsk_op_state(const nsk_operator* h, int64_t* m_eff, int64_t* appended, int64_t* nzeroed, int64_t* zeroed_rows,
                 int64_t cap) {
  if (int rc = check_op(h)) return rc;
  const Operator& op = *OP(h);
  if (m_eff) *m_eff = op.m_eff();
  if (appended) *appended = op.appended;
  if (nzeroed) *nzeroed = static_cast<int64_t>(op.zeroed.size());
  if (zeroed_rows)
    for (int64_t i = 0; i < cap && i < static_cast<int64_t>(op.zeroed.size()); ++i)
      zeroed_rows[i] = op.zeroed[static_cast<size_t>(i)];
  return nsk::OK;
}

int nsk_update_row(nsk_operator* h, int scalar_sa, int64_t n, int scalar_row, const void* a_row, void* SA,
                   int64_t ldsa, void* stream) {
  if (int rc = check_op(h)) return rc;
  Operator& op = *OP(h);
  if (n < 0 || ldsa < op.s || (n > 0 && (!a_row || !SA))) return nsk::fail(nsk::EINVAL_, "update_row: bad arguments");
  if (op.kind == nsk::SRDCT && scalar_row == NSK_COMPLEX)
    return nsk::fail(nsk::EINVAL_, "update_row: srdct sketch carries real data only");
  if (scalar_sa == NSK_REAL && scalar_row == NSK_COMPLEX)
    return nsk::fail(nsk::EINVAL_, "update_row: a complex row needs a complex sketch (promote SA first)");
  cudaStream_t st = ST(stream);
  nsk::Scratch g;
  NSK_CUDA_OK(g.alloc(sizeof(double) * op.s, st));
  // (1/sqrt s) g, g = Gaussians #(p*s + i) of stream (seed, 1): column m + p of S.
  if (int rc = nsk::sketch_column(op, op.m_eff(), g.as<double>(), 1, st)) return rc;
  if (int rc = nsk::rank1_update(static_cast<double*>(SA), ldsa, scalar_sa == NSK_COMPLEX ? 2 : 1, op.s, n,
                                 g.as<double>(), 1, static_cast<const double*>(a_row),
                                 scalar_row == NSK_COMPLEX ? 2 : 1, 1.0, st))
    return rc;
  NSK_CUDA_OK(cudaStreamSynchronize(st));
  ++op.appended;
  ++op.state_version;
  return nsk::OK;
}

int nsk_downdate_row(nsk_operator* h, int64_t j, int scalar_sa, int64_t n, int scalar_row, const void* a_row,
                     void* SA, int64_t ldsa, void* stream) {
  if (int rc = check_op(h)) return rc;
  Operator& op = *OP(h);
  if (j < 0 || j >= op.m_eff()) return nsk::fail(nsk::ERANGE_, "downdate_row: row index out of range");
  if (op.is_zeroed(j))
    return nsk::fail(nsk::EINVAL_, "downdate_row: row " + std::to_string(j) + " already removed");
  if (n < 0 || ldsa < op.s || (n > 0 && (!a_row || !SA))) return nsk::fail(nsk::EINVAL_, "downdate_row: bad arguments");
  const int nc_col = (op.kind == nsk::SRFT && j < op.m) ? 2 : 1;
  if (scalar_sa == NSK_REAL && (nc_col == 2 || scalar_row == NSK_COMPLEX))
    return nsk::fail(nsk::EINVAL_, "downdate_row: the update is complex, pass a complex sketch");
  cudaStream_t st = ST(stream);
  nsk::Scratch col;
  NSK_CUDA_OK(col.alloc(sizeof(double) * op.s * nc_col, st));
  if (int rc = nsk::sketch_column(op, j, col.as<double>(), nc_col, st)) return rc;  // S e_j before zeroing
  if (int rc = nsk::rank1_update(static_cast<double*>(SA), ldsa, scalar_sa == NSK_COMPLEX ? 2 : 1, op.s, n,
                                 col.as<double>(), nc_col, static_cast<const double*>(a_row),
                                 scalar_row == NSK_COMPLEX ? 2 : 1, -1.0, st))
    return rc;
  NSK_CUDA_OK(cudaStreamSynchronize(st));
  op.zeroed.insert(std::lower_bound(op.zeroed.begin(), op.zeroed.end(), j), j);
  ++op.state_version;
  const int64_t live = op.m_eff() - static_cast<int64_t>(op.zeroed.size());
  if (live < 2 * op.s)  // sketch.cpp:296-299
    std::fprintf(stderr, "nullsketch: warning: sketch operator down to %lld live rows (s = %lld); quality degrades "
                         "as rows are removed\n",
                 static_cast<long long>(live), static_cast<long long>(op.s));
  return nsk::OK;
}

int nsk_update_column(const nsk_operator* h, int scalar, int64_t m, const void* a_col, void* out, void* stream) {
  if (int rc = check_op(h)) return rc;
  const Operator& op = *OP(h);
  if (int rc = validate_apply(op, scalar, m, 1, a_col, m, out, op.s, false)) return rc;
  cudaStream_t st = ST(stream);
  const int nc = scalar == NSK_COMPLEX ? 2 : 1;
  nsk::Scratch c;
  NSK_CUDA_OK(c.alloc(sizeof(double) * (m > 0 ? m : 1) * nc, st));
  NSK_CUDA_OK(cudaMemcpyAsync(c.p, a_col, sizeof(double) * m * nc, cudaMemcpyDeviceToDevice, st));
  if (int rc = nsk::mask_zeroed(op, c.as<double>(), nc, st)) return rc;  // sketch.cpp:244-251
  nsk::RowMap rows{0, 1, m};
  return dispatch_apply(op, nc, rows, 1, c.as<double>(), m > 0 ? m : 1, static_cast<double*>(out), op.s, st);
}

// Host-buffer variants (the C++ mirror's update_row / downdate_row /
// update_column): stage SA and the row or column in, call the device entry
// point on the library's host stream, copy SA or the sketched column back.
int nsk_update_row_host(nsk_operator* h, int scalar_sa, int64_t n, int scalar_row, const void* a_row, void* SA,
                        int64_t ldsa) {
  if (int rc = check_op(h)) return rc;
  const Operator& op = *OP(h);
  if (n < 0 || ldsa < op.s || (n > 0 && (!a_row || !SA))) return nsk::fail(nsk::EINVAL_, "update_row: bad arguments");
  cudaStream_t st = host_stream();
  const int nc_sa = scalar_sa == NSK_COMPLEX ? 2 : 1, nc_row = scalar_row == NSK_COMPLEX ? 2 : 1;
  nsk::Scratch dsa, drow;
  double *pSA = nullptr, *pRow = nullptr;
  if (int rc = copy_in(SA, op.s, n, ldsa, nc_sa, &pSA, dsa, st)) return rc;
  if (int rc = copy_in(a_row, 1, n, 1, nc_row, &pRow, drow, st)) return rc;
  if (int rc = nsk_update_row(h, scalar_sa, n, scalar_row, pRow, pSA, op.s, st)) return rc;
  if (int rc = copy_out(SA, ldsa, pSA, op.s, n, nc_sa, st)) return rc;
  NSK_CUDA_OK(cudaStreamSynchronize(st));
  return nsk::OK;
}

int nsk_downdate_row_host(nsk_operator* h, int64_t j, int scalar_sa, int64_t n, int scalar_row, const void* a_row,
                          void* SA, int64_t ldsa) {
  if (int rc = check_op(h)) return rc;
  const Operator& op = *OP(h);
  if (n < 0 || ldsa < op.s || (n > 0 && (!a_row || !SA)))
    return nsk::fail(nsk::EINVAL_, "downdate_row: bad arguments");
  cudaStream_t st = host_stream();
  const int nc_sa = scalar_sa == NSK_COMPLEX ? 2 : 1, nc_row = scalar_row == NSK_COMPLEX ? 2 : 1;
  nsk::Scratch dsa, drow;
  double *pSA = nullptr, *pRow = nullptr;
  if (int rc = copy_in(SA, op.s, n, ldsa, nc_sa, &pSA, dsa, st)) return rc;
  if (int rc = copy_in(a_row, 1, n, 1, nc_row, &pRow, drow, st)) return rc;
  if (int rc = nsk_downdate_row(h, j, scalar_sa, n, scalar_row, pRow, pSA, op.s, st)) return rc;
  if (int rc = copy_out(SA, ldsa, pSA, op.s, n, nc_sa, st)) return rc;
  NSK_CUDA_OK(cudaStreamSynchronize(st));
  return nsk::OK;
}

int nsk_update_column_host(const nsk_operator* h, int scalar, int64_t m, const void* a_col, void* out) {
  if (int rc = check_op(h)) return rc;
  const Operator& op = *OP(h);
  if (m < 0 || (m > 0 && !a_col) || !out) return nsk::fail(nsk::EINVAL_, "update_column: bad arguments");
  cudaStream_t st = host_stream();
  const int nc = scalar == NSK_COMPLEX ? 2 : 1, nc_out = out_ncomp(op, nc);
  nsk::Scratch dcol, dout;
  double* pCol = nullptr;
  if (int rc = copy_in(a_col, m, 1, m > 0 ? m : 1, nc, &pCol, dcol, st)) return rc;
  NSK_CUDA_OK(dout.alloc(sizeof(double) * op.s * nc_out, st));
  if (int rc = nsk_update_column(h, scalar, m, pCol, dout.p, st)) return rc;
  if (int rc = copy_out(out, op.s, dout.as<double>(), op.s, 1, nc_out, st)) return rc;
  NSK_CUDA_OK(cudaStreamSynchronize(st));
  return nsk::OK;
}

// ---- total least squares (tls.cpp:26-62) -----------------------------------
// Shared tail of the sketched and exact solvers: M (rows x (n + k), ld ldm) is
// S [A|B] or the R factor of [A|B].  Trailing k right singular vectors and
// the full spectrum of M, sigma_n of its leading n columns, the existence
// check (tls.cpp:46-50), the V_k2 condition estimate and X = -V_k1 V_k2^{-1}.
static int tls_finish(int nc, int64_t rows, const double* M, int64_t ldm, int64_t n, int64_t k, double cond_limit,
                      int allow_marginal, void* X, int64_t ldx, void* Vk, int64_t ldv, double* sigma, double* info,
                      cudaStream_t st) {
  const int64_t nk = n + k;
  nsk::Scratch siga, v2s, v2w;
  NSK_CUDA_OK(siga.alloc(sizeof(double) * n, st));
  NSK_CUDA_OK(v2s.alloc(sizeof(double) * k, st));
  NSK_CUDA_OK(v2w.alloc(sizeof(double) * k * k * nc, st));
  // The two SVDs of tls.cpp:110-111 share one QR (R of the leading n columns is the leading block of
  // R) and their Jacobi stages run concurrently (jacobi_trailing_pair).
  if (int rc = nsk::jacobi_trailing_pair(nc, rows, nk, M, ldm, k, static_cast<double*>(Vk), ldv, sigma, n,
                                         siga.as<double>(), st))
    return rc;
  std::vector<double> s_aug(static_cast<size_t>(nk)), s_a(static_cast<size_t>(n));
  NSK_CUDA_OK(cudaMemcpyAsync(s_aug.data(), sigma, sizeof(double) * nk, cudaMemcpyDeviceToHost, st));
  NSK_CUDA_OK(cudaMemcpyAsync(s_a.data(), siga.p, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
  NSK_CUDA_OK(cudaStreamSynchronize(st));
  double tail = 0.0;
  for (int64_t i = n; i < nk; ++i) tail += s_aug[static_cast<size_t>(i)] * s_aug[static_cast<size_t>(i)];
  info[0] = std::sqrt(tail);                   // tls_residual
  info[2] = s_a[static_cast<size_t>(n - 1)];   // sigma_n(A) (of the sketch / of R)
  info[3] = s_aug[static_cast<size_t>(n)];     // sigma_{n+1}([A|B])
  if (!(info[2] > info[3]) && !allow_marginal)
    return nsk::fail(NSK_ETLS_EXISTENCE, "tls: solution existence check failed: sigma_n(A) = " +
                                             std::to_string(info[2]) + " is not above sigma_{n+1}([A|B]) = " +
                                             std::to_string(info[3]));
  // Condition estimate of the k x k corner V_k2 (tls.cpp:32-37), then X = -V_k1 V_k2^{-1}.
  NSK_CUDA_OK(cudaMemcpy2DAsync(v2w.p, sizeof(double) * k * nc, static_cast<double*>(Vk) + n * nc,
                                sizeof(double) * ldv * nc, sizeof(double) * k * nc, k, cudaMemcpyDeviceToDevice, st));
  if (int rc = nsk::jacobi_trailing(nc, k, k, v2w.as<double>(), k, 0, nullptr, 1, v2s.as<double>(), st)) return rc;
  std::vector<double> sv2(static_cast<size_t>(k));
  NSK_CUDA_OK(cudaMemcpyAsync(sv2.data(), v2s.p, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
  NSK_CUDA_OK(cudaStreamSynchronize(st));
  const double smin = sv2[static_cast<size_t>(k - 1)];
  info[1] = smin == 0.0 ? HUGE_VAL : sv2[0] / smin;
  if (!(info[1] <= cond_limit))
    return nsk::fail(NSK_ETLS_CONDITION, "tls: V_k2 is ill conditioned (cond estimate " + std::to_string(info[1]) +
                                             "); X = -V_k1 V_k2^{-1} is unreliable");
  return nsk::tls_corner(nc, static_cast<const double*>(Vk), ldv, n, k, static_cast<double*>(X), ldx, st);
}

// ---- sketched total least squares (tls.cpp:97-113) ------------------------

int nsk_tls_solve_sketched(const nsk_operator* h, int scalar, int64_t m, int64_t n, int64_t k, const void* A,
                           int64_t lda, const void* B, int64_t ldb, double cond_limit, int allow_marginal, void* X,
                           int64_t ldx, void* Vk, int64_t ldv, double* sigma, double* info, void* stream) {
  if (k > 64) return nsk::fail(nsk::EINVAL_, "tls: this build supports at most 64 right-hand sides");
  if (int rc = check_op(h)) return rc;
  const Operator& op = *OP(h);
  if (k < 1) return nsk::fail(nsk::EINVAL_, "tls: B must have at least one column");
  if (n < k) return nsk::fail(nsk::EINVAL_, "tls: need n >= k");
  if (m < n + k) return nsk::fail(nsk::EINVAL_, "tls: need m >= n + k");
  if (op.m_eff() != m) return nsk::fail(nsk::EINVAL_, "tls: sketch operator row count does not match [A|B]");
  if (op.s < n + k) return nsk::fail(nsk::EINVAL_, "tls: sketch size below n + k");
  if (int rc = validate_apply(op, scalar, m, n, A, lda, reinterpret_cast<const void*>(1), op.s, false)) return rc;
  if (int rc = validate_apply(op, scalar, m, k, B, ldb, reinterpret_cast<const void*>(1), op.s, false)) return rc;
  if (!X || !Vk || !sigma || !info || ldx < n || ldv < n + k) return nsk::fail(nsk::EINVAL_, "tls: bad outputs");
  cudaStream_t st = ST(stream);
  const int nc_in = scalar == NSK_COMPLEX ? 2 : 1, nc = out_ncomp(op, nc_in);
  const int64_t nk = n + k;
  nsk::Scratch sa;
  NSK_CUDA_OK(sa.alloc(sizeof(double) * op.s * nk * nc, st));
  nsk::RowMap rows{0, 1, m};
  // S [A | B] without forming [A | B] (tls.cpp:108-109): one pass over both blocks.
  if (int rc = dispatch_apply2(op, nc_in, rows, n, static_cast<const double*>(A), lda, k,
                               static_cast<const double*>(B), ldb, sa.as<double>(), op.s, st))
    return rc;
  return tls_finish(nc, op.s, sa.as<double>(), op.s, n, k, cond_limit, allow_marginal, X, ldx, Vk, ldv, sigma, info,
                    st);
}

// ---- exact total least squares (tls.cpp:83-95) ----------------------------
// Thin QR of [A|B] on the device (tall_qr.cu), then the same SVD tail on the
// (n + k) x (n + k) triangle.
int nsk_tls_solve_exact(int scalar, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B,
                        int64_t ldb, double cond_limit, int allow_marginal, void* X, int64_t ldx, void* Vk,
                        int64_t ldv, double* sigma, double* info, void* stream) {
  if (k > 64) return nsk::fail(nsk::EINVAL_, "tls: this build supports at most 64 right-hand sides");
  if (scalar != NSK_REAL && scalar != NSK_COMPLEX) return nsk::fail(nsk::EINVAL_, "tls: bad scalar kind");
  if (k < 1) return nsk::fail(nsk::EINVAL_, "tls: B must have at least one column");
  if (n < k) return nsk::fail(nsk::EINVAL_, "tls: need n >= k");
  if (m < n + k) return nsk::fail(nsk::EINVAL_, "tls: need m >= n + k");
  if (!A || !B || lda < m || ldb < m) return nsk::fail(nsk::EINVAL_, "tls: bad A / B");
  if (!X || !Vk || !sigma || !info || ldx < n || ldv < n + k) return nsk::fail(nsk::EINVAL_, "tls: bad outputs");
  cudaStream_t st = ST(stream);
  const int nc = scalar == NSK_COMPLEX ? 2 : 1;
  const int64_t nk = n + k;
  nsk::Scratch r;
  NSK_CUDA_OK(r.alloc(sizeof(double) * nk * nk * nc, st));
  if (int rc = nsk::tall_qr_r(nc, m, n, static_cast<const double*>(A), lda, k, static_cast<const double*>(B), ldb,
                              r.as<double>(), st))
    return rc;
  return tls_finish(nc, nk, r.as<double>(), nk, n, k, cond_limit, allow_marginal, X, ldx, Vk, ldv, sigma, info, st);
}

int nsk_tls_solve_exact_host(int scalar, int64_t m, int64_t n, int64_t k, const void* A, int64_t lda, const void* B,
                             int64_t ldb, double cond_limit, int allow_marginal, void* X, int64_t ldx, void* Vk,
                             int64_t ldv, double* sigma, double* info) {
  if (k > 64) return nsk::fail(nsk::EINVAL_, "tls: this build supports at most 64 right-hand sides");
  if (lda < m || ldb < m || k < 1 || n < 1) return nsk::fail(nsk::EINVAL_, "tls: bad dimensions");
  cudaStream_t st = host_stream();
  const int nc = scalar == NSK_COMPLEX ? 2 : 1;
  nsk::Scratch a, b, x, v, sg;
  double *dA = nullptr, *dB = nullptr;
  if (int rc = copy_in(A, m, n, lda, nc, &dA, a, st)) return rc;
  if (int rc = copy_in(B, m, k, ldb, nc, &dB, b, st)) return rc;
  NSK_CUDA_OK(x.alloc(sizeof(double) * n * k * nc, st));
  NSK_CUDA_OK(v.alloc(sizeof(double) * (n + k) * k * nc, st));
  NSK_CUDA_OK(sg.alloc(sizeof(double) * (n + k), st));
  const int rc = nsk_tls_solve_exact(scalar, m, n, k, dA, m, dB, m, cond_limit, allow_marginal, x.p, n, v.p, n + k,
                                     sg.as<double>(), info, st);
  if (rc != NSK_OK && rc != NSK_ETLS_CONDITION) return rc;
  if (rc == NSK_OK && X) {
    if (int r2 = copy_out(X, ldx, x.as<double>(), n, k, nc, st)) return r2;
  }
  if (Vk) {
    if (int r2 = copy_out(Vk, ldv, v.as<double>(), n + k, k, nc, st)) return r2;
  }
  if (sigma) NSK_CUDA_OK(cudaMemcpyAsync(sigma, sg.p, sizeof(double) * (n + k), cudaMemcpyDeviceToHost, st));
  NSK_CUDA_OK(cudaStreamSynchronize(st));
  return rc;
}

int nsk_tls_solve_sketched_host(const nsk_operator* h, int scalar, int64_t m, int64_t n, int64_t k, const void* A,
                                int64_t lda, const void* B, int64_t ldb, double cond_limit, int allow_marginal,
                                void* X, int64_t ldx, void* Vk, int64_t ldv, double* sigma, double* info) {
  if (k > 64) return nsk::fail(nsk::EINVAL_, "tls: this build supports at most 64 right-hand sides");
  if (int rc = check_op(h)) return rc;
  const Operator& op = *OP(h);
  if (lda < m || ldb < m || k < 1 || n < 1) return nsk::fail(nsk::EINVAL_, "tls: bad dimensions");
  if (n < k) return nsk::fail(nsk::EINVAL_, "tls: need n >= k");
  if (m < n + k) return nsk::fail(nsk::EINVAL_, "tls: need m >= n + k");
  if (op.m_eff() != m) return nsk::fail(nsk::EINVAL_, "tls: sketch operator row count does not match [A|B]");
  if (op.s < n + k) return nsk::fail(nsk::EINVAL_, "tls: sketch size below n + k");
  if (int rc = validate_apply(op, scalar, m, n, A, lda, reinterpret_cast<const void*>(1), op.s, false)) return rc;
  if (int rc = validate_apply(op, scalar, m, k, B, ldb, reinterpret_cast<const void*>(1), op.s, false)) return rc;
  if (!info) return nsk::fail(nsk::EINVAL_, "tls: bad outputs");
  cudaStream_t st = host_stream();
  const int nc_in = scalar == NSK_COMPLEX ? 2 : 1, nc = out_ncomp(op, nc_in);
  nsk::Scratch a, b, sa, x, v, sg;
  // S [A | B] straight from host memory: A's H2D overlaps its sketch (host_sketch)
  NSK_CUDA_OK(sa.alloc(sizeof(double) * op.s * (n + k) * nc, st));
  if (int rc = host_sketch(op, nc_in, m, n, A, lda, a, sa.as<double>(), st, k, B, ldb, &b)) return rc;
  NSK_CUDA_OK(x.alloc(sizeof(double) * n * k * nc, st));
  NSK_CUDA_OK(v.alloc(sizeof(double) * (n + k) * k * nc, st));
  NSK_CUDA_OK(sg.alloc(sizeof(double) * (n + k), st));
  const int rc = tls_finish(nc, op.s, sa.as<double>(), op.s, n, k, cond_limit, allow_marginal, x.p, n, v.p, n + k,
                            sg.as<double>(), info, st);
  if (rc != NSK_OK && rc != NSK_ETLS_CONDITION) return rc;
  if (rc == NSK_OK && X) {
    if (int r2 = copy_out(X, ldx, x.as<double>(), n, k, nc, st)) return r2;
  }
  if (Vk) {
    if (int r2 = copy_out(Vk, ldv, v.as<double>(), n + k, k, nc, st)) return r2;
  }
  if (sigma) NSK_CUDA_OK(cudaMemcpyAsync(sigma, sg.p, sizeof(double) * (n + k), cudaMemcpyDeviceToHost, st));
  NSK_CUDA_OK(cudaStreamSynchronize(st));
  return rc;
}

}  // extern "C"
