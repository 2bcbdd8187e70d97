// h2d.cpp -- host -> device transfer of a caller's column-major matrix for the
// host-buffer entry points (nsk_apply_host, nsk_solve_k_host, ...).
//
// The reference's callers hold ordinary (pageable) Eigen buffers
// (matrix.hpp:32-105).  A cudaMemcpy from pageable memory is staged by the
// driver at ~11 GB/s on the B200 hosts; registering the buffer
// (cudaHostRegister) costs ~0.25 s per 2 GiB (tools/micro/h2d_paths.cu).  So a
// pageable source is streamed through a ring of 16 pinned 16 MiB slots: 8 host
// threads pack tiles of the matrix into free slots with streaming stores while
// the copy engine DMAs the filled ones (~51 GB/s for a 2 GiB matrix, against
// 55.6 GB/s from a pinned source and ~42 GB/s with ordinary memcpy stores;
// ring / slot / thread counts swept on the B200 host).  A pinned source (cudaHostAlloc / cudaHostRegister memory) is
// DMAed directly.  Either way the matrix moves in row chunks and the compute
// stream waits per chunk, so the caller can sketch chunk c while chunk c + 1
// is in flight.  On the device the chunks are laid out chunk-major: chunk c
// (rows [c chunk, c chunk + rows)) is a rows x n column-major block with
// leading dimension rows at element offset c chunk n -- with one chunk, plain
// column-major with ld m -- so the staged DMAs are contiguous runs.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <emmintrin.h>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "nsk_internal.hpp"

namespace nsk {

namespace {

constexpr int RING_MAX = 32;
// pinned slots and bytes per slot (NSK_STAGE_RING / NSK_STAGE_SLOT_MB override; defaults measured best)
int ring_slots() {
  static const int r = [] {
    const char* e = std::getenv("NSK_STAGE_RING");
    const int v = e ? std::atoi(e) : 16;
    return v >= 2 && v <= RING_MAX ? v : 16;
  }();
  return r;
}
size_t slot_bytes() {
  static const size_t b = [] {
    const char* e = std::getenv("NSK_STAGE_SLOT_MB");
    const long v = e ? std::atol(e) : 16;
    return static_cast<size_t>(v >= 1 && v <= 256 ? v : 16) << 20;
  }();
  return b;
}

struct Staging {
  std::mutex mu;  // one staged transfer at a time per process
  char* buf = nullptr;
};

// Copy into the pinned ring with streaming (non-temporal) stores: the slot is only read back by the
// copy engine, so allocating its lines in the CPU caches (and reading them first, for ordinary stores)
// would only add host memory traffic.  Head and tail up to a 16-byte boundary go through memcpy.
void copy_stream_nt(char* dst, const char* src, size_t n) {
  size_t head = (16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15;
  if (head > n) head = n;
  std::memcpy(dst, src, head);
  dst += head;
  src += head;
  n -= head;
  const size_t blocks = n / 64;
  for (size_t b = 0; b < blocks; ++b) {
    const __m128i x0 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src));
    const __m128i x1 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + 16));
    const __m128i x2 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + 32));
    const __m128i x3 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst), x0);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + 16), x1);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + 32), x2);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + 48), x3);
    src += 64;
    dst += 64;
  }
  std::memcpy(dst, src, n - blocks * 64);
}

bool stage_nt() {  // NSK_STAGE_NT=0: plain memcpy (A/B)
  static const bool v = [] {
    const char* e = std::getenv("NSK_STAGE_NT");
    return !(e && e[0] == '0');
  }();
  return v;
}

// Host threads packing the ring (NSK_STAGE_THREADS overrides; default 8, measured best of 4/8/16).
int stage_threads() {
  static const int t = [] {
    const char* e = std::getenv("NSK_STAGE_THREADS");
    const int v = e ? std::atoi(e) : 8;
    return v >= 1 && v <= 64 ? v : 8;
  }();
  return t;
}

Staging& staging() {
  static Staging s;
  return s;
}

struct Tile {
  int64_t r0, nr, c0, nc;
  int64_t chunk_end;  // > 0: last tile of the row chunk ending at this row
};

}  // namespace

namespace {
struct PinnedScratch {
  std::mutex mu;
  void* buf = nullptr;
  size_t have = 0;
};
PinnedScratch& pinned_state() {
  static PinnedScratch p;
  return p;
}
}  // namespace

std::unique_lock<std::mutex> pinned_scratch(size_t bytes, void** out) {
  PinnedScratch& ps = pinned_state();
  void*& buf = ps.buf;
  size_t& have = ps.have;
  std::unique_lock<std::mutex> lock(ps.mu);
  *out = nullptr;
  if (bytes > have) {
    if (buf) cudaFreeHost(buf);
    buf = nullptr;
    have = 0;
    if (cudaHostAlloc(&buf, bytes, cudaHostAllocPortable) != cudaSuccess) {
      cudaGetLastError();
      buf = nullptr;
      return lock;
    }
    have = bytes;
  }
  *out = buf;
  return lock;
}

// Frees the process-wide pinned host buffers (staging ring, schedule scratch) when no transfer uses
// them; the next host-buffer call allocates them again.
void release_pinned_host() {
  {
    Staging& stg = staging();
    std::lock_guard<std::mutex> lock(stg.mu);
    if (stg.buf) cudaFreeHost(stg.buf);
    stg.buf = nullptr;
  }
  PinnedScratch& ps = pinned_state();
  std::lock_guard<std::mutex> lock(ps.mu);
  if (ps.buf) cudaFreeHost(ps.buf);
  ps.buf = nullptr;
  ps.have = 0;
}

// One non-blocking copy stream per device for the life of the process (per-thread streams leaked with
// every short-lived calling thread).  Callers order their work on it with events only, so concurrent
// host-buffer calls share it safely (the copy engine serialises their DMAs anyway).
cudaStream_t copy_stream() {
  constexpr int MAXDEV = 64;
  static std::mutex mu;
  static cudaStream_t cs[MAXDEV] = {};
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur < 0 || cur >= MAXDEV) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!cs[cur] && cudaStreamCreateWithFlags(&cs[cur], cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    cs[cur] = nullptr;
  }
  return cs[cur];
}

// This thread's non-blocking compute stream on the current device for the host-buffer entry points
// (concurrent callers on different threads run independently); destroyed when the thread exits.
cudaStream_t thread_stream() {
  struct PerThread {
    cudaStream_t s[64] = {};
    ~PerThread() {
      for (cudaStream_t x : s)
        if (x) cudaStreamDestroy(x);
    }
  };
  thread_local PerThread t;
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur < 0 || cur >= 64) return nullptr;
  if (!t.s[cur] && cudaStreamCreateWithFlags(&t.s[cur], cudaStreamNonBlocking) != cudaSuccess) {
    cudaGetLastError();
    t.s[cur] = nullptr;
  }
  return t.s[cur];
}

bool host_is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

namespace {

// st waits for everything issued on cs so far.
int join_streams(cudaStream_t cs, cudaStream_t st) {
  cudaEvent_t e;
  NSK_CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  NSK_CUDA_OK(cudaEventRecord(e, cs));
  NSK_CUDA_OK(cudaStreamWaitEvent(st, e, 0));
  cudaEventDestroy(e);
  return OK;
}

// The chunk ending now on cs: its landing event goes to on_chunk (which owns it and makes its own
// stream wait on it), or st waits for it here when there is no callback.
int chunk_landed(int64_t r0, int64_t rows, cudaStream_t cs, cudaStream_t st, const ChunkFn& on_chunk) {
  if (!on_chunk) return join_streams(cs, st);
  cudaEvent_t e;
  NSK_CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  if (cudaError_t err = cudaEventRecord(e, cs)) {
    cudaEventDestroy(e);
    return cuda_fail(err, "chunk event");
  }
  return on_chunk(r0, rows, e);
}

int h2d_pinned(const char* A, int64_t m, int64_t n, int64_t lda, size_t elem, char* dA, int64_t chunk,
               int64_t dcols, cudaStream_t cs, cudaStream_t st, const ChunkFn& on_chunk) {
  for (int64_t r0 = 0; r0 < m; r0 += chunk) {
    const int64_t rows = std::min(chunk, m - r0);
    // chunk-major destination: chunk c is its own rows x dcols column-major block (ld = rows) at row
    // offset r0 * dcols, A in its first n columns
    NSK_CUDA_OK(cudaMemcpy2DAsync(dA + r0 * dcols * elem, elem * rows, A + r0 * elem, elem * lda, elem * rows, n,
                                  cudaMemcpyHostToDevice, cs));
    if (int rc = chunk_landed(r0, rows, cs, st, on_chunk)) return rc;
  }
  return OK;
}

int h2d_staged(const char* A, int64_t m, int64_t n, int64_t lda, size_t elem, char* dA, int64_t chunk,
               int64_t dcols, cudaStream_t cs, cudaStream_t st, const ChunkFn& on_chunk) {
  Staging& stg = staging();
  std::lock_guard<std::mutex> lock(stg.mu);
  const int RING = ring_slots();
  const size_t SLOT = slot_bytes();
  if (!stg.buf) NSK_CUDA_OK(cudaHostAlloc(reinterpret_cast<void**>(&stg.buf), SLOT * RING, cudaHostAllocPortable));
  // tiles: row chunks, each split into slot-sized (rows x cols) pieces
  std::vector<Tile> tiles;
  for (int64_t r0 = 0; r0 < m; r0 += chunk) {
    const int64_t rows = std::min(chunk, m - r0);
    const int64_t tr = std::max<int64_t>(1, std::min<int64_t>(rows, static_cast<int64_t>(SLOT / elem)));
    for (int64_t q0 = r0; q0 < r0 + rows; q0 += tr) {
      const int64_t nr = std::min(tr, r0 + rows - q0);
      const int64_t tc = std::max<int64_t>(1, static_cast<int64_t>(SLOT / (elem * nr)));
      for (int64_t c0 = 0; c0 < n; c0 += tc) tiles.push_back({q0, nr, c0, std::min(tc, n - c0), 0});
    }
    tiles.back().chunk_end = r0 + rows;
  }
  const size_t T = tiles.size();
  std::vector<std::atomic<int>> filled(T);
  for (auto& f : filled) f.store(0, std::memory_order_relaxed);
  std::atomic<size_t> owner[RING_MAX];
  for (int s = 0; s < RING; ++s) owner[s].store(static_cast<size_t>(s), std::memory_order_relaxed);
  std::atomic<size_t> next{0};
  std::atomic<bool> abort{false};
  const bool nt = stage_nt();
  const int nthreads = static_cast<int>(std::min<size_t>(
      std::min<unsigned>(static_cast<unsigned>(stage_threads()), std::max(1u, std::thread::hardware_concurrency())), T));
  std::vector<std::thread> workers;
  for (int w = 0; w < nthreads; ++w)
    workers.emplace_back([&]() {
      for (;;) {
        const size_t t = next.fetch_add(1);
        if (t >= T) return;
        const int s = static_cast<int>(t % RING);
        while (owner[s].load(std::memory_order_acquire) != t) {
          if (abort.load(std::memory_order_relaxed)) return;
          std::this_thread::yield();
        }
        const Tile& tl = tiles[t];
        char* dst = stg.buf + s * SLOT;
        const size_t seg = static_cast<size_t>(tl.nr) * elem;
        for (int64_t c = 0; c < tl.nc; ++c) {
          if (nt)
            copy_stream_nt(dst + c * seg, A + (tl.r0 + (tl.c0 + c) * lda) * elem, seg);
          else
            std::memcpy(dst + c * seg, A + (tl.r0 + (tl.c0 + c) * lda) * elem, seg);
        }
        if (nt) _mm_sfence();  // the streaming stores are visible before the slot is marked filled
        filled[t].store(1, std::memory_order_release);
      }
    });
  cudaEvent_t ev[RING_MAX];
  int rc = OK;
  int made = 0;
  for (; made < RING && rc == OK; ++made)
    if (cudaError_t e = cudaEventCreateWithFlags(&ev[made], cudaEventDisableTiming)) rc = cuda_fail(e, "staging event");
  for (size_t t = 0; t < T && rc == OK; ++t) {
    const int s = static_cast<int>(t % RING);
    while (!filled[t].load(std::memory_order_acquire)) std::this_thread::yield();
    const Tile& tl = tiles[t];
    // chunk-major destination (see h2d_pinned): a tile spanning the chunk's rows is one contiguous run
    const int64_t cr0 = tl.r0 / chunk * chunk, crows = std::min(chunk, m - cr0);
    char* dst = dA + (cr0 * dcols + (tl.r0 - cr0) + tl.c0 * crows) * elem;
    cudaError_t e = tl.nr == crows
                        ? cudaMemcpyAsync(dst, stg.buf + s * SLOT, elem * tl.nr * tl.nc, cudaMemcpyHostToDevice, cs)
                        : cudaMemcpy2DAsync(dst, elem * crows, stg.buf + s * SLOT, elem * tl.nr, elem * tl.nr, tl.nc,
                                            cudaMemcpyHostToDevice, cs);
    if (e == cudaSuccess) e = cudaEventRecord(ev[s], cs);
    // the previous tile's DMA runs ahead of this one: once it is done its slot goes to the tile RING later
    if (e == cudaSuccess && t >= 1) {
      const int ps = static_cast<int>((t - 1) % RING);
      e = cudaEventSynchronize(ev[ps]);
      if (e == cudaSuccess) owner[ps].store(t - 1 + RING, std::memory_order_release);
    }
    if (e != cudaSuccess) {
      rc = cuda_fail(e, "staged host-to-device copy");
      break;
    }
    if (tl.chunk_end > 0) {
      const int64_t cend = tl.chunk_end, cstart = (cend - 1) / chunk * chunk;
      rc = chunk_landed(cstart, cend - cstart, cs, st, on_chunk);
    }
  }
  if (rc != OK) abort.store(true);
  for (auto& w : workers) w.join();
  // the ring is reused by the next call: its last DMAs must be done
  if (cudaError_t e = cudaStreamSynchronize(cs); e != cudaSuccess && rc == OK) rc = cuda_fail(e, "staged copy");
  for (int i = 0; i < made; ++i) cudaEventDestroy(ev[i]);
  return rc;
}

}  // namespace

int h2d_rows(const void* A, int64_t m, int64_t n, int64_t lda, size_t elem, void* dA, int64_t chunk,
             cudaStream_t st, const ChunkFn& on_chunk, int64_t dcols) {
  if (m <= 0 || n <= 0) return OK;
  if (chunk <= 0 || chunk > m) chunk = m;
  if (dcols < n) dcols = n;
  cudaStream_t cs = copy_stream();
  if (!cs) return fail(ECUDA, "host-to-device copy: no copy stream");
  // the destination (stream-ordered allocation on st) exists before the copies start
  if (int rc = join_streams(st, cs)) return rc;
  const char* a = static_cast<const char*>(A);
  char* d = static_cast<char*>(dA);
  const bool small = static_cast<double>(m) * static_cast<double>(n) * static_cast<double>(elem) < 4.0 * (1 << 20);
  if (host_is_pinned(A) || small) return h2d_pinned(a, m, n, lda, elem, d, chunk, dcols, cs, st, on_chunk);
  return h2d_staged(a, m, n, lda, elem, d, chunk, dcols, cs, st, on_chunk);
}

}  // namespace nsk
