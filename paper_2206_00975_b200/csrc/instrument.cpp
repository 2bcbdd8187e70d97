// instrument.cpp -- launch counter and optional CUDA-event timing of the
// dominant kernel of each apply (used by bench.py for the roofline figure).
#include <atomic>
#include <mutex>
#include <vector>

#include "../../include/nullsketch_b200.h"
#include "nsk_internal.hpp"

namespace nsk {
namespace {
std::atomic<int64_t> g_launches{0};
std::atomic<int> g_timing{0};
struct EvPair {
  cudaEvent_t a = nullptr, b = nullptr;
};
thread_local std::vector<EvPair> t_pending;
thread_local std::vector<EvPair> t_free;
thread_local const char* t_name = "";
}  // namespace

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

cudaMemPool_t scratch_pool() {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!pools[dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    uint64_t keep = UINT64_MAX;  // private pool: retained blocks only ever serve this library
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    pools[dev] = pool;
  }
  return pools[dev];
}

KernelTimer::KernelTimer(cudaStream_t s, const char* name, bool enabled) : st(s) {
  if (!enabled) return;
  if (!g_timing.load(std::memory_order_relaxed)) return;
  t_name = name;
  EvPair p;
  if (!t_free.empty()) {
    p = t_free.back();
    t_free.pop_back();
  } else {
    cudaEventCreate(&p.a);
    cudaEventCreate(&p.b);
  }
  cudaEventRecord(p.a, st);
  t_pending.push_back(p);
  pair = &t_pending.back();
}

void KernelTimer::stop() {
  if (!pair) return;
  cudaEventRecord(t_pending.back().b, st);
  pair = nullptr;
}

}  // namespace nsk

extern "C" {

int64_t nsk_kernel_launches(void) { return nsk::g_launches.load(); }

void nsk_timing_enable(int on) { nsk::g_timing.store(on ? 1 : 0); }

const char* nsk_timing_kernel(void) { return nsk::t_name; }

int nsk_release_scratch(void) {
  cudaMemPool_t pool = nsk::scratch_pool();
  if (!pool) return nsk::fail(nsk::ECUDA, "no scratch pool on this device");
  if (cudaError_t e = cudaDeviceSynchronize()) return nsk::cuda_fail(e, "release scratch");
  if (cudaError_t e = cudaMemPoolTrimTo(pool, 0)) return nsk::cuda_fail(e, "release scratch");
  nsk::release_pinned_host();
  return nsk::OK;
}

int nsk_timing_collect(double* total_ms, int64_t* count) {
  double tot = 0.0;
  int64_t c = 0;
  for (auto& p : nsk::t_pending) {
    cudaError_t e = cudaEventSynchronize(p.b);
    if (e != cudaSuccess) return nsk::cuda_fail(e, "timing collect");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.a, p.b);
    tot += ms;
    ++c;
    nsk::t_free.push_back(p);
  }
  nsk::t_pending.clear();
  if (total_ms) *total_ms = tot;
  if (count) *count = c;
  return nsk::OK;
}

}  // extern "C"
