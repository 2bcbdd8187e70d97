// Host -> device paths for a 2 GiB pageable buffer (the e2e input of configs[1]):
//   (a) cudaMemcpyAsync straight from pageable memory (driver staging)
//   (b) cudaHostRegister + copy + cudaHostUnregister
//   (c) T host threads memcpy pageable -> a ring of pinned staging chunks, DMA from the ring
//   (d) reference: pinned source
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a h2d_paths.cu -o h2d_paths -lpthread
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) {                                                            \
      std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));   \
      std::exit(1);                                                                    \
    }                                                                                  \
  } while (0)

int main(int argc, char** argv) {
  const size_t bytes = size_t(2) << 30;
  char* h = static_cast<char*>(std::malloc(bytes));
  std::memset(h, 1, bytes);
  char* d;
  CK(cudaMalloc(&d, bytes));
  cudaStream_t st;
  CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  auto report = [&](const char* name, double t) { std::printf("%-44s %8.2f ms  %6.1f GB/s\n", name, t * 1e3, bytes / t / 1e9); };
  for (int rep = 0; rep < 2; ++rep) {
    double t0 = now();
    CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    report("(a) pageable cudaMemcpyAsync", now() - t0);
  }
  for (int rep = 0; rep < 2; ++rep) {
    double t0 = now();
    CK(cudaHostRegister(h, bytes, cudaHostRegisterDefault));
    double t1 = now();
    CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    double t2 = now();
    CK(cudaHostUnregister(h));
    double t3 = now();
    report("(b) register + copy + unregister", t3 - t0);
    std::printf("    register %.2f ms copy %.2f ms unregister %.2f ms\n", (t1 - t0) * 1e3, (t2 - t1) * 1e3,
                (t3 - t2) * 1e3);
  }
  for (int T : {4, 8, 16}) {
    for (size_t chunk : {size_t(8) << 20, size_t(32) << 20}) {
      const int ring = 2 * T;
      char* pin;
      CK(cudaMallocHost(&pin, chunk * ring));
      std::vector<cudaEvent_t> ev(ring);
      for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      const size_t nchunks = (bytes + chunk - 1) / chunk;
      for (int rep = 0; rep < 2; ++rep) {
        double t0 = now();
        // chunk c goes through ring slot c % ring; worker threads fill, the main thread DMAs in order
        std::vector<std::atomic<int>> filled(nchunks);
        for (auto& f : filled) f.store(0);
        std::vector<std::atomic<int>> slot_free(ring);
        for (auto& f : slot_free) f.store(1);
        std::atomic<size_t> next{0};
        std::vector<std::thread> th;
        std::vector<std::atomic<size_t>> slot_owner(ring);
        for (int s = 0; s < ring; ++s) slot_owner[s].store(s);
        for (int t = 0; t < T; ++t)
          th.emplace_back([&]() {
            for (;;) {
              size_t c = next.fetch_add(1);
              if (c >= nchunks) return;
              const int s = static_cast<int>(c % ring);
              while (slot_owner[s].load(std::memory_order_acquire) != c) std::this_thread::yield();
              size_t len = c + 1 == nchunks ? bytes - c * chunk : chunk;
              std::memcpy(pin + s * chunk, h + c * chunk, len);
              filled[c].store(1, std::memory_order_release);
            }
          });
        for (size_t c = 0; c < nchunks; ++c) {
          const int s = static_cast<int>(c % ring);
          while (!filled[c].load(std::memory_order_acquire)) std::this_thread::yield();
          size_t len = c + 1 == nchunks ? bytes - c * chunk : chunk;
          CK(cudaMemcpyAsync(d + c * chunk, pin + s * chunk, len, cudaMemcpyHostToDevice, st));
          CK(cudaEventRecord(ev[s], st));
          // the previous chunk's DMA is queued ahead of this one: once it is done, its slot goes to the
          // chunk `ring` places later (one DMA running, one queued, the workers fill ahead)
          if (c >= 1) {
            const int ps = static_cast<int>((c - 1) % ring);
            CK(cudaEventSynchronize(ev[ps]));
            if (c - 1 + ring < nchunks) slot_owner[ps].store(c - 1 + ring, std::memory_order_release);
          }
        }
        CK(cudaStreamSynchronize(st));
        for (auto& x : th) x.join();
        char name[96];
        std::snprintf(name, sizeof(name), "(c) %2d threads, %2zu MiB staging chunks", T, chunk >> 20);
        report(name, now() - t0);
      }
      for (auto& e : ev) cudaEventDestroy(e);
      cudaFreeHost(pin);
    }
  }
  char* hp;
  CK(cudaMallocHost(&hp, bytes));
  std::memset(hp, 1, bytes);
  for (int rep = 0; rep < 2; ++rep) {
    double t0 = now();
    CK(cudaMemcpyAsync(d, hp, bytes, cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
    report("(d) pinned cudaMemcpyAsync", now() - t0);
  }
  return 0;
}
