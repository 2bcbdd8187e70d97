// operator.cpp -- SketchOperator state: draw, descriptor, device tables.
//
// Mirrors SketchOperator::draw / descriptor / from_descriptor of the
// reference (/root/reference/proj/src/sketch.cpp:103-128, 303-337).  The
// Gaussian matrix is never materialised (the reference stores s*m doubles,
// sketch.cpp:117-121); signs and hash buckets are regenerated on the device
// from stream (seed, 0).  Only the sorted sample of s indices is stored.
#include <algorithm>
#include <cstdlib>
#include <chrono>
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <string>
#include <unordered_map>

#include "nsk_internal.hpp"

namespace nsk {

namespace {
thread_local std::string g_last_error;
std::atomic<uint64_t> g_next_id{1};

inline uint32_t host_philox_word(PhiloxKey key, uint64_t i) {
  uint64_t ctr = i >> 2;
  uint32_t c0 = static_cast<uint32_t>(ctr), c1 = static_cast<uint32_t>(ctr >> 32), c2 = 0, c3 = 0;
  uint32_t k0 = key.k0, k1 = key.k1;
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = 0xD2511F53ULL * c0, p1 = 0xCD9E8D57ULL * c2;
    uint32_t n0 = static_cast<uint32_t>(p1 >> 32) ^ c1 ^ k0;
    uint32_t n1 = static_cast<uint32_t>(p1);
    uint32_t n2 = static_cast<uint32_t>(p0 >> 32) ^ c3 ^ k1;
    uint32_t n3 = static_cast<uint32_t>(p0);
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  const uint32_t w[4] = {c0, c1, c2, c3};
  return w[i & 3];
}
}  // namespace

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(ECUDA, std::string("CUDA error ") + cudaGetErrorName(e) + " (" +
                         cudaGetErrorString(e) + ") in " + what);
}

const char* last_error() { return g_last_error.c_str(); }

const char* kind_name(int kind) {
  switch (kind) {
    case GAUSSIAN: return "gaussian";
    case SRFT: return "srft";
    case SRDCT: return "srdct";
    case SRHT: return "srht";
    case COUNTSKETCH: return "countsketch";
  }
  return "unknown";
}

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (!cached[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    cached[dev] = v > 0 ? v : 148;
  }
  return cached[dev];
}

// rng.hpp:108-121 with the O(m) iota array replaced by a map of the touched
// positions: position p holds p unless it was swapped.  Step i draws the u64
// made of stream words m+2i (low) and m+2i+1 (high) -- the m sign words come
// first (sketch.cpp:122-126).
std::vector<int64_t> sample_without_replacement(PhiloxKey key, int64_t m, int64_t s) {
  std::unordered_map<int64_t, int64_t> moved;
  moved.reserve(static_cast<size_t>(2 * s + 1));
  auto get = [&](int64_t p) {
    auto it = moved.find(p);
    return it == moved.end() ? p : it->second;
  };
  for (int64_t i = 0; i < s; ++i) {
    const uint64_t w = static_cast<uint64_t>(m) + 2u * static_cast<uint64_t>(i);
    const uint64_t u = (static_cast<uint64_t>(host_philox_word(key, w + 1)) << 32) |
                       host_philox_word(key, w);
    const uint64_t below = static_cast<uint64_t>(
        (static_cast<unsigned __int128>(u) * static_cast<uint64_t>(m - i)) >> 64);
    const int64_t j = i + static_cast<int64_t>(below);
    const int64_t vi = get(i), vj = get(j);
    moved[i] = vj;
    moved[j] = vi;
  }
  std::vector<int64_t> out(static_cast<size_t>(s));
  for (int64_t i = 0; i < s; ++i) out[static_cast<size_t>(i)] = get(i);
  std::sort(out.begin(), out.end());
  return out;
}

int draw_operator(int kind, int64_t s, int64_t m, uint64_t seed, Operator** out) {
  if (!out) return fail(EINVAL_, "sketch draw: null output handle");
  *out = nullptr;
  if (kind < GAUSSIAN || kind > COUNTSKETCH)
    return fail(EINVAL_, "unknown sketch kind: " + std::to_string(kind));
  if (s < 1 || m < 1) return fail(EINVAL_, "sketch draw: s and m must be positive");
  if ((kind == SRFT || kind == SRDCT || kind == SRHT) && s > m)
    return fail(EINVAL_, "sketch draw: subsampled transforms need s <= m");
  if (kind == SRHT && (m & (m - 1)) != 0)
    return fail(EINVAL_, "sketch draw: srht needs m to be a power of two (no zero padding)");
  if (s > (int64_t(1) << 31) || m > (int64_t(1) << 40))
    return fail(EINVAL_, "sketch draw: sizes beyond the supported range");
  Operator* op = new (std::nothrow) Operator();
  if (!op) return fail(ENOMEM_, "sketch draw: out of host memory");
  op->kind = kind;
  op->s = s;
  op->m = m;
  op->seed = seed;
  op->id = g_next_id.fetch_add(1);
  op->key0 = make_key(seed, 0);
  op->key1 = make_key(seed, 1);
  if (kind == SRFT || kind == SRDCT || kind == SRHT) {
    op->idx = sample_without_replacement(op->key0, m, s);
  }
  if (kind == SRHT) {
    int lb = 0;
    while ((int64_t(1) << lb) < m && lb < 10) ++lb;
    op->srht_lo_bits = lb;
    std::vector<int32_t> order(static_cast<size_t>(s));
    for (int64_t r = 0; r < s; ++r) order[static_cast<size_t>(r)] = static_cast<int32_t>(r);
    const int64_t mask = (int64_t(1) << lb) - 1;
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
      return (op->idx[a] & mask) < (op->idx[b] & mask);
    });
    // Bank-balanced slot order for the kernel's shared-memory gather: slot t is
    // read by lane t % 32, and the value of row r_lo sits at double offset
    // r_lo + 2 (r_lo / 64) in the 2048-row kernel with 16-byte loads
    // (srht_kernel16, the usual path for m >= 2048) and at r_lo + r_lo / 32 in
    // the 8-byte kernels, i.e. in 8-byte bank pair (offset % 16).  Fill each
    // half-warp (16 consecutive slots) with distinct bank pairs where the
    // sample allows it, taking rows in increasing r_lo within each class.
    if (lb == 10) {
      const bool v16 = m >= 2048;
      std::vector<std::vector<int32_t>> cls(16);
      for (int32_t r : order) {
        const int64_t lo = op->idx[static_cast<size_t>(r)] & (v16 ? 2047 : mask);
        cls[static_cast<size_t>((v16 ? lo + 2 * (lo >> 6) : lo + (lo >> 5)) & 15)].push_back(r);
      }
      // Spread every class evenly over the ceil(s / 16) half-warps: half-warp h takes
      // ceil(remaining_c / half-warps left) rows of class c, trimmed or topped up to 16 by
      // the classes whose share is furthest from a whole row.  A half-warp costs as many
      // wavefronts as its largest class multiplicity (97 -> 80 for the 64 half-warps of
      // configs[1]; 76 is the bound set by the largest class).
      std::vector<size_t> head(16, 0);
      std::vector<int32_t> balanced;
      balanced.reserve(order.size());
      const int64_t nh = (s + 15) / 16;
      for (int64_t h = 0; h < nh; ++h) {
        const double hl = static_cast<double>(nh - h);
        int64_t cnt[16], take[16], sum = 0, avail = 0;
        for (int c = 0; c < 16; ++c) {
          cnt[c] = static_cast<int64_t>(cls[static_cast<size_t>(c)].size() - head[static_cast<size_t>(c)]);
          take[c] = (cnt[c] + (nh - h) - 1) / (nh - h);
          sum += take[c];
          avail += cnt[c];
        }
        while (sum > 16) {
          int best = -1;
          double bv = 0.0;
          for (int c = 0; c < 16; ++c)
            if (take[c] > 0) {
              const double v = static_cast<double>(cnt[c]) / hl - static_cast<double>(take[c] - 1);
              if (best < 0 || v < bv) {
                best = c;
                bv = v;
              }
            }
          --take[best];
          --sum;
        }
        while (sum < 16 && sum < avail) {
          int best = -1;
          double bv = 0.0;
          for (int c = 0; c < 16; ++c)
            if (cnt[c] > take[c]) {
              const double v = static_cast<double>(cnt[c]) / hl - static_cast<double>(take[c]);
              if (best < 0 || v > bv) {
                best = c;
                bv = v;
              }
            }
          ++take[best];
          ++sum;
        }
        for (int c = 0; c < 16; ++c)
          for (int64_t t = 0; t < take[c]; ++t)
            balanced.push_back(cls[static_cast<size_t>(c)][head[static_cast<size_t>(c)]++]);
      }
      order.swap(balanced);
    }
    op->srht_slot.resize(static_cast<size_t>(s));
    op->srht_row.resize(static_cast<size_t>(s));
    for (int64_t t = 0; t < s; ++t) {
      op->srht_row[static_cast<size_t>(t)] = order[static_cast<size_t>(t)];
      op->srht_slot[static_cast<size_t>(t)] =
          static_cast<uint32_t>(op->idx[static_cast<size_t>(order[static_cast<size_t>(t)])]);
    }
  }
  *out = op;
  return OK;
}

const DeviceTables* Operator::tables(int64_t row_lo, int64_t row_hi) const {
  int devno = 0;
  if (cudaGetDevice(&devno) != cudaSuccess) return nullptr;
  if (row_hi < 0) row_hi = m;
  const bool window = kind == COUNTSKETCH && row_hi > row_lo;
  std::lock_guard<std::mutex> lock(mu);
  for (auto& t : dev)
    if (t.device == devno && (!window || (t.cs_base <= row_lo && row_hi <= t.cs_base + t.cs_rows))) return &t;
  DeviceTables t;
  t.device = devno;
  // a failed build frees what it allocated (the next call retries from scratch)
  auto bail = [&t]() -> const DeviceTables* {
    void* ptrs[] = {t.idx, t.srht_slot, t.srht_row, t.sign_mask, t.cs_table, t.sign_bits, t.srtt_freq, t.srtt_row,
                    t.srdct_sgn, t.srft_sgn, t.dct_freq, t.dct_row, t.cs_ent, t.cs_cnt};
    for (void* q : ptrs)
      if (q) cudaFree(q);
    return nullptr;
  };
  if (window) {  // tile-aligned window around the requested rows
    t.cs_base = row_lo / CS_T * CS_T;
    t.cs_rows = std::min<int64_t>(m, (row_hi + CS_T - 1) / CS_T * CS_T) - t.cs_base;
  }
  auto up = [](void** dst, const void* src, size_t bytes) {
    if (bytes == 0) return cudaSuccess;
    cudaError_t e = cudaMalloc(dst, bytes);
    if (e != cudaSuccess) return e;
    return cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice);
  };
  cudaError_t e = cudaSuccess;
  if (!idx.empty()) e = up(reinterpret_cast<void**>(&t.idx), idx.data(), idx.size() * 8);
  if (e == cudaSuccess && !srht_slot.empty())
    e = up(reinterpret_cast<void**>(&t.srht_slot), srht_slot.data(), srht_slot.size() * 4);
  if (e == cudaSuccess && !srht_row.empty())
    e = up(reinterpret_cast<void**>(&t.srht_row), srht_row.data(), srht_row.size() * 4);
  if (e != cudaSuccess) {
    cuda_fail(e, "operator table upload");
    return bail();
  }
  if (kind == SRHT && m >= 1024 && build_sign_mask(key0, m, &t.sign_mask) != OK) return bail();
  if (kind == COUNTSKETCH && s <= 65536 && build_cs_table(key0, m, s, t.cs_base, t.cs_rows, &t.cs_table) != OK)
    return bail();
  if (kind == COUNTSKETCH && t.cs_rows > 0 && cs_owner_eligible(s, m)) {
    // Owner schedule over the window's full CS_T-row tiles, from the device row table.
    const bool dbg = std::getenv("NSK_TABLES_DEBUG") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    const auto t0 = now();
    const int64_t ntiles = t.cs_rows / CS_T;
    // one pinned buffer: [table (ntiles CS_T u32) | schedule entries | counts]
    const size_t per_tile = static_cast<size_t>(CS_WARPS) * CS_GMAX * 32;
    const size_t tab_b = static_cast<size_t>(ntiles) * CS_T * 4, ent_b = static_cast<size_t>(ntiles) * per_tile * 8,
                 cnt_b = static_cast<size_t>(ntiles) * CS_WARPS;
    void* hbuf = nullptr;
    auto hold = pinned_scratch(tab_b + ent_b + cnt_b, &hbuf);
    if (!hbuf) {
      fail(ENOMEM_, "countsketch schedule: pinned host scratch");
      return bail();
    }
    uint32_t* tab = static_cast<uint32_t*>(hbuf);
    uint64_t* ent = reinterpret_cast<uint64_t*>(static_cast<char*>(hbuf) + tab_b);
    uint8_t* cnt = reinterpret_cast<uint8_t*>(ent) + ent_b;
    if (cudaMemcpy(tab, t.cs_table, tab_b, cudaMemcpyDeviceToHost) != cudaSuccess) {
      cuda_fail(cudaGetLastError(), "countsketch table readback");
      return bail();
    }
    const auto t1 = now();
    if (ntiles > 0 && build_cs_schedule_into(tab, ntiles, CS_T, s, ent, cnt) == OK) {
      const auto t2 = now();
      if (up(reinterpret_cast<void**>(&t.cs_ent), ent, ent_b) != cudaSuccess ||
          up(reinterpret_cast<void**>(&t.cs_cnt), cnt, cnt_b) != cudaSuccess) {
        cuda_fail(cudaGetLastError(), "countsketch schedule upload");
        return bail();
      }
      t.cs_ntiles = ntiles;
      if (dbg) {
        auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
        std::fprintf(stderr, "nsk tables: cs readback %.1f ms, schedule %.1f ms, upload %.1f ms (%zu MB)\n",
                     ms(t0, t1), ms(t1, t2), ms(t2, now()), ent_b >> 20);
      }
    }  // else: the streaming kernel covers every tile
  }
  if ((kind == SRFT || kind == SRDCT) && build_sign_bits(key0, m, &t.sign_bits) != OK) return bail();
  if (kind == SRFT && build_srft_sgn(t.sign_bits, m, &t.srft_sgn) != OK) return bail();
  if (kind == SRDCT && build_srdct_sgn(t.sign_bits, m, &t.srdct_sgn) != OK) return bail();
  if ((kind == SRFT || kind == SRDCT) && !idx.empty()) {
    // Slots sorted by FFT bin (idx mod 1024) for the tile kernel (srtt_tile.cu).
    std::vector<int32_t> order(idx.size());
    for (size_t r = 0; r < idx.size(); ++r) order[r] = static_cast<int32_t>(r);
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
      return (idx[static_cast<size_t>(a)] & 1023) < (idx[static_cast<size_t>(b)] & 1023);
    });
    std::vector<int64_t> freq(idx.size());
    for (size_t r = 0; r < idx.size(); ++r) freq[r] = idx[static_cast<size_t>(order[r])];
    if (up(reinterpret_cast<void**>(&t.srtt_freq), freq.data(), freq.size() * 8) != cudaSuccess ||
        up(reinterpret_cast<void**>(&t.srtt_row), order.data(), order.size() * 4) != cudaSuccess) {
      cuda_fail(cudaGetLastError(), "srtt slot table upload");
      return bail();
    }
  }
  if (kind == SRDCT && !idx.empty()) {
    // Makhoul index of each sample (srdct_stream.cu): y_{2n} = v_n, y_{2n+1} = v_{m-1-n}.
    std::vector<int64_t> nv(idx.size());
    for (size_t r = 0; r < idx.size(); ++r) {
      const int64_t a = idx[r];
      nv[r] = (a & 1) == 0 ? a / 2 : m - 1 - (a - 1) / 2;
    }
    std::vector<int32_t> order(idx.size());
    for (size_t r = 0; r < idx.size(); ++r) order[r] = static_cast<int32_t>(r);
    std::stable_sort(order.begin(), order.end(), [&](int32_t a, int32_t b) {
      return (nv[static_cast<size_t>(a)] & 1023) < (nv[static_cast<size_t>(b)] & 1023);
    });
    std::vector<int64_t> freq(idx.size());
    for (size_t r = 0; r < idx.size(); ++r) freq[r] = nv[static_cast<size_t>(order[r])];
    if (up(reinterpret_cast<void**>(&t.dct_freq), freq.data(), freq.size() * 8) != cudaSuccess ||
        up(reinterpret_cast<void**>(&t.dct_row), order.data(), order.size() * 4) != cudaSuccess) {
      cuda_fail(cudaGetLastError(), "srdct slot table upload");
      return bail();
    }
  }
  dev.push_back(t);
  return &dev.back();
}

bool Operator::is_zeroed(int64_t j) const { return std::binary_search(zeroed.begin(), zeroed.end(), j); }

int Operator::zero_mask(const uint32_t** out) const {
  *out = nullptr;
  if (zeroed.empty()) return OK;
  int devno = 0;
  NSK_CUDA_OK(cudaGetDevice(&devno));
  std::lock_guard<std::mutex> lock(mu);
  if (zmask_version != state_version) {  // operator changed: drop every device copy
    if (!zmask_dev.empty()) cudaDeviceSynchronize();  // earlier applies may still read them
    for (auto& d : zmask_dev) {
      cudaSetDevice(d.first);
      cudaFree(d.second);
    }
    cudaSetDevice(devno);
    zmask_dev.clear();
    zmask_version = state_version;
  }
  for (auto& d : zmask_dev)
    if (d.first == devno) {
      *out = d.second;
      return OK;
    }
  const int64_t words = (m_eff() + 31) / 32;
  std::vector<uint32_t> bits(static_cast<size_t>(words), 0u);
  for (int64_t j : zeroed) bits[static_cast<size_t>(j >> 5)] |= 1u << (j & 31);
  uint32_t* d = nullptr;
  NSK_CUDA_OK(cudaMalloc(&d, sizeof(uint32_t) * words));
  if (cudaError_t e = cudaMemcpy(d, bits.data(), sizeof(uint32_t) * words, cudaMemcpyHostToDevice)) {
    cudaFree(d);
    return cuda_fail(e, "zeroed-row mask upload");
  }
  zmask_dev.emplace_back(devno, d);
  *out = d;
  return OK;
}

Operator::~Operator() {
  int cur = 0;
  cudaGetDevice(&cur);
  for (auto& t : shard_tabs) {
    cudaSetDevice(t.device);
    void* ptrs[] = {t.bits, t.sgn, t.freq, t.row, t.post};
    for (void* q : ptrs)
      if (q) cudaFree(q);
  }
  for (auto& d : zmask_dev) {
    cudaSetDevice(d.first);
    cudaFree(d.second);
  }
  for (auto& t : dev) {
    cudaSetDevice(t.device);
    if (t.idx) cudaFree(t.idx);
    if (t.srht_slot) cudaFree(t.srht_slot);
    if (t.srht_row) cudaFree(t.srht_row);
    if (t.sign_mask) cudaFree(t.sign_mask);
    if (t.cs_table) cudaFree(t.cs_table);
    if (t.sign_bits) cudaFree(t.sign_bits);
    if (t.srtt_freq) cudaFree(t.srtt_freq);
    if (t.srtt_row) cudaFree(t.srtt_row);
    if (t.srft_sgn) cudaFree(t.srft_sgn);
    if (t.srdct_sgn) cudaFree(t.srdct_sgn);
    if (t.dct_freq) cudaFree(t.dct_freq);
    if (t.dct_row) cudaFree(t.dct_row);
    if (t.cs_ent) cudaFree(t.cs_ent);
    if (t.cs_cnt) cudaFree(t.cs_cnt);
  }
  cudaSetDevice(cur);
}

}  // namespace nsk
