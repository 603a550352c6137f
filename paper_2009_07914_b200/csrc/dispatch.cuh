// dispatch.cuh -- launch plumbing: persistent-grid sizing and the runtime
// (layout, key width, value width, group width) -> template dispatch.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <mutex>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "common.cuh"

namespace chb {

// Optional CUDA-event timing of the probe kernels (bench.py: the dominant
// kernel's own duration, on the stream it runs on).
struct KernelTimer {
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
};

struct Launch {
  cudaStream_t stream;
  int device;
  int sms;
  KernelTimer* timer = nullptr;
  // probe kernels over a device-counted list (staged.cu fallback): when set, the
  // batch size is *n_dev (n is only the capacity) and results go to dst[out_idx[i]]
  const unsigned long long* n_dev = nullptr;
  const uint32_t* out_idx = nullptr;
  // per-element in-window offset to resume at (WINDOW: window 0 is known to hold
  // neither the key nor a free slot, so the probe starts at window 1)
  const uint32_t* o_start = nullptr;
  // cap on the CTAs of a chunk-scheduled kernel (0: one full wave).  A narrower
  // wave keeps the in-flight band of a region-ordered batch inside L2.
  int max_blocks = 0;
  // optional device counter of non-INSERTED statuses written by an insert
  unsigned long long* exc = nullptr;
};

struct TypeSel {
  int layout;  // SOA / AOS / PACKED
  int kbytes;  // 4 or 8
  int vbytes;  // 4 or 8
  int g;       // group width 1..32
};

// error reporting into the C ABI's thread-local message (api.cu)
void set_error(const std::string& msg);

inline int cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return 0;
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return -5;  // CH_EIO
}

// Resident CTAs per SM for a kernel at 256 threads (cached per kernel).
inline int occupancy(const void* kern, int threads) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> cache;
  std::lock_guard<std::mutex> g(mu);
  auto it = cache.find(kern);
  if (it != cache.end()) return it->second;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, 0) != cudaSuccess || occ < 1) occ = 1;
  cache[kern] = occ;
  return occ;
}

// Kernel launches issued by this library (bench.py reports them per timed region).
void count_launch(uint64_t n = 1);

// Persistent grid: one wave of CTAs (SMs x resident CTAs/SM), or fewer for
// small batches; kernels grid-stride over items.
template <typename F>
int launch_persistent(const Launch& lc, const void* kern, uint64_t items, int lanes_per_item, F&& fn,
                      int threads = 256) {
  if (items == 0) return 0;
  const uint64_t want = (items * (uint64_t)lanes_per_item + threads - 1) / threads;
  const uint64_t full = (uint64_t)lc.sms * (uint64_t)occupancy(kern, threads);
  const uint64_t blocks = want < full ? want : full;
  fn(dim3((unsigned)blocks), dim3(threads));
  count_launch();
  return cuda_check(cudaGetLastError(), "kernel launch");
}

// Chunk-scheduled probe kernels (sched.cuh): reset the table's work queue,
// then one wave of CTAs (no more CTAs than chunks).
template <typename F>
int launch_chunked(const Launch& lc, const TableRef& T, const void* kern, uint64_t items, int chunk, F&& fn,
                   int threads = 256) {
  if (items == 0) return 0;
  int rc = cuda_check(cudaMemsetAsync(T.work, 0, sizeof(unsigned long long), lc.stream), "queue reset");
  if (rc) return rc;
  const uint64_t want = (items + chunk - 1) / chunk;
  uint64_t full = (uint64_t)lc.sms * (uint64_t)occupancy(kern, threads);
  if (lc.max_blocks > 0 && (uint64_t)lc.max_blocks < full) full = (uint64_t)lc.max_blocks;
  const uint64_t blocks = want < full ? want : full;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (lc.timer && cudaEventCreate(&e0) == cudaSuccess && cudaEventCreate(&e1) == cudaSuccess)
    cudaEventRecord(e0, lc.stream);
  fn(dim3((unsigned)blocks), dim3(threads));
  count_launch();
  if (e1) {
    cudaEventRecord(e1, lc.stream);
    lc.timer->ev.emplace_back(e0, e1);
  }
  return cuda_check(cudaGetLastError(), "kernel launch");
}

template <typename T>
struct TypeTag {
  using type = T;
};

template <template <Layout, typename, typename, int> class KS, Layout LAY, typename K, typename V, typename F>
int dispatch_g(int g, F&& f) {
  switch (g) {
    case 1: return f(TypeTag<KS<LAY, K, V, 1>>{});
    case 2: return f(TypeTag<KS<LAY, K, V, 2>>{});
    case 4: return f(TypeTag<KS<LAY, K, V, 4>>{});
    case 8: return f(TypeTag<KS<LAY, K, V, 8>>{});
    case 16: return f(TypeTag<KS<LAY, K, V, 16>>{});
    case 32: return f(TypeTag<KS<LAY, K, V, 32>>{});
  }
  set_error("group_width must be one of 1,2,4,8,16,32");
  return -22;
}

template <template <Layout, typename, typename, int> class KS, typename F>
int dispatch_types(const TypeSel& ts, F&& f) {
  if (ts.layout == PACKED) {
    if (ts.kbytes == 4 && ts.vbytes == 4) return dispatch_g<KS, PACKED, uint32_t, uint32_t>(ts.g, f);
    set_error("packed layout needs 32-bit keys and values");
    return -22;
  }
#define CHB_KV(LAY)                                                                       \
  if (ts.kbytes == 4 && ts.vbytes == 4) return dispatch_g<KS, LAY, uint32_t, uint32_t>(ts.g, f); \
  if (ts.kbytes == 4 && ts.vbytes == 8) return dispatch_g<KS, LAY, uint32_t, uint64_t>(ts.g, f); \
  if (ts.kbytes == 8 && ts.vbytes == 4) return dispatch_g<KS, LAY, uint64_t, uint32_t>(ts.g, f); \
  if (ts.kbytes == 8 && ts.vbytes == 8) return dispatch_g<KS, LAY, uint64_t, uint64_t>(ts.g, f);
  if (ts.layout == SOA) { CHB_KV(SOA) }
  if (ts.layout == AOS) { CHB_KV(AOS) }
#undef CHB_KV
  set_error("unsupported layout / width combination");
  return -22;
}

// ---- entry points implemented in the .cu files (called by api.cu) ----
int single_clear(const Launch& lc, const TableRef& T, const TypeSel& ts);
int single_insert(const Launch& lc, const TableRef& T, const TypeSel& ts, const void* keys, const void* vals,
                  uint64_t n, uint8_t* status, int64_t* slot_out, int mode);
int single_lookup(const Launch& lc, const TableRef& T, const TypeSel& ts, const void* keys, uint64_t n,
                  void* vals_out, uint8_t* flag, int64_t* slot_out, uint32_t* att_out, uint32_t* win_out,
                  int mode);
int multi_insert(const Launch& lc, const TableRef& T, const TypeSel& ts, const void* keys, const void* vals,
                 uint64_t n, uint8_t* status);
// multi-value scans: hot chains handed to the CTA walker (multi.cu); the counters scratch of
// multi_scan holds 4 words and this many 24-byte entries
constexpr uint64_t kMultiHugeCap = 1ull << 16;
constexpr size_t multi_scan_counter_bytes() { return 32 + kMultiHugeCap * 24; }
// stash (count pass, mode 0): the first stash_s values of every query resolved by the thread
// pass, and per query {key, count, attempts, windows}; the retrieve pass (mode 1) copies them
// for queries whose key and count still match instead of walking again (MultiStashMeta)
struct MultiStashMeta {
  unsigned long long key;
  uint32_t total, att, win, pad;
};
int multi_scan(const Launch& lc, const TableRef& T, const TypeSel& ts, const void* keys, uint64_t n,
               uint32_t* counts, const uint64_t* offsets, void* vals_out, int mode, uint32_t* long_list,
               unsigned long long* counters, int64_t* slot_out = nullptr,
               void* stash = nullptr, void* stash_meta = nullptr, uint32_t stash_s = 0);
size_t for_all_scratch_bytes(uint64_t c);
int table_for_all(const Launch& lc, const TableRef& T, const TypeSel& ts, void* keys_out, void* vals_out,
                  int64_t* slots_out, uint64_t cap, uint64_t* d_count, void* scratch, size_t scratch_bytes);
int table_reduce(const Launch& lc, const TableRef& T, const TypeSel& ts, unsigned long long* out);
int exclusive_scan_u32(const Launch& lc, const uint32_t* counts, uint64_t n, uint64_t* out, void* scratch,
                       size_t scratch_bytes);
size_t exclusive_scan_scratch_bytes(uint64_t n);
// stable LSD radix sort of (key, payload) pairs by the whole key (rsort.cu)
size_t radix_sort_scratch_bytes(uint64_t n, int kbytes, int pbytes);
template <typename K, typename P>
int radix_sort_pairs(const Launch& lc, const K* kin, const P* pin, K* kout, P* pout, uint64_t n, void* scratch,
                     size_t scratch_bytes);
int exclusive_scan_u64(const Launch& lc, const uint64_t* counts, uint64_t n, uint64_t* out, void* scratch,
                       size_t scratch_bytes);

}  // namespace chb
