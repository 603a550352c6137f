// bucket.cuh -- bucket-list geometry and per-batch bookkeeping shared by
// bucket.cu (kernels) and api.cu (table ownership).
#pragma once
#include "common.cuh"

namespace chb {

constexpr uint64_t COUNT_BITS = 20, TAIL_BITS = 42;
constexpr uint64_t COUNT_MAX = (1ull << COUNT_BITS) - 1, TAIL_MAX = (1ull << TAIL_BITS) - 1;
constexpr uint64_t H_UNINIT = 0, H_BLOCKED = 1, H_READY = 2, H_FULL = 3;
constexpr uint32_t FIT_DEFERRED = 0xFFFFFFFFu;

__device__ __forceinline__ uint64_t pack_handle(uint64_t state, uint64_t count, uint64_t tail) {
  return (state << (COUNT_BITS + TAIL_BITS)) | (count << TAIL_BITS) | tail;
}

struct Growth {            // exact growth geometry, host-computed (GrowthPolicy, :73-126)
  const uint64_t* sizes;   // s_b
  const uint64_t* sums;    // s_0 + ... + s_b
  uint64_t m;              // table length; sums[m-1] >= COUNT_MAX
  // bisect_left(sums, count) + 1  (:113-119)
  __device__ __forceinline__ uint64_t buckets_for(uint64_t count) const {
    if (count == 0) return 0;
    uint64_t lo = 0, hi = m;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (__ldg(sums + mid) < count) lo = mid + 1;
      else hi = mid;
    }
    return lo + 1;
  }
  // capacity_of(b): values held by buckets 0..b-1
  __device__ __forceinline__ uint64_t before(uint64_t b) const { return b ? __ldg(sums + b - 1) : 0; }
  // the same through a generic pointer (sums may point to shared memory)
  __device__ __forceinline__ uint64_t buckets_for_gen(uint64_t count) const {
    if (count == 0) return 0;
    uint64_t lo = 0, hi = m;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (sums[mid] < count) lo = mid + 1;
      else hi = mid;
    }
    return lo + 1;
  }
  __device__ __forceinline__ uint64_t before_gen(uint64_t b) const { return b ? sums[b - 1] : 0; }
  __device__ __forceinline__ uint64_t size(uint64_t b) const { return __ldg(sizes + b); }
  // arena cells of buckets [b0, b1] (bucket b > 0 spends one cell on the prev link)
  __device__ __forceinline__ uint64_t cells(uint64_t b0, uint64_t b1) const {
    return before(b1 + 1) - before(b0) + (b1 - b0 + 1) - (b0 == 0 ? 1 : 0);
  }
};

struct BucketInfo {        // per key-store slot, valid during one batch
  uint64_t region;         // arena offset of the first newly allocated bucket
  uint64_t tail_old;       // tail bucket before the batch
  uint32_t c0;             // value count before the batch
  uint32_t fit;            // values of this batch that get a cell
  uint64_t need;           // arena cells this batch allocates
  uint64_t new_count;      // published count
  uint32_t overflow;       // count limit hit -> handle becomes FULL
  uint32_t pad;
};

struct BucketRef {
  TableRef T;              // key store (value cells = handles)
  void* arena;
  uint64_t pool_cap;
  unsigned long long* bump;
  uint32_t* bcnt;          // per slot batch counts, zero at rest
  BucketInfo* info;
  ulonglong2* winfo;       // per slot, final for the batch: {region | c0 << 42, tail_old | fit << 42}
  unsigned long long* first_fail;
  Growth gr;
};

}  // namespace chb
