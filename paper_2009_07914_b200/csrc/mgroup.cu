// mgroup.cu -- grouped bulk insert for multi-value tables (multi_table.py:113-152, 207-226).
//
// The reference inserts every pair on its own: each copy of a key walks the key's COPS
// sequence past all earlier copies to the first free slot, so a key with m copies costs
// O(m^2) slot visits, and on a GPU its m copies race for the same free slot (one CAS
// winner per slot).  With Zipf-distributed keys (BASELINE configs[2]: 2^27 pairs over
// 2^23 ranks, the hottest key ~23K copies) that serialises the batch (1.7 G pairs/s).
//
// Here the batch is grouped by key first -- a radix sort of (key, position) pairs
// (CUB's DeviceRadixSort as a sort primitive; a hash-table grouping pass was tried
// first and cost 26 ms of random DRAM traffic) -- and then ONE warp per distinct key
// walks the key's sequence once: it loads a 32-slot window (a slot per lane), claims
// the free cells it needs with CAS in lane (= sequence) order, and writes the group's
// values into the cells it won.  The result is the state the reference reaches by
// inserting the m copies one after another (they fill the first m free slots of the
// sequence), i.e. a valid linearisation of the concurrent batch; per-copy probe
// counters are computed from the sequence positions, exactly as the reference counts
// them (single_table.py:197).
#include <cub/device/device_radix_sort.cuh>
#include <type_traits>

#include "dispatch.cuh"

namespace chb {

constexpr int MG_THREADS = 256;

// sort payload: the pair's position, and (32-bit values) the value itself, so the
// placing warps read a group's values contiguously instead of gathering them
template <typename P, typename V>
__global__ void k_mg_payload(P* __restrict__ x, const V* __restrict__ vals, uint64_t n) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    if constexpr (sizeof(P) == 8) x[i] = (P)i << 32 | (P)(uint32_t)vals[i];
    else x[i] = (P)i;
  }
}
template <typename P>
__device__ __forceinline__ uint32_t pay_idx(P p) { return sizeof(P) == 8 ? (uint32_t)(p >> 32) : (uint32_t)p; }

// head[i] = 1 where a run of equal keys starts in the sorted batch
template <typename K>
__global__ void k_mg_heads(const K* __restrict__ sk, uint64_t n, uint32_t* __restrict__ head) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    head[i] = (i == 0 || sk[i] != sk[i - 1]) ? 1u : 0u;
}

// gstart[g] = first sorted position of group g; gstart[ngroups] = n
__global__ void k_mg_starts(const uint32_t* __restrict__ head, const uint64_t* __restrict__ hoff, uint64_t n,
                            uint32_t* __restrict__ gstart) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    if (head[i]) gstart[hoff[i]] = (uint32_t)i;
  if (blockIdx.x == 0 && threadIdx.x == 0) gstart[hoff[n]] = (uint32_t)n;
}

// key of slot q (through L2: other SMs claim cells concurrently)
template <Layout LAY, typename K, typename V>
__device__ __forceinline__ K mg_key(const TableRef& T, uint64_t q) {
  if constexpr (LAY == PACKED) {
    return (K)__ldcg(reinterpret_cast<const uint32_t*>(T.slots) + 2 * q);
  } else if constexpr (LAY == SOA) {
    return __ldcg(static_cast<const K*>(T.slots) + q);
  } else {
    return __ldcg(&static_cast<const CellT<K, V>*>(T.slots)[q].k);
  }
}

// claim a free cell for key k (key only); true if this call won it
template <Layout LAY, typename K, typename V>
__device__ __forceinline__ bool mg_claim(const TableRef& T, uint64_t q, K expected, K k) {
  if constexpr (LAY == PACKED) {
    const uint64_t exp = (uint64_t)expected;  // free packed cells carry value 0 (layout.py:103, 231)
    return atomic_cas(static_cast<uint64_t*>(T.slots) + q, exp, (uint64_t)k) == exp;
  } else if constexpr (LAY == SOA) {
    return atomic_cas(static_cast<K*>(T.slots) + q, expected, k) == expected;
  } else {
    return atomic_cas(&static_cast<CellT<K, V>*>(T.slots)[q].k, expected, k) == expected;
  }
}

template <Layout LAY, typename K, typename V>
__device__ __forceinline__ void mg_store_value(const TableRef& T, uint64_t q, V v) {
  if constexpr (LAY == PACKED) {
    reinterpret_cast<uint32_t*>(T.slots)[2 * q + 1] = (uint32_t)v;  // value << 32 | key, little endian
  } else {
    *LayoutOps<LAY, K, V>::value_ptr(T, q) = v;
  }
}

// One warp per distinct key (groups taken from a global counter): walk the key's
// sequence window by window and claim the group's m cells in sequence order.  Statuses
// are pre-set to INSERTED; copies that find the sequence exhausted become TABLE_FULL,
// sentinel keys INVALID_KEY.
template <Layout LAY, typename K, typename V, typename P>
__global__ void __launch_bounds__(MG_THREADS) k_mg_place(TableRef T, const K* __restrict__ sk,
                                                         const P* __restrict__ sidx,
                                                         const uint32_t* __restrict__ gstart,
                                                         const uint64_t* __restrict__ ngroups_p,
                                                         unsigned long long* __restrict__ next,
                                                         const V* __restrict__ vals, uint8_t* __restrict__ status,
                                                         int g) {
  const int lane = threadIdx.x & 31;
  const uint32_t below = (1u << lane) - 1u;
  const K e = (K)T.e, tomb = (K)T.t;
  const uint32_t ug = (uint32_t)g;
  const uint64_t ngroups = *ngroups_p;
  long long ops = 0, att = 0, win = 0, occ = 0;
  for (;;) {
    unsigned long long gi = 0;
    if (lane == 0) gi = atomicAdd(next, 1ull);
    gi = __shfl_sync(0xffffffffu, gi, 0);
    if (gi >= ngroups) break;
    const uint32_t base = gstart[gi], m = gstart[gi + 1] - base;
    const K k = sk[base];
    if (k == e || k == tomb) {  // INVALID_KEY, no accounting (multi_table.py:213-215)
      for (uint32_t x = lane; x < m; x += 32) status[pay_idx(sidx[base + x])] = ST_INVALID;
      continue;
    }
    const ProbeStart ps = probe_start(T, (uint64_t)k);
    uint64_t ws = ps.h;
    uint32_t j = 0, o = 0, placed = 0;
    while (placed < m) {
      uint64_t q = ws + lane;
      if (q >= T.c) q -= T.c;
      const K c = mg_key<LAY, K, V>(T, q);
      const bool fr = (uint32_t)lane >= o && (c == e || c == tomb);  // lowest free first (:136-139)
      const uint32_t fm = __ballot_sync(0xffffffffu, fr);
      const uint32_t want = m - placed;
      const bool sel = fr && __popc(fm & below) < want;
      const bool won = sel && mg_claim<LAY, K, V>(T, q, c, k);
      const uint32_t wm = __ballot_sync(0xffffffffu, won);
      if (won) {
        const uint32_t idx = placed + __popc(wm & below);
        const P pv = sidx[base + idx];
        mg_store_value<LAY, K, V>(T, q, sizeof(P) == 8 ? (V)(uint32_t)pv : vals[pay_idx(pv)]);
        att += (long long)((uint64_t)j * WINDOW + chunk_end((uint32_t)lane, ug));
        win += (long long)(j + 1);
      }
      placed += __popc(wm);
      const uint32_t sm = __ballot_sync(0xffffffffu, sel);
      // continue after the last cell this step tried (lost ones are occupied now)
      o = sm ? 32u - __clz(sm) : 32u;
      if (o >= WINDOW && placed < m) {
        o = 0;
        ++j;
        if (j >= T.max_windows) break;
        ws += ps.step;
        if (ws >= T.c) ws -= T.c;
      }
    }
    if (lane == 0) {
      ops += m;
      occ += placed;
      const uint64_t lost = m - placed;  // sequence exhausted: TABLE_FULL, whole budget walked
      att += (long long)(lost * (uint64_t)T.max_windows * WINDOW);
      win += (long long)(lost * T.max_windows);
    }
    for (uint32_t x = placed + lane; x < m; x += 32) status[pay_idx(sidx[base + x])] = ST_TABLE_FULL;
  }
  const long long v[4] = {ops, att, win, occ};
  long long* const dst[4] = {(long long*)&T.ctr->ops, (long long*)&T.ctr->attempts, (long long*)&T.ctr->windows,
                             &T.ctr->occupied};
  cta_add<4>(v, dst);
}

static uint64_t al256(uint64_t x) { return (x + 255) & ~(uint64_t)255; }

template <typename K, typename P>
static size_t sort_temp_bytes(uint64_t n) {
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, (const K*)nullptr, (K*)nullptr, (const P*)nullptr, (P*)nullptr,
                                  (int)n);
  return tb;
}

size_t mgroup_scratch_bytes(uint64_t n, int kbytes, int vbytes) {
  const size_t sort_b = kbytes == 8 ? sort_temp_bytes<uint64_t, uint64_t>(n) : sort_temp_bytes<uint32_t, uint64_t>(n);
  (void)vbytes;
  return al256(sort_b) + al256(n * kbytes) + 2 * al256(n * 8) + al256(n * 4) + al256((n + 1) * 8) +
         al256(exclusive_scan_scratch_bytes(n)) + al256((n + 1) * 4) + 256;
}

template <Layout LAY, typename K, typename V>
static int mgroup_impl(const Launch& lc, const TableRef& T, int g, const K* keys, const V* vals, uint64_t n,
                       uint8_t* status, void* scratch, size_t scratch_bytes) {
  if (n >= (1ull << 31)) {
    set_error("grouped insert: batch too large for a 32-bit sort");
    return -22;
  }
  char* q = static_cast<char*>(scratch);
  const auto take = [&](uint64_t bytes) {
    char* r = q;
    q += al256(bytes);
    return (void*)r;
  };
  using P = typename std::conditional<sizeof(V) == 4, uint64_t, uint32_t>::type;
  size_t sort_b = sort_temp_bytes<K, P>(n);
  void* sort_tmp = take(sort_b);
  K* sk = (K*)take(n * sizeof(K));
  P* idx = (P*)take(n * 8);
  P* sidx = (P*)take(n * 8);
  uint32_t* head = (uint32_t*)take(n * 4);
  uint64_t* hoff = (uint64_t*)take((n + 1) * 8);
  const size_t scan_b = exclusive_scan_scratch_bytes(n);
  void* scan = take(scan_b);
  uint32_t* gstart = (uint32_t*)take((n + 1) * 4);
  unsigned long long* next = (unsigned long long*)take(64);
  if ((size_t)(q - static_cast<char*>(scratch)) > scratch_bytes) {
    set_error("grouped insert scratch too small");
    return -22;
  }
  int rc = cuda_check(cudaMemsetAsync(status, ST_INSERTED, n, lc.stream), "memset");
  if (!rc) rc = cuda_check(cudaMemsetAsync(next, 0, 8, lc.stream), "memset");
  if (rc) return rc;
  const unsigned grid = (unsigned)(lc.sms * 8);
  k_mg_payload<P, V><<<grid, MG_THREADS, 0, lc.stream>>>(idx, vals, n);
  count_launch();
  rc = cuda_check(cub::DeviceRadixSort::SortPairs(sort_tmp, sort_b, keys, sk, idx, sidx, (int)n, 0,
                                                  (int)(8 * sizeof(K)), lc.stream),
                  "sort by key");
  count_launch(sizeof(K) == 8 ? 8 : 4);  // onesweep passes (approximate launch count)
  if (rc) return rc;
  k_mg_heads<K><<<grid, MG_THREADS, 0, lc.stream>>>(sk, n, head);
  count_launch();
  if ((rc = exclusive_scan_u32(lc, head, n, hoff, scan, scan_b))) return rc;
  k_mg_starts<<<grid, MG_THREADS, 0, lc.stream>>>(head, hoff, n, gstart);
  count_launch();
  if ((rc = cuda_check(cudaGetLastError(), "group runs"))) return rc;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (lc.timer && cudaEventCreate(&e0) == cudaSuccess && cudaEventCreate(&e1) == cudaSuccess)
    cudaEventRecord(e0, lc.stream);
  k_mg_place<LAY, K, V, P><<<grid, MG_THREADS, 0, lc.stream>>>(T, sk, sidx, gstart, hoff + n, next, vals, status,
                                                                g);
  count_launch();
  if (e1) {
    cudaEventRecord(e1, lc.stream);
    lc.timer->ev.emplace_back(e0, e1);
  }
  return cuda_check(cudaGetLastError(), "grouped place");
}

template <Layout LAY, typename K, typename V, int G>
struct MGroupKernels {
  static int insert(const Launch& lc, const TableRef& T, const void* keys, const void* vals, uint64_t n,
                    uint8_t* status, void* scratch, size_t scratch_bytes) {
    return mgroup_impl<LAY, K, V>(lc, T, G, (const K*)keys, (const V*)vals, n, status, scratch, scratch_bytes);
  }
};

int multi_insert_grouped(const Launch& lc, const TableRef& T, const TypeSel& ts, const void* keys, const void* vals,
                         uint64_t n, uint8_t* status, void* scratch, size_t scratch_bytes) {
  return dispatch_types<MGroupKernels>(ts, [&](auto tag) {
    return decltype(tag)::type::insert(lc, T, keys, vals, n, status, scratch, scratch_bytes);
  });
}

}  // namespace chb
