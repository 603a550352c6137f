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
#include <cstdlib>
#include <type_traits>

#include "dispatch.cuh"
#include "probe.cuh"

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

// Big groups first: their index list (m >= MG_BIG), so the longest walks start while the
// table is emptiest and no hot key is left as the kernel's tail.
constexpr uint32_t MG_BIG = 256;
constexpr uint32_t MG_SMALL = 8;  // groups below this are placed a thread per group (k_mg_small)
__global__ void k_mg_big(const uint32_t* __restrict__ gstart, const uint64_t* __restrict__ ngroups_p,
                         uint32_t* __restrict__ big, unsigned long long* __restrict__ nbig) {
  const uint64_t ng = *ngroups_p;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ng; i += stride)
    if (gstart[i + 1] - gstart[i] >= MG_BIG) big[atomicAdd(nbig, 1ull)] = (uint32_t)i;
}

// One warp per distinct key (big groups first, then the rest in sorted order, taken from
// a global counter): walk the key's sequence and claim the group's m cells in sequence
// order -- one window per step while few copies remain, MW windows per step (independent
// loads, claims assigned across the windows in order) while many do.  Statuses are
// pre-set to INSERTED; copies that find the sequence exhausted become TABLE_FULL,
// sentinel keys INVALID_KEY.
template <Layout LAY, typename K, typename V, typename P>
__global__ void __launch_bounds__(MG_THREADS) k_mg_place(TableRef T, const K* __restrict__ sk,
                                                         const P* __restrict__ sidx,
                                                         const uint32_t* __restrict__ gstart,
                                                         const uint64_t* __restrict__ ngroups_p,
                                                         const uint32_t* __restrict__ big,
                                                         const unsigned long long* __restrict__ nbig_p,
                                                         unsigned long long* __restrict__ next,
                                                         const V* __restrict__ vals, uint8_t* __restrict__ status,
                                                         int g, int mw_max) {
  constexpr int MW = 4;
  const int lane = threadIdx.x & 31;
  const uint32_t below = (1u << lane) - 1u;
  const K e = (K)T.e, tomb = (K)T.t;
  const uint32_t ug = (uint32_t)g;
  const uint64_t ngroups = *ngroups_p, nbig = *nbig_p;
  long long ops = 0, att = 0, win = 0, occ = 0;
  // one group: walk its key's sequence and claim m cells
  auto place = [&](uint64_t gi) {
    const uint32_t base = gstart[gi], m = gstart[gi + 1] - base;
    const K k = sk[base];
    if (k == e || k == tomb) {  // INVALID_KEY, no accounting (multi_table.py:213-215)
      for (uint32_t x = lane; x < m; x += 32) status[pay_idx(sidx[base + x])] = ST_INVALID;
      return;
    }
    const ProbeStart ps = probe_start(T, (uint64_t)k);
    uint64_t ws = ps.h;
    uint32_t j = 0, o = 0, placed = 0;
    bool exhausted = false;
    while (placed < m && !exhausted) {
      const uint32_t nw = m - placed > 32 ? (uint32_t)mw_max : 1u;
      K c[MW];
      uint64_t wsv[MW];
      uint64_t sv = ws;
#pragma unroll
      for (int v = 0; v < MW; ++v) {  // independent loads of nw windows
        wsv[v] = sv;
        c[v] = k;  // "not free"
        if ((uint32_t)v < nw && j + v < T.max_windows) {
          uint64_t q = sv + lane;
          if (q >= T.c) q -= T.c;
          c[v] = mg_key<LAY, K, V>(T, q);
        }
        sv += ps.step;
        if (sv >= T.c) sv -= T.c;
      }
      uint32_t taken = 0, last_v = 0, last_sel = 0;
      bool any_sel = false, stop = false;
#pragma unroll
      for (int v = 0; v < MW; ++v) {
        // a lost claim ends the step: its copy belongs to the next free cell in sequence
        // order, which may be a later cell of the same window (not one of a later window)
        if ((uint32_t)v >= nw || stop) continue;
        const bool fr = (v > 0 || (uint32_t)lane >= o) && (c[v] == e || c[v] == tomb);  // lowest free first
        const uint32_t fm = __ballot_sync(0xffffffffu, fr);
        const uint32_t want = m - placed - taken;
        const bool sel = fr && __popc(fm & below) < want;
        uint64_t q = wsv[v] + lane;
        if (q >= T.c) q -= T.c;
        const bool won = sel && mg_claim<LAY, K, V>(T, q, c[v], k);
        const uint32_t wm = __ballot_sync(0xffffffffu, won);
        if (won) {
          const uint32_t idx = placed + taken + __popc(wm & below);
          const P pv = sidx[base + idx];
          mg_store_value<LAY, K, V>(T, q, sizeof(P) == 8 ? (V)(uint32_t)pv : vals[pay_idx(pv)]);
          att += (long long)((uint64_t)(j + v) * WINDOW + chunk_end((uint32_t)lane, ug));
          win += (long long)(j + v + 1);
        }
        taken += __popc(wm);
        const uint32_t sm = __ballot_sync(0xffffffffu, sel);
        if (sm) {
          any_sel = true;
          last_v = (uint32_t)v;
          last_sel = 32u - __clz(sm);
        }
        if (sm != wm) stop = true;
      }
      placed += taken;
      if (placed >= m) break;
      // continue after the last cell tried (lost ones are occupied now); windows whose
      // free cells were all taken are behind us
      uint32_t adv;
      if (any_sel && last_sel < WINDOW) {
        adv = last_v;
        o = last_sel;
      } else {
        adv = any_sel ? last_v + 1 : nw;
        o = 0;
      }
      for (uint32_t v = 0; v < adv; ++v) {
        ++j;
        ws += ps.step;
        if (ws >= T.c) ws -= T.c;
      }
      if (j >= T.max_windows) exhausted = true;
    }
    if (lane == 0) {
      ops += m;
      occ += placed;
      const uint64_t lost = m - placed;  // sequence exhausted: TABLE_FULL, whole budget walked
      att += (long long)(lost * (uint64_t)T.max_windows * WINDOW);
      win += (long long)(lost * T.max_windows);
    }
    for (uint32_t x = placed + lane; x < m; x += 32) status[pay_idx(sidx[base + x])] = ST_TABLE_FULL;
  };
  // big groups first, one per grab (their walks are long: spread them over the warps)
  for (;;) {
    unsigned long long gi = 0;
    if (lane == 0) gi = atomicAdd(next, 1ull);
    gi = __shfl_sync(0xffffffffu, gi, 0);
    if (gi >= nbig) break;
    place(big[gi]);
  }
  // the rest in sorted order, 32 groups per grab: with few copies per key (r ~ 1) one
  // grab per group made the shared counter the kernel's limit (16.7 M atomics on one word)
  for (;;) {
    unsigned long long g0 = 0;
    if (lane == 0) g0 = atomicAdd(next + 2, 32ull);
    g0 = __shfl_sync(0xffffffffu, g0, 0);
    if (g0 >= ngroups) break;
    const uint64_t g1 = g0 + 32 < ngroups ? g0 + 32 : ngroups;
    for (uint64_t gi = g0; gi < g1; ++gi) {
      const uint32_t m = gstart[gi + 1] - gstart[gi];
      if (m < MG_BIG && m >= MG_SMALL) place(gi);  // big ones were placed above, small ones by k_mg_small
    }
  }
  const long long v[4] = {ops, att, win, occ};
  long long* const dst[4] = {(long long*)&T.ctr->ops, (long long*)&T.ctr->attempts, (long long*)&T.ctr->windows,
                             &T.ctr->occupied};
  cta_add<4>(v, dst);
}

// Groups of fewer than MG_SMALL copies (all of them when keys are unique, r = 1): one
// THREAD per group walks the sequence with 8-slot (64 B) spans and claims the group's cells
// one after another -- a warp per group left 31 lanes idle per claimed cell and measured
// 6.6 ms for 2^24 single-copy groups (latency-bound with ~9.5 K groups in flight).
// A lost CAS re-reads the span from the lost cell (single_table.py:232-233 order).
template <Layout LAY, typename K, typename V, typename P>
__global__ void __launch_bounds__(MG_THREADS) k_mg_small(TableRef T, const K* __restrict__ sk,
                                                         const P* __restrict__ sidx,
                                                         const uint32_t* __restrict__ gstart,
                                                         const uint64_t* __restrict__ ngroups_p,
                                                         const V* __restrict__ vals, uint8_t* __restrict__ status,
                                                         int g) {
  using Pr = Probe<LAY, K, V, 8>;
  using Ops = typename Pr::Ops;
  const K e = (K)T.e, tomb = (K)T.t;
  const uint32_t ug = (uint32_t)g;
  const uint64_t ngroups = *ngroups_p;
  long long ops = 0, att = 0, win = 0, occ = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t gi = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; gi < ngroups; gi += stride) {
    const uint32_t base = gstart[gi], m = gstart[gi + 1] - base;
    if (m >= MG_SMALL) continue;
    const K k = sk[base];
    if (k == e || k == tomb) {
      for (uint32_t x = 0; x < m; ++x) status[pay_idx(sidx[base + x])] = ST_INVALID;
      continue;
    }
    const ProbeStart ps = probe_start(T, (uint64_t)k);
    Cursor cur;
    cur.init(ps.h);
    uint32_t placed = 0;
    bool exhausted = false;
    while (placed < m) {
      typename Pr::Step st;
      Pr::load(T, cur, k, st);
      uint32_t fm = st.em | st.tm;
      bool lost = false;
      while (fm && placed < m) {
        const uint32_t u = lowest_bit(fm);
        const P pv = sidx[base + placed];
        const V val = sizeof(P) == 8 ? (V)(uint32_t)pv : vals[pay_idx(pv)];
        bool won = false;
        Ops::claim(T, st.base + u, ((st.em >> u) & 1u) ? e : tomb, k, val, true, &won);
        if (!won) {  // another claimant took it: re-read from this cell
          cur.o = Pr::offset_of(cur, st, u);
          lost = true;
          break;
        }
        att += (long long)(cur.attempts + chunk_end(Pr::offset_of(cur, st, u), ug));
        win += (long long)cur.windows_seen;
        ++placed;
        fm &= fm - 1;
      }
      if (placed >= m) break;
      if (!lost && !Pr::advance(T, cur, st, ps.step)) {
        exhausted = true;
        break;
      }
    }
    ops += m;
    occ += placed;
    if (exhausted) {  // TABLE_FULL for the rest, whole budget walked (as k_mg_place)
      const uint64_t left = m - placed;
      att += (long long)(left * (uint64_t)T.max_windows * WINDOW);
      win += (long long)(left * T.max_windows);
      for (uint32_t x = placed; x < m; ++x) status[pay_idx(sidx[base + x])] = ST_TABLE_FULL;
    }
  }
  const long long v[4] = {ops, att, win, occ};
  long long* const dst[4] = {(long long*)&T.ctr->ops, (long long*)&T.ctr->attempts, (long long*)&T.ctr->windows,
                             &T.ctr->occupied};
  cta_add<4>(v, dst);
}

static uint64_t al256(uint64_t x) { return (x + 255) & ~(uint64_t)255; }
static int g_mw = [] {
  const char* e = getenv("CH_MG_MW");
  const int v = e ? atoi(e) : 4;
  return v >= 1 && v <= 4 ? v : 4;
}();

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
         al256(exclusive_scan_scratch_bytes(n)) + 2 * al256((n + 1) * 4) + 256;
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
  uint32_t* big = (uint32_t*)take((n + 1) * 4);
  unsigned long long* next = (unsigned long long*)take(64);  // [0] big-group grab, [1] big groups, [2] grab
  if ((size_t)(q - static_cast<char*>(scratch)) > scratch_bytes) {
    set_error("grouped insert scratch too small");
    return -22;
  }
  int rc = cuda_check(cudaMemsetAsync(status, ST_INSERTED, n, lc.stream), "memset");
  if (!rc) rc = cuda_check(cudaMemsetAsync(next, 0, 24, lc.stream), "memset");  // big grab, nbig, small grab
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
  k_mg_big<<<grid, MG_THREADS, 0, lc.stream>>>(gstart, hoff + n, big, next + 1);
  count_launch();
  if ((rc = cuda_check(cudaGetLastError(), "group runs"))) return rc;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (lc.timer && cudaEventCreate(&e0) == cudaSuccess && cudaEventCreate(&e1) == cudaSuccess)
    cudaEventRecord(e0, lc.stream);
  k_mg_place<LAY, K, V, P><<<grid, MG_THREADS, 0, lc.stream>>>(T, sk, sidx, gstart, hoff + n, big, next + 1, next,
                                                                vals, status, g, g_mw);
  count_launch();
  k_mg_small<LAY, K, V, P><<<grid, MG_THREADS, 0, lc.stream>>>(T, sk, sidx, gstart, hoff + n, vals, status, g);
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
