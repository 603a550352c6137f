// mgroup.cu -- grouped bulk insert for multi-value tables (multi_table.py:113-152, 207-226).
//
// The reference inserts every pair on its own: each copy of a key walks the key's COPS
// sequence past all earlier copies to the first free slot, so a key with m copies costs
// O(m^2) slot visits, and on a GPU its m copies race for the same free slot (one CAS
// winner per slot).  With Zipf-distributed keys (BASELINE configs[2]: 2^27 pairs over
// 2^23 ranks, the hottest key ~23K copies) that serialises the batch (1.7 G pairs/s).
//
// Here the batch is grouped by key first -- a stable radix sort of (key, position) pairs
// (rsort.cu; CUB's DeviceRadixSort with CH_MG_CUB=1; a hash-table grouping pass was
// tried first and cost 26 ms of random DRAM traffic) -- and then ONE warp per distinct key
// walks the key's sequence once: it loads a 32-slot window (a slot per lane), claims
// the free cells it needs with CAS in lane (= sequence) order, and writes the group's
// values into the cells it won.  The result is the state the reference reaches by
// inserting the m copies one after another (they fill the first m free slots of the
// sequence), i.e. a valid linearisation of the concurrent batch; per-copy probe
// counters are computed from the sequence positions, exactly as the reference counts
// them (single_table.py:197).
#include <cub/device/device_radix_sort.cuh>
#include <algorithm>
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

// Runs of equal keys in the sorted batch, in one pass: gstart[g] = first sorted position of
// group g, gstart[ngroups] = n, *ngroups.  Tiles of 4096 keys in start order (atomic tile
// counter); a warp owns 256 consecutive keys (eight ballots of run heads), a block scan
// over the warps numbers the tile's heads and a decoupled look-back by warp 0 (one status
// word per tile: flag << 62 | heads, 32 predecessors per step) numbers the tile's first head.  (Was: head flags, a scan of
// 2^27 u32 into u64 and a scatter -- 1.2 ms of the 2^27 Zipf insert.)
constexpr int MR_T = 512, MR_I = 8;
constexpr uint32_t MR_TILE = MR_T * MR_I;
constexpr uint64_t MR_AGG = 1ull << 62, MR_INC = 2ull << 62, MR_VAL = (1ull << 62) - 1;
template <typename K>
__global__ void __launch_bounds__(MR_T) k_mg_runs(const K* __restrict__ sk, uint64_t n, uint32_t* __restrict__ gstart,
                                                  unsigned long long* __restrict__ ngroups,
                                                  unsigned long long* __restrict__ status,
                                                  unsigned int* __restrict__ next_tile) {
  __shared__ uint32_t s_t, wsum[MR_T / 32];
  __shared__ unsigned long long s_pre;
  if (threadIdx.x == 0) s_t = atomicAdd(next_tile, 1u);
  __syncthreads();
  const uint32_t t = s_t;
  const uint64_t base = (uint64_t)t * MR_TILE;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  K k[MR_I];
  K before = 0;  // the key just before the warp's first (lane 0)
#pragma unroll
  for (int r = 0; r < MR_I; ++r) {
    const uint64_t i = base + warp * 32u * MR_I + (uint32_t)r * 32u + lane;
    k[r] = i < n ? sk[i] : (K)0;
  }
  {
    const uint64_t i0 = base + warp * 32u * MR_I;
    if (lane == 0 && i0 > 0 && i0 < n) before = sk[i0 - 1];
  }
  uint32_t bal[MR_I], cnt = 0;
#pragma unroll
  for (int r = 0; r < MR_I; ++r) {
    const uint64_t i = base + warp * 32u * MR_I + (uint32_t)r * 32u + lane;
    K prev = __shfl_up_sync(0xffffffffu, k[r], 1);
    const K last = __shfl_sync(0xffffffffu, k[r], 31);  // the next round's lane 0 compares with it
    if (lane == 0) prev = before;
    before = last;
    const bool head = i < n && (i == 0 || k[r] != prev);
    bal[r] = __ballot_sync(0xffffffffu, head);
    cnt += (uint32_t)__popc(bal[r]);
  }
  if (lane == 0) wsum[warp] = cnt;
  __syncthreads();
  uint32_t woff = 0, tot = 0;
#pragma unroll
  for (int w = 0; w < MR_T / 32; ++w) {
    const uint32_t x = wsum[w];
    woff += w < (int)warp ? x : 0u;
    tot += x;
  }
  if (warp == 0) {  // publish, then look back with the whole warp (32 predecessors per step)
    volatile unsigned long long* const st = status;
    if (lane == 0) st[t] = (t == 0 ? MR_INC : MR_AGG) | tot;
    uint64_t pre = 0;
    for (int64_t j = (int64_t)t - 1; j >= 0;) {
      const int64_t q = j - (int64_t)lane;
      const uint64_t sv = q >= 0 ? st[q] : MR_INC;  // before tile 0: an inclusive zero
      const unsigned inc = __ballot_sync(0xffffffffu, (sv & MR_INC) != 0);
      const unsigned nr = __ballot_sync(0xffffffffu, (sv & ~MR_VAL) == 0);
      const unsigned upto = inc ? (inc & (0u - inc)) * 2u - 1u : 0xffffffffu;  // lanes through the nearest INC
      if (nr & upto) continue;  // an unpublished tile on the way: read again
      uint64_t v = (lane < 32u && ((upto >> lane) & 1u)) ? (sv & MR_VAL) : 0ull;
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
      pre += v;
      if (inc) break;
      j -= 32;
    }
    if (lane == 0) {
      if (t) st[t] = MR_INC | (pre + tot);
      s_pre = pre;
      if (base + MR_TILE >= n) {  // the last tile: the sentinel start and the group count
        gstart[pre + tot] = (uint32_t)n;
        *ngroups = pre + tot;
      }
    }
  }
  __syncthreads();
  uint64_t g = s_pre + woff;
#pragma unroll
  for (int r = 0; r < MR_I; ++r) {
    const uint64_t i = base + warp * 32u * MR_I + (uint32_t)r * 32u + lane;
    if ((bal[r] >> lane) & 1u) gstart[g + (uint32_t)__popc(bal[r] & lt)] = (uint32_t)i;
    g += (uint32_t)__popc(bal[r]);
  }
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
constexpr uint32_t MG_HUGE = 8192;  // groups this large are placed a CTA per group (k_mg_place_cta)
__global__ void k_mg_big(const uint32_t* __restrict__ gstart, const uint64_t* __restrict__ ngroups_p,
                         uint32_t* __restrict__ big, unsigned long long* __restrict__ nbig,
                         uint32_t* __restrict__ huge, unsigned long long* __restrict__ nhuge) {
  const uint64_t ng = *ngroups_p;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < ng; i += stride) {
    const uint32_t m = gstart[i + 1] - gstart[i];
    if (m >= MG_HUGE) huge[atomicAdd(nhuge, 1ull)] = (uint32_t)i;
    else if (m >= MG_BIG) big[atomicAdd(nbig, 1ull)] = (uint32_t)i;
  }
}

// The hottest groups (>= MG_HUGE copies: a Zipf s = 0.75 batch of 2^27 pairs has keys with
// ~6 * 10^5) placed one CTA per group, 128 windows per step (16 warps x 8, independent loads:
// the window starts h + j step are known up front): a block scan of the windows' free cells
// hands the group's next copies the first free cells in sequence order, every lane claims its
// cell with CAS, and the values go to the cells won, in sequence order.  A cell lost to another
// key is occupied afterwards, so the copies still fill the first free cells of the sequence
// (the reference inserting them one after another, the others' claims linearised first); the
// next step resumes after the last cell tried.  Runs before k_mg_place, on the emptiest table.
template <Layout LAY, typename K, typename V, typename P>
__global__ void __launch_bounds__(512) k_mg_place_cta(TableRef T, const K* __restrict__ sk,
                                                      const P* __restrict__ sidx,
                                                      const uint32_t* __restrict__ gstart,
                                                      const uint32_t* __restrict__ huge,
                                                      const unsigned long long* __restrict__ nhuge_p,
                                                      unsigned long long* __restrict__ grab,
                                                      const V* __restrict__ vals, uint8_t* __restrict__ status, int g) {
  constexpr uint32_t NWARP = 16, WPW = 8, WSTEP = NWARP * WPW;
  __shared__ uint32_t s_free[WSTEP], s_pre[WSTEP], s_won[WSTEP], s_wpre[WSTEP];
  __shared__ uint32_t s_tot, s_wtot, s_lastx, s_lastlane;
  __shared__ unsigned long long s_item;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint32_t below = (1u << lane) - 1u;
  const K e = (K)T.e, tomb = (K)T.t;
  const uint32_t ug = (uint32_t)g;
  const unsigned long long nh = *nhuge_p;
  long long ops = 0, att = 0, win = 0, occ = 0;
  // exclusive scan of x[0..WSTEP) by warp 0 into pre; returns the total (all warp-0 lanes)
  auto scan128 = [&](const uint32_t* x, uint32_t* pre) -> uint32_t {
    uint32_t run = 0;
    for (uint32_t x0 = 0; x0 < WSTEP; x0 += 32) {
      const uint32_t cx = x[x0 + lane];
      uint32_t inc = cx;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
        if ((int)lane >= d) inc += y;
      }
      pre[x0 + lane] = run + inc - cx;
      run += __shfl_sync(0xffffffffu, inc, 31);
    }
    return run;
  };
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(grab, 1ull);
    __syncthreads();
    const unsigned long long item = s_item;
    __syncthreads();
    if (item >= nh) break;
    const uint32_t gi = huge[item];
    const uint32_t base = gstart[gi], m = gstart[gi + 1] - base;
    const K k = sk[base];
    if (k == e || k == tomb) {  // INVALID_KEY, no accounting (multi_table.py:213-215)
      for (uint32_t x = threadIdx.x; x < m; x += blockDim.x) status[pay_idx(sidx[base + x])] = ST_INVALID;
      continue;
    }
    const ProbeStart ps = probe_start(T, (uint64_t)k);
    uint64_t jb = 0, wsb = ps.h;
    uint32_t o = 0, placed = 0;
    bool exhausted = false;
    while (placed < m && !exhausted) {  // CTA-uniform
      const uint32_t need = m - placed;
      uint64_t ws = T.modc.mod(wsb + (uint64_t)(warp * WPW) * ps.step);
      K c[WPW];
      uint32_t fmv[WPW];
#pragma unroll
      for (uint32_t v = 0; v < WPW; ++v) {
        const uint64_t jj = jb + warp * WPW + v;
        uint64_t q = ws + lane;
        if (q >= T.c) q -= T.c;
        c[v] = jj < T.max_windows ? mg_key<LAY, K, V>(T, q) : k;  // past the budget: "not free"
        ws += ps.step;
        if (ws >= T.c) ws -= T.c;
      }
#pragma unroll
      for (uint32_t v = 0; v < WPW; ++v) {
        const uint32_t x = warp * WPW + v;
        const bool fr = (x > 0 || lane >= o) && (c[v] == e || c[v] == tomb);  // lowest free first
        fmv[v] = __ballot_sync(0xffffffffu, fr);
        if (lane == 0) s_free[x] = __popc(fmv[v]);
      }
      __syncthreads();
      if (warp == 0) {
        const uint32_t tot = scan128(s_free, s_pre);
        if (lane == 0) s_tot = tot;
      }
      __syncthreads();
      // the first `need` free cells in sequence order: claim them
      const uint32_t tot = s_tot, take = need < tot ? need : tot;
      uint32_t wonv[WPW];
      ws = T.modc.mod(wsb + (uint64_t)(warp * WPW) * ps.step);
#pragma unroll
      for (uint32_t v = 0; v < WPW; ++v) {
        const uint32_t x = warp * WPW + v;
        const uint32_t rank = s_pre[x] + __popc(fmv[v] & below);
        const bool sel = ((fmv[v] >> lane) & 1u) && rank < take;
        uint64_t q = ws + lane;
        if (q >= T.c) q -= T.c;
        const bool won = sel && mg_claim<LAY, K, V>(T, q, c[v], k);
        wonv[v] = __ballot_sync(0xffffffffu, won);
        if (lane == 0) s_won[x] = __popc(wonv[v]);
        if (sel && rank == take - 1) {  // the last cell tried
          s_lastx = x;
          s_lastlane = lane;
        }
        ws += ps.step;
        if (ws >= T.c) ws -= T.c;
      }
      __syncthreads();
      if (warp == 0) {
        const uint32_t wt = scan128(s_won, s_wpre);
        if (lane == 0) s_wtot = wt;
      }
      __syncthreads();
      // values of the copies, in sequence order of the cells won
      ws = T.modc.mod(wsb + (uint64_t)(warp * WPW) * ps.step);
#pragma unroll
      for (uint32_t v = 0; v < WPW; ++v) {
        const uint32_t x = warp * WPW + v;
        if ((wonv[v] >> lane) & 1u) {
          const uint32_t idx = placed + s_wpre[x] + __popc(wonv[v] & below);
          const P pv = sidx[base + idx];
          uint64_t q = ws + lane;
          if (q >= T.c) q -= T.c;
          mg_store_value<LAY, K, V>(T, q, sizeof(P) == 8 ? (V)(uint32_t)pv : vals[pay_idx(pv)]);
          const uint64_t jj = jb + x;
          att += (long long)(jj * WINDOW + chunk_end(lane, ug));
          win += (long long)(jj + 1);
        }
        ws += ps.step;
        if (ws >= T.c) ws -= T.c;
      }
      placed += s_wtot;
      // resume after the last cell tried, or after these windows when every free cell was tried
      if (placed < m) {
        if (take < tot) {
          const uint32_t lx = s_lastx, ll = s_lastlane;
          jb += lx;
          wsb = T.modc.mod(wsb + (uint64_t)lx * ps.step);
          o = ll + 1;
          if (o >= WINDOW) {
            o = 0;
            jb += 1;
            wsb += ps.step;
            if (wsb >= T.c) wsb -= T.c;
          }
        } else {
          jb += WSTEP;
          wsb = T.modc.mod(wsb + (uint64_t)WSTEP * ps.step);
          o = 0;
        }
        if (jb >= T.max_windows) exhausted = true;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) {
      ops += m;
      occ += placed;
      const uint64_t lost = m - placed;  // sequence exhausted: TABLE_FULL, whole budget walked
      att += (long long)(lost * (uint64_t)T.max_windows * WINDOW);
      win += (long long)(lost * T.max_windows);
    }
    for (uint32_t x = placed + threadIdx.x; x < m; x += blockDim.x) status[pay_idx(sidx[base + x])] = ST_TABLE_FULL;
  }
  const long long v[4] = {ops, att, win, occ};
  long long* const dst[4] = {(long long*)&T.ctr->ops, (long long*)&T.ctr->attempts, (long long*)&T.ctr->windows,
                             &T.ctr->occupied};
  cta_add<4>(v, dst);
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

// CH_MG_CUB=1: CUB's DeviceRadixSort for the grouping sort instead of rsort.cu's
static bool g_mg_cub = [] {
  const char* e = getenv("CH_MG_CUB");
  return e && e[0] == '1';
}();

template <typename K, typename P>
static size_t sort_temp_bytes(uint64_t n) {
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, (const K*)nullptr, (K*)nullptr, (const P*)nullptr, (P*)nullptr,
                                  (int)n);
  return std::max(tb, radix_sort_scratch_bytes(n, (int)sizeof(K), (int)sizeof(P)));
}

size_t mgroup_scratch_bytes(uint64_t n, int kbytes, int vbytes) {
  const size_t sort_b = kbytes == 8 ? sort_temp_bytes<uint64_t, uint64_t>(n) : sort_temp_bytes<uint32_t, uint64_t>(n);
  (void)vbytes;
  return al256(sort_b) + al256(n * kbytes) + 2 * al256(n * 8) + al256((n + MR_TILE - 1) / MR_TILE * 8 + 64) +
         al256(8) + 2 * al256((n + 1) * 4) + 256 + al256((n / MG_HUGE + 1) * 4);
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
  const uint64_t rtiles = (n + MR_TILE - 1) / MR_TILE;
  unsigned long long* rstat = (unsigned long long*)take(rtiles * 8 + 64);  // run look-back, tile counter
  unsigned int* rnext = (unsigned int*)(rstat + rtiles);
  uint64_t* ngroups = (uint64_t*)take(8);
  uint32_t* gstart = (uint32_t*)take((n + 1) * 4);
  uint32_t* big = (uint32_t*)take((n + 1) * 4);
  unsigned long long* next = (unsigned long long*)take(64);  // [0] big grab, [1] big groups, [2] grab, [3] huge, [4] huge grab
  uint32_t* huge = (uint32_t*)take((n / MG_HUGE + 1) * 4);
  if ((size_t)(q - static_cast<char*>(scratch)) > scratch_bytes) {
    set_error("grouped insert scratch too small");
    return -22;
  }
  int rc = cuda_check(cudaMemsetAsync(status, ST_INSERTED, n, lc.stream), "memset");
  if (!rc) rc = cuda_check(cudaMemsetAsync(next, 0, 40, lc.stream), "memset");  // grabs and list counts
  if (rc) return rc;
  const unsigned grid = (unsigned)(lc.sms * 8);
  k_mg_payload<P, V><<<grid, MG_THREADS, 0, lc.stream>>>(idx, vals, n);
  count_launch();
  if (g_mg_cub) {
    rc = cuda_check(cub::DeviceRadixSort::SortPairs(sort_tmp, sort_b, keys, sk, idx, sidx, (int)n, 0,
                                                    (int)(8 * sizeof(K)), lc.stream),
                    "sort by key");
    count_launch(sizeof(K) == 8 ? 8 : 4);  // onesweep passes (approximate launch count)
  } else {
    rc = radix_sort_pairs<K, P>(lc, keys, idx, sk, sidx, n, sort_tmp, sort_b);  // stable, by key
  }
  if (rc) return rc;
  if ((rc = cuda_check(cudaMemsetAsync(rstat, 0, rtiles * 8 + 64, lc.stream), "memset"))) return rc;
  k_mg_runs<K><<<(unsigned)rtiles, MR_T, 0, lc.stream>>>(sk, n, gstart, (unsigned long long*)ngroups, rstat, rnext);
  count_launch();
  k_mg_big<<<grid, MG_THREADS, 0, lc.stream>>>(gstart, ngroups, big, next + 1, huge, next + 3);
  count_launch();
  if ((rc = cuda_check(cudaGetLastError(), "group runs"))) return rc;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (lc.timer && cudaEventCreate(&e0) == cudaSuccess && cudaEventCreate(&e1) == cudaSuccess)
    cudaEventRecord(e0, lc.stream);
  k_mg_place_cta<LAY, K, V, P><<<(unsigned)lc.sms, 512, 0, lc.stream>>>(T, sk, sidx, gstart, huge, next + 3, next + 4,
                                                                        vals, status, g);
  count_launch();
  k_mg_place<LAY, K, V, P><<<grid, MG_THREADS, 0, lc.stream>>>(T, sk, sidx, gstart, ngroups, big, next + 1, next,
                                                                vals, status, g, g_mw);
  count_launch();
  k_mg_small<LAY, K, V, P><<<grid, MG_THREADS, 0, lc.stream>>>(T, sk, sidx, gstart, ngroups, vals, status, g);
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
