// multi.cu -- multi-value COPS kernels (multi_table.py):
//   K4 insert: claim the first free slot of the key's sequence, no presence check (:113-152)
//   K5 count:  matches before the first empty (:171-203, :228-254)
//   K6 write:  re-walk, emit the values in probe order at offsets[q] (:256-295)
// plus the device exclusive scan that turns counts into offsets (:28-30).
#include "dispatch.cuh"
#include "probe.cuh"
#include "sched.cuh"

namespace chb {

constexpr int OUT_NONE_M = -1;

template <Layout LAY, typename K, typename V, int G>
__global__ void __launch_bounds__(256) k_multi_insert(TableRef T, const K* __restrict__ keys,
                                                      const V* __restrict__ vals, uint64_t n,
                                                      uint8_t* __restrict__ status) {
  using P = Probe<LAY, K, V, G>;
  using Ops = typename P::Ops;
  constexpr int MCHUNK = chunk_for<K, V>();
  __shared__ ChunkState cs;
  __shared__ K s_keys[MCHUNK];
  __shared__ uint32_t s_hw[MCHUNK], s_sw[MCHUNK];
  __shared__ uint8_t s_ho[MCHUNK];
  const StartSlots ss{s_hw, s_sw, s_ho};
  __shared__ V s_vals[MCHUNK];
  __shared__ uint8_t s_status[MCHUNK];
  constexpr int lane = 0;  // one thread per key (probe.cuh)
  long long occ = 0, ops = 0, att = 0, win = 0;
  while (chunk_begin<MCHUNK>(cs, T.work, n)) {
    stage_keys(s_keys, ss, keys, cs, T);
    stage_in(s_vals, vals, cs);
    __syncthreads();
    bool active = false;
    uint32_t li = 0;
    K key = 0;
    V val = 0;
    ProbeStart ps{0, 0};
    Cursor cur;
    cur.init(0);
    for (;;) {
      if (!active) {
        for (;;) {
          li = atomicAdd(&cs.next, 1u);
          if (li >= cs.cnt) break;
          key = s_keys[li];
          if (key != (K)T.e && key != (K)T.t) break;
          if (lane == 0) s_status[li] = ST_INVALID;
        }
        if (li >= cs.cnt) break;
        val = s_vals[li];
        ps = ss.get(li);
        cur.init(ps.h);
        active = true;
      }
      typename P::Step st;
      // the key mask is irrelevant here; pass a sentinel so no slot matches
      P::load(T, cur, (K)T.e, st);
      const uint32_t fr = st.em | st.tm;
      int outcome = OUT_NONE_M;
      uint32_t o_term = 0;
      if (fr) {
        const uint32_t u = lowest_bit(fr);  // lowest free, empty or tombstone (:136-139)
        const K expected = ((st.em >> u) & 1u) ? (K)T.e : (K)T.t;
        bool won = false;
        Ops::claim(T, st.base + u, expected, key, val, true, &won);
        o_term = P::offset_of(cur, st, u);
        if (won) outcome = 0;
        else cur.attempts += G;  // lost the race: re-read the chunk (:149-150)
      } else if (!P::advance(T, cur, st, ps.step)) {
        outcome = 2;
      }
      if (outcome != OUT_NONE_M) {
        ops += 1;
        att += (long long)(cur.attempts + (outcome == 0 ? chunk_end(o_term, G) : 0));
        win += (long long)cur.windows_seen;
        if (outcome == 0) occ += 1;
        if (lane == 0) s_status[li] = outcome == 0 ? ST_INSERTED : ST_TABLE_FULL;
        active = false;
      }
    }
    __syncthreads();
    stage_out(status, s_status, cs);
  }
  const long long v[4] = {ops, att, win, occ};
  long long* const dst[4] = {(long long*)&T.ctr->ops, (long long*)&T.ctr->attempts,
                             (long long*)&T.ctr->windows, &T.ctr->occupied};
  cta_add<4>(v, dst);
}

// MODE 0: counts[i]; MODE 1: write values at offsets[i] (probe order)
// Thread per query, 8-slot spans (bandwidth-lean for the many short chains).  Queries
// still open after `budget` windows are handed to the warp walker (k_multi_walk) through
// a device-counted list, unaccounted here (the walker restarts and accounts them).
template <Layout LAY, typename K, typename V, int G, int MODE>
__global__ void __launch_bounds__(256) k_multi_scan(TableRef T, const K* __restrict__ keys, uint64_t n,
                                                    uint32_t* __restrict__ counts,
                                                    const uint64_t* __restrict__ offsets,
                                                    V* __restrict__ out, int64_t* __restrict__ slot_out,
                                                    uint32_t budget, uint32_t* __restrict__ long_list,
                                                    unsigned long long* __restrict__ long_count,
                                                    V* __restrict__ stash, MultiStashMeta* __restrict__ meta,
                                                    uint32_t S) {
  using P = Probe<LAY, K, V, G>;
  using Ops = typename P::Ops;
  constexpr int MCHUNK = chunk_for<K, V>();
  __shared__ ChunkState cs;
  __shared__ K s_keys[MCHUNK];
  __shared__ uint32_t s_hw[MCHUNK], s_sw[MCHUNK];
  __shared__ uint8_t s_ho[MCHUNK];
  const StartSlots ss{s_hw, s_sw, s_ho};
  __shared__ uint32_t s_cnt[MODE == 0 ? MCHUNK : 1];
  __shared__ uint32_t s_long[MCHUNK];
  __shared__ uint32_t s_nlong;
  __shared__ unsigned long long s_lbase;
  constexpr int lane = 0;  // one thread per key (probe.cuh)
  long long att = 0, win = 0;
  while (chunk_begin<MCHUNK>(cs, T.work, n)) {
    if (threadIdx.x == 0) s_nlong = 0;
    stage_keys(s_keys, ss, keys, cs, T);
    __syncthreads();
    bool active = false;
    uint32_t li = 0;
    K key = 0;
    ProbeStart ps{0, 0};
    Cursor cur;
    cur.init(0);
    uint64_t total = 0, base_off = 0, want = 0;
    for (;;) {
      if (!active) {
        for (;;) {
          li = atomicAdd(&cs.next, 1u);
          if (li >= cs.cnt) break;
          key = s_keys[li];
          bool skip = key == (K)T.e || key == (K)T.t;
          if (MODE == 1 && !skip) {  // nothing to collect (:279-280)
            base_off = offsets[cs.base + li];
            want = offsets[cs.base + li + 1] - base_off;
            skip = want == 0;
          }
          if (!skip) break;
          if (MODE == 0 && lane == 0) s_cnt[li] = 0;
          if (MODE == 0 && meta) meta[cs.base + li].win = 0;
        }
        if (li >= cs.cnt) break;
        ps = ss.get(li);
        cur.init(ps.h);
        total = 0;
        active = true;
      }
      typename P::Step st;
      P::load(T, cur, key, st);
      const uint32_t km = st.km & below_lowest(st.em);
      if (MODE == 1 && km) {
        // the values of the matches, in probe order
        uint64_t r = total;
        for (uint32_t m = km; m; m &= m - 1, ++r) {
          // a writer racing the counting pass: keep the segment length (:285-286)
          if (r < want) {
            out[base_off + r] = P::value(T, st, lowest_bit(m));
            if (slot_out) slot_out[base_off + r] = (int64_t)(st.base + lowest_bit(m));  // for_each (:299-328)
          }
        }
      }
      if (MODE == 0 && stash && km && total < S) {  // the first S values, in probe order
        uint64_t r = total;
        V* const sq = stash + (uint64_t)(cs.base + li) * S;
        for (uint32_t m = km; m && r < S; m &= m - 1, ++r) sq[r] = P::value(T, st, lowest_bit(m));
      }
      total += (uint64_t)__popc(km);
      bool done = false;
      uint64_t attempts = 0;
      if (st.em) {
        done = true;
        attempts = cur.attempts + chunk_end(P::offset_of(cur, st, lowest_bit(st.em)), G);
      } else if (!P::advance(T, cur, st, ps.step)) {
        done = true;
        attempts = cur.attempts;
      } else if (budget && cur.j >= budget) {  // a long chain: to the warp walker
        s_long[atomicAdd(&s_nlong, 1u)] = (uint32_t)(cs.base + li);
        if (MODE == 0 && lane == 0) s_cnt[li] = 0;
        if (MODE == 0 && meta) meta[cs.base + li].win = 0;
        active = false;
        continue;
      }
      if (done) {
        if (MODE == 0 && lane == 0) s_cnt[li] = (uint32_t)total;
        if (MODE == 0 && meta) {
          MultiStashMeta mt;
          mt.key = (unsigned long long)key;
          mt.total = (uint32_t)total;
          mt.att = (uint32_t)attempts;
          mt.win = total <= S ? (uint32_t)cur.windows_seen : 0u;  // 0: not stashed
          mt.pad = 0;
          meta[cs.base + li] = mt;
        }
        att += (long long)attempts;
        win += (long long)cur.windows_seen;
        active = false;
      }
    }
    __syncthreads();
    if (MODE == 0) stage_out(counts, s_cnt, cs);
    if (long_list) {
      if (threadIdx.x == 0) s_lbase = s_nlong ? atomicAdd(long_count, (unsigned long long)s_nlong) : 0ull;
      __syncthreads();
      for (uint32_t x = threadIdx.x; x < s_nlong; x += blockDim.x) long_list[s_lbase + x] = s_long[x];
    }
  }
  // ops are accounted per bulk call on the host side (multi_table.py:249,290: ops += n)
  const long long v[2] = {att, win};
  long long* const dst[2] = {(long long*)&T.ctr->attempts, (long long*)&T.ctr->windows};
  cta_add<2>(v, dst);
}

// K5 / K6 as one warp per query (the count pass and the write pass walk the same
// sequence): a lane per slot of a 32-slot window, matches in window (= probe) order
// before the first empty, tombstones passed (multi_table.py:171-203).  After the first
// window the warp loads WW windows per step (independent loads) so a hot key's long
// chain costs chain / (32 WW) dependent steps; windows after the first empty are read
// but ignored.  A thread per query walked a 23K-copy chain alone (the batch's tail).
template <Layout LAY, typename K, typename V>
__device__ __forceinline__ uint64_t mw_load(const TableRef& T, uint64_t q) {
  if constexpr (LAY == PACKED) return __ldcg(static_cast<const unsigned long long*>(T.slots) + q);
  else if constexpr (LAY == SOA) return (uint64_t)__ldcg(static_cast<const K*>(T.slots) + q);
  else return (uint64_t)__ldcg(&static_cast<const CellT<K, V>*>(T.slots)[q].k);
}
template <Layout LAY, typename K, typename V>
__device__ __forceinline__ V mw_value(const TableRef& T, uint64_t q, uint64_t word) {
  if constexpr (LAY == PACKED) return (V)(word >> 32);
  else if constexpr (LAY == SOA) return __ldcg(static_cast<const V*>(T.vals) + q);
  else return __ldcg(&static_cast<const CellT<K, V>*>(T.slots)[q].v);
}

// A chain still open after HUGE_W windows (a Zipf-hot key: ~10^5 copies at s = 0.75 walk
// ~2.5 * 10^4 windows) is handed to k_multi_walk_cta with its position and running count.
constexpr uint32_t HUGE_W = 256;
struct HugeEntry {
  uint32_t qi, j;              // query, next window index
  unsigned long long total;    // matches so far
  unsigned long long ws;       // start slot of window j
};

template <Layout LAY, typename K, typename V, int MODE>
__global__ void __launch_bounds__(256) k_multi_walk(TableRef T, const K* __restrict__ keys, uint64_t n,
                                                    uint32_t* __restrict__ counts,
                                                    const uint64_t* __restrict__ offsets, V* __restrict__ out,
                                                    int64_t* __restrict__ slot_out,
                                                    unsigned long long* __restrict__ next, int g,
                                                    const uint32_t* __restrict__ list,
                                                    const unsigned long long* __restrict__ n_dev,
                                                    HugeEntry* __restrict__ huge,
                                                    unsigned long long* __restrict__ n_huge, uint64_t huge_cap) {
  if (n_dev) n = *n_dev;
  constexpr int WW = 4;
  const int lane = threadIdx.x & 31;
  const uint32_t below = (1u << lane) - 1u;
  const K e = (K)T.e, tomb = (K)T.t;
  const uint32_t ug = (uint32_t)g;
  long long att = 0, win = 0;
  for (;;) {
    unsigned long long qi = 0;
    if (lane == 0) qi = atomicAdd(next, 1ull);
    qi = __shfl_sync(0xffffffffu, qi, 0);
    if (qi >= n) break;
    if (list) qi = list[qi];
    const K k = keys[qi];
    uint64_t base = 0, want = 0;
    bool skip = k == e || k == tomb;
    if (MODE == 1 && !skip) {  // nothing to collect (multi_table.py:279-280)
      base = offsets[qi];
      want = offsets[qi + 1] - base;
      skip = want == 0;
    }
    if (skip) {
      if (MODE == 0 && lane == 0) counts[qi] = 0;
      continue;
    }
    const ProbeStart ps = probe_start(T, (uint64_t)k);
    uint64_t ws = ps.h, total = 0, attempts = 0, windows = 0;
    uint32_t j = 0, nw = 1;  // windows per step: 1 first, then WW
    bool done = false;
    while (!done) {
      uint64_t w[WW];
      uint64_t wsv[WW];
      uint64_t s = ws;
#pragma unroll
      for (int v = 0; v < WW; ++v) {
        wsv[v] = s;
        if ((uint32_t)v < nw && j + v < T.max_windows) {
          uint64_t q = s + lane;
          if (q >= T.c) q -= T.c;
          w[v] = mw_load<LAY, K, V>(T, q);
        } else {
          w[v] = 0;
        }
        s += ps.step;
        if (s >= T.c) s -= T.c;
      }
#pragma unroll
      for (int v = 0; v < WW; ++v) {
        if (done || (uint32_t)v >= nw) continue;
        if (j + v >= T.max_windows) {  // budget walked without an empty (probing.py:214-217)
          attempts = (uint64_t)T.max_windows * WINDOW;
          windows = T.max_windows;
          done = true;
          continue;
        }
        const K c = (K)w[v];
        const uint32_t em = __ballot_sync(0xffffffffu, c == e);
        const uint32_t km = __ballot_sync(0xffffffffu, c == k) & below_lowest(em);
        if (MODE == 1 && ((km >> lane) & 1u)) {
          const uint64_t r = total + __popc(km & below);
          uint64_t q = wsv[v] + lane;
          if (q >= T.c) q -= T.c;
          if (r < want) {  // racing writer: keep the length
            out[base + r] = mw_value<LAY, K, V>(T, q, w[v]);
            if (slot_out) slot_out[base + r] = (int64_t)q;
          }
        }
        total += __popc(km);
        if (em) {
          attempts = (uint64_t)(j + v) * WINDOW + chunk_end(lowest_bit(em), ug);
          windows = j + v + 1;
          done = true;
        }
      }
      j += nw;
      ws = wsv[0];
      for (uint32_t v = 0; v < nw; ++v) {
        ws += ps.step;
        if (ws >= T.c) ws -= T.c;
      }
      nw = nw * 2 < (uint32_t)WW ? nw * 2 : (uint32_t)WW;  // 1, 2, 4, 4, ... windows per step
      if (!done && huge && j >= HUGE_W) {  // a hot key: the CTA walker continues it
        unsigned long long slot = 0;
        if (lane == 0) slot = atomicAdd(n_huge, 1ull);
        slot = __shfl_sync(0xffffffffu, slot, 0);
        if (slot < huge_cap) {
          if (lane == 0) huge[slot] = HugeEntry{(uint32_t)qi, j, (unsigned long long)total, (unsigned long long)ws};
          break;
        }
        huge = nullptr;  // list full: walk it here
      }
    }
    if (!done) continue;  // handed off
    if (lane == 0) {
      if (MODE == 0) counts[qi] = (uint32_t)total;
      att += (long long)attempts;
      win += (long long)windows;
    }
  }
  // ops are accounted per bulk call on the host side (multi_table.py:249,290: ops += n)
  const long long v[2] = {att, win};
  long long* const dst[2] = {(long long*)&T.ctr->attempts, (long long*)&T.ctr->windows};
  cta_add<2>(v, dst);
}

// K5 / K6 for the hot keys: one CTA per chain, 128 windows per step (16 warps x 8 windows,
// all loads independent: the window starts h + j step are known up front), a block-wide cut
// at the first window holding an empty and a scan of the per-window match counts, so the
// values land in probe order.  The chain of a key with 10^5 copies takes ~200 steps instead
// of ~6 * 10^3 dependent steps of the warp walker.
template <Layout LAY, typename K, typename V, int MODE>
__global__ void __launch_bounds__(512) k_multi_walk_cta(TableRef T, const K* __restrict__ keys,
                                                        uint32_t* __restrict__ counts,
                                                        const uint64_t* __restrict__ offsets, V* __restrict__ out,
                                                        int64_t* __restrict__ slot_out,
                                                        const HugeEntry* __restrict__ huge,
                                                        const unsigned long long* __restrict__ n_huge,
                                                        unsigned long long* __restrict__ grab, int g) {
  constexpr uint32_t NWARP = 16, WPW = 8, WSTEP = NWARP * WPW;
  __shared__ uint32_t s_cnt[WSTEP], s_emp[WSTEP], s_pre[WSTEP];
  __shared__ unsigned long long s_item;
  __shared__ uint32_t s_cut, s_sum;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint32_t below = (1u << lane) - 1u;
  const K e = (K)T.e;
  const uint32_t ug = (uint32_t)g;
  const unsigned long long nh = *n_huge;
  long long att = 0, win = 0;
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(grab, 1ull);
    __syncthreads();
    const unsigned long long item = s_item;
    __syncthreads();
    if (item >= nh) break;
    const HugeEntry he = huge[item];
    const K k = keys[he.qi];
    const ProbeStart ps = probe_start(T, (uint64_t)k);
    uint64_t base = 0, want = ~0ull;
    if (MODE == 1) {
      base = offsets[he.qi];
      want = offsets[he.qi + 1] - base;
    }
    uint64_t total = he.total, jb = he.j, wsb = he.ws;
    for (;;) {  // CTA-uniform
      // this warp's first window: wsb + (warp WPW) step mod c
      uint64_t ws = T.modc.mod(wsb + (uint64_t)(warp * WPW) * ps.step);
      uint64_t words[WPW];
      uint32_t kms[WPW];
#pragma unroll
      for (uint32_t v = 0; v < WPW; ++v) {
        const uint64_t jj = jb + warp * WPW + v;
        uint64_t q = ws + lane;
        if (q >= T.c) q -= T.c;
        words[v] = jj < T.max_windows ? mw_load<LAY, K, V>(T, q) : 0;
        ws += ps.step;
        if (ws >= T.c) ws -= T.c;
      }
#pragma unroll
      for (uint32_t v = 0; v < WPW; ++v) {
        const uint64_t jj = jb + warp * WPW + v;
        const K c = (K)words[v];
        const uint32_t em = __ballot_sync(0xffffffffu, c == e);
        const uint32_t km = __ballot_sync(0xffffffffu, c == k) & below_lowest(em);
        kms[v] = km;
        if (lane == 0) {
          s_cnt[warp * WPW + v] = __popc(km);
          // 1 + lowest empty lane; 33: the window budget ends here (probing.py:214-217)
          s_emp[warp * WPW + v] = jj >= T.max_windows ? 33u : (em ? lowest_bit(em) + 1u : 0u);
        }
      }
      __syncthreads();
      if (warp == 0) {  // the cut (first window with an empty or past the budget) and the scan
        uint32_t cut = WSTEP;
        for (uint32_t x0 = 0; x0 < WSTEP; x0 += 32) {
          const unsigned hb = __ballot_sync(0xffffffffu, s_emp[x0 + lane] != 0);
          if (hb) {
            cut = x0 + __ffs(hb) - 1;
            break;
          }
        }
        uint32_t run = 0;
        for (uint32_t x0 = 0; x0 < WSTEP; x0 += 32) {
          const uint32_t x = x0 + lane;
          const uint32_t cx = x <= cut && s_emp[x] != 33u ? s_cnt[x] : 0u;
          uint32_t inc = cx;
#pragma unroll
          for (int d = 1; d < 32; d <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, d);
            if ((int)lane >= d) inc += y;
          }
          s_pre[x] = run + inc - cx;
          run += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) {
          s_cut = cut;
          s_sum = run;
        }
      }
      __syncthreads();
      const uint32_t cut = s_cut;
      if (MODE == 1) {
        uint64_t ws2 = T.modc.mod(wsb + (uint64_t)(warp * WPW) * ps.step);
#pragma unroll
        for (uint32_t v = 0; v < WPW; ++v) {
          const uint32_t x = warp * WPW + v;
          if (x <= cut && s_emp[x] != 33u && ((kms[v] >> lane) & 1u)) {
            const uint64_t r = total + s_pre[x] + __popc(kms[v] & below);
            uint64_t q = ws2 + lane;
            if (q >= T.c) q -= T.c;
            if (r < want) {  // racing writer: keep the length (multi_table.py:285-286)
              out[base + r] = mw_value<LAY, K, V>(T, q, words[v]);
              if (slot_out) slot_out[base + r] = (int64_t)q;
            }
          }
          ws2 += ps.step;
          if (ws2 >= T.c) ws2 -= T.c;
        }
      }
      total += s_sum;
      if (cut < WSTEP) {
        if (threadIdx.x == 0) {
          const uint32_t em1 = s_emp[cut];
          const uint64_t jc = jb + cut;
          if (em1 == 33u) {
            att += (long long)(T.max_windows * WINDOW);
            win += (long long)T.max_windows;
          } else {
            att += (long long)(jc * WINDOW + chunk_end(em1 - 1u, ug));
            win += (long long)(jc + 1);
          }
          if (MODE == 0) counts[he.qi] = (uint32_t)total;
        }
        __syncthreads();
        break;
      }
      jb += WSTEP;
      wsb = T.modc.mod(wsb + (uint64_t)WSTEP * ps.step);
      __syncthreads();
    }
  }
  const long long v[2] = {att, win};
  long long* const dst[2] = {(long long*)&T.ctr->attempts, (long long*)&T.ctr->windows};
  cta_add<2>(v, dst);
}

// Retrieve pass from the count pass's stash: a thread per query whose key and count still
// match its stash entry copies the values (and accounts the walk the count pass recorded,
// the same walk the reference's second pass repeats, multi_table.py:256-295); the rest go to
// the warp walker's list.
template <typename K, typename V>
__global__ void __launch_bounds__(256) k_multi_stash_copy(TableRef T, const K* __restrict__ keys, uint64_t n,
                                                          const uint64_t* __restrict__ offsets, V* __restrict__ out,
                                                          const V* __restrict__ stash,
                                                          const MultiStashMeta* __restrict__ meta, uint32_t S,
                                                          uint32_t* __restrict__ long_list,
                                                          unsigned long long* __restrict__ long_count) {
  long long att = 0, win = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t n_up = (n + 31) & ~(uint64_t)31;  // whole warps in the loop (ballots)
  const uint32_t lane = threadIdx.x & 31u;
  for (uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; q < n_up; q += stride) {
    bool walk = false, copy = false;
    uint64_t base = 0, m = 0;
    if (q < n) {
      base = offsets[q];
      m = offsets[q + 1] - base;
      if (m) {
        const MultiStashMeta mt = meta[q];
        if (mt.win && mt.key == (unsigned long long)keys[q] && mt.total == m && m <= S) {
          copy = true;
          att += mt.att;
          win += mt.win;
        } else {
          walk = true;
        }
      }
    }
    // the warp copies its 32 queries' values one query at a time (coalesced rows)
    unsigned cm = __ballot_sync(0xffffffffu, copy);
    while (cm) {
      const int j = __ffs(cm) - 1;
      cm &= cm - 1;
      const uint64_t qj = __shfl_sync(0xffffffffu, q, j), bj = __shfl_sync(0xffffffffu, base, j);
      const uint32_t mj = (uint32_t)__shfl_sync(0xffffffffu, m, j);
      const V* sq = stash + qj * S;
      for (uint32_t r = lane; r < mj; r += 32) out[bj + r] = sq[r];
    }
    const unsigned b = __ballot_sync(0xffffffffu, walk);
    if (b) {
      unsigned long long w0 = 0;
      if (lane == (uint32_t)(__ffs(b) - 1)) w0 = atomicAdd(long_count, (unsigned long long)__popc(b));
      w0 = __shfl_sync(0xffffffffu, w0, __ffs(b) - 1);
      if (walk) long_list[w0 + __popc(b & ((1u << lane) - 1u))] = (uint32_t)q;
    }
  }
  const long long v[2] = {att, win};
  long long* const dst[2] = {(long long*)&T.ctr->attempts, (long long*)&T.ctr->windows};
  cta_add<2>(v, dst);
}

template <Layout LAY, typename K, typename V, int G>
struct MultiKernels {
  static int insert(const Launch& lc, const TableRef& T, const void* keys, const void* vals, uint64_t n,
                    uint8_t* status) {
    auto kern = k_multi_insert<LAY, K, V, G>;
    return launch_chunked(lc, T, (const void*)kern, n, (chunk_for<K, V>()), [&](dim3 g, dim3 b) {
      kern<<<g, b, 0, lc.stream>>>(T, (const K*)keys, (const V*)vals, n, status);
    });
  }
  // thread pass (first kBudget windows), then the warp walker over the queries it handed off,
  // then the CTA walker over the chains the warps handed off (counters: [0] long list, [1] warp
  // grab, [2] hot list, [3] CTA grab, then kHugeCap hot-list entries)
  static constexpr uint32_t kBudget = 4;
  static constexpr uint64_t kHugeCap = kMultiHugeCap;
  static int scan(const Launch& lc, const TableRef& T, const void* keys, uint64_t n, uint32_t* counts,
                  const uint64_t* offsets, void* out, int mode, uint32_t* long_list,
                  unsigned long long* counters, int64_t* slot_out, void* stash, void* meta, uint32_t S) {
    if (n == 0) return 0;
    int rc = cuda_check(cudaMemsetAsync(counters, 0, 4 * sizeof(unsigned long long), lc.stream), "memset");
    if (rc) return rc;
    if (mode == 0) {
      auto kern = k_multi_scan<LAY, K, V, G, 0>;
      rc = launch_chunked(lc, T, (const void*)kern, n, (chunk_for<K, V>()), [&](dim3 g, dim3 b) {
        kern<<<g, b, 0, lc.stream>>>(T, (const K*)keys, n, counts, offsets, (V*)out, slot_out, kBudget, long_list,
                                     counters, (V*)stash, (MultiStashMeta*)meta, S);
      });
    } else if (stash && meta && out && !slot_out) {  // the count pass's stash: copy, walk the rest
      k_multi_stash_copy<K, V><<<(unsigned)(lc.sms * 8), 256, 0, lc.stream>>>(
          T, (const K*)keys, n, offsets, (V*)out, (const V*)stash, (const MultiStashMeta*)meta, S, long_list, counters);
      count_launch();
      rc = cuda_check(cudaGetLastError(), "multi stash copy");
    } else {
      auto kern = k_multi_scan<LAY, K, V, G, 1>;
      rc = launch_chunked(lc, T, (const void*)kern, n, (chunk_for<K, V>()), [&](dim3 g, dim3 b) {
        kern<<<g, b, 0, lc.stream>>>(T, (const K*)keys, n, counts, offsets, (V*)out, slot_out, kBudget, long_list,
                                     counters, nullptr, nullptr, 0u);
      });
    }
    if (rc) return rc;
    const unsigned grid = (unsigned)(lc.sms * 8);
    HugeEntry* huge = reinterpret_cast<HugeEntry*>(counters + 4);
    if (mode == 0)
      k_multi_walk<LAY, K, V, 0><<<grid, 256, 0, lc.stream>>>(T, (const K*)keys, n, counts, offsets, (V*)out,
                                                             slot_out, counters + 1, G, long_list, counters,
                                                             huge, counters + 2, kHugeCap);
    else
      k_multi_walk<LAY, K, V, 1><<<grid, 256, 0, lc.stream>>>(T, (const K*)keys, n, counts, offsets, (V*)out,
                                                             slot_out, counters + 1, G, long_list, counters,
                                                             huge, counters + 2, kHugeCap);
    count_launch();
    if ((rc = cuda_check(cudaGetLastError(), "multi walk"))) return rc;
    const unsigned grid2 = (unsigned)(lc.sms * 2);  // CTAs take hot chains from a counter; most exit at once
    if (mode == 0)
      k_multi_walk_cta<LAY, K, V, 0><<<grid2, 512, 0, lc.stream>>>(T, (const K*)keys, counts, offsets, (V*)out,
                                                                  slot_out, huge, counters + 2, counters + 3, G);
    else
      k_multi_walk_cta<LAY, K, V, 1><<<grid2, 512, 0, lc.stream>>>(T, (const K*)keys, counts, offsets, (V*)out,
                                                                  slot_out, huge, counters + 2, counters + 3, G);
    count_launch();
    return cuda_check(cudaGetLastError(), "multi walk (hot chains)");
  }
};

int multi_insert(const Launch& lc, const TableRef& T, const TypeSel& ts, const void* keys, const void* vals,
                 uint64_t n, uint8_t* status) {
  return dispatch_types<MultiKernels>(
      ts, [&](auto tag) { return decltype(tag)::type::insert(lc, T, keys, vals, n, status); });
}
int multi_scan(const Launch& lc, const TableRef& T, const TypeSel& ts, const void* keys, uint64_t n,
               uint32_t* counts, const uint64_t* offsets, void* vals_out, int mode, uint32_t* long_list,
               unsigned long long* counters, int64_t* slot_out, void* stash, void* stash_meta, uint32_t stash_s) {
  return dispatch_types<MultiKernels>(ts, [&](auto tag) {
    return decltype(tag)::type::scan(lc, T, keys, n, counts, offsets, vals_out, mode, long_list, counters,
                                     slot_out, stash, stash_meta, stash_s);
  });
}

}  // namespace chb
