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
template <Layout LAY, typename K, typename V, int G, int MODE>
__global__ void __launch_bounds__(256) k_multi_scan(TableRef T, const K* __restrict__ keys, uint64_t n,
                                                    uint32_t* __restrict__ counts,
                                                    const uint64_t* __restrict__ offsets,
                                                    V* __restrict__ out) {
  using P = Probe<LAY, K, V, G>;
  using Ops = typename P::Ops;
  constexpr int MCHUNK = chunk_for<K, V>();
  __shared__ ChunkState cs;
  __shared__ K s_keys[MCHUNK];
  __shared__ uint32_t s_hw[MCHUNK], s_sw[MCHUNK];
  __shared__ uint8_t s_ho[MCHUNK];
  const StartSlots ss{s_hw, s_sw, s_ho};
  __shared__ uint32_t s_cnt[MODE == 0 ? MCHUNK : 1];
  constexpr int lane = 0;  // one thread per key (probe.cuh)
  long long att = 0, win = 0;
  while (chunk_begin<MCHUNK>(cs, T.work, n)) {
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
          if (r < want) out[base_off + r] = P::value(T, st, lowest_bit(m));
        }
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
      }
      if (done) {
        if (MODE == 0 && lane == 0) s_cnt[li] = (uint32_t)total;
        att += (long long)attempts;
        win += (long long)cur.windows_seen;
        active = false;
      }
    }
    __syncthreads();
    if (MODE == 0) stage_out(counts, s_cnt, cs);
  }
  // ops are accounted per bulk call on the host side (multi_table.py:249,290: ops += n)
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
  static int scan(const Launch& lc, const TableRef& T, const void* keys, uint64_t n, uint32_t* counts,
                  const uint64_t* offsets, void* out, int mode) {
    if (mode == 0) {
      auto kern = k_multi_scan<LAY, K, V, G, 0>;
      return launch_chunked(lc, T, (const void*)kern, n, (chunk_for<K, V>()), [&](dim3 g, dim3 b) {
        kern<<<g, b, 0, lc.stream>>>(T, (const K*)keys, n, counts, offsets, (V*)out);
      });
    }
    auto kern = k_multi_scan<LAY, K, V, G, 1>;
    return launch_chunked(lc, T, (const void*)kern, n, (chunk_for<K, V>()), [&](dim3 g, dim3 b) {
      kern<<<g, b, 0, lc.stream>>>(T, (const K*)keys, n, counts, offsets, (V*)out);
    });
  }
};

int multi_insert(const Launch& lc, const TableRef& T, const TypeSel& ts, const void* keys, const void* vals,
                 uint64_t n, uint8_t* status) {
  return dispatch_types<MultiKernels>(
      ts, [&](auto tag) { return decltype(tag)::type::insert(lc, T, keys, vals, n, status); });
}
int multi_scan(const Launch& lc, const TableRef& T, const TypeSel& ts, const void* keys, uint64_t n,
               uint32_t* counts, const uint64_t* offsets, void* vals_out, int mode) {
  return dispatch_types<MultiKernels>(ts, [&](auto tag) {
    return decltype(tag)::type::scan(lc, T, keys, n, counts, offsets, vals_out, mode);
  });
}

}  // namespace chb
