// single.cu -- single-value COPS kernels: K0 clear, K1 insert / find_or_claim,
// K2 retrieve, K3 erase, find (slot_of + probe stats).
//
// Every kernel is a persistent grid-stride loop of probe GROUPS (L lanes).  The
// loop is flattened into one step per iteration: a group that resolves its key
// immediately fetches the next one, so a warp never idles on the longest probe
// of its 32 keys (memory-level parallelism is what bounds random-access work).
#include "dispatch.cuh"
#include "probe.cuh"

namespace chb {

// ------------------------------------------------------------------ K0
template <Layout LAY, typename K, typename V>
__global__ void __launch_bounds__(256) k_clear(TableRef T, int zero_values) {
  const uint64_t stride = gridDim.x * (uint64_t)blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < T.c; i += stride) {
    if constexpr (LAY == PACKED) {
      static_cast<uint64_t*>(T.slots)[i] = (uint64_t)(K)T.e;  // pack_pair(e, 0) (layout.py:103)
    } else if constexpr (LAY == SOA) {
      static_cast<K*>(T.slots)[i] = (K)T.e;
      static_cast<V*>(T.vals)[i] = 0;
    } else {
      CellT<K, V> c;
      c.k = (K)T.e;
      c.v = 0;
      static_cast<CellT<K, V>*>(T.slots)[i] = c;
    }
  }
}

// ------------------------------------------------------------------ K1
// MODE 0: insert_bulk (single_table.py:355-374, _insert_at :279-290)
// MODE 1: find_or_claim (single_table.py:292-311): value cell untouched,
//         slot written to slot_out (the bucket list's key store).
enum Outcome : int { OUT_NONE = -1, OUT_CLAIMED = 0, OUT_FOUND = 1, OUT_FULL = 2 };

template <Layout LAY, typename K, typename V, int G, int MODE>
__global__ void __launch_bounds__(256) k_insert(TableRef T, const K* __restrict__ keys,
                                                const V* __restrict__ vals, uint64_t n,
                                                uint8_t* __restrict__ status,
                                                int64_t* __restrict__ slot_out) {
  using P = Probe<LAY, K, V, G>;
  using Ops = typename P::Ops;
  auto tile = cg::tiled_partition<P::L>(cg::this_thread_block());
  const int lane = P::L > 1 ? (int)tile.thread_rank() : 0;
  const uint64_t ngroups = (gridDim.x * (uint64_t)blockDim.x) / P::L;
  uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / P::L;
  long long occ = 0, tomb = 0, ops = 0, att = 0, win = 0;

  bool active = false;
  K key = 0;
  V val = 0;
  ProbeStart ps{0, 0};
  Cursor cur;
  cur.init(0);
  int64_t pending = -1;

  for (;;) {
    if (!active) {
      while (i < n) {
        key = ld_stream(keys + i);
        if (key != (K)T.e && key != (K)T.t) break;
        if (lane == 0) {  // sentinel keys: INVALID_KEY, no accounting (single_table.py:369-370)
          status[i] = ST_INVALID;
          if (MODE == 1) slot_out[i] = -1;
        }
        i += ngroups;
      }
      if (i >= n) break;
      if (MODE == 0) val = ld_stream(vals + i);
      ps = probe_start(T, key);
      cur.init(ps.h);
      pending = -1;
      active = true;
    }

    typename P::Step st;
    P::load(T, tile, cur, key, st);

    int outcome = OUT_NONE;
    uint64_t oslot = 0;
    bool was_tomb = false;
    bool add_chunk = true;   // final chunk accounting (false after a whole cycle)
    uint32_t o_term = 0;

    const uint32_t kb = st.km & below_lowest(st.em);
    if (kb) {  // key present before the first empty: duplicate (single_table.py:198-200)
      const uint32_t u = lowest_bit(kb);
      outcome = OUT_FOUND;
      oslot = st.base + u;
      o_term = P::offset_of(cur, st, u);
    } else {
      int64_t target = -1;
      K expected = (K)T.e;
      if (pending < 0) {
        const uint32_t fr = st.em | st.tm;
        if (fr) {
          const uint32_t u = lowest_bit(fr);
          if (((st.tm >> u) & 1u) && st.em == 0) {
            pending = (int64_t)(st.base + u);  // tombstone only: defer (:210-214)
          } else {
            target = (int64_t)(st.base + u);
            expected = ((st.em >> u) & 1u) ? (K)T.e : (K)T.t;
          }
        }
      } else if (st.em) {
        target = pending;  // an empty bounds the duplicate scan: claim the tombstone (:219-223)
        expected = (K)T.t;
      }
      bool exhausted = false;
      if (target < 0) {
        if (!P::advance(T, cur, st, ps.step)) {
          exhausted = true;
          if (pending >= 0) {  // whole cycle without an empty: claim the tombstone (:238-244)
            target = pending;
            expected = (K)T.t;
          } else {
            outcome = OUT_FULL;
            add_chunk = false;
          }
        }
      }
      if (target >= 0) {
        // the lane holding the target slot (any lane for a deferred tombstone) does the CAS
        const bool in_span = (uint64_t)target >= st.base && (uint64_t)target < st.base + P::A;
        const int owner = in_span ? (int)(((uint64_t)target - st.base) / P::SPL) : 0;
        bool won = false;
        K seen = 0;
        if (lane == owner) seen = Ops::claim(T, (uint64_t)target, expected, key, val, MODE == 0, &won);
        won = tile_bcast(tile, won, owner);
        seen = tile_bcast(tile, seen, owner);
        if (!exhausted) o_term = P::offset_of(cur, st, lowest_bit(st.em));
        else add_chunk = false;
        if (won) {
          outcome = OUT_CLAIMED;
          oslot = (uint64_t)target;
          was_tomb = expected == (K)T.t;
        } else if (seen == key) {
          outcome = OUT_FOUND;
          oslot = (uint64_t)target;
        } else if (target == pending) {
          // lost the deferred tombstone: restart the whole probe (:229-231, :244)
          cur.attempts += add_chunk ? chunk_end(o_term, G) : 0;
          cur.ws = ps.h;
          cur.j = 0;
          cur.o = 0;
          cur.windows_seen += 1;
          pending = -1;
        } else {
          cur.attempts += G;  // lost to another key: the chunk is re-read (:232-233)
        }
      }
    }

    if (outcome != OUT_NONE) {
      ops += 1;
      att += (long long)(cur.attempts + (add_chunk ? chunk_end(o_term, G) : 0));
      win += (long long)cur.windows_seen;
      if (lane == 0) {
        status[i] = outcome == OUT_CLAIMED ? ST_INSERTED : outcome == OUT_FOUND ? ST_DUPLICATE : ST_TABLE_FULL;
        if (MODE == 1) slot_out[i] = outcome == OUT_FULL ? -1 : (int64_t)oslot;
      }
      if (outcome == OUT_CLAIMED) {
        occ += 1;
        if (was_tomb) tomb -= 1;
      }
      active = false;
      i += ngroups;
    }
  }
  if (P::L > 1 && lane != 0) occ = tomb = ops = att = win = 0;
  const long long v[5] = {ops, att, win, occ, tomb};
  long long* const dst[5] = {(long long*)&T.ctr->ops, (long long*)&T.ctr->attempts,
                             (long long*)&T.ctr->windows, &T.ctr->occupied, &T.ctr->tombstones};
  cta_add<5>(v, dst);
}

// ------------------------------------------------------------------ K2
// MODE 0: retrieve_bulk (single_table.py:376-408): value + found flag
// MODE 1: find (slot_of / retrieve_with_stats, :317-336): slot, attempts, windows
// MODE 2: erase (:338-351): retire the key (layout.py:224-243)
template <Layout LAY, typename K, typename V, int G, int MODE>
__global__ void __launch_bounds__(256) k_lookup(TableRef T, const K* __restrict__ keys, uint64_t n,
                                                V* __restrict__ vals_out, uint8_t* __restrict__ flag,
                                                int64_t* __restrict__ slot_out,
                                                uint32_t* __restrict__ att_out,
                                                uint32_t* __restrict__ win_out) {
  using P = Probe<LAY, K, V, G>;
  using Ops = typename P::Ops;
  auto tile = cg::tiled_partition<P::L>(cg::this_thread_block());
  const int lane = P::L > 1 ? (int)tile.thread_rank() : 0;
  const uint64_t ngroups = (gridDim.x * (uint64_t)blockDim.x) / P::L;
  uint64_t i = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) / P::L;
  long long ops = 0, att = 0, win = 0, occ = 0, tomb = 0;

  bool active = false;
  K key = 0;
  ProbeStart ps{0, 0};
  Cursor cur;
  cur.init(0);

  for (;;) {
    if (!active) {
      while (i < n) {
        key = ld_stream(keys + i);
        if (key != (K)T.e && key != (K)T.t) break;
        if (MODE == 0) ops += lane == 0;  // retrieve_bulk counts every query (:403)
        if (lane == 0) {
          if (MODE == 0) { st_stream(vals_out + i, (V)0); st_stream(flag + i, (uint8_t)0); }
          if (MODE == 1) {
            slot_out[i] = -1;
            if (vals_out) vals_out[i] = 0;
            if (att_out) att_out[i] = 0;
            if (win_out) win_out[i] = 0;
          }
          if (MODE == 2) flag[i] = 0;
        }
        i += ngroups;
      }
      if (i >= n) break;
      ps = probe_start(T, key);
      cur.init(ps.h);
      active = true;
    }

    typename P::Step st;
    P::load(T, tile, cur, key, st);
    const uint32_t kb = st.km & below_lowest(st.em);
    bool done = false, found = false;
    uint32_t u = 0;
    uint64_t attempts = 0;
    if (kb) {
      u = lowest_bit(kb);
      found = done = true;
      attempts = cur.attempts + chunk_end(P::offset_of(cur, st, u), G);
    } else if (st.em) {
      done = true;
      attempts = cur.attempts + chunk_end(P::offset_of(cur, st, lowest_bit(st.em)), G);
    } else if (!P::advance(T, cur, st, ps.step)) {
      done = true;
      attempts = cur.attempts;
    }
    if (!done) continue;

    const int owner = (int)(u / P::SPL);
    const int s = (int)(u % P::SPL);
    if (MODE == 0) {
      V v = 0;
      if (found && lane == owner) v = Ops::template value<P::SPL>(T, st.base + u, st.sl, s);
      if (lane == owner) {
        st_stream(vals_out + i, found ? v : (V)0);
        st_stream(flag + i, (uint8_t)found);
      }
    } else if (MODE == 1) {
      if (vals_out) {
        V v = 0;
        if (found && lane == owner) v = Ops::template value<P::SPL>(T, st.base + u, st.sl, s);
        if (lane == owner) vals_out[i] = v;
      }
      if (lane == 0) {
        slot_out[i] = found ? (int64_t)(st.base + u) : -1;
        if (att_out) att_out[i] = (uint32_t)attempts;
        if (win_out) win_out[i] = (uint32_t)cur.windows_seen;
      }
    } else {
      bool won = false;
      if (found && lane == owner) won = Ops::template retire<P::SPL>(T, st.base + u, st.sl, s);
      won = tile_bcast(tile, won, owner);
      if (lane == 0) flag[i] = won;
      if (won) { occ -= 1; tomb += 1; }
    }
    ops += 1;
    att += (long long)attempts;
    win += (long long)cur.windows_seen;
    active = false;
    i += ngroups;
  }
  if (P::L > 1 && lane != 0) ops = att = win = occ = tomb = 0;
  const long long v[5] = {ops, att, win, occ, tomb};
  long long* const dst[5] = {(long long*)&T.ctr->ops, (long long*)&T.ctr->attempts,
                             (long long*)&T.ctr->windows, &T.ctr->occupied, &T.ctr->tombstones};
  cta_add<5>(v, dst);
}

// ------------------------------------------------------------- launchers
template <Layout LAY, typename K, typename V, int G>
struct SingleKernels {
  static int clear(const Launch& lc, const TableRef& T) {
    auto kern = k_clear<LAY, K, V>;
    return launch_persistent(lc, (const void*)kern, T.c, 1, [&](dim3 g, dim3 b) {
      kern<<<g, b, 0, lc.stream>>>(T, 1);
    });
  }
  static int insert(const Launch& lc, const TableRef& T, const void* keys, const void* vals, uint64_t n,
                    uint8_t* status, int64_t* slot_out, int mode) {
    using P = Probe<LAY, K, V, G>;
    if (mode == 0) {
      auto kern = k_insert<LAY, K, V, G, 0>;
      return launch_persistent(lc, (const void*)kern, n, P::L, [&](dim3 g, dim3 b) {
        kern<<<g, b, 0, lc.stream>>>(T, (const K*)keys, (const V*)vals, n, status, slot_out);
      });
    }
    auto kern = k_insert<LAY, K, V, G, 1>;
    return launch_persistent(lc, (const void*)kern, n, P::L, [&](dim3 g, dim3 b) {
      kern<<<g, b, 0, lc.stream>>>(T, (const K*)keys, (const V*)vals, n, status, slot_out);
    });
  }
  static int lookup(const Launch& lc, const TableRef& T, const void* keys, uint64_t n, void* vals_out,
                    uint8_t* flag, int64_t* slot_out, uint32_t* att_out, uint32_t* win_out, int mode) {
    using P = Probe<LAY, K, V, G>;
#define CHB_LOOKUP(M)                                                                                  \
  {                                                                                                    \
    auto kern = k_lookup<LAY, K, V, G, M>;                                                             \
    return launch_persistent(lc, (const void*)kern, n, P::L, [&](dim3 g, dim3 b) {                     \
      kern<<<g, b, 0, lc.stream>>>(T, (const K*)keys, n, (V*)vals_out, flag, slot_out, att_out, win_out); \
    });                                                                                                \
  }
    if (mode == 0) CHB_LOOKUP(0)
    if (mode == 1) CHB_LOOKUP(1)
    CHB_LOOKUP(2)
#undef CHB_LOOKUP
  }
};

int single_clear(const Launch& lc, const TableRef& T, const TypeSel& ts) {
  return dispatch_types<SingleKernels>(ts, [&](auto tag) { return decltype(tag)::type::clear(lc, T); });
}
int single_insert(const Launch& lc, const TableRef& T, const TypeSel& ts, const void* keys, const void* vals,
                  uint64_t n, uint8_t* status, int64_t* slot_out, int mode) {
  return dispatch_types<SingleKernels>(ts, [&](auto tag) {
    return decltype(tag)::type::insert(lc, T, keys, vals, n, status, slot_out, mode);
  });
}
int single_lookup(const Launch& lc, const TableRef& T, const TypeSel& ts, const void* keys, uint64_t n,
                  void* vals_out, uint8_t* flag, int64_t* slot_out, uint32_t* att_out, uint32_t* win_out,
                  int mode) {
  return dispatch_types<SingleKernels>(ts, [&](auto tag) {
    return decltype(tag)::type::lookup(lc, T, keys, n, vals_out, flag, slot_out, att_out, win_out, mode);
  });
}

}  // namespace chb
