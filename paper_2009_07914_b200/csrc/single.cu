// single.cu -- single-value COPS kernels: K0 clear, K1 insert / find_or_claim,
// K2 retrieve, K3 erase, find (slot_of + probe stats).
//
// Every probe kernel is a persistent grid of CTAs that claim CHUNK-element
// slices of the batch (sched.cuh).  Inside a chunk the probe GROUPS (L lanes)
// run a flattened loop: one probe step per iteration, and a group that
// resolves its key immediately takes the next one from the chunk, so no warp
// idles on the longest probe of its keys.
#include "dispatch.cuh"
#include "probe.cuh"
#include "sched.cuh"

namespace chb {

constexpr int CHUNK_FIND = 512;

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

// find_or_claim also stages an int64 slot per element
template <typename K, typename V, int MODE>
constexpr int insert_chunk() { return MODE == 1 ? 1024 : chunk_for<K, V>(); }

#ifndef CH_AB_PROBE_MINB
#define CH_AB_PROBE_MINB 4  // 5 (<= 51 registers) measured slower for the staged fallback (2.14 -> 2.43 ms)
#endif
template <Layout LAY, typename K, typename V, int G, int MODE>
__global__ void __launch_bounds__(256, CH_AB_PROBE_MINB) k_insert(TableRef T, const K* __restrict__ keys,
                                                const V* __restrict__ vals, uint64_t n,
                                                uint8_t* __restrict__ status,
                                                int64_t* __restrict__ slot_out,
                                                const unsigned long long* __restrict__ n_dev,
                                                const uint32_t* __restrict__ out_idx,
                                                const uint32_t* __restrict__ o_start,
                                                unsigned long long* __restrict__ exc) {
  if (n_dev) n = *n_dev;
  using P = Probe<LAY, K, V, G>;
  using Ops = typename P::Ops;
  constexpr int CHUNK = insert_chunk<K, V, MODE>();
  long long nexc = 0;  // statuses other than INSERTED (staged.cu skips its status gathers without any)
  __shared__ ChunkState cs;
  __shared__ K s_keys[CHUNK];
  __shared__ uint32_t s_hw[CHUNK], s_sw[CHUNK];
  __shared__ uint8_t s_ho[CHUNK];
  const StartSlots ss{s_hw, s_sw, s_ho};
  __shared__ V s_vals[MODE == 0 ? CHUNK : 1];
  __shared__ uint8_t s_status[CHUNK];
  __shared__ int64_t s_slot[MODE == 1 ? CHUNK : 1];
  constexpr int lane = 0;  // one thread per key (probe.cuh)
  long long occ = 0, tomb = 0, ops = 0, att = 0, win = 0;

  __shared__ uint16_t q_li[CHUNK];
  __shared__ uint8_t q_o[CHUNK];
  __shared__ uint32_t q_cnt;
  using F = FastSpan<LAY, K, V>;

  while (chunk_begin<CHUNK>(cs, T.work, n)) {
    if (threadIdx.x == 0) q_cnt = 0;
    stage_keys(s_keys, ss, keys, cs, T);
    if (MODE == 0) stage_in(s_vals, vals, cs);
    __syncthreads();

    // ---- fast pass: one 128 B step per key; claims the first slot when it is an
    // empty with no tombstone before it (the common case), otherwise queues the key
    for (uint32_t fi = threadIdx.x; fi < cs.cnt; fi += blockDim.x) {
      const K fkey = s_keys[fi];
      if (fkey == (K)T.e || fkey == (K)T.t) {  // INVALID_KEY, no accounting (single_table.py:369-370)
        s_status[fi] = ST_INVALID;
        if (MODE == 1) s_slot[fi] = -1;
        continue;
      }
      const ProbeStart fps = ss.get(fi);
      F fs;
      // o0 = WINDOW: the staged pass saw window 0 hold neither the key nor a free
      // cell, so the fast span runs at window 1's start (staged.cu)
      const uint32_t o0 = o_start ? o_start[cs.base + fi] : 0u;
      const uint32_t jw = o0 ? 1u : 0u;
      uint32_t o_next = o0;
      uint64_t fws = fps.h;
      if (jw) {
        fws += fps.step;
        if (fws >= T.c) fws -= T.c;
      }
      if ((o0 == 0 || (o0 == WINDOW && T.max_windows > 1)) && fs.load(T, fws, fkey)) {
        const uint32_t kb = fs.km & below_lowest(fs.em);
        int res = OUT_NONE;
        uint32_t u = 0;
        if (kb) {
          u = lowest_bit(kb);
          res = OUT_FOUND;
        } else if (fs.em && !(fs.tm & below_lowest(fs.em))) {
          u = lowest_bit(fs.em);
          bool won = false;
          const K seen = Ops::claim(T, fs.base + u, (K)T.e, fkey, MODE == 0 ? s_vals[fi] : (V)0, MODE == 0, &won);
          if (won) res = OUT_CLAIMED;
          else if (seen == fkey) res = OUT_FOUND;
        } else if (!fs.em && !fs.tm) {
          o_next = o0 + fs.n_use;  // nothing free and no key in the span: continue after it
        }
        if (res != OUT_NONE) {
          ops += 1;
          att += (long long)(jw * WINDOW + chunk_end(u - fs.lo, G));
          win += 1 + jw;
          s_status[fi] = res == OUT_CLAIMED ? ST_INSERTED : ST_DUPLICATE;
          if (MODE == 1) s_slot[fi] = (int64_t)(fs.base + u);
          if (res == OUT_CLAIMED) occ += 1;
          continue;
        }
      }
      const uint32_t qi = atomicAdd(&q_cnt, 1u);
      q_li[qi] = (uint16_t)fi;
      q_o[qi] = (uint8_t)o_next;
    }
    __syncthreads();
    const uint32_t nq = q_cnt;

    bool active = false;
    uint32_t li = 0;
    K key = 0;
    V val = 0;
    ProbeStart ps{0, 0};
    Cursor cur;
    cur.init(0);
    int64_t pending = -1;
    for (;;) {
      if (!active) {
        const uint32_t qi = atomicAdd(&cs.next, 1u);
        if (qi >= nq) break;
        li = q_li[qi];
        key = s_keys[li];
        if (MODE == 0) val = s_vals[li];
        ps = ss.get(li);
        pending = -1;
        if (!cursor_seek(T, cur, ps.h, ps.step, q_o[qi])) {  // budget spent without a free slot
          ops += 1;
          att += (long long)cur.attempts;
          win += (long long)cur.windows_seen;
          s_status[li] = ST_TABLE_FULL;
          if (MODE == 1) s_slot[li] = -1;
          continue;
        }
        active = true;
      }

      typename P::Step st;
      P::load(T, cur, key, st);

      int outcome = OUT_NONE;
      uint64_t oslot = 0;
      bool was_tomb = false;
      bool add_chunk = true;  // final chunk accounting (false after a whole cycle)
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
          bool won = false;
          const K seen = Ops::claim(T, (uint64_t)target, expected, key, val, MODE == 0, &won);
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
          s_status[li] = outcome == OUT_CLAIMED ? ST_INSERTED : outcome == OUT_FOUND ? ST_DUPLICATE : ST_TABLE_FULL;
          if (MODE == 1) s_slot[li] = outcome == OUT_FULL ? -1 : (int64_t)oslot;
        }
        if (outcome == OUT_CLAIMED) {
          occ += 1;
          if (was_tomb) tomb -= 1;
        }
        active = false;
      }
    }
    __syncthreads();
    stage_out_ix(status, s_status, cs, out_idx);
    if (MODE == 1) stage_out(slot_out, s_slot, cs);
    if (exc)
      for (uint32_t j = threadIdx.x; j < cs.cnt; j += blockDim.x) nexc += s_status[j] != ST_INSERTED;
  }
  const long long v[6] = {ops, att, win, occ, tomb, nexc};
  long long* const dst[6] = {(long long*)&T.ctr->ops, (long long*)&T.ctr->attempts,
                             (long long*)&T.ctr->windows, &T.ctr->occupied, &T.ctr->tombstones, (long long*)exc};
  cta_add<6>(v, dst);
}

// ------------------------------------------------------------------ K2
// MODE 0: retrieve_bulk (single_table.py:376-408): value + found flag
// MODE 1: find (slot_of / retrieve_with_stats, :317-336): slot, attempts, windows, value
// MODE 2: erase (:338-351): retire the key (layout.py:224-243)
//
// Per chunk: a SIMT-uniform fast pass resolves every key whose answer lies in
// the first 128 B of window 0 (FastSpan); the rest are queued and finished by
// the flattened general loop.
template <Layout LAY, typename K, typename V, int G, int MODE>
__global__ void __launch_bounds__(256, CH_AB_PROBE_MINB) k_lookup(TableRef T, const K* __restrict__ keys, uint64_t n,
                                                V* __restrict__ vals_out, uint8_t* __restrict__ flag,
                                                int64_t* __restrict__ slot_out,
                                                uint32_t* __restrict__ att_out,
                                                uint32_t* __restrict__ win_out,
                                                const unsigned long long* __restrict__ n_dev,
                                                const uint32_t* __restrict__ out_idx,
                                                const uint32_t* __restrict__ o_start) {
  if (n_dev) n = *n_dev;
  using P = Probe<LAY, K, V, G>;
  using F = FastSpan<LAY, K, V>;
  constexpr int CH = MODE == 1 ? CHUNK_FIND : chunk_for<K, V>();
  __shared__ ChunkState cs;
  __shared__ K s_keys[CH];
  __shared__ uint32_t s_hw[CH], s_sw[CH];
  __shared__ uint8_t s_ho[CH];
  const StartSlots ss{s_hw, s_sw, s_ho};
  __shared__ V s_vals[MODE == 2 ? 1 : CH];
  __shared__ uint8_t s_flag[MODE == 1 ? 1 : CH];
  __shared__ int64_t s_slot[MODE == 1 ? CH : 1];
  __shared__ uint32_t s_att[MODE == 1 ? CH : 1];
  __shared__ uint32_t s_win[MODE == 1 ? CH : 1];
  __shared__ uint16_t q_li[CH];
  __shared__ uint8_t q_o[CH];
  __shared__ uint32_t q_cnt;
  long long ops = 0, att = 0, win = 0, occ = 0, tomb = 0;

  // record the outcome of one key (found at slot `slot` / absent), `attempts` in g-units
  auto finish = [&](uint32_t li, bool found, uint64_t slot, V value, bool erased, uint64_t attempts,
                    uint64_t windows) {
    if (MODE == 0) {
      s_vals[li] = found ? value : (V)0;
      s_flag[li] = (uint8_t)found;
    } else if (MODE == 1) {
      s_vals[li] = found ? value : (V)0;
      s_slot[li] = found ? (int64_t)slot : -1;
      s_att[li] = (uint32_t)attempts;
      s_win[li] = (uint32_t)windows;
    } else {
      s_flag[li] = erased;
      if (erased) { occ -= 1; tomb += 1; }
    }
    ops += 1;
    att += (long long)attempts;
    win += (long long)windows;
  };

  while (chunk_begin<CH>(cs, T.work, n)) {
    if (threadIdx.x == 0) q_cnt = 0;
    stage_keys(s_keys, ss, keys, cs, T);
    __syncthreads();

    // ---- fast pass: one 128 B step for every key of the chunk
    for (uint32_t li = threadIdx.x; li < cs.cnt; li += blockDim.x) {
      const K key = s_keys[li];
      if (key == (K)T.e || key == (K)T.t) {
        if (MODE == 0) { ops += 1; s_vals[li] = 0; s_flag[li] = 0; }  // retrieve_bulk counts every query (:403)
        if (MODE == 1) { s_slot[li] = -1; s_att[li] = 0; s_win[li] = 0; s_vals[li] = 0; }
        if (MODE == 2) s_flag[li] = 0;
        continue;
      }
      // o0 = WINDOW: window 0 is known to hold neither the key nor an empty (staged.cu):
      // the fast span runs at window 1's start
      const uint32_t o0 = o_start ? o_start[cs.base + li] : 0u;
      uint32_t o_next = o0;
      if (o0 == 0 || (o0 == WINDOW && T.max_windows > 1)) {
        const uint32_t jw = o0 ? 1u : 0u;
        const ProbeStart fps = ss.get(li);
        uint64_t fws = fps.h;
        if (jw) {
          fws += fps.step;
          if (fws >= T.c) fws -= T.c;
        }
        F fs;
        if (fs.load(T, fws, key)) {
          const uint32_t kb = fs.km & below_lowest(fs.em);
          if (kb) {
            const uint32_t u = lowest_bit(kb);
            const bool erased = MODE == 2 ? fs.retire(T, u) : false;
            finish(li, true, fs.base + u, MODE == 2 ? (V)0 : fs.value(T, u), erased,
                   jw * WINDOW + chunk_end(u - fs.lo, G), 1 + jw);
            continue;
          }
          if (fs.em) {
            finish(li, false, 0, (V)0, false, jw * WINDOW + chunk_end(lowest_bit(fs.em) - fs.lo, G), 1 + jw);
            continue;
          }
          o_next = o0 + fs.n_use;
        }
      }
      const uint32_t qi = atomicAdd(&q_cnt, 1u);
      q_li[qi] = (uint16_t)li;
      q_o[qi] = (uint8_t)o_next;
    }
    __syncthreads();

    // ---- general loop over the queued keys (flattened, one step per iteration)
    bool active = false;
    uint32_t li = 0;
    K key = 0;
    ProbeStart ps{0, 0};
    Cursor cur;
    cur.init(0);
    const uint32_t nq = q_cnt;
    for (;;) {
      if (!active) {
        uint32_t qi = atomicAdd(&cs.next, 1u);
        if (qi >= nq) break;
        li = q_li[qi];
        key = s_keys[li];
        ps = ss.get(li);
        if (!cursor_seek(T, cur, ps.h, ps.step, q_o[qi])) {  // window budget spent: absent
          finish(li, false, 0, (V)0, false, cur.attempts, cur.windows_seen);
          continue;
        }
        active = true;
      }
      typename P::Step st;
      P::load(T, cur, key, st);
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
      const bool erased = MODE == 2 && found ? P::retire(T, st, u) : false;
      finish(li, found, st.base + u, (MODE != 2 && found) ? P::value(T, st, u) : (V)0, erased, attempts,
             cur.windows_seen);
      active = false;
    }
    __syncthreads();
    if (MODE == 0) {
      stage_out_ix(vals_out, s_vals, cs, out_idx);
      stage_out_ix(flag, s_flag, cs, out_idx);
    } else if (MODE == 1) {
      stage_out(slot_out, s_slot, cs);
      if (att_out) stage_out(att_out, s_att, cs);
      if (win_out) stage_out(win_out, s_win, cs);
      if (vals_out) stage_out(vals_out, s_vals, cs);
    } else {
      stage_out_ix(flag, s_flag, cs, out_idx);  // erase (staged.cu passes out_idx for its deferred keys)
    }
  }
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
    if (mode == 0) {
      auto kern = k_insert<LAY, K, V, G, 0>;
      return launch_chunked(lc, T, (const void*)kern, n, insert_chunk<K, V, 0>(), [&](dim3 g, dim3 b) {
        kern<<<g, b, 0, lc.stream>>>(T, (const K*)keys, (const V*)vals, n, status, slot_out, lc.n_dev,
                                     lc.out_idx, lc.o_start, lc.exc);
      });
    }
    auto kern = k_insert<LAY, K, V, G, 1>;
    return launch_chunked(lc, T, (const void*)kern, n, insert_chunk<K, V, 1>(), [&](dim3 g, dim3 b) {
      kern<<<g, b, 0, lc.stream>>>(T, (const K*)keys, (const V*)vals, n, status, slot_out, lc.n_dev,
                                     lc.out_idx, lc.o_start, lc.exc);
    });
  }
  static int lookup(const Launch& lc, const TableRef& T, const void* keys, uint64_t n, void* vals_out,
                    uint8_t* flag, int64_t* slot_out, uint32_t* att_out, uint32_t* win_out, int mode) {
#define CHB_LOOKUP(M, CH)                                                                              \
  {                                                                                                    \
    auto kern = k_lookup<LAY, K, V, G, M>;                                                             \
    return launch_chunked(lc, T, (const void*)kern, n, CH, [&](dim3 g, dim3 b) {                       \
      kern<<<g, b, 0, lc.stream>>>(T, (const K*)keys, n, (V*)vals_out, flag, slot_out, att_out, win_out,   \
                                   lc.n_dev, lc.out_idx, lc.o_start);                                  \
    });                                                                                                \
  }
    if (mode == 0) CHB_LOOKUP(0, (chunk_for<K, V>()))
    if (mode == 1) CHB_LOOKUP(1, CHUNK_FIND)
    CHB_LOOKUP(2, (chunk_for<K, V>()))
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
