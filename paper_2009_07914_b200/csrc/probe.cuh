// probe.cuh -- the COPS probe step shared by every table kernel.
//
// One step: the prober loads the aligned span containing the next unexamined
// slot of its key's sequence and builds three bit masks over the span (bit u
// <=> slot base+u): key matches, empties and tombstones, restricted to the
// slots that belong to the current window at or after the cursor.  Callers
// decide in sequence order (lowest bit first), which is the reference's
// lowest-index-first rule (single_table.py:198-223).
//
// B200 mapping.  The paper probes with a cooperative group of g lanes, one
// slot per lane, combined by ballots.  A B200 thread can issue 256-bit loads,
// so here ONE thread owns a key and loads the whole span itself with up to
// four 32 B vector loads issued back to back (one memory latency per step).
// There is no cross-lane reduction at all: on sm_100a the tile shuffles of
// divergent probe groups compiled to ~150 SHFL + 50 WARPSYNC.COLLECTIVE per
// loop body (profiles/r01_sass_tile_shuffles.txt).  The span is group_width
// slots capped at 128 B; the reference's per-g probe counters stay exact
// because they are computed from sequence positions (chunk_end), not from the
// hardware span.
#pragma once
#include "common.cuh"

namespace chb {

template <Layout LAY, typename K, typename V, int G>
struct Probe {
  using Ops = LayoutOps<LAY, K, V>;
  static constexpr int A_MAX = 128 / Ops::UNIT > 0 ? 128 / Ops::UNIT : 1;
  static constexpr int A = G < A_MAX ? G : A_MAX;                   // slots per step (power of 2, divides 32)
  static constexpr int SPL = A < Ops::SPL_MAX ? A : Ops::SPL_MAX;   // slots per vector load
  static constexpr int NV = A / SPL;                                // vector loads per step
  static constexpr int L = 1;
  using Slots = typename Ops::template Slots<SPL>;
  static_assert(SPL * NV == A && A >= 1 && A <= 32 && (32 % A) == 0, "bad span");

  struct Step {
    uint64_t base;   // aligned span start slot
    uint32_t lo;     // first useful bit
    uint32_t n_use;  // useful bits
    uint32_t km, em, tm;
    Slots sl[NV];
  };

  __device__ __forceinline__ static void load(const TableRef& T, const Cursor& cur, K key, Step& st) {
    const uint64_t q = cur.slot(T);
    st.base = q & ~(uint64_t)(A - 1);
    st.lo = (uint32_t)(q - st.base);
    const uint32_t room = WINDOW - cur.o;
    st.n_use = (A - st.lo) < room ? (A - st.lo) : room;
    const uint32_t hi = st.lo + st.n_use;
#pragma unroll
    for (int v = 0; v < NV; ++v) st.sl[v] = Ops::template load<SPL>(T, st.base + (uint64_t)v * SPL);
    uint32_t km = 0, em = 0, tm = 0;
    const K e = (K)T.e, t = (K)T.t;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
#pragma unroll
      for (int s = 0; s < SPL; ++s) {
        const uint32_t u = (uint32_t)(v * SPL + s);
        const K k = st.sl[v].key(s);
        km |= (uint32_t)(k == key) << u;
        em |= (uint32_t)(k == e) << u;
        tm |= (uint32_t)(k == t) << u;
      }
    }
    const uint32_t range = (hi >= 32 ? 0xFFFFFFFFu : ((1u << hi) - 1u)) & ~((1u << st.lo) - 1u);
    st.km = km & range;
    st.em = em & range;
    st.tm = tm & range;
  }

  // value / retire of span bit u (register-only part selection)
  __device__ __forceinline__ static V value(const TableRef& T, const Step& st, uint32_t u) {
    const int part = (int)(u / SPL), s = (int)(u % SPL);
    if constexpr (NV == 1) return Ops::template value<SPL>(T, st.base + u, st.sl[0], s);
    V r = 0;
#pragma unroll
    for (int v = 0; v < NV; ++v)
      if (v == part) r = Ops::template value<SPL>(T, st.base + u, st.sl[v], s);
    return r;
  }
  __device__ __forceinline__ static bool retire(const TableRef& T, const Step& st, uint32_t u) {
    const int part = (int)(u / SPL), s = (int)(u % SPL);
    bool won = false;
#pragma unroll
    for (int v = 0; v < NV; ++v)
      if (v == part) won = Ops::template retire<SPL>(T, st.base + u, st.sl[v], s);
    return won;
  }

  // in-window offset of span bit u
  __device__ __forceinline__ static uint32_t offset_of(const Cursor& cur, const Step& st, uint32_t u) {
    return cur.o + (u - st.lo);
  }

  // Move past the examined part of the span.  Returns false when the
  // max_outer_attempts windows are exhausted (probing.py:214-217).
  __device__ __forceinline__ static bool advance(const TableRef& T, Cursor& cur, const Step& st, uint64_t step) {
    cur.o += st.n_use;
    if (cur.o == WINDOW) {
      cur.attempts += WINDOW;
      cur.j += 1;
      if (cur.j >= T.max_windows) return false;
      cur.windows_seen += 1;
      cur.ws += step;
      if (cur.ws >= T.c) cur.ws -= T.c;
      cur.o = 0;
    }
    return true;
  }
};

// First-step fast path: the 128 B that start at the window start (rounded down
// to 32 B), i.e. >= 13 useful slots of window 0 for 8 B slots, in four
// independent 256-bit loads.  Kernels run it for every key of a chunk in a
// SIMT-uniform pre-pass; only keys it cannot resolve enter the divergent
// general loop (profiles: ~22 -> ~8 warp-instructions per retrieved key).
template <Layout LAY, typename K, typename V>
struct FastSpan {
  using Ops = LayoutOps<LAY, K, V>;
  static constexpr int SPL = Ops::SPL_MAX;                               // slots per 32 B load
  static constexpr int FAST = (128 / Ops::UNIT) < 32 ? (128 / Ops::UNIT) : 32;
  static constexpr int NV = FAST / SPL;
  using Slots = typename Ops::template Slots<SPL>;
  static_assert(NV * SPL == FAST && FAST <= 32, "bad fast span");

  uint64_t base;
  uint32_t lo, n_use;
  uint32_t km, em, tm;
  Slots sl[NV];

  // false when the span would run past the end of the slot array (rare; the
  // caller then takes the general path from the window start)
  __device__ __forceinline__ bool load(const TableRef& T, uint64_t q0, K key) {
    base = q0 & ~(uint64_t)(SPL - 1);
    if (base + FAST > T.c) return false;
    lo = (uint32_t)(q0 - base);
    n_use = FAST - lo;  // <= 32, all inside window 0
#pragma unroll
    for (int v = 0; v < NV; ++v) sl[v] = Ops::template load<SPL>(T, base + (uint64_t)v * SPL);
    uint32_t k_ = 0, e_ = 0, t_ = 0;
    const K e = (K)T.e, t = (K)T.t;
#pragma unroll
    for (int v = 0; v < NV; ++v) {
#pragma unroll
      for (int s = 0; s < SPL; ++s) {
        const uint32_t u = (uint32_t)(v * SPL + s);
        const K k = sl[v].key(s);
        k_ |= (uint32_t)(k == key) << u;
        e_ |= (uint32_t)(k == e) << u;
        t_ |= (uint32_t)(k == t) << u;
      }
    }
    const uint32_t range = (FAST >= 32 ? 0xFFFFFFFFu : ((1u << FAST) - 1u)) & ~((1u << lo) - 1u);
    km = k_ & range;
    em = e_ & range;
    tm = t_ & range;
    return true;
  }
  __device__ __forceinline__ V value(const TableRef& T, uint32_t u) const {
    const int part = (int)(u / SPL), s = (int)(u % SPL);
    V r = 0;
#pragma unroll
    for (int v = 0; v < NV; ++v)
      if (v == part) r = Ops::template value<SPL>(T, base + u, sl[v], s);
    return r;
  }
  __device__ __forceinline__ bool retire(const TableRef& T, uint32_t u) const {
    const int part = (int)(u / SPL), s = (int)(u % SPL);
    bool won = false;
#pragma unroll
    for (int v = 0; v < NV; ++v)
      if (v == part) won = Ops::template retire<SPL>(T, base + u, sl[v], s);
    return won;
  }
};

// Position a fresh cursor (window 0 at h) at in-window offset o; returns false
// if that exhausts the window budget.
// (o < 2 WINDOW: the fast pass examines at most window 0 or the start of window 1)
__device__ __forceinline__ bool cursor_seek(const TableRef& T, Cursor& cur, uint64_t h, uint64_t step, uint32_t o) {
  cur.init(h);
  while (o >= WINDOW) {
    cur.attempts += WINDOW;
    cur.j += 1;
    if (cur.j >= T.max_windows) return false;
    cur.windows_seen += 1;
    cur.ws += step;
    if (cur.ws >= T.c) cur.ws -= T.c;
    o -= WINDOW;
  }
  cur.o = o;
  return true;
}

__device__ __forceinline__ uint32_t lowest_bit(uint32_t m) { return (uint32_t)__ffs(m) - 1; }
// bits strictly below the lowest set bit of m (all bits when m == 0)
__device__ __forceinline__ uint32_t below_lowest(uint32_t m) { return m ? ((m & (0u - m)) - 1u) : 0xFFFFFFFFu; }

}  // namespace chb
