// probe.cuh -- the COPS probe step shared by every table kernel.
//
// One step: the group loads the aligned span containing the next unexamined
// slot of the key's sequence, and reduces three group-uniform bit masks over
// the span (bit u <=> slot base+u): key matches, empties and tombstones,
// restricted to the slots that belong to the current window at or after the
// cursor.  Callers decide in sequence order (lowest bit first), which is the
// reference's lowest-index-first rule (single_table.py:198-223).
#pragma once
#include "common.cuh"

namespace chb {

template <Layout LAY, typename K, typename V, int G>
struct Probe {
  using Geo = Geometry<LAY, K, V, G>;
  using Ops = typename Geo::Ops;
  static constexpr int SPL = Geo::SPL;
  static constexpr int L = Geo::L;
  static constexpr int A = Geo::A;
  using Slots = typename Ops::template Slots<SPL>;

  struct Step {
    uint64_t base;   // aligned span start slot
    uint32_t lo;     // first useful bit
    uint32_t n_use;  // useful bits
    uint32_t km, em, tm;
    Slots sl;        // this lane's SPL slots
  };

  template <typename Tile>
  __device__ __forceinline__ static void load(const TableRef& T, const Tile& tile, const Cursor& cur,
                                              K key, Step& st) {
    const uint64_t q = cur.slot(T);
    st.base = q & ~(uint64_t)(A - 1);
    st.lo = (uint32_t)(q - st.base);
    const uint32_t room = WINDOW - cur.o;
    st.n_use = (A - st.lo) < room ? (A - st.lo) : room;
    const uint32_t hi = st.lo + st.n_use;
    const int lane = L > 1 ? (int)tile.thread_rank() : 0;
    st.sl = Ops::template load<SPL>(T, st.base + (uint64_t)lane * SPL);
    uint32_t km = 0, em = 0, tm = 0;
    const K e = (K)T.e, t = (K)T.t;
#pragma unroll
    for (int s = 0; s < SPL; ++s) {
      const uint32_t u = (uint32_t)(lane * SPL + s);
      const bool in = u >= st.lo && u < hi;
      const K k = st.sl.key(s);
      km |= (uint32_t)(in && k == key) << u;
      em |= (uint32_t)(in && k == e) << u;
      tm |= (uint32_t)(in && k == t) << u;
    }
    st.km = tile_or<L>(tile, km);
    st.em = tile_or<L>(tile, em);
    st.tm = tile_or<L>(tile, tm);
  }

  // in-window offset of span bit u
  __device__ __forceinline__ static uint32_t offset_of(const Cursor& cur, const Step& st, uint32_t u) {
    return cur.o + (u - st.lo);
  }

  // Move past the examined part of the span.  Returns false when the
  // max_outer_attempts windows are exhausted (probing.py:214-217).
  __device__ __forceinline__ static bool advance(const TableRef& T, Cursor& cur, const Step& st,
                                                 uint64_t step) {
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

__device__ __forceinline__ uint32_t lowest_bit(uint32_t m) { return (uint32_t)__ffs(m) - 1; }
// bits strictly below the lowest set bit of m (all bits when m == 0)
__device__ __forceinline__ uint32_t below_lowest(uint32_t m) { return m ? ((m & (0u - m)) - 1u) : 0xFFFFFFFFu; }

template <typename X, typename Tile>
__device__ __forceinline__ X tile_bcast(const Tile& tile, X v, int src) {
  if constexpr (Tile::num_threads() > 1) return tile.shfl(v, src);
  return v;
}

}  // namespace chb
