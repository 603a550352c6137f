// common.cuh -- device-side building blocks of the B200 COPS hash tables.
//
// Semantics follow the reference package coophash:
//   mix64 / HashFn            probing.py:79-117
//   dh_step                   probing.py:220-229
//   window starts (h + j*step) mod c, window width 32   single_table.py:192
//   sentinels e = 2^kb-1, t = 2^kb-2                     layout.py:50-53
//   packed word = value << 32 | key                      layout.py:56-62
//
// Hardware mapping (B200-first, not the reference's chunking): a probe group
// of L lanes examines an ALIGNED span of A = group_width slots per step, each
// lane issuing one vector load of SPL consecutive slots (8..256 bit).  Slots
// before the window start inside the first span are masked off, so the slot
// sequence visited is exactly the reference's unaligned COPS order
// (probing.py:266-284); only the memory transactions are aligned.  DRAM on
// B200 is random-access-rate bound for <= 64 B requests (profiles/randbench),
// so an aligned span is one request however few slots of it are useful.
#pragma once
#include <cooperative_groups.h>
#include <cstdint>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

namespace chb {

constexpr uint32_t WINDOW = 32;
constexpr uint64_t STEP_SEED = 0x9E3779B97F4A7C15ull;

// Per-element status codes == InsertStatus order (single_table.py:48-53).
enum : uint8_t { ST_INSERTED = 0, ST_DUPLICATE = 1, ST_TABLE_FULL = 2, ST_INVALID = 3, ST_OOM = 4 };

enum Layout : int { SOA = 0, AOS = 1, PACKED = 2 };

// Device-resident counters; reduced per CTA, one atomic per CTA per field.
struct DevCounters {
  unsigned long long ops;
  unsigned long long attempts;
  unsigned long long windows;
  long long occupied;
  long long tombstones;
  long long total_values;   // bucket list
  unsigned long long pool_used;  // bucket list: successfully allocated slots
  unsigned long long error;      // sticky device error flags (bit 0: contention timeout)
  unsigned long long deferred;   // staged keys finished by the COPS kernels (staged.cu)
};

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t key) {
  uint64_t x = key + STEP_SEED;
  x ^= x >> 33;
  x *= 0xFF51AFD7ED558CCDull;
  x ^= x >> 33;
  x *= 0xC4CEB9FE1A85EC53ull;
  x ^= x >> 33;
  return x;
}

// x mod d by Barrett reduction with m = floor(2^64 / d) (d >= 2): the quotient
// estimate is off by at most one, so a single conditional subtract is exact.
struct FastMod {
  uint64_t d, m;
  __host__ static FastMod make(uint64_t d_) {
    FastMod f;
    f.d = d_;
    f.m = d_ >= 2 ? (uint64_t)(((unsigned __int128)1 << 64) / d_) : 0;
    return f;
  }
  __device__ __forceinline__ uint64_t mod(uint64_t x) const {
    if (d < 2) return 0;
    uint64_t q = __umul64hi(x, m);
    uint64_t r = x - q * d;
    return r >= d ? r - d : r;
  }
  // d < 2^31 (and >= 2): the remainder before the correction is below 2d < 2^32,
  // so it is exact in the low words (one 32-bit multiply instead of a 64-bit one)
  __device__ __forceinline__ uint32_t mod31(uint64_t x) const {
    const uint32_t q = (uint32_t)__umul64hi(x, m);
    const uint32_t r = (uint32_t)x - q * (uint32_t)d;
    return r >= (uint32_t)d ? r - (uint32_t)d : r;
  }
  __device__ __forceinline__ uint64_t mod_any(uint64_t x) const { return (d >> 31) ? mod(x) : (uint64_t)mod31(x); }
};

// Everything a kernel needs to walk a table.  Passed by value.
struct TableRef {
  void* slots;      // PACKED: u64 words; SOA: key array; AOS: cell array
  void* vals;       // SOA: value array (unused otherwise)
  uint64_t c;       // capacity = 32 p
  uint64_t p;       // prime window count
  uint64_t max_windows;
  uint64_t e, t;    // sentinels
  FastMod modc, modpm1;
  DevCounters* ctr;
  unsigned long long* work;  // chunk queue of the running probe kernel (sched.cuh)
};

struct ProbeStart {
  uint64_t h, step;
};

__device__ __forceinline__ ProbeStart probe_start(const TableRef& T, uint64_t key) {
  ProbeStart s;
  s.h = T.modc.mod_any(mix64(key));  // HashFn(0).value(key) % c
  s.step = T.p == 2 ? (uint64_t)WINDOW : (uint64_t)WINDOW * (1 + T.modpm1.mod_any(mix64(STEP_SEED ^ key)));
  return s;
}

// ----------------------------------------------------------------- loads
// Table words are read through L2 only (.cg): L1 is not coherent with the
// CAS traffic of other SMs, and random probes get no L1 reuse anyway.

template <int BYTES>
struct Vec;
template <> struct Vec<4> { uint32_t w[1]; };
template <> struct Vec<8> { uint64_t w[1]; };
template <> struct Vec<16> { uint64_t w[2]; };
template <> struct Vec<32> { uint64_t w[4]; };

template <int BYTES>
__device__ __forceinline__ Vec<BYTES> ld_cg(const void* p);
template <> __device__ __forceinline__ Vec<4> ld_cg<4>(const void* p) {
  Vec<4> v;
  asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v.w[0]) : "l"(p));
  return v;
}
template <> __device__ __forceinline__ Vec<8> ld_cg<8>(const void* p) {
  Vec<8> v;
  asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v.w[0]) : "l"(p));
  return v;
}
template <> __device__ __forceinline__ Vec<16> ld_cg<16>(const void* p) {
  Vec<16> v;
  asm volatile("ld.global.cg.v2.u64 {%0,%1}, [%2];" : "=l"(v.w[0]), "=l"(v.w[1]) : "l"(p));
  return v;
}
template <> __device__ __forceinline__ Vec<32> ld_cg<32>(const void* p) {
  Vec<32> v;
  asm volatile("ld.global.cg.v4.u64 {%0,%1,%2,%3}, [%4];"
               : "=l"(v.w[0]), "=l"(v.w[1]), "=l"(v.w[2]), "=l"(v.w[3])
               : "l"(p));
  return v;
}

// Batch inputs / outputs.  Probe groups consume keys and emit results at
// different times (each resolves its key after a different number of steps),
// so neighbouring elements of one 128 B line are touched by many warps over a
// short interval.  Evict-first (.cs) hints made L2 drop such lines between
// touches -- every 4 B key re-fetched a 128 B line and every 1-4 B result
// became a DRAM read-modify-write (profiles/r01_launches_loc_v1.csv).  Default
// caching lets L2 merge them: one line fill / write-back per 128 B.
template <typename X>
__device__ __forceinline__ X ld_stream(const X* p) { return __ldg(p); }
template <typename X>
__device__ __forceinline__ void st_stream(X* p, X v) { *p = v; }

__device__ __forceinline__ uint32_t atomic_cas(uint32_t* p, uint32_t cmp, uint32_t val) {
  return atomicCAS(reinterpret_cast<unsigned int*>(p), cmp, val);
}
__device__ __forceinline__ uint64_t atomic_cas(uint64_t* p, uint64_t cmp, uint64_t val) {
  return atomicCAS(reinterpret_cast<unsigned long long*>(p), (unsigned long long)cmp,
                   (unsigned long long)val);
}

// ------------------------------------------------------------- layouts
// A layout exposes:
//   SPL_MAX           max slots one lane loads with a single (<= 32 B) vector load
//   load<SPL>(T, s)   keys (and whatever else is cheap) of slots s..s+SPL
//   claim(...)        CAS a free key cell, write the value (layout.py:174-205)
//   value(...)        the value of a slot whose key matched
//   retire(...)       CAS key -> tombstone (layout.py:224-243)

// Register-only selection of element s from a small array (a runtime index
// into a register array would spill it to the stack).
template <typename X, int N>
__device__ __forceinline__ X reg_select(const X (&a)[N], int s) {
  X r = a[0];
#pragma unroll
  for (int i = 1; i < N; ++i) r = (i == s) ? a[i] : r;
  return r;
}

template <typename K, typename V>
struct CellT {
  K k;
  V v;
};

template <Layout LAY, typename K, typename V>
struct LayoutOps;

// Packed AoS: one u64 word per slot, value << 32 | key (layout.py:56-66,195-205).
template <>
struct LayoutOps<PACKED, uint32_t, uint32_t> {
  using K = uint32_t;
  using V = uint32_t;
  static constexpr int UNIT = 8;
  static constexpr int SPL_MAX = 4;
  template <int SPL>
  struct Slots {
    uint64_t w[SPL];
    __device__ __forceinline__ K key(int s) const { return (K)w[s]; }
    __device__ __forceinline__ V val(int s) const { return (V)(reg_select(w, s) >> 32); }
    __device__ __forceinline__ uint64_t word(int s) const { return reg_select(w, s); }
  };
  template <int SPL>
  __device__ __forceinline__ static Slots<SPL> load(const TableRef& T, uint64_t s) {
    Slots<SPL> r;
    auto v = ld_cg<SPL * 8>(static_cast<const uint64_t*>(T.slots) + s);
#pragma unroll
    for (int i = 0; i < SPL; ++i) r.w[i] = v.w[i];
    return r;
  }
  // CAS a free cell (empty or tombstone; their packed words carry value 0)
  // to (key, value) in one atomic step (layout.py:195-205).  Returns the key
  // observed in the cell; *won tells whether this call claimed it.
  __device__ __forceinline__ static K claim(const TableRef& T, uint64_t slot, K expected, K key, V value,
                                            bool write_value, bool* won) {
    const uint64_t exp = (uint64_t)expected;
    const uint64_t desired = ((uint64_t)(write_value ? value : 0) << 32) | key;
    const uint64_t old = atomic_cas(static_cast<uint64_t*>(T.slots) + slot, exp, desired);
    *won = old == exp;
    return (K)old;
  }
  template <int SPL>
  __device__ __forceinline__ static V value(const TableRef&, uint64_t, const Slots<SPL>& seen, int s) {
    return seen.val(s);
  }
  template <int SPL>
  __device__ __forceinline__ static bool retire(const TableRef& T, uint64_t slot, const Slots<SPL>& seen,
                                                int s) {
    const uint64_t tomb = (uint64_t)(K)T.t;  // packed tombstone zeroes the value (layout.py:231)
    const uint64_t w = seen.word(s);
    return atomic_cas(static_cast<uint64_t*>(T.slots) + slot, w, tomb) == w;
  }
  __device__ __forceinline__ static V* value_ptr(const TableRef&, uint64_t) { return nullptr; }
};

// SoA: separate key and value arrays (layout.py:95-98).
template <typename K_, typename V_>
struct LayoutOps<SOA, K_, V_> {
  using K = K_;
  using V = V_;
  static constexpr int UNIT = sizeof(K);
  static constexpr int SPL_MAX = 32 / sizeof(K);
  template <int SPL>
  struct Slots {
    K k[SPL];
    __device__ __forceinline__ K key(int s) const { return k[s]; }
  };
  template <int SPL>
  __device__ __forceinline__ static Slots<SPL> load(const TableRef& T, uint64_t s) {
    Slots<SPL> r;
    constexpr int BYTES = SPL * sizeof(K);
    auto v = ld_cg<BYTES>(static_cast<const K*>(T.slots) + s);
    const K* kk = reinterpret_cast<const K*>(&v);
#pragma unroll
    for (int i = 0; i < SPL; ++i) r.k[i] = kk[i];
    return r;
  }
  // CAS the key cell, then a plain value store (layout.py:174-193, 162-170)
  __device__ __forceinline__ static K claim(const TableRef& T, uint64_t slot, K expected, K key, V value,
                                            bool write_value, bool* won) {
    const K old = atomic_cas(static_cast<K*>(T.slots) + slot, expected, key);
    *won = old == expected;
    if (*won && write_value) static_cast<V*>(T.vals)[slot] = value;
    return old;
  }
  template <int SPL>
  __device__ __forceinline__ static V value(const TableRef& T, uint64_t slot, const Slots<SPL>&, int) {
    return __ldcg(static_cast<const V*>(T.vals) + slot);
  }
  template <int SPL>
  __device__ __forceinline__ static bool retire(const TableRef& T, uint64_t slot, const Slots<SPL>& seen,
                                                int s) {
    const K k = reg_select(seen.k, s);
    return atomic_cas(static_cast<K*>(T.slots) + slot, k, (K)T.t) == k;
  }
  __device__ __forceinline__ static V* value_ptr(const TableRef& T, uint64_t slot) {
    return static_cast<V*>(T.vals) + slot;
  }
};

// AoS: interleaved (key, value) cells (layout.py:99-101).
template <typename K_, typename V_>
struct LayoutOps<AOS, K_, V_> {
  using K = K_;
  using V = V_;
  using Cell = CellT<K, V>;
  static constexpr int UNIT = sizeof(Cell);
  static constexpr int SPL_MAX = 32 / sizeof(Cell);
  template <int SPL>
  struct Slots {
    Cell c[SPL];
    __device__ __forceinline__ K key(int s) const { return c[s].k; }
  };
  template <int SPL>
  __device__ __forceinline__ static Slots<SPL> load(const TableRef& T, uint64_t s) {
    Slots<SPL> r;
    constexpr int BYTES = SPL * sizeof(Cell);
    auto v = ld_cg<BYTES>(static_cast<const Cell*>(T.slots) + s);
    const Cell* cc = reinterpret_cast<const Cell*>(&v);
#pragma unroll
    for (int i = 0; i < SPL; ++i) r.c[i] = cc[i];
    return r;
  }
  __device__ __forceinline__ static K claim(const TableRef& T, uint64_t slot, K expected, K key, V value,
                                            bool write_value, bool* won) {
    Cell* cell = static_cast<Cell*>(T.slots) + slot;
    const K old = atomic_cas(&cell->k, expected, key);
    *won = old == expected;
    if (*won && write_value) cell->v = value;
    return old;
  }
  template <int SPL>
  __device__ __forceinline__ static V value(const TableRef& T, uint64_t slot, const Slots<SPL>& seen, int s) {
    // the loaded cell carries the value; re-read it through L2 in case the
    // claimant's value store landed after our window load (split layouts).
    return __ldcg(&static_cast<const Cell*>(T.slots)[slot].v);
  }
  template <int SPL>
  __device__ __forceinline__ static bool retire(const TableRef& T, uint64_t slot, const Slots<SPL>& seen,
                                                int s) {
    K ks[SPL];
#pragma unroll
    for (int i = 0; i < SPL; ++i) ks[i] = seen.c[i].k;
    const K k = reg_select(ks, s);
    return atomic_cas(&static_cast<Cell*>(T.slots)[slot].k, k, (K)T.t) == k;
  }
  __device__ __forceinline__ static V* value_ptr(const TableRef& T, uint64_t slot) {
    return &static_cast<Cell*>(T.slots)[slot].v;
  }
};

// --------------------------------------------------------- probe group
// Geometry of one probe group for span A = G (the table's group_width).
template <Layout LAY, typename K, typename V, int G>
struct Geometry {
  using Ops = LayoutOps<LAY, K, V>;
  static constexpr int SPL = G < Ops::SPL_MAX ? G : Ops::SPL_MAX;  // slots per lane
  static constexpr int L = G / SPL;                                 // lanes per group
  static constexpr int A = G;                                       // aligned span (slots)
  static_assert(L * SPL == G, "span must be lanes * slots-per-lane");
  static_assert(L >= 1 && L <= 32, "bad group");
};

// OR-reduce a per-lane mask over the L lanes of a tile.
template <int L, typename Tile>
__device__ __forceinline__ uint32_t tile_or(const Tile& tile, uint32_t x) {
  if constexpr (L > 1) {
#pragma unroll
    for (int d = 1; d < L; d <<= 1) x |= tile.shfl_xor(x, d);
  }
  return x;
}

// Probe cursor: tracks the position along the reference's sequence
// (window j, in-window offset o) and the reference-unit probe counters.
struct Cursor {
  uint64_t ws;     // current window start slot
  uint32_t j;      // window index (restarts keep counting windows, as the reference)
  uint32_t o;      // in-window offset of the next unexamined slot
  uint64_t windows_seen;
  uint64_t attempts;
  __device__ __forceinline__ void init(uint64_t h) {
    ws = h; j = 0; o = 0; windows_seen = 1; attempts = 0;
  }
  // next slot index and this step's aligned block
  __device__ __forceinline__ uint64_t slot(const TableRef& T) const {
    uint64_t q = ws + o;
    return q >= T.c ? q - T.c : q;
  }
};

// Reference-unit probe count (single_table.py:197): g-sized chunks from the
// window start; an op that stops at in-window offset o in window j has probed
// 32 j + (o / g + 1) g slots (plus whatever full windows it walked before).
__device__ __forceinline__ uint64_t chunk_end(uint32_t o, uint32_t g) { return (uint64_t)((o & ~(g - 1u)) + g); }  // g = 2^k

// ------------------------------------------------------ CTA reductions
template <typename X>
__device__ __forceinline__ X warp_sum(X v) {
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
  return v;
}

// Sum NV per-thread values over the CTA and atomically add them to dst[].
// Must be called by all threads of the CTA (after the grid-stride loop).
template <int NV>
__device__ __forceinline__ void cta_add(const long long (&v)[NV], long long* const (&dst)[NV]) {
  __shared__ long long red[NV][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  long long w[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) w[i] = warp_sum(v[i]);
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) red[i][warp] = w[i];
  }
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      long long x = lane < nw ? red[i][lane] : 0;
      x = warp_sum(x);
      if (lane == 0 && x != 0 && dst[i]) atomicAdd(reinterpret_cast<unsigned long long*>(dst[i]),
                                                   (unsigned long long)x);
    }
  }
}

}  // namespace chb
