// staged.cu -- shared-memory-staged execution of big packed single-value batches.
//
// Why.  A bulk insert / retrieve over a table larger than L2 is a random-access
// workload: every key touches one or two 128 B lines of a 2 GiB slot array, so a
// probe-per-key kernel is bound by the DRAM random-access rate (~40 G 32-64 B
// requests/s on B200, profiles/randbench_2g.txt), not by bandwidth.  Ordering the
// batch so that each L2-sized region is probed by consecutive CTAs (locality.cu)
// still left the probe kernels L2-latency bound (4 L2 requests per key).
//
// What.  The batch is partitioned by the REGION of R = 2^13 slots (64 KiB of
// packed words) that its first window starts in.  One CTA then owns one region:
// it stages the region in shared memory with one TMA bulk copy, resolves every
// key of the region against it (the reference's window-0 rule, single_table.py:
// 171-245 / 247-269, shared-memory CAS of the key word for claims), and writes the region
// back with one bulk copy.  Every table byte crosses HBM once per batch, in 64 KiB
// transfers; keys that window 0 cannot decide (window full, a tombstone before
// the first empty, an insert window crossing the region end) are appended to a
// device-counted list and finished by the unchanged COPS probe kernels
// (single.cu) after the region pass -- a valid linearisation of the concurrent
// batch, since nothing is ever removed from a table during an insert or lookup.
//
// Pipeline (all passes stream; n keys):
//   L1      tile partition by super-region (256 regions)      k_st_split<1>
//           into fixed areas; on overflow the exact count-based L1 is redone by
//           gated kernels (count, scan, plan)                 k_st_count, k_st_plan
//   plan    per-super-region L2 tile map                      k_st_plan_oa
//   L2      tile partition by region, per super-region tiles  k_st_split<2>
//           into fixed region areas; over-full runs -> the COPS kernels
//   region  shared-memory probe of window 0                   k_st_probe
//   rest    deferred keys through the COPS kernels            single.cu (n_dev, out_idx, o_start)
//   back    results (status / value + found) to the caller's order: the inverse
//           of each tile partition, gathering that tile's runs   k_st_gather<2>, <1>
// A tile partition buckets a 4096-element tile in shared memory, writes whole
// (bucket, tile) runs, and records where each element went (u16 rank inside the
// tile, per-tile run table), so results return by gathering the same runs --
// every pass reads and writes coalesced and no position is carried per key.
#include <algorithm>
#include <climits>
#include <cstdlib>

#include "dispatch.cuh"

namespace chb {

constexpr int ST_LOG_R = 13;
constexpr uint32_t ST_R = 1u << ST_LOG_R;  // region slots
constexpr uint32_t ST_HALO = WINDOW;       // lookups read window 0 past the region end
constexpr int ST_S2 = 8;                   // regions per super-region = 2^ST_S2
constexpr int PT = 512, PI = 8;            // partition CTA: threads x items
constexpr uint32_t PTILE = (uint32_t)PT * PI;
constexpr uint32_t PBINS = 512;
constexpr int RT = 512;                    // region CTA threads
constexpr uint32_t ST_MAX_REGIONS = 51200; // count histogram in shared memory (200 KiB)
static_assert((ST_MAX_REGIONS >> ST_S2) <= (uint32_t)PT, "tile_super: one super-region per thread");

// Start slot of window wj (0 or 1) of key's COPS sequence: h, or h + step mod c
// (probing.py:202-220; step = 32 (1 + stephash mod (p-1)), p = 2 -> 32).  c < 2^32.
__device__ __forceinline__ uint32_t window_start(const TableRef& T, uint32_t key, int wj) {
  uint64_t ws = T.modc.mod_any(mix64((uint64_t)key));
  if (wj) {
    ws += T.p == 2 ? (uint64_t)WINDOW : (uint64_t)WINDOW * (1 + T.modpm1.mod_any(mix64(STEP_SEED ^ (uint64_t)key)));
    if (ws >= T.c) ws -= T.c;
  }
  return (uint32_t)ws;
}
__device__ __forceinline__ uint32_t region_of_key(const TableRef& T, uint32_t key, int wj) {
  return window_start(T, key, wj) >> ST_LOG_R;
}

// ------------------------------------------------------------- TMA helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// shared-memory atomic add as plain PTX (the compiler wraps atomicAdd in its own warp
// aggregation, ~17 instructions, even where one lane issues it)
__device__ __forceinline__ uint32_t atom_add_shared(uint32_t* p, uint32_t v) {
  uint32_t r;
  asm volatile("atom.shared.add.u32 %0, [%1], %2;" : "=r"(r) : "r"(smem_addr(p)), "r"(v) : "memory");
  return r;
}


__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(phase)
        : "memory");
  }
}
// global -> shared bulk copy (TMA, no tensor map), completion on an mbarrier
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
// shared -> global bulk copy; waits until the shared-memory source has been read (the
// global writes complete on their own before the kernel does)
__device__ __forceinline__ void bulk_store_wait(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void fence_smem_to_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// shared -> global bulk copy issued now, its shared-memory read awaited later (bulk_read_wait)
__device__ __forceinline__ void bulk_store_issue(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_read_wait() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
// bulk prefetch of [p, p + bytes) into L2 (one thread; 16-byte granules, size < 2^32)
__device__ __forceinline__ void l2_prefetch(const void* p, size_t bytes) {
  if (!bytes) return;
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(p) & ~(uintptr_t)15;
  const uintptr_t a1 = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~(uintptr_t)15;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((uint32_t)(a1 - a0)) : "memory");
}

// ------------------------------------------------------------- count
// Region histogram of the batch (dynamic shared memory, one counter per region).
// gate: run only when *gate != 0 (the count-mode redo of an overflowed level-1 pass).
__global__ void __launch_bounds__(1024) k_st_count(TableRef T, const uint32_t* __restrict__ keys, uint64_t n,
                                                   uint32_t regions, uint32_t* __restrict__ gcount,
                                                   const unsigned long long* __restrict__ n_dev, int wj,
                                                   const int* __restrict__ gate) {
  extern __shared__ uint32_t s_cnt[];
  if (gate && *gate == 0) return;
  if (n_dev) n = *n_dev;
  for (uint32_t i = threadIdx.x; i < regions; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  // 16-byte loads (four keys each, 4 in flight per thread) over the aligned body
  const uint64_t head = ((16 - ((uintptr_t)keys & 15)) & 15) / 4;  // keys before the first 16 B boundary
  const uint64_t h0 = head < n ? head : n;
  const uint64_t nv = (n - h0) / 4;
  const uint4* kv = reinterpret_cast<const uint4*>(keys + h0);
  uint64_t i = tid;
  for (; i + 3 * stride < nv; i += 4 * stride) {
    uint4 q[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) q[u] = __ldcs(kv + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      atomicAdd(&s_cnt[region_of_key(T, q[u].x, wj)], 1u);
      atomicAdd(&s_cnt[region_of_key(T, q[u].y, wj)], 1u);
      atomicAdd(&s_cnt[region_of_key(T, q[u].z, wj)], 1u);
      atomicAdd(&s_cnt[region_of_key(T, q[u].w, wj)], 1u);
    }
  }
  for (; i < nv; i += stride) {
    const uint4 q = __ldcs(kv + i);
    atomicAdd(&s_cnt[region_of_key(T, q.x, wj)], 1u);
    atomicAdd(&s_cnt[region_of_key(T, q.y, wj)], 1u);
    atomicAdd(&s_cnt[region_of_key(T, q.z, wj)], 1u);
    atomicAdd(&s_cnt[region_of_key(T, q.w, wj)], 1u);
  }
  // unaligned head and the tail past the last full vector
  if (tid < h0) atomicAdd(&s_cnt[region_of_key(T, keys[tid], wj)], 1u);
  const uint64_t t0 = h0 + nv * 4;
  if (tid < n - t0) atomicAdd(&s_cnt[region_of_key(T, keys[t0 + tid], wj)], 1u);
  __syncthreads();
  for (uint32_t r = threadIdx.x; r < regions; r += blockDim.x)
    if (s_cnt[r]) atomicAdd(&gcount[r], s_cnt[r]);
}

struct DeferOut {
  uint32_t *k, *v, *x;
  uint32_t* o;
  unsigned long long* count;
};

// Partition state of one forward round.  Count mode: region offsets (foff) from the
// count pass; cursors hold absolute positions.  Overallocated mode (the common big
// batch, no count pass): super-region b owns [b cs, (b + 1) cs) of the level-1 order and
// region r owns [r cr, (r + 1) cr) of the region order; cursors count from there.  A
// level-1 run that does not fit raises `flag` and the count-mode level 1 is redone
// (gated kernels, no host round trip); a level-2 run that does not fit is handed to
// the COPS kernels through list A with result positions past regions * cr.
struct Part {
  const uint64_t* foff;      // count mode: region offsets (regions + 1); nullptr when overallocated
  uint32_t* sbase;           // per super-region: first element of its level-1 area
  uint32_t* scnt;            // per super-region: elements
  uint32_t* tstart;          // per super-region: first level-2 tile; [supers] = level-2 tiles
  uint32_t* cur1;            // level-1 run cursors
  uint32_t* cur2;            // level-2 run cursors
  uint32_t* lim2;            // overallocated: smallest start of an overflowing run per region
  uint32_t cs, cr;           // overallocated capacities per super-region / region (0: count mode)
  int* flag;                 // level-1 overflow
  const int* gate;           // count-mode redo kernels run only when *gate != 0 (nullptr: always)
  unsigned long long* ovf2;  // level-2 overflow results: positions ovf2_base + ...
  uint32_t ovf2_base;
  DeferOut da;               // level-2 overflow keys -> list A (resume at window 0)
  uint32_t pfd;              // level 1, a CTA per tile: prefetch tile t + pfd into L2 (0: off)
};

// tstart from per-super-region element counts (one CTA of PT threads)
__device__ __forceinline__ void plan_tiles(const uint32_t* scnt, uint32_t supers, uint32_t* tstart) {
  __shared__ uint32_t wt[PT / 32];
  uint32_t carry = 0;
  for (uint32_t b0 = 0; b0 < supers; b0 += PT) {
    const uint32_t b = b0 + threadIdx.x;
    const uint32_t v = b < supers ? (scnt[b] + PTILE - 1) / PTILE : 0u;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) wt[warp] = x;
    __syncthreads();
    uint32_t before = carry, tot = 0;
    for (int w = 0; w < PT / 32; ++w) {
      if (w < warp) before += wt[w];
      tot += wt[w];
    }
    if (b < supers) tstart[b] = before + x - v;
    carry += tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) tstart[supers] = carry;
}

// Count mode: cursors (super-region starts; region starts when level 2 is count mode
// too) and the level-2 tile map: the L2 pass cuts every super-region into its own
// 4096-element tiles, so a tile never spans two super-regions (<= 256 buckets).
__global__ void __launch_bounds__(PT) k_st_plan(Part P, uint32_t regions, uint32_t supers, int init_cur2) {
  if (P.gate && *P.gate == 0) return;
  const uint64_t* foff = P.foff;
  if (init_cur2)
    for (uint32_t i = threadIdx.x; i < regions; i += PT) P.cur2[i] = (uint32_t)foff[i];
  for (uint32_t b = threadIdx.x; b < supers; b += PT) {
    const uint64_t s = foff[(uint64_t)b << ST_S2];
    const uint64_t e = foff[((uint64_t)(b + 1) << ST_S2) < regions ? ((uint64_t)(b + 1) << ST_S2) : regions];
    P.cur1[b] = (uint32_t)s;
    P.sbase[b] = (uint32_t)s;
    P.scnt[b] = (uint32_t)(e - s);
  }
  __syncthreads();
  plan_tiles(P.scnt, supers, P.tstart);
}

// Overallocated level 1 done without overflow: super-region geometry from its cursors
// (after an overflow the count-mode plan has set it already).
__global__ void __launch_bounds__(PT) k_st_plan_oa(Part P, uint32_t supers) {
  if (*P.flag) return;
  for (uint32_t b = threadIdx.x; b < supers; b += PT) {
    P.sbase[b] = b * P.cs;
    P.scnt[b] = P.cur1[b];
  }
  __syncthreads();
  plan_tiles(P.scnt, supers, P.tstart);
}

// Geometry of partition tile `t` of level L.  Level 1 tiles are the input cut in
// PTILE pieces; level 2 tiles are each super-region (input: level-1 order) cut in
// PTILE pieces.  Returns false for CTAs past the last tile.
constexpr uint32_t NO_SUPER = 0xffffffffu;

struct TileGeo {
  uint64_t pos0;   // first element (position in this level's input order)
  uint32_t cnt;    // elements
  uint32_t cbase;  // cursor index of bucket 0 (level 2: first region of the super-region)
};

template <int L>
__device__ __forceinline__ bool tile_geo(uint32_t t, uint64_t n, const Part& P, const uint32_t* sup,
                                         TileGeo& g) {
  if (L == 1) {
    g.pos0 = (uint64_t)t * PTILE;
    if (g.pos0 >= n) return false;
    g.cnt = (uint32_t)((n - g.pos0) < PTILE ? (n - g.pos0) : PTILE);
    g.cbase = 0;
    return true;
  }
  const uint32_t lo = sup[0];  // the tile's super-region and its first tile (tile_super)
  if (lo == NO_SUPER) return false;
  const uint32_t off = (t - sup[1]) * PTILE, cnt = sup[3];
  g.pos0 = (uint64_t)sup[2] + off;
  g.cnt = (cnt - off) < PTILE ? (cnt - off) : PTILE;
  g.cbase = lo << ST_S2;
  return true;
}

// Level 2: the super-region owning tile t (tstart[b] <= t < tstart[b + 1]), found by
// the CTA in one compare per thread (a per-thread binary search was 7% of the
// split's instructions); sup[0] = the super-region or NO_SUPER, sup[1] = its first tile.
__device__ __forceinline__ void tile_super(uint32_t t, const Part& P, uint32_t supers, uint32_t* sup) {
  // every load before the first branch: one L2 round trip (supers <= blockDim.x)
  const uint32_t* tstart = P.tstart;
  const uint32_t tot = tstart[supers];
  const uint32_t i = threadIdx.x;
  const bool own = i < supers;
  const uint32_t a = own ? tstart[i] : 0u, b = own ? tstart[i + 1] : 0u;
  const uint32_t sb = own ? P.sbase[i] : 0u, sc = own ? P.scnt[i] : 0u;
  if (t >= tot) {  // past the last tile (CTA-uniform)
    sup[0] = NO_SUPER;
    return;
  }
  if (a <= t && t < b) {
    sup[0] = i;
    sup[1] = a;
    sup[2] = sb;
    sup[3] = sc;
  }
  __syncthreads();
}

// PT-thread exclusive scan of v (one value per thread); returns the prefix.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* wt) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) wt[warp] = x;
  __syncthreads();
  // warp totals scanned with shuffles (a per-thread loop over the warps was 5% of
  // the split's instructions)
  uint32_t y = lane < PT / 32 ? wt[lane] : 0u;
#pragma unroll
  for (int d = 1; d < PT / 32; d <<= 1) {
    const uint32_t z = __shfl_up_sync(0xffffffffu, y, d);
    if (lane >= d) y += z;
  }
  const uint32_t before = warp ? __shfl_sync(0xffffffffu, y, warp - 1) : 0u;
  return before + x - v;
}

__device__ __forceinline__ void cp_async4(void* sdst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_addr(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Tile partition, level L (1: by super-region, 2: by region).  Besides the
// bucketed keys (+ values, + the window start inside the region at level 2) it
// records the inverse: inv[pos] = the element's slot in the tile's bucketed
// order, th/tg[t * nb + b] = length / destination of the tile's run of bucket b.
// NPAY u32 payload arrays ride along (0: lookup keys, 1: + values, 2: + the
// round-1 position of a round-2 key, or of a lookup key in round 2 with NPAY=1
// meaning the position).  Round 2 (wj = 1) partitions the deferred keys by their
// window-1 start; its count lives on the device (n_dev) and it needs no inverse.
#ifndef CH_AB_P0_MINB
#define CH_AB_P0_MINB 4  // level 1 of lookup keys: 4 CTAs/SM without spills (0.98 -> 0.95 ms)
#endif
#ifndef CH_AB_L2P_MINB
#define CH_AB_L2P_MINB 2  // level 2 with payloads: no spills at 2 CTAs/SM (1.83 -> 1.72 ms)
#endif
#ifndef CH_AB_SPLIT_MINB
#define CH_AB_SPLIT_MINB 3  // 3 CTAs per SM (<= 42 registers, small spills): 26.5 -> 27.1 G ops/s
#endif
template <int L, int NPAY>
__global__ void __launch_bounds__(PT, (L == 2 && NPAY >= 1) ? CH_AB_L2P_MINB : (L == 1 && NPAY == 0) ? CH_AB_P0_MINB : CH_AB_SPLIT_MINB) k_st_split(TableRef T, uint64_t n, Part P, uint32_t supers,
                                                    uint32_t ntiles,
                                                    const uint32_t* __restrict__ kin,
                                                    const uint32_t* __restrict__ vin,
                                                    const uint32_t* __restrict__ pin,
                                                    const uint32_t* __restrict__ rin, uint32_t* __restrict__ kout,
                                                    uint32_t* __restrict__ vout, uint32_t* __restrict__ pout,
                                                    uint32_t* __restrict__ rout,
                                                    uint16_t* __restrict__ lo_out, uint16_t* __restrict__ inv,
                                                    uint16_t* __restrict__ th, uint32_t* __restrict__ tg, uint32_t nb,
                                                    const unsigned long long* __restrict__ n_dev, int wj,
                                                    uint8_t* __restrict__ bid) {
  constexpr bool VALS = NPAY >= 1;
  constexpr bool POS = NPAY >= 2;
  constexpr bool RES = NPAY >= 3;
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* sK = reinterpret_cast<uint32_t*>(smem);
  uint32_t* sV = sK + PTILE;
  uint32_t* sP = sV + (VALS ? PTILE : 0);
  uint32_t* sR = sP + (POS ? PTILE : 0);
  uint16_t* sD = reinterpret_cast<uint16_t*>(sR + (RES ? PTILE : 0));
  uint16_t* sL = sD + PTILE;   // level 2 only: window start in bucketed order
  uint16_t* sLi = sL + PTILE;  // level 2 only: window start in input order
  if (P.gate && *P.gate == 0) return;
  if (n_dev) n = *n_dev;
  __shared__ uint32_t hist[PBINS], boff[PBINS], gbase[PBINS], dbase[PBINS];
  __shared__ uint8_t smode[PBINS];  // 0: run written, 1: dropped (level-1 overflow), 2: to list A
  __shared__ uint32_t wt[PT / 32];
  __shared__ uint32_t s_sup[4];
  const uint32_t cap = L == 1 ? P.cs : P.cr;
  uint32_t* const cursor = L == 1 ? P.cur1 : P.cur2;
  // persistent CTAs (a gated redo exits in one wave)
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    if (L == 1 && P.pfd && threadIdx.x == 0) {  // the tile a CTA starts one wave from now, into L2
      const uint64_t q0 = (uint64_t)(t + P.pfd) * PTILE;
      if (q0 < n) {
        const uint64_t cn = (n - q0) < PTILE ? (n - q0) : PTILE;
        l2_prefetch(kin + q0, cn * 4);
        if (VALS) l2_prefetch(vin + q0, cn * 4);
      }
    }
    if (L == 2) tile_super(t, P, supers, s_sup);
    TileGeo g;
    if (!tile_geo<L>(t, n, P, s_sup, g)) break;  // tiles past the end are past it for every later t
    if (L == 2 && P.pfd && threadIdx.x == 0) {  // the same super-region's tile one wave ahead
      const uint64_t q0 = g.pos0 + (uint64_t)P.pfd * PTILE, end = (uint64_t)s_sup[2] + s_sup[3];
      if (q0 < end) {
        const uint64_t cn = (end - q0) < PTILE ? (end - q0) : PTILE;
        l2_prefetch(kin + q0, cn * 4);
        if (VALS) l2_prefetch(vin + q0, cn * 4);
      }
    }
    hist[threadIdx.x] = 0;  // PBINS == PT
    // d: bucket | rank << 16 (one register per item); level 2 with payloads keeps
    // bucket | window start << 16 and the rank apart (measured faster than staging the
    // window start in shared memory there: 1.83 vs 1.97 ms)
    constexpr bool LOREG = L == 2 && VALS;
    uint32_t k[PI], v[PI], q[PI], w[PI], d[PI], r[LOREG ? PI : 1];
#pragma unroll
    for (int it = 0; it < PI; ++it) {  // all loads in flight before any use
      const uint32_t li = (uint32_t)it * PT + threadIdx.x;
      k[it] = li < g.cnt ? __ldcs(kin + g.pos0 + li) : 0u;
      if (VALS) v[it] = li < g.cnt ? __ldcs(vin + g.pos0 + li) : 0u;
      if (POS) q[it] = li < g.cnt ? __ldcs(pin + g.pos0 + li) : 0u;
      if (RES) w[it] = li < g.cnt ? __ldcs(rin + g.pos0 + li) : 0u;
    }
    __syncthreads();  // hist zeroed
#pragma unroll
    for (int it = 0; it < PI; ++it) {
      const uint32_t li = (uint32_t)it * PT + threadIdx.x;
      if (li >= g.cnt) continue;
      const uint32_t h = window_start(T, k[it], wj);
      const uint32_t b = L == 1 ? (h >> ST_LOG_R) >> ST_S2 : (h >> ST_LOG_R) - g.cbase;
      if (LOREG) {
        r[it] = atomicAdd(&hist[b], 1u);
        d[it] = b | (h & (ST_R - 1)) << 16;
      } else {
        d[it] = b | atomicAdd(&hist[b], 1u) << 16;
        if (L == 2) sLi[li] = (uint16_t)(h & (ST_R - 1));  // the window start waits in shared memory
      }
    }
    __syncthreads();
    const uint32_t hv = hist[threadIdx.x];
    const uint32_t bg = g.cbase + threadIdx.x;  // the bucket's cursor (super-region / region)
    // the run's global position: the atomic's round trip overlaps the bucketing below
    uint32_t old = hv ? atomicAdd(&cursor[bg], hv) : 0u;
    const uint32_t bo = block_excl_scan(hv, wt);
    boff[threadIdx.x] = bo;
    __syncthreads();
#pragma unroll
    for (int it = 0; it < PI; ++it) {
      const uint32_t li = (uint32_t)it * PT + threadIdx.x;
      if (li >= g.cnt) continue;
      const uint32_t b = d[it] & 0xFFFFu;
      const uint32_t j = boff[b] + (LOREG ? r[LOREG ? it : 0] : d[it] >> 16);
      sK[j] = k[it];
      if (VALS) sV[j] = v[it];
      if (POS) sP[j] = q[it];
      if (RES) sR[j] = w[it];
      sD[j] = (uint16_t)b;
      if (L == 2) sL[j] = LOREG ? (uint16_t)(d[it] >> 16) : sLi[li];
      if (inv) inv[g.pos0 + li] = (uint16_t)j;
    }
    uint8_t mode = 0;
    uint32_t gb = (cap ? bg * cap : 0u) + old;
    if (cap && hv && old + hv > cap) {  // the bucket's area is full (skewed batch)
      if (L == 1) {
        *P.flag = 1;  // the count-mode level 1 runs again
        mode = 1;
      } else {
        atomicMin(&P.lim2[bg], old);  // the region's keys end before this run
        gb = P.ovf2_base + (uint32_t)atomicAdd(P.ovf2, (unsigned long long)hv);
        dbase[threadIdx.x] = (uint32_t)atomicAdd(P.da.count, (unsigned long long)hv) - bo;
        mode = 2;
      }
    }
    smode[threadIdx.x] = mode;
    gbase[threadIdx.x] = gb - bo;  // run destination minus its tile offset (u32 wrap is fine)
    if (th && threadIdx.x < nb) {
      th[(uint64_t)t * nb + threadIdx.x] = (uint16_t)hv;
      tg[(uint64_t)t * nb + threadIdx.x] = gb;
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < g.cnt; j += PT) {
      const uint32_t b = sD[j];
      if (bid) bid[g.pos0 + j] = (uint8_t)b;  // the gather's bucket of bucketed slot j
      const uint32_t dst = gbase[b] + j;
      const uint8_t md = smode[b];
      if (md == 0) {
        kout[dst] = sK[j];
        if (VALS) vout[dst] = sV[j];
        if (POS) pout[dst] = sP[j];
        if (RES) rout[dst] = sR[j];
        if (L == 2) lo_out[dst] = sL[j];
      } else if (L == 2 && md == 2) {  // COPS kernels from window 0; result at dst
        const uint32_t a = dbase[b] + j;
        P.da.k[a] = sK[j];
        if (VALS) P.da.v[a] = sV[j];
        P.da.x[a] = dst;
        P.da.o[a] = 0;
      }
    }
    __syncthreads();  // shared buffers are reused by the next tile
  }
}

// Inverse of k_st_split<L>: bring the tile's results back from its runs and
// emit them in the tile's input order.  The tile's bucketed order is rebuilt in
// shared memory (bucket id per slot), every thread then gathers PI slots with
// all loads in flight (consecutive slots of a run are consecutive addresses;
// default caching: a sector is shared by the runs of neighbouring tiles).
// VAL: u32 value + u8 flag, otherwise u8 only (insert status).
#ifndef CH_AB_GATHER_MINB
#define CH_AB_GATHER_MINB 3  // 3 CTAs per SM (<= 42 registers): 57-58 registers ran 2 and measured slower
#endif
template <int L, bool VAL>
__global__ void __launch_bounds__(PT, CH_AB_GATHER_MINB) k_st_gather(uint64_t n, Part P, uint32_t supers, uint32_t ntiles,
                                                  const uint16_t* __restrict__ inv,
                                                  const uint16_t* __restrict__ th, const uint32_t* __restrict__ tg,
                                                  uint32_t nb, const uint32_t* __restrict__ src_v,
                                                  const uint8_t* __restrict__ src_f, uint32_t* __restrict__ dst_v,
                                                  uint8_t* __restrict__ dst_f,
                                                  const unsigned long long* __restrict__ exc,
                                                  const uint8_t* __restrict__ bid) {
  __shared__ uint32_t sV[VAL ? PTILE : 1];
  __shared__ uint8_t sF[PTILE];
  __shared__ uint16_t sB[VAL ? 1 : PTILE];  // statuses: bucket of each bucketed slot
  __shared__ uint32_t gsrc[PBINS];
  __shared__ uint32_t wt[PT / 32];
  const uint32_t t = blockIdx.x;
  __shared__ uint32_t s_sup[4];
  if (t >= ntiles) return;
  // every status INSERTED (insert without exceptions): nothing to move back
  const bool skip = !VAL && exc && *exc == 0;
  // the run table depends on t only: in flight while the geometry resolves
  const bool rt = !skip && threadIdx.x < nb;
  const uint32_t hv = rt ? th[(uint64_t)t * nb + threadIdx.x] : 0u;
  const uint32_t gs = rt ? tg[(uint64_t)t * nb + threadIdx.x] : 0u;
  if (L == 2) {
    if (skip) return;  // level 1 writes the statuses
    tile_super(t, P, supers, s_sup);
  }
  TileGeo g;
  if (t >= ntiles || !tile_geo<L>(t, n, P, s_sup, g)) return;
  if (skip) {
    if (L == 1) {  // 16-byte stores where the tile's status range is aligned
      uint8_t* d = dst_f + g.pos0;
      const uint32_t head = (uint32_t)((16u - ((uintptr_t)d & 15u)) & 15u) < g.cnt ? (uint32_t)((16u - ((uintptr_t)d & 15u)) & 15u) : g.cnt;
      for (uint32_t li = threadIdx.x; li < head; li += PT) d[li] = ST_INSERTED;
      const uint32_t nv = (g.cnt - head) / 16;
      const uint4 fill = make_uint4(0x01010101u * ST_INSERTED, 0x01010101u * ST_INSERTED, 0x01010101u * ST_INSERTED,
                                    0x01010101u * ST_INSERTED);
      for (uint32_t q = threadIdx.x; q < nv; q += PT) reinterpret_cast<uint4*>(d + head)[q] = fill;
      for (uint32_t li = head + nv * 16 + threadIdx.x; li < g.cnt; li += PT) d[li] = ST_INSERTED;
    }
    return;
  }
  // ib: inverse rank | bucket of bucketed slot it * PT + tid << 16.  Lookups (VAL) take the
  // buckets from the split (bid, 1 B per key: 1.03 -> 0.94 ms per level at 2^28); inserts,
  // whose gathers run only after exceptions, rebuild them from the run table (thread b
  // writes its run's slots).  Full, aligned lookup tiles (vec) write the caller's order four
  // keys per thread: 16-byte value and 4-byte flag stores, 8-byte inverse-rank loads.
  const bool vec = VAL && L == 1 && g.cnt == PTILE && ((g.pos0 & 3) == 0) && (((uintptr_t)(dst_v + g.pos0) & 15) == 0) &&
                   (((uintptr_t)(dst_f + g.pos0) & 3) == 0);
  uint32_t ib[PI];
  uint2 iv4[PI / 4];
  if (vec) {
#pragma unroll
    for (int h = 0; h < PI / 4; ++h)
      iv4[h] = __ldcs(reinterpret_cast<const uint2*>(inv + g.pos0) + h * PT + threadIdx.x);
#pragma unroll
    for (int it = 0; it < PI; ++it) ib[it] = (uint32_t)__ldcs(bid + g.pos0 + (uint32_t)it * PT + threadIdx.x) << 16;
  } else {
#pragma unroll
    for (int it = 0; it < PI; ++it) {  // inverse ranks (and bucket ids) load alongside the run table
      const uint32_t li = (uint32_t)it * PT + threadIdx.x;
      ib[it] = li < g.cnt ? (uint32_t)__ldcs(inv + g.pos0 + li) |
                                (VAL ? (uint32_t)__ldcs(bid + g.pos0 + li) << 16 : 0u)
                          : 0u;
    }
  }
  const uint32_t bo = block_excl_scan(hv, wt);
  gsrc[threadIdx.x] = gs - bo;  // run source minus its tile offset
  if (!VAL) {
    __syncthreads();
    for (uint32_t x = 0; x < hv; ++x) sB[bo + x] = (uint16_t)threadIdx.x;
    __syncthreads();
#pragma unroll
    for (int it = 0; it < PI; ++it) ib[it] |= (uint32_t)sB[(uint32_t)it * PT + threadIdx.x] << 16;
  }
  __syncthreads();
  uint32_t v[PI];
  uint8_t fl[PI];
#pragma unroll
  for (int it = 0; it < PI; ++it) {
    const uint32_t j = (uint32_t)it * PT + threadIdx.x;
    if (j < g.cnt) {
      const uint32_t src = gsrc[ib[it] >> 16] + j;
      if (VAL) v[it] = src_v[src];
      fl[it] = src_f[src];
    }
  }
#pragma unroll
  for (int it = 0; it < PI; ++it) {
    const uint32_t j = (uint32_t)it * PT + threadIdx.x;
    if (j < g.cnt) {
      if (VAL) sV[j] = v[it];
      sF[j] = fl[it];
    }
  }
  __syncthreads();
  if (vec) {
#pragma unroll
    for (int h = 0; h < PI / 4; ++h) {
      const uint32_t li = 4u * ((uint32_t)h * PT + threadIdx.x);
      const uint32_t j0 = iv4[h].x & 0xFFFFu, j1 = iv4[h].x >> 16, j2 = iv4[h].y & 0xFFFFu, j3 = iv4[h].y >> 16;
      *reinterpret_cast<uint4*>(dst_v + g.pos0 + li) = make_uint4(sV[j0], sV[j1], sV[j2], sV[j3]);
      *reinterpret_cast<uint32_t*>(dst_f + g.pos0 + li) =
          (uint32_t)sF[j0] | (uint32_t)sF[j1] << 8 | (uint32_t)sF[j2] << 16 | (uint32_t)sF[j3] << 24;
    }
    return;
  }
#pragma unroll
  for (int it = 0; it < PI; ++it) {
    const uint32_t li = (uint32_t)it * PT + threadIdx.x;
    if (li < g.cnt) {
      const uint32_t j = ib[it] & 0xFFFFu;
      if (VAL) dst_v[g.pos0 + li] = sV[j];
      dst_f[g.pos0 + li] = sF[j];
    }
  }
}

// The status gathers (inserts): the same inverse as k_st_gather, run as a few persistent
// CTAs over the tiles; without exceptions (the common case) level 1 fills the caller's
// statuses with INSERTED grid-stride and nothing else runs -- no 65 K-CTA launch.
template <int L, bool VAL>
__global__ void __launch_bounds__(PT, CH_AB_GATHER_MINB) k_st_gather_st(uint64_t n, Part P, uint32_t supers, uint32_t ntiles,
                                                  const uint16_t* __restrict__ inv,
                                                  const uint16_t* __restrict__ th, const uint32_t* __restrict__ tg,
                                                  uint32_t nb, const uint32_t* __restrict__ src_v,
                                                  const uint8_t* __restrict__ src_f, uint32_t* __restrict__ dst_v,
                                                  uint8_t* __restrict__ dst_f,
                                                  const unsigned long long* __restrict__ exc,
                                                  const uint8_t* __restrict__ bid) {
  __shared__ uint32_t sV[VAL ? PTILE : 1];
  __shared__ uint8_t sF[PTILE];
  __shared__ uint16_t sB[VAL ? 1 : PTILE];  // statuses: bucket of each bucketed slot
  __shared__ uint32_t gsrc[PBINS];
  __shared__ uint32_t wt[PT / 32];
  __shared__ uint32_t s_sup[4];
  // every status INSERTED (insert without exceptions): nothing to move back; level 1 fills
  // the caller's statuses grid-stride with 16-byte stores (the status gathers run as a few
  // persistent CTAs, so the common case costs no 65 K-CTA launch)
  if (!VAL && exc && *exc == 0) {
    if (L == 1) {
      const uint32_t head = (uint32_t)((16u - ((uintptr_t)dst_f & 15u)) & 15u) < n ? (uint32_t)((16u - ((uintptr_t)dst_f & 15u)) & 15u) : (uint32_t)n;
      const uint64_t gtid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, gstr = (uint64_t)gridDim.x * blockDim.x;
      if (gtid < head) dst_f[gtid] = ST_INSERTED;
      const uint64_t nv = (n - head) / 16;
      const uint4 fill = make_uint4(0x01010101u * ST_INSERTED, 0x01010101u * ST_INSERTED, 0x01010101u * ST_INSERTED,
                                    0x01010101u * ST_INSERTED);
      for (uint64_t q = gtid; q < nv; q += gstr) reinterpret_cast<uint4*>(dst_f + head)[q] = fill;
      for (uint64_t li = head + nv * 16 + gtid; li < n; li += gstr) dst_f[li] = ST_INSERTED;
    }
    return;
  }
  auto one_tile = [&](const uint32_t t) {
  // the run table depends on t only: in flight while the geometry resolves
  const bool rt = threadIdx.x < nb;
  const uint32_t hv = rt ? th[(uint64_t)t * nb + threadIdx.x] : 0u;
  const uint32_t gs = rt ? tg[(uint64_t)t * nb + threadIdx.x] : 0u;
  if (L == 2) tile_super(t, P, supers, s_sup);
  TileGeo g;
  if (t >= ntiles || !tile_geo<L>(t, n, P, s_sup, g)) return;
  // ib: inverse rank | bucket of bucketed slot it * PT + tid << 16.  Lookups (VAL) take the
  // buckets from the split (bid, 1 B per key: 1.03 -> 0.94 ms per level at 2^28); inserts,
  // whose gathers run only after exceptions, rebuild them from the run table (thread b
  // writes its run's slots).  Full, aligned lookup tiles (vec) write the caller's order four
  // keys per thread: 16-byte value and 4-byte flag stores, 8-byte inverse-rank loads.
  const bool vec = VAL && L == 1 && g.cnt == PTILE && ((g.pos0 & 3) == 0) && (((uintptr_t)(dst_v + g.pos0) & 15) == 0) &&
                   (((uintptr_t)(dst_f + g.pos0) & 3) == 0);
  uint32_t ib[PI];
  uint2 iv4[PI / 4];
  if (vec) {
#pragma unroll
    for (int h = 0; h < PI / 4; ++h)
      iv4[h] = __ldcs(reinterpret_cast<const uint2*>(inv + g.pos0) + h * PT + threadIdx.x);
#pragma unroll
    for (int it = 0; it < PI; ++it) ib[it] = (uint32_t)__ldcs(bid + g.pos0 + (uint32_t)it * PT + threadIdx.x) << 16;
  } else {
#pragma unroll
    for (int it = 0; it < PI; ++it) {  // inverse ranks (and bucket ids) load alongside the run table
      const uint32_t li = (uint32_t)it * PT + threadIdx.x;
      ib[it] = li < g.cnt ? (uint32_t)__ldcs(inv + g.pos0 + li) |
                                (VAL ? (uint32_t)__ldcs(bid + g.pos0 + li) << 16 : 0u)
                          : 0u;
    }
  }
  const uint32_t bo = block_excl_scan(hv, wt);
  gsrc[threadIdx.x] = gs - bo;  // run source minus its tile offset
  if (!VAL) {
    __syncthreads();
    for (uint32_t x = 0; x < hv; ++x) sB[bo + x] = (uint16_t)threadIdx.x;
    __syncthreads();
#pragma unroll
    for (int it = 0; it < PI; ++it) ib[it] |= (uint32_t)sB[(uint32_t)it * PT + threadIdx.x] << 16;
  }
  __syncthreads();
  uint32_t v[PI];
  uint8_t fl[PI];
#pragma unroll
  for (int it = 0; it < PI; ++it) {
    const uint32_t j = (uint32_t)it * PT + threadIdx.x;
    if (j < g.cnt) {
      const uint32_t src = gsrc[ib[it] >> 16] + j;
      if (VAL) v[it] = src_v[src];
      fl[it] = src_f[src];
    }
  }
#pragma unroll
  for (int it = 0; it < PI; ++it) {
    const uint32_t j = (uint32_t)it * PT + threadIdx.x;
    if (j < g.cnt) {
      if (VAL) sV[j] = v[it];
      sF[j] = fl[it];
    }
  }
  __syncthreads();
  if (vec) {
#pragma unroll
    for (int h = 0; h < PI / 4; ++h) {
      const uint32_t li = 4u * ((uint32_t)h * PT + threadIdx.x);
      const uint32_t j0 = iv4[h].x & 0xFFFFu, j1 = iv4[h].x >> 16, j2 = iv4[h].y & 0xFFFFu, j3 = iv4[h].y >> 16;
      *reinterpret_cast<uint4*>(dst_v + g.pos0 + li) = make_uint4(sV[j0], sV[j1], sV[j2], sV[j3]);
      *reinterpret_cast<uint32_t*>(dst_f + g.pos0 + li) =
          (uint32_t)sF[j0] | (uint32_t)sF[j1] << 8 | (uint32_t)sF[j2] << 16 | (uint32_t)sF[j3] << 24;
    }
    return;
  }
#pragma unroll
  for (int it = 0; it < PI; ++it) {
    const uint32_t li = (uint32_t)it * PT + threadIdx.x;
    if (li < g.cnt) {
      const uint32_t j = ib[it] & 0xFFFFu;
      if (VAL) dst_v[g.pos0 + li] = sV[j];
      dst_f[g.pos0 + li] = sF[j];
    }
  }
  };
  // lookups: one CTA per tile; statuses: persistent CTAs over the tiles
  for (uint32_t t = blockIdx.x; t < ntiles; t += VAL ? ntiles : gridDim.x) {
    one_tile(t);
    if (!VAL) __syncthreads();  // shared buffers are reused by the next tile
  }
}

// ------------------------------------------------------------- region pass
// Keys that window 0 cannot decide are buffered in shared memory and appended to
// the device-counted list in batches (one global atomic per flush: a per-warp
// atomic on one counter serialised the whole pass).
constexpr uint32_t DBUF = 256;    // deferred entries buffered per CTA
#ifndef CH_AB_STEP
#define CH_AB_STEP 8
#endif
constexpr uint32_t STEP = CH_AB_STEP;  // slots one key examines per step
constexpr uint32_t TILE_PAD = 8;  // a step may read up to STEP-1 slots past its window

template <bool VALS, uint32_t CAP>
struct DeferBuf {
  uint32_t k[CAP];
  uint32_t v[VALS ? CAP : 1];
  uint32_t x[CAP];
  uint8_t o[CAP];
  uint32_t n;
  unsigned long long gb;
};


template <bool VALS, uint32_t CAP>
__device__ __forceinline__ void defer_push(DeferBuf<VALS, CAP>& B, const DeferOut& D, uint32_t k, uint32_t v,
                                           uint32_t x, uint32_t o) {
  const uint32_t s = atom_add_shared(&B.n, 1u);
  if (s < CAP) {
    B.k[s] = k;
    if (VALS) B.v[s] = v;
    B.x[s] = x;
    B.o[s] = (uint8_t)o;
  } else {  // buffer full (pathological batches): straight to the list
    const unsigned long long g = atomicAdd(D.count, 1ull);
    D.k[g] = k;
    if (VALS) D.v[g] = v;
    D.x[g] = x;
    D.o[g] = o;
  }
}

// CTA-uniform: flush when half full (or when forced and non-empty)
template <bool VALS, uint32_t CAP>
__device__ __forceinline__ void defer_flush(DeferBuf<VALS, CAP>& B, const DeferOut& D, bool force) {
  __syncthreads();
  const uint32_t dn = B.n < CAP ? B.n : CAP;
  __syncthreads();  // everyone has read B.n
  if (!(dn >= CAP / 2 || (force && dn))) return;
  if (threadIdx.x == 0) {
    B.gb = atomicAdd(D.count, (unsigned long long)dn);
    B.n = 0;
  }
  __syncthreads();
  const unsigned long long gb = B.gb;
  for (uint32_t i = threadIdx.x; i < dn; i += blockDim.x) {
    D.k[gb + i] = B.k[i];
    if (VALS) D.v[gb + i] = B.v[i];
    D.x[gb + i] = B.x[i];
    D.o[gb + i] = B.o[i];
  }
  __syncthreads();
}

// both deferral buffers of a region at once (one pair of barriers instead of two)
template <bool VALS, uint32_t CAP>
__device__ __forceinline__ void defer_flush2(DeferBuf<VALS, CAP>& B1, const DeferOut& D1, DeferBuf<VALS, CAP>& B2,
                                             const DeferOut& D2) {
  __syncthreads();
  const uint32_t n1 = B1.n < CAP ? B1.n : CAP, n2 = B2.n < CAP ? B2.n : CAP;
  __syncthreads();  // everyone has read the counts
  if (!(n1 | n2)) return;
  if (threadIdx.x == 0) {
    if (n1) B1.gb = atomicAdd(D1.count, (unsigned long long)n1);
    if (n2) B2.gb = atomicAdd(D2.count, (unsigned long long)n2);
    B1.n = 0;
    B2.n = 0;
  }
  __syncthreads();
  const unsigned long long g1 = B1.gb, g2 = B2.gb;
  for (uint32_t i = threadIdx.x; i < n1 + n2; i += blockDim.x) {
    const bool a = i < n1;
    DeferBuf<VALS, CAP>& Bx = a ? B1 : B2;
    const DeferOut& Dx = a ? D1 : D2;
    const uint32_t j = a ? i : i - n1;
    const unsigned long long gd = (a ? g1 : g2) + j;
    Dx.k[gd] = Bx.k[j];
    if (VALS) Dx.v[gd] = Bx.v[j];
    Dx.x[gd] = Bx.x[j];
    Dx.o[gd] = Bx.o[j];
  }
}

__device__ __forceinline__ uint32_t lds32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_addr(p)) : "memory");
  return v;
}

// Region pass.  Results are written at the key's region-ordered position (the
// gather passes return them to the caller's order): MODE 0 insert the status,
// MODE 1 lookup the value and found flag.
//
// Every lane of a warp holds one open key and advances it STEP slots of window 0
// per iteration (the same work for every lane); a lane whose key resolved takes
// the next one from the warp's key chunks (32 keys loaded coalesced into
// registers, the following chunk already in flight, handed out with shuffles;
// chunks come from a per-region counter, so warps balance themselves).  No
// barrier between the tile load and the write-back: a staged-segment version
// with rounds and a shared-memory queue spent 26% of its stalls at segment
// barriers and 10% of its instructions on the queue (profiles/r01_ncu_staged_probe).
// R2 (round 2): the keys are round 1's deferred ones, probed in window 1, and each
// carries the position its result belongs to (pos).  Deferrals go to DA when the
// COPS kernel must re-examine the window (start crossing the region end, a
// tombstone before the first empty) and to DB when the window is full (round 1:
// those are round 2's input; round 2: DB == DA, the COPS kernel's list).
constexpr uint32_t DBUF_B = 1024;  // window-full deferrals buffered per region (~4.6% of ~7.8K keys)
constexpr uint32_t NONE = 0xffffffffu;

// Lookups scan a byte per slot: 0 for the empty sentinel, 1..255 from the key word
// otherwise, so a step reads 8 slots' fingerprints with three 4-byte loads instead of
// eight key words (the random shared-memory gathers were the region pass's limit).
#ifndef CH_AB_FSTEP
#define CH_AB_FSTEP 16
#endif
constexpr uint32_t FSTEP = CH_AB_FSTEP;  // slots per lookup step (multiple of 8)
constexpr uint32_t FP_BYTES = ((ST_R + ST_HALO + TILE_PAD + FSTEP + 16) + 15) & ~15u;
__device__ __forceinline__ uint32_t slot_fp(uint32_t key, uint32_t e) {
  if (key == e) return 0u;
  const uint32_t f = (key * 0x9E3779B1u) >> 24;
  return f ? f : 1u;
}
__device__ __forceinline__ uint32_t zero_bytes(uint32_t v) { return (v - 0x01010101u) & ~v & 0x80808080u; }

template <int MODE, bool R2>
__global__ void __launch_bounds__(RT, 2) k_st_probe(TableRef T, Part P,
                                                    const uint32_t* __restrict__ keys,
                                                    const uint32_t* __restrict__ vals,
                                                    const uint32_t* __restrict__ pos,
                                                    const uint16_t* __restrict__ los, uint8_t* __restrict__ status,
                                                    uint32_t* __restrict__ res_val, uint8_t* __restrict__ res_flag,
                                                    DeferOut DA, DeferOut DB, int g,
                                                    unsigned long long* __restrict__ exc) {
  constexpr bool INS = MODE == 0;
  constexpr uint32_t HALO = INS ? 0u : ST_HALO;
  constexpr uint32_t OW = R2 ? WINDOW : 0u;  // sequence offset of the window probed here
  extern __shared__ __align__(128) unsigned char dsm[];
  uint64_t* tile = reinterpret_cast<uint64_t*>(dsm);
  uint32_t* fp32 = reinterpret_cast<uint32_t*>(tile + ST_R + HALO + TILE_PAD);  // lookups: fingerprints
  __shared__ DeferBuf<INS, DBUF_B> B;  // -> DB
  __shared__ DeferBuf<INS, DBUF> BA;   // -> DA
  __shared__ uint32_t s_next;
  __shared__ __align__(8) uint64_t bar;
  __shared__ int dirty;
  const uint32_t f = blockIdx.x;
  uint64_t k0;
  uint32_t m;
  if (P.foff) {  // count mode
    k0 = P.foff[f];
    m = (uint32_t)(P.foff[f + 1] - k0);
  } else {  // overallocated: the region's area, up to its first overflowing run
    k0 = (uint64_t)f * P.cr;
    const uint32_t c2 = P.cur2[f], l2 = P.lim2[f];
    m = c2 < l2 ? c2 : l2;
  }
  if (m == 0) return;  // no key starts in this region
  const uint64_t rbase = (uint64_t)f << ST_LOG_R;
  const uint32_t len = (uint32_t)((T.c - rbase) < ST_R ? (T.c - rbase) : ST_R);
  uint64_t* slots = static_cast<uint64_t*>(T.slots);
  if (threadIdx.x == 0) {
    dirty = 0;
    B.n = 0;
    BA.n = 0;
    s_next = 0;
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, (len + HALO) * 8u);
    bulk_load(tile, slots + rbase, len * 8u, &bar);
    if (HALO) {  // window 0 of the region's last keys runs into the next region (or wraps)
      const uint64_t hb = rbase + len < T.c ? rbase + len : 0;
      bulk_load(tile + len, slots + hb, HALO * 8u, &bar);
    }
  }
  __syncthreads();  // the mbarrier is initialised before anyone waits on it
  const uint32_t e = (uint32_t)T.e, t = (uint32_t)T.t;
  const uint32_t ug = (uint32_t)g;
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t ops = 0, att = 0, win = 0, occ = 0, ndef = 0, nexc = 0;  // per thread: < 2^32 even for 2^32 keys
  bool claimed_any = false;
  const bool adj = t + 1u == e;  // default sentinels: "free" is one subtract and compare, (c - t) <= 1

  // one probe step of key k from in-window offset o (updated); true while the key
  // stays open (nothing decisive in these slots, or a lost claim)
  // packed slot s: key word tw[2 s], value word tw[2 s + 1] (little-endian u64)
  uint32_t* const tw = reinterpret_cast<uint32_t*>(tile);
  auto step = [&](uint32_t k, uint32_t v, uint32_t lo, uint32_t ri, uint32_t& o) -> bool {
    if constexpr (!INS) {  // fingerprints of FSTEP slots: decisive = the key's fingerprint or empty
      const uint32_t x = lo + o, a = x >> 2, sh = (x & 3u) * 8u;
      const uint32_t rep = v;  // lookups carry the key's fingerprint in every byte of v
      uint32_t wv[FSTEP / 4 + 1];
#pragma unroll
      for (int q = 0; q <= (int)FSTEP / 4; ++q) wv[q] = fp32[a + q];
      // lowest flagged byte of each zero_bytes() is exact (false flags only sit above a true one)
      uint64_t mk[FSTEP / 8];
#pragma unroll
      for (int q = 0; q < (int)FSTEP / 8; ++q) {
        const uint32_t b0 = __funnelshift_r(wv[2 * q], wv[2 * q + 1], sh);
        const uint32_t b1 = __funnelshift_r(wv[2 * q + 1], wv[2 * q + 2], sh);
        mk[q] = (uint64_t)(zero_bytes(b0 ^ rep) | zero_bytes(b0)) |
                (uint64_t)(zero_bytes(b1 ^ rep) | zero_bytes(b1)) << 32;
      }
      const uint32_t room = WINDOW - o;
      uint32_t u = FSTEP;
#pragma unroll
      for (int q = (int)FSTEP / 8 - 1; q >= 0; --q)
        if (mk[q]) u = 8u * q + ((uint32_t)(__ffsll((long long)mk[q]) - 1) >> 3);
      if (u >= room) {  // nothing decisive inside the window's remaining slots
        o += FSTEP;
        if (o < WINDOW) return true;
        defer_push(B, DB, k, v, ri, OW + WINDOW);  // window 0 has neither the key nor an empty
        ndef += 1;
        return false;
      }
      o += u;
      const uint32_t s2 = 2 * (lo + o);
      const uint32_t c = tw[s2];
      if (c != k && c != e) {  // fingerprint collision: scan on after it
        o += 1;
        if (o < WINDOW) return true;
        defer_push(B, DB, k, v, ri, OW + WINDOW);
        ndef += 1;
        return false;
      }
      const bool hit = c == k;
      res_val[ri] = hit ? tw[s2 + 1] : 0u;
      res_flag[ri] = (uint8_t)hit;
      ops += 1;
      att += OW + chunk_end(o, ug);
      win += R2 ? 2 : 1;
      return false;
    } else {
    // key words only: a 4-byte gather per slot (the shared pipe is the kernel's limit)
    uint32_t w[STEP];
#pragma unroll
    for (int q = 0; q < (int)STEP; ++q) w[q] = INS ? lds32(tw + 2 * (lo + o + q)) : tw[2 * (lo + o + q)];
    // first decisive slot and its key word, scanning backwards with selects
    const uint32_t room = WINDOW - o;  // slots left in the window
    uint32_t u = STEP, c = 0;
#pragma unroll
    for (int q = (int)STEP - 1; q >= 0; --q) {
      const uint32_t x = w[q];
      bool d;
      if (INS) d = (x == k) | (adj ? (x - t) <= 1u : ((x == e) | (x == t)));
      else d = (x == k) | (x == e);  // lookups pass tombstones
      d = d && (uint32_t)q < room;
      u = d ? (uint32_t)q : u;
      c = d ? x : c;
    }
    if (u == STEP) {
      o += STEP;
      if (o < WINDOW) return true;
      // the window holds neither the key nor a free cell: resume at the next one
      defer_push(B, DB, k, v, ri, OW + WINDOW);
      ndef += 1;
      return false;
    }
    o += u;
    const uint32_t s2 = 2 * (lo + o);
    if (INS) {
      if (c == k) {  // present before the first free cell (single_table.py:198-200)
        status[ri] = ST_DUPLICATE;
        nexc += 1;
      } else if (c == t) {  // tombstone first: the deferred-claim rule (:201-223), COPS kernel
        defer_push(BA, DA, k, v, ri, OW);
        ndef += 1;
        return false;
      } else {
        // claim the key word (32-bit CAS); the value word follows with a plain store:
        // nothing in this pass reads values, and the write-back runs after a barrier
        if (atomicCAS(tw + s2, e, k) != e) {  // another key took it: re-read from this slot (:232-233)
          att += ug;
          return true;
        }
        tw[s2 + 1] = v;
        occ += 1;
        claimed_any = true;  // status: INSERTED is pre-set (staged_insert)
      }
    } else {
      const bool hit = c == k;
      res_val[ri] = hit ? tw[s2 + 1] : 0u;
      res_flag[ri] = (uint8_t)hit;
    }
    ops += 1;
    att += OW + chunk_end(o, ug);
    win += R2 ? 2 : 1;
    return false;
    }
  };

  // key chunks: 32 consecutive keys of the region's list, one per lane
  // chunk pairs from a per-region counter (one atomic per 64 keys, issued as PTX by
  // lane 0: the compiler's warp aggregation of atomicAdd cost ~17 instructions per
  // chunk); a statically interleaved assignment measured slower for inserts (the
  // warps' CAS work is uneven)
  uint32_t pair_b = 0;
  auto grab = [&]() -> uint32_t {
    uint32_t b;
    if (pair_b & 32u) {
      b = pair_b;
      pair_b = 0;
    } else {
      uint32_t a = 0;
      if (lane == 0)
        asm volatile("atom.shared.add.u32 %0, [%1], 64;" : "=r"(a) : "r"(smem_addr(&s_next)) : "memory");
      b = __shfl_sync(0xffffffffu, a, 0);
      pair_b = b + 32u;
    }
    return b < m ? b : NONE;
  };
  uint32_t ck = e, cv = 0, cp = 0, cl = 0, nk = e, nv = 0, np = 0, nl = 0;
  auto fetch = [&](uint32_t b, uint32_t& kk, uint32_t& vv, uint32_t& pp, uint32_t& ll) {
    const uint32_t i = b + lane;
    if (b != NONE && i < m) {
      kk = __ldcs(keys + k0 + i);
      ll = __ldcs(los + k0 + i);
      if (INS) vv = __ldcs(vals + k0 + i);
      if (R2) pp = __ldcs(pos + k0 + i);
    }
  };
  uint32_t cbase = grab();
  fetch(cbase, ck, cv, cp, cl);
  uint32_t nbase = cbase == NONE ? NONE : grab();
  fetch(nbase, nk, nv, np, nl);
  uint32_t ptr = 0;  // entries of the current chunk handed out
  mbar_wait(&bar, 0);
  if (!INS) {  // fingerprints of the staged slots (4 per word; slots past the halo are never decisive)
    const uint32_t words = (len + HALO + TILE_PAD + 3) >> 2;
    for (uint32_t i = threadIdx.x; i < words; i += RT) {
      uint32_t f = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) f |= slot_fp(tw[2 * (4 * i + u)], e) << (8 * u);
      fp32[i] = f;
    }
    for (uint32_t i = words + threadIdx.x; i < FP_BYTES / 4; i += RT) fp32[i] = 0xFFFFFFFFu;
    __syncthreads();
  }

  bool act = false;
  const uint32_t k0u = (uint32_t)k0;  // positions stay below 2^32 (staged_supported)
  uint32_t k = 0, v = 0, lo = 0, ri = 0, o = 0;
  for (;;) {
    const unsigned need = __ballot_sync(0xffffffffu, !act);
    if (need && cbase != NONE) {
      const uint32_t take = ptr + __popc(need & ((1u << lane) - 1u));  // < 64
      const uint32_t src = take & 31u;
      const bool fromc = take < 32u;
      // (the source lane cannot choose the chunk: it does not know the taker's take)
      auto pick = [&](uint32_t cur, uint32_t nxt) {
        const uint32_t a = __shfl_sync(0xffffffffu, cur, src), b = __shfl_sync(0xffffffffu, nxt, src);
        return fromc ? a : b;
      };
      const uint32_t xk = pick(ck, nk), xl = pick(cl, nl);
      const uint32_t xv = INS ? pick(cv, nv) : 0u, xp = R2 ? pick(cp, np) : 0u;
      const uint32_t tb = fromc ? cbase : nbase;
      const bool got = !act && tb != NONE && tb + src < m;
      ptr += __popc(need);
      if (ptr >= 32u) {  // current chunk used up: the next one moves in, another is fetched
        ptr -= 32u;
        cbase = nbase;
        ck = nk, cv = nv, cp = np, cl = nl;
        nbase = cbase == NONE ? NONE : grab();
        fetch(nbase, nk, nv, np, nl);
      }
      if (got) {
        k = xk, lo = xl, o = 0;
        v = INS ? xv : slot_fp(xk, e) * 0x01010101u;
        ri = R2 ? xp : k0u + tb + src;
        if (k == e || k == t) {  // sentinels are never stored (single_table.py:369-370, 391-393)
          if (INS) {
            status[ri] = ST_INVALID;
            nexc += 1;
          } else {
            res_val[ri] = 0;
            res_flag[ri] = 0;
            ops += 1;  // retrieve_bulk counts every query (:403)
          }
        } else if (INS && lo + WINDOW > len) {  // the window leaves the staged region
          defer_push(BA, DA, k, v, ri, OW);
          ndef += 1;
        } else {
          act = true;
        }
      }
    }
    if (act) act = step(k, v, lo, ri, o);
    if (cbase == NONE && !__any_sync(0xffffffffu, act)) break;
  }
  defer_flush(B, DB, true);  // syncs
  defer_flush(BA, DA, true);
  if (INS) {
    if (claimed_any) dirty = 1;
    fence_smem_to_async();
    __syncthreads();
    if (threadIdx.x == 0 && dirty) bulk_store_wait(slots + rbase, tile, len * 8u);
  }
  const long long cv6[6] = {(long long)ops, (long long)att, (long long)win, (long long)occ, (long long)nexc,
                            (long long)ndef};
  long long* const dst[6] = {(long long*)&T.ctr->ops, (long long*)&T.ctr->attempts, (long long*)&T.ctr->windows,
                             &T.ctr->occupied, INS ? (long long*)exc : nullptr, (long long*)&T.ctr->deferred};
  cta_add<6>(cv6, dst);
}

// Region pass for lookups, uniform rounds.  Every key of the region takes exactly one
// 16-slot fingerprint step from window 0's start (thread i: the region's keys i, i + RT,
// ...; coalesced key / lo loads one round ahead, coalesced result stores); a key the step
// does not decide is pushed (warp-aggregated) to a shared queue with its offset, and the
// queue is drained after the rounds with as many steps as each entry needs (a full window
// ends at offset 32, so at most two more).  Same rule, results and counters as
// k_st_probe<1, false>, without its per-step refill (ballot / shuffles / chunk cursors).
//
// Fingerprints here are 7 bits (fp7: 0..127) and an empty slot is 0x80, so one step flags
// "the key's fingerprint or empty" with four integer ops per 4 slots (zero-byte test of
// b ^ rep, OR the high bits of b), and the 16 per-slot flags are packed into one 16-bit
// mask with two multiplies per 8 slots (flag_mask8), whose lowest set bit is the first
// decisive slot.
constexpr uint32_t LQ_CAP = 2048;  // queued keys per region (~8% of ~7.8 K at load 0.95)
constexpr uint32_t FP_EMPTY = 0x80u;
#ifndef CH_LQ_THREADS
#define CH_LQ_THREADS 768
#endif
constexpr uint32_t LQT = CH_LQ_THREADS;  // lookup region CTA threads (2 CTAs per SM)

__device__ __forceinline__ uint32_t fp7(uint32_t key) { return (key * 0x9E3779B1u) >> 25; }
// bit 7 of each byte: the byte equals the key's fingerprint (rep = fp7 * 0x01010101) or is
// empty; the lowest flag is exact (the zero-byte borrow only creates flags above a true one)
__device__ __forceinline__ uint32_t fp_flags(uint32_t b, uint32_t rep) {
  const uint32_t x = b ^ rep;
  return ((x - 0x01010101u) & ~x & 0x80808080u) | (b & 0x80808080u);
}
// flags of slots 0..3 (f0) and 4..7 (f1) -> slot i at bit 24 + i.  Each product places
// byte j's flag at 24 + j (f0 >> 4) or 28 + j (f1); every other partial-product bit lands
// below bit 24 and no two partial products share a bit, so the sum carries nothing.
__device__ __forceinline__ uint32_t flag_mask8(uint32_t f0, uint32_t f1) {
  return (f0 >> 4) * 0x00204081u + f1 * 0x00204081u;
}

// ERASE: the same pass retires the keys it finds (single_table.py:338-351): a shared-memory CAS
// of the key's word to the tombstone, the erased flag in res_flag, and the region written back
// when anything was retired.  Keys whose window crosses the region end go to the COPS erase
// (after every region is written back: the halo belongs to the next region's CTA).
template <bool ERASE>
__global__ void __launch_bounds__(LQT, 2) k_st_lookup_q(TableRef T, Part P, const uint32_t* __restrict__ keys,
                                                       const uint16_t* __restrict__ los,
                                                       uint32_t* __restrict__ res_val, uint8_t* __restrict__ res_flag,
                                                       DeferOut DB, int g) {
  constexpr uint32_t HALO = ST_HALO;
  extern __shared__ __align__(128) unsigned char dsm[];
  uint64_t* tile = reinterpret_cast<uint64_t*>(dsm);
  uint32_t* fp32 = reinterpret_cast<uint32_t*>(tile + ST_R + HALO + TILE_PAD);
  uint32_t* qk = fp32 + FP_BYTES / 4;  // queue: key, region index, lo | offset << 16
  uint32_t* qi = qk + LQ_CAP;
  uint32_t* qlo = qi + LQ_CAP;
  __shared__ DeferBuf<false, DBUF_B> B;
  __shared__ uint32_t s_qn;
  __shared__ int s_dirty;
  __shared__ __align__(8) uint64_t bar;
  const uint32_t f = blockIdx.x;
  uint64_t k0;
  uint32_t m;
  if (P.foff) {
    k0 = P.foff[f];
    m = (uint32_t)(P.foff[f + 1] - k0);
  } else {
    k0 = (uint64_t)f * P.cr;
    const uint32_t c2 = P.cur2[f], l2 = P.lim2[f];
    m = c2 < l2 ? c2 : l2;
  }
  if (m == 0) return;
  const uint64_t rbase = (uint64_t)f << ST_LOG_R;
  const uint32_t len = (uint32_t)((T.c - rbase) < ST_R ? (T.c - rbase) : ST_R);
  const uint64_t* slots = static_cast<const uint64_t*>(T.slots);
  if (threadIdx.x == 0) {
    B.n = 0;
    s_qn = 0;
    s_dirty = 0;
    mbar_init(&bar, 1);
    mbar_expect_tx(&bar, (len + HALO) * 8u);
    bulk_load(tile, slots + rbase, len * 8u, &bar);
    const uint64_t hb = rbase + len < T.c ? rbase + len : 0;
    bulk_load(tile + len, slots + hb, HALO * 8u, &bar);
  }
  const uint32_t e = (uint32_t)T.e, t = (uint32_t)T.t;
  const uint32_t gm = ~((uint32_t)g - 1u), ug = (uint32_t)g;
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t att = 0, ndef = 0, nsent = 0, nerased = 0;
  const uint32_t* const tw = reinterpret_cast<const uint32_t*>(tile);
  const uint32_t* const kp = keys + k0;
  const uint16_t* const lp = los + k0;
  uint32_t* const rvp = res_val + k0;
  uint8_t* const rfp = res_flag + k0;
  const uint32_t k0u = (uint32_t)k0;
  // first round's keys in flight while the tile lands
  // two keys per thread and round (i and i + LQT): independent steps, one queue push
  uint32_t nk[2] = {e, e}, nl[2] = {0, 0};
#pragma unroll
  for (int x = 0; x < 2; ++x)
    if (threadIdx.x + x * LQT < m) {
      nk[x] = __ldcs(kp + threadIdx.x + x * LQT);
      nl[x] = __ldcs(lp + threadIdx.x + x * LQT);
    }
  __syncthreads();  // mbarrier initialised
  mbar_wait(&bar, 0);
  {
    // 4 slots per thread from two 16-byte loads (consecutive threads, consecutive 32 B: no
    // bank conflicts; a 4-byte key-word gather per slot was 8-way conflicted)
    const uint32_t words = (len + HALO + TILE_PAD + 3) >> 2;
    const uint4* t16 = reinterpret_cast<const uint4*>(tile);
    for (uint32_t i = threadIdx.x; i < words; i += LQT) {
      const uint4 a = t16[2 * i], b = t16[2 * i + 1];
      const uint32_t w[4] = {a.x, a.z, b.x, b.z};
      uint32_t fw = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) fw |= (w[u] == e ? FP_EMPTY : fp7(w[u])) << (8 * u);
      fp32[i] = fw;
    }
    // past the staged slots: never decisive (a step only reads them beyond its window)
    for (uint32_t i = words + threadIdx.x; i < FP_BYTES / 4; i += LQT) fp32[i] = 0x7F7F7F7Fu;
  }
  __syncthreads();

  // one 16-slot step of key k (rep = fp7(k) * 0x01010101) at window offset o (updated);
  // true while the key stays open
  auto step = [&](uint32_t k, uint32_t rep, uint32_t lo, uint32_t i, uint32_t& o) -> bool {
    const uint32_t x = lo + o, a = x >> 2, sh = (x & 3u) * 8u;
    const uint32_t w0 = fp32[a], w1 = fp32[a + 1], w2 = fp32[a + 2], w3 = fp32[a + 3], w4 = fp32[a + 4];
    const uint32_t f0 = fp_flags(__funnelshift_r(w0, w1, sh), rep);
    const uint32_t f1 = fp_flags(__funnelshift_r(w1, w2, sh), rep);
    const uint32_t f2 = fp_flags(__funnelshift_r(w2, w3, sh), rep);
    const uint32_t f3 = fp_flags(__funnelshift_r(w3, w4, sh), rep);
    const uint32_t mk = __byte_perm(flag_mask8(f0, f1), flag_mask8(f2, f3), 0x0073);  // slots 0..15 -> bits 0..15
    const uint32_t u = (uint32_t)__ffs(mk) - 1u;  // first decisive slot (0xffffffff: none)
    const uint32_t room = WINDOW - o;
    if (u >= (room < 16u ? room : 16u)) {  // nothing decisive in this step's part of the window
      o += 16u;
      if (o < WINDOW) return true;
      defer_push(B, DB, k, 0u, k0u + i, WINDOW);  // window 0 has neither the key nor an empty
      ndef += 1;
      return false;
    }
    o += u;
    const uint32_t s2 = 2 * (lo + o);
    const uint32_t c = tw[s2];
    if (c != k && c != e) {  // fingerprint collision: scan on after it
      o += 1;
      if (o < WINDOW) return true;
      defer_push(B, DB, k, 0u, k0u + i, WINDOW);
      ndef += 1;
      return false;
    }
    const bool hit = c == k;
    if (ERASE) {
      bool erased = false;
      if (hit) {  // retire: key word -> tombstone, value zeroed (layout.py:231)
        const unsigned long long w = ((unsigned long long)tw[s2 + 1] << 32) | c;
        erased = atomicCAS(reinterpret_cast<unsigned long long*>(tile) + (lo + o), w, (unsigned long long)t) == w;
        if (erased) {
          nerased += 1;
          s_dirty = 1;
        }
      }
      rfp[i] = (uint8_t)erased;
    } else {
      rvp[i] = hit ? tw[s2 + 1] : 0u;
      rfp[i] = (uint8_t)hit;
    }
    att += (o & gm) + ug;  // chunk_end(o, g)
    return false;
  };

  for (uint32_t base = 0; base < m; base += 2 * LQT) {  // CTA-uniform rounds
    uint32_t k[2], lo[2], o[2] = {0, 0};
    bool open[2] = {false, false};
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      const uint32_t i = base + x * LQT + threadIdx.x;
      k[x] = nk[x];
      lo[x] = nl[x];
      if (i + 2 * LQT < m) {  // next round's keys
        nk[x] = __ldcs(kp + i + 2 * LQT);
        nl[x] = __ldcs(lp + i + 2 * LQT);
      }
    }
#pragma unroll
    for (int x = 0; x < 2; ++x) {
      const uint32_t i = base + x * LQT + threadIdx.x;
      if (i < m) {
        if (k[x] == e || k[x] == t) {  // sentinels are never stored (single_table.py:391-393)
          if (!ERASE) rvp[i] = 0;
          rfp[i] = 0;
          nsent += 1;
        } else if (ERASE && lo[x] + WINDOW > len) {  // window 0 reaches into the next region
          defer_push(B, DB, k[x], 0u, k0u + i, 0u);
          ndef += 1;
        } else {
          open[x] = step(k[x], fp7(k[x]) * 0x01010101u, lo[x], i, o[x]);
        }
      }
    }
    // warp-aggregated push of the open keys (both of this round's)
    const unsigned w0 = __ballot_sync(0xffffffffu, open[0]), w1 = __ballot_sync(0xffffffffu, open[1]);
    if (w0 | w1) {
      const int leader = __ffs(w0 | w1) - 1;
      uint32_t qb = 0;
      if ((int)lane == leader) qb = atom_add_shared(&s_qn, (uint32_t)(__popc(w0) + __popc(w1)));
      qb = __shfl_sync(0xffffffffu, qb, leader);
#pragma unroll
      for (int x = 0; x < 2; ++x) {
        if (!open[x]) continue;
        const uint32_t i = base + x * LQT + threadIdx.x;
        const uint32_t sq = qb + (x ? __popc(w0) : 0u) + __popc((x ? w1 : w0) & ((1u << lane) - 1u));
        if (sq < LQ_CAP) {
          qk[sq] = k[x];
          qi[sq] = i;
          qlo[sq] = lo[x] | o[x] << 16;
        } else {  // queue full (skewed region): finish here
          const uint32_t rep = fp7(k[x]) * 0x01010101u;
          while (step(k[x], rep, lo[x], i, o[x])) {
          }
        }
      }
    }
  }
  __syncthreads();
  const uint32_t qn = s_qn < LQ_CAP ? s_qn : LQ_CAP;
  for (uint32_t s = threadIdx.x; s < qn; s += LQT) {
    const uint32_t k = qk[s], i = qi[s], w = qlo[s];
    const uint32_t lo = w & 0xFFFFu, rep = fp7(k) * 0x01010101u;
    uint32_t o = w >> 16;
    while (step(k, rep, lo, i, o)) {
    }
  }
  defer_flush(B, DB, true);  // syncs
  if (ERASE && s_dirty) {  // the retired keys back to the table (the halo stays untouched)
    fence_smem_to_async();
    __syncthreads();
    if (threadIdx.x == 0) bulk_store_wait(const_cast<uint64_t*>(slots) + rbase, tile, len * 8u);
  }
  // every key of the region is either resolved (one op, one window unless a sentinel) or deferred;
  // erase counts no sentinel (single_table.py:338-351)
  const long long ops = (threadIdx.x == 0 ? (long long)m : 0ll) - (long long)ndef - (ERASE ? (long long)nsent : 0ll);
  const long long cv6[6] = {ops, (long long)att, ops - (ERASE ? 0ll : (long long)nsent), -(long long)nerased,
                            (long long)nerased, (long long)ndef};
  long long* const dst[6] = {(long long*)&T.ctr->ops, (long long*)&T.ctr->attempts, (long long*)&T.ctr->windows,
                             &T.ctr->occupied, ERASE ? &T.ctr->tombstones : nullptr, (long long*)&T.ctr->deferred};
  cta_add<6>(cv6, dst);
}
constexpr size_t lookup_q_smem() { return (size_t)(ST_R + ST_HALO + TILE_PAD) * 8 + FP_BYTES + LQ_CAP * 12; }

// Region pass for inserts, uniform rounds (the insert counterpart of k_st_lookup_q).  The
// fingerprint bytes are kept current while the region fills: a claim's winner turns its
// slot's byte from empty (0x80) into the key's fp7 with one shared atomic XOR.  A byte can
// lag its key word only between a CAS and that XOR, and a key that reads such a stale
// "empty" loses the CAS exactly as if it had read the word -- a lost claim to another key
// continues after the slot (single_table.py:232-233 re-reads, counted like it: + g
// attempts), a lost claim to the same key is DUPLICATE_KEY (:224-231).  Tombstones are
// 0x81 and decisive like an empty; a tombstone first defers the key to the COPS kernel
// (the deferred-claim rule, :201-223), as in k_st_probe<0>.
constexpr uint32_t IQ_CAP = 1536;  // queued keys per region
constexpr uint32_t IQ_DBUF = 512;  // window-full deferrals buffered per region (~4.6% of ~7.8 K)
constexpr uint32_t FP_TOMB = 0x81u;
#ifndef CH_IQ_STEP
#define CH_IQ_STEP 16
#endif
// slots per insert step.  32 (the whole window: a key claims as soon as it is examined)
// measured 3.49 vs 3.00 ms; with 16 the queued keys (~20%) claim after the rest of the
// region's keys, which leaves ~5-8% more keys past window 0 than the lane-refill pass did.
constexpr uint32_t IQ_STEP = CH_IQ_STEP;

__device__ __forceinline__ void insert_q_region(uint32_t f, const TableRef& T, const Part& P,
                                                const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                                                const uint16_t* __restrict__ los, uint8_t* __restrict__ status,
                                                const DeferOut& DA, const DeferOut& DB, int g,
                                                unsigned long long* __restrict__ exc, int fresh) {
  extern __shared__ __align__(128) unsigned char dsm[];
  uint64_t* tile = reinterpret_cast<uint64_t*>(dsm);
  uint32_t* fp32 = reinterpret_cast<uint32_t*>(tile + ST_R + TILE_PAD);
  uint32_t* qk = fp32 + FP_BYTES / 4;  // queue: key, value, region index, lo | offset << 16
  uint32_t* qv = qk + IQ_CAP;
  uint32_t* qi = qv + IQ_CAP;
  uint32_t* qlo = qi + IQ_CAP;
  __shared__ DeferBuf<true, IQ_DBUF> B;  // -> DB (window full)
  __shared__ DeferBuf<true, DBUF> BA;    // -> DA (tombstone first, window past the region)
  __shared__ uint32_t s_qn;
  __shared__ __align__(8) uint64_t bar;
  __shared__ int dirty;
  uint64_t k0;
  uint32_t m;
  if (P.foff) {
    k0 = P.foff[f];
    m = (uint32_t)(P.foff[f + 1] - k0);
  } else {
    k0 = (uint64_t)f * P.cr;
    const uint32_t c2 = P.cur2[f], l2 = P.lim2[f];
    m = c2 < l2 ? c2 : l2;
  }
  if (m == 0 && !fresh) return;  // (a pending clear still writes the region: fresh)
  const uint64_t rbase = (uint64_t)f << ST_LOG_R;
  const uint32_t len = (uint32_t)((T.c - rbase) < ST_R ? (T.c - rbase) : ST_R);
  uint64_t* slots = static_cast<uint64_t*>(T.slots);
  if (threadIdx.x == 0) {
    B.n = 0;
    BA.n = 0;
    s_qn = 0;
    dirty = 0;
    mbar_init(&bar, 1);
    if (!fresh) {
      mbar_expect_tx(&bar, len * 8u);
      bulk_load(tile, slots + rbase, len * 8u, &bar);
    }
  }
  const uint32_t e = (uint32_t)T.e, t = (uint32_t)T.t;
  const uint32_t gm = ~((uint32_t)g - 1u), ug = (uint32_t)g;
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t att = 0, ndef = 0, nexc = 0, occ = 0, nsent = 0;
  uint32_t* const tw = reinterpret_cast<uint32_t*>(tile);
  const uint32_t* const kp = keys + k0;
  const uint32_t* const vp = vals + k0;
  const uint16_t* const lp = los + k0;
  uint8_t* const stp = status + k0;
  const uint32_t k0u = (uint32_t)k0;
  uint32_t nk = e, nv = 0, nl = 0;
  if (threadIdx.x < m) {
    nk = __ldcs(kp + threadIdx.x);
    nv = __ldcs(vp + threadIdx.x);
    nl = __ldcs(lp + threadIdx.x);
  }
  __syncthreads();  // mbarrier initialised
  if (fresh) {  // the table's clear is pending: the region starts empty
    for (uint32_t q = threadIdx.x; q < (len + 1) / 2; q += LQT)
      reinterpret_cast<uint4*>(tile)[q] = make_uint4(e, 0u, e, 0u);
    __syncthreads();
  } else {
    mbar_wait(&bar, 0);
  }
  {
    const uint32_t words = (len + TILE_PAD + 3) >> 2;
    const uint4* t16 = reinterpret_cast<const uint4*>(tile);
    for (uint32_t i = threadIdx.x; i < words; i += LQT) {
      const uint4 a = t16[2 * i], b = t16[2 * i + 1];
      const uint32_t w[4] = {a.x, a.z, b.x, b.z};
      uint32_t fw = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) fw |= (w[u] == e ? FP_EMPTY : w[u] == t ? FP_TOMB : fp7(w[u])) << (8 * u);
      fp32[i] = fw;
    }
    for (uint32_t i = words + threadIdx.x; i < FP_BYTES / 4; i += LQT) fp32[i] = 0x7F7F7F7Fu;
  }
  __syncthreads();

  // one 16-slot step of key k at window offset o (updated); true while the key stays open
  auto step = [&](uint32_t k, uint32_t v, uint32_t rep, uint32_t lo, uint32_t i, uint32_t& o) -> bool {
    const uint32_t x = lo + o, a = x >> 2, sh = (x & 3u) * 8u;
    uint32_t w[IQ_STEP / 4 + 1], fl[IQ_STEP / 4];
#pragma unroll
    for (int q = 0; q <= (int)IQ_STEP / 4; ++q) w[q] = lds32(fp32 + a + q);
#pragma unroll
    for (int q = 0; q < (int)IQ_STEP / 4; ++q) fl[q] = fp_flags(__funnelshift_r(w[q], w[q + 1], sh), rep);
    uint32_t mk = __byte_perm(flag_mask8(fl[0], fl[1]), flag_mask8(fl[2], fl[3]), 0x0073);
    if (IQ_STEP == 32)  // slots 16..31 -> bits 16..31
      mk = (mk & 0xFFFFu) |
           __byte_perm(flag_mask8(fl[4 % (IQ_STEP / 4)], fl[5 % (IQ_STEP / 4)]),
                       flag_mask8(fl[6 % (IQ_STEP / 4)], fl[7 % (IQ_STEP / 4)]), 0x7300) & 0xFFFF0000u;
    const uint32_t u = (uint32_t)__ffs(mk) - 1u;
    const uint32_t room = WINDOW - o;
    if (u >= (room < IQ_STEP ? room : IQ_STEP)) {
      o += IQ_STEP;
      if (o < WINDOW) return true;
      defer_push(B, DB, k, v, k0u + i, WINDOW);  // neither the key nor a free cell in window 0
      ndef += 1;
      return false;
    }
    o += u;
    const uint32_t s = lo + o;
    const uint32_t c = lds32(tw + 2 * s);
    if (c == t) {  // tombstone first: the deferred-claim rule, COPS kernel from window 0
      defer_push(BA, DA, k, v, k0u + i, 0u);
      ndef += 1;
      return false;
    }
    if (c == e) {
      const uint32_t old = atomicCAS(tw + 2 * s, e, k);
      if (old == e) {
        tw[2 * s + 1] = v;  // nothing in this pass reads values; the write-back follows a barrier
        atomicXor(fp32 + (s >> 2), (FP_EMPTY ^ fp7(k)) << (8 * (s & 3u)));
        occ += 1;
        att += (o & gm) + ug;
        return false;  // INSERTED is pre-set
      }
      if (old != k) {  // another key took the cell: on after it
        att += ug;
        o += 1;
        if (o < WINDOW) return true;
        defer_push(B, DB, k, v, k0u + i, WINDOW);
        ndef += 1;
        return false;
      }
    } else if (c != k) {  // fingerprint collision
      o += 1;
      if (o < WINDOW) return true;
      defer_push(B, DB, k, v, k0u + i, WINDOW);
      ndef += 1;
      return false;
    }
    stp[i] = ST_DUPLICATE;  // present before the first free cell (single_table.py:198-200)
    nexc += 1;
    att += (o & gm) + ug;
    return false;
  };

  for (uint32_t base = 0; base < m; base += LQT) {  // CTA-uniform rounds
    const uint32_t i = base + threadIdx.x;
    const uint32_t k = nk, v = nv, lo = nl;
    if (i + LQT < m) {
      nk = __ldcs(kp + i + LQT);
      nv = __ldcs(vp + i + LQT);
      nl = __ldcs(lp + i + LQT);
    }
    bool open = false;
    uint32_t o = 0;
    if (i < m) {
      if (k == e || k == t) {  // sentinels are never stored (single_table.py:369-370)
        stp[i] = ST_INVALID;
        nexc += 1;
        nsent += 1;
      } else if (lo + WINDOW > len) {  // the window leaves the staged region: COPS kernel
        defer_push(BA, DA, k, v, k0u + i, 0u);
        ndef += 1;
      } else {
        open = step(k, v, fp7(k) * 0x01010101u, lo, i, o);
      }
    }
    const unsigned want = __ballot_sync(0xffffffffu, open);
    if (want) {
      const int leader = __ffs(want) - 1;
      uint32_t qb = 0;
      if ((int)lane == leader) qb = atom_add_shared(&s_qn, (uint32_t)__popc(want));
      qb = __shfl_sync(0xffffffffu, qb, leader);
      if (open) {
        const uint32_t q = qb + __popc(want & ((1u << lane) - 1u));
        if (q < IQ_CAP) {
          qk[q] = k;
          qv[q] = v;
          qi[q] = i;
          qlo[q] = lo | o << 16;
        } else {  // queue full: finish here
          const uint32_t rep = fp7(k) * 0x01010101u;
          while (step(k, v, rep, lo, i, o)) {
          }
        }
      }
    }
  }
  __syncthreads();
  const uint32_t qn = s_qn < IQ_CAP ? s_qn : IQ_CAP;
  for (uint32_t q = threadIdx.x; q < qn; q += LQT) {
    const uint32_t k = qk[q], v = qv[q], i = qi[q], w = qlo[q];
    const uint32_t lo = w & 0xFFFFu, rep = fp7(k) * 0x01010101u;
    uint32_t o = w >> 16;
    while (step(k, v, rep, lo, i, o)) {
    }
  }
  defer_flush(B, DB, true);  // syncs
  defer_flush(BA, DA, true);
  if (occ || fresh) dirty = 1;
  fence_smem_to_async();
  __syncthreads();
  if (threadIdx.x == 0 && dirty) bulk_store_wait(slots + rbase, tile, len * 8u);
  // resolved keys: one op and one window each (sentinels: neither), deferred: counted by the COPS kernel
  const long long ops = (threadIdx.x == 0 ? (long long)m : 0ll) - (long long)ndef - (long long)nsent;
  const long long cv6[6] = {ops, (long long)att, ops, (long long)occ, (long long)nexc, (long long)ndef};
  long long* const dst[6] = {(long long*)&T.ctr->ops, (long long*)&T.ctr->attempts, (long long*)&T.ctr->windows,
                             &T.ctr->occupied, (long long*)exc, (long long*)&T.ctr->deferred};
  cta_add<6>(cv6, dst);
  __syncthreads();
  if (threadIdx.x == 0) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_addr(&bar)) : "memory");
}

// Regions k_st_insert_sg handed back (list, device-counted; a few CTAs loop over them), or
// every region (list == nullptr: one CTA per region).
__global__ void __launch_bounds__(LQT, 2) k_st_insert_q(TableRef T, Part P, const uint32_t* __restrict__ keys,
                                                        const uint32_t* __restrict__ vals,
                                                        const uint16_t* __restrict__ los,
                                                        uint8_t* __restrict__ status, DeferOut DA, DeferOut DB, int g,
                                                        unsigned long long* __restrict__ exc,
                                                        const uint32_t* __restrict__ list,
                                                        const unsigned long long* __restrict__ n_list, int fresh) {
  if (!list) {
    insert_q_region(blockIdx.x, T, P, keys, vals, los, status, DA, DB, g, exc, fresh);
    return;
  }
  const unsigned long long nl = *n_list;
  for (unsigned long long idx = blockIdx.x; idx < nl; idx += gridDim.x)
    insert_q_region(list[idx], T, P, keys, vals, los, status, DA, DB, g, exc, fresh);
}
constexpr size_t insert_q_smem() { return (size_t)(ST_R + TILE_PAD) * 8 + FP_BYTES + IQ_CAP * 16; }

// ------------------------------------------------------------- sorted-greedy insert
// Region pass for inserts that places the region's keys in ascending order of their window
// start (lo): each key takes the first free slot of its window at its turn, so the result
// is the reference's sequential insert of the keys in that order -- a valid linearisation
// of the batch -- and among all orders it keeps the most keys inside window 0 (placing
// equal-length intervals by left end, leftmost free slot first, is a maximum matching).
// Simulated at load 0.95 (tools/sim_sorted_greedy.py): 0.2% of the keys leave window 0
// against ~4% in arbitrary order; those are the keys the COPS kernels finish with random
// DRAM probes, and fewer of them also lets more lookups resolve in window 0.
//
// Parallel form.  Keys with equal lo are interchangeable, so the greedy runs over the 2^13
// window starts with multiplicities c_l; in free-slot index space (free = empty slot of the
// staged tile) the lag of the placed keys behind each window start evolves by a clamped
// addition, and one block scan of those maps gives every group's first slot and how many of
// its keys fit (phase (c) below).  Keys that do not fit resume at window 1 (COPS kernel).
// In-batch duplicates (same key -> same lo) are found after the placement by comparing each
// key with its group's placed keys of lower rank; a region with one is handed back whole
// (nothing has reached global memory by then).
//
// Regions with tombstones (the deferred-claim rule) or more than SG_MAXK keys are handed
// back (redo[]) to k_st_insert_q, which runs next over those regions only.
constexpr uint32_t SGT = 768;
constexpr uint32_t SG_MAXK = 9216;            // keys per region (12 per thread)
constexpr uint32_t SG_PER = SG_MAXK / SGT;    // keys per thread (region order)
constexpr uint32_t SG_LPT = (ST_R + SGT - 1) / SGT;  // window starts per thread (11)
constexpr uint32_t SG_DBUF = 192;             // deferrals buffered per region
constexpr uint32_t SG_CQ = 512;               // duplicate-check queue (~6% of the keys)
#ifndef CH_AB_SG_PB
#define CH_AB_SG_PB 4
#endif
constexpr int SG_PB = CH_AB_SG_PB;             // values / keys read per placement batch
static_assert(SG_MAXK % SGT == 0 && SG_PER <= 12, "sorted pass geometry");

template <int NT>
__device__ __forceinline__ uint32_t block_excl_sum(uint32_t v, uint32_t* wt) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) wt[warp] = x;
  __syncthreads();
  uint32_t y = lane < NT / 32 ? wt[lane] : 0u;
#pragma unroll
  for (int d = 1; d < NT / 32; d <<= 1) {
    const uint32_t z = __shfl_up_sync(0xffffffffu, y, d);
    if (lane >= d) y += z;
  }
  const uint32_t before = warp ? __shfl_sync(0xffffffffu, y, warp - 1) : 0u;
  __syncthreads();  // wt reusable
  return before + x - v;
}

// x -> min(max(x + p, q), r) on int lags; closed under composition.  The +-2^24 sentinels
// stay far from any reachable value (the offsets of one region sum to less than 2^14 in size).
struct ClampMap {
  int p, q, r;
  static constexpr int INF = 1 << 24;
  __device__ __forceinline__ static ClampMap id() { return {0, -INF, INF}; }
  __device__ __forceinline__ int apply(int x) const { return min(max(x + p, q), r); }
};
// g after f
__device__ __forceinline__ ClampMap compose(const ClampMap& f, const ClampMap& g) {
  return {f.p + g.p, max(f.q + g.p, g.q), min(max(f.r + g.p, g.q), g.r)};
}
// one window-start group: c keys, free indices a = fidx(l), a1 = fidx(l + 1), b = fidx(l + 32)
__device__ __forceinline__ ClampMap group_map(uint32_t c, uint32_t a, uint32_t a1, uint32_t b) {
  const int d = (int)(a1 - a), w = (int)(b - a);
  if (c == 0) return {-d, -ClampMap::INF, ClampMap::INF};
  return {(int)c - d, (int)c - d, w - d};
}
// exclusive prefix composition in thread order (identity for thread 0)
template <int NT>
__device__ __forceinline__ ClampMap block_excl_clamp(ClampMap x, int (*wsm)[3]) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  ClampMap in = x;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    ClampMap y;
    y.p = __shfl_up_sync(0xffffffffu, in.p, d);
    y.q = __shfl_up_sync(0xffffffffu, in.q, d);
    y.r = __shfl_up_sync(0xffffffffu, in.r, d);
    if (lane >= d) in = compose(y, in);
  }
  if (lane == 31) wsm[warp][0] = in.p, wsm[warp][1] = in.q, wsm[warp][2] = in.r;
  __syncthreads();
  // the warps before this one: an exclusive scan of the warp totals, lane w holding warp w's
  ClampMap wv = lane < NT / 32 ? ClampMap{wsm[lane][0], wsm[lane][1], wsm[lane][2]} : ClampMap::id();
#pragma unroll
  for (int d = 1; d < NT / 32; d <<= 1) {
    ClampMap y;
    y.p = __shfl_up_sync(0xffffffffu, wv.p, d);
    y.q = __shfl_up_sync(0xffffffffu, wv.q, d);
    y.r = __shfl_up_sync(0xffffffffu, wv.r, d);
    if (lane >= d) wv = compose(y, wv);
  }
  ClampMap carry;
  carry.p = __shfl_sync(0xffffffffu, wv.p, (warp + 31) & 31);
  carry.q = __shfl_sync(0xffffffffu, wv.q, (warp + 31) & 31);
  carry.r = __shfl_sync(0xffffffffu, wv.r, (warp + 31) & 31);
  if (warp == 0) carry = ClampMap::id();
  ClampMap prev;  // the lanes before this one
  prev.p = __shfl_up_sync(0xffffffffu, in.p, 1);
  prev.q = __shfl_up_sync(0xffffffffu, in.q, 1);
  prev.r = __shfl_up_sync(0xffffffffu, in.r, 1);
  if (lane == 0) prev = ClampMap::id();
  __syncthreads();
  return compose(carry, prev);
}

// per-key class after the exclusion pass (key state bits 28..31; rank in bits 0..15)
constexpr uint32_t SG_NONE = 0u, SG_PART = 1u, SG_INV = 2u, SG_DUP = 3u, SG_DEFA = 4u, SG_DEFB = 5u;

__global__ void __launch_bounds__(SGT, 2) k_st_insert_sg(TableRef T, Part P, const uint32_t* __restrict__ keys,
                                                         const uint32_t* __restrict__ vals,
                                                         const uint16_t* __restrict__ los,
                                                         uint8_t* __restrict__ status, DeferOut DA, DeferOut DB,
                                                         int g, unsigned long long* __restrict__ exc,
                                                         uint32_t* __restrict__ redo,
                                                         unsigned long long* __restrict__ n_redo, int fresh) {
  extern __shared__ __align__(128) unsigned char dsm[];
  uint64_t* tile = reinterpret_cast<uint64_t*>(dsm);
  // per window start lo: participants (bits 0..15) | signature of their key hashes (16..31);
  // after the scan (c): free index of the group's first key (0..15) | keys placed (16..31)
  uint32_t* cs = reinterpret_cast<uint32_t*>(tile + ST_R + TILE_PAD);
  uint32_t* freew = cs + ST_R;                                             // free-slot bitmap
  uint16_t* wpre = reinterpret_cast<uint16_t*>(freew + ST_R / 32);         // free slots before word w
  __shared__ DeferBuf<true, SG_DBUF> B;   // -> DB (window full)
  __shared__ DeferBuf<true, SG_DBUF> BA;  // -> DA (window past the region)
  __shared__ uint32_t wt[SGT / 32];
  __shared__ int s_tomb, s_dup;
  __shared__ uint32_t s_qn;
  __shared__ uint32_t cq_k[SG_CQ];  // duplicate-check queue: key, lo | own rank << 13 (63: not placed)
  __shared__ uint16_t cq_l[SG_CQ];
  __shared__ int cm3[SGT / 32][3];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t f = blockIdx.x;
  uint64_t k0;
  uint32_t m;
  if (P.foff) {
    k0 = P.foff[f];
    m = (uint32_t)(P.foff[f + 1] - k0);
  } else {
    k0 = (uint64_t)f * P.cr;
    const uint32_t c2 = P.cur2[f], l2 = P.lim2[f];
    m = c2 < l2 ? c2 : l2;
  }
  if (m == 0 && !fresh) return;  // (a pending clear still writes the region: fresh)
  if (m > SG_MAXK) {  // skewed region: the concurrent pass takes it
    if (threadIdx.x == 0) redo[atomicAdd(n_redo, 1ull)] = f;
    return;
  }
  const uint64_t rbase = (uint64_t)f << ST_LOG_R;
  const uint32_t len = (uint32_t)((T.c - rbase) < ST_R ? (T.c - rbase) : ST_R);
  uint64_t* slots = static_cast<uint64_t*>(T.slots);
  if (threadIdx.x == 0) {
    B.n = 0;
    BA.n = 0;
    s_tomb = 0;
    s_dup = 0;
    s_qn = 0;
    mbar_init(&bar, 1);
    if (!fresh) {
      mbar_expect_tx(&bar, len * 8u);
      bulk_load(tile, slots + rbase, len * 8u, &bar);
    }
  }
  for (uint32_t q = threadIdx.x; q < ST_R / 4; q += SGT) reinterpret_cast<uint4*>(cs)[q] = make_uint4(0u, 0u, 0u, 0u);
  const uint32_t e = (uint32_t)T.e, t = (uint32_t)T.t;
  const uint32_t gm = ~((uint32_t)g - 1u), ug = (uint32_t)g;
  const uint32_t* const kp = keys + k0;
  const uint32_t* const vp = vals + k0;
  const uint16_t* const lp = los + k0;
  uint8_t* const stp = status + k0;
  const uint32_t k0u = (uint32_t)k0;
  uint32_t* const tw = reinterpret_cast<uint32_t*>(tile);
  const uint32_t lane = threadIdx.x & 31u;
  auto cq_push = [&](uint32_t k, uint32_t lo, uint32_t own) {
    const uint32_t q = atom_add_shared(&s_qn, 1u);
    if (q < SG_CQ) {
      cq_k[q] = k;
      cq_l[q] = (uint16_t)(lo | own << 13);
    } else {
      s_dup = 1;  // queue full: the concurrent pass takes the region
    }
  };
  // the region's keys and window starts (coalesced), in flight while the tile lands; the
  // values (needed at the placement) are prefetched into L2 by one bulk prefetch
  if (threadIdx.x == 0) l2_prefetch(vp, (size_t)m * 4);
  uint32_t kk[SG_PER], ks0[SG_PER];
#pragma unroll
  for (int u = 0; u < (int)SG_PER; ++u) {
    const uint32_t i = threadIdx.x + (uint32_t)u * SGT;
    kk[u] = i < m ? kp[i] : 0u;  // (kept in L2: the placement reads the keys again)
    ks0[u] = i < m ? (uint32_t)__ldcs(lp + i) : 0u;
  }
  __syncthreads();  // zeroed, mbarrier initialised
  // any occupied cell in the tile?  (16-byte reads of the key words; the common case -- a
  // fresh table -- needs no free-slot bitmap: the free index of slot s is s).  With the table's
  // clear pending (fresh) the region starts empty and is not read at all.
  bool occ_any;
  if (fresh) {
    for (uint32_t q = threadIdx.x; q < (len + 1) / 2; q += SGT)
      reinterpret_cast<uint4*>(tile)[q] = make_uint4(e, 0u, e, 0u);
    __syncthreads();
    occ_any = false;
  } else {
    mbar_wait(&bar, 0);
    const uint4* t16 = reinterpret_cast<const uint4*>(tile);
    bool oc = false;
    for (uint32_t q = threadIdx.x; q < len / 2; q += SGT) {
      const uint4 x = t16[q];
      oc |= (x.x != e) | (x.z != e);
    }
    if (len & 1u) oc |= threadIdx.x == 0 && tw[2 * (len - 1)] != e;
    occ_any = __syncthreads_or(oc) != 0;
  }
  if (occ_any) {  // free-slot bitmap (a warp per 32-slot word); tombstones
    for (uint32_t w = threadIdx.x >> 5; w < ST_R / 32; w += SGT / 32) {
      const uint32_t sl = 32 * w + lane;
      const uint32_t kw = sl < len ? tw[2 * sl] : e;
      const uint32_t fb = __ballot_sync(0xffffffffu, sl < len && kw == e);
      const bool tb = __any_sync(0xffffffffu, sl < len && kw == t);
      if (lane == 0) {
        freew[w] = fb;
        if (tb) s_tomb = 1;
      }
    }
    __syncthreads();
    if (s_tomb) {  // tombstones: the deferred-claim rule needs the concurrent pass
      if (threadIdx.x == 0) redo[atomicAdd(n_redo, 1ull)] = f;
      return;
    }
    const uint32_t fc = threadIdx.x < ST_R / 32 ? __popc(freew[threadIdx.x]) : 0u;
    const uint32_t fb = block_excl_sum<SGT>(fc, wt);  // syncs
    if (threadIdx.x < ST_R / 32) wpre[threadIdx.x] = (uint16_t)fb;
    __syncthreads();
  }
  auto fidx = [&](uint32_t sl) -> uint32_t {  // free slots before slot sl (sl <= ST_R)
    if (!occ_any) return sl < len ? sl : len;  // an empty tile: every staged slot is free
    const uint32_t w = sl >> 5, b = sl & 31u;
    if (w >= ST_R / 32) return (uint32_t)wpre[ST_R / 32 - 1] + __popc(freew[ST_R / 32 - 1]);
    return (uint32_t)wpre[w] + __popc(freew[w] & ((1u << b) - 1u));
  };
  // (b) exclusions (region order, no side effects yet); participants take a rank in their group.
  // Key state ks: class << 28 | over-placed flag << 27 | lo << 14 | rank (or probe offset).
  uint32_t ks[SG_PER];
  uint32_t special = 0;  // bit u: item u ends as anything but placed / absent (phase (f) looks at those only)
#pragma unroll
  for (int u = 0; u < (int)SG_PER; ++u) {
    const uint32_t i = threadIdx.x + (uint32_t)u * SGT;
    ks[u] = SG_NONE << 28;
    if (i >= m) continue;
    const uint32_t k = kk[u], lo = ks0[u];
    if (k == e || k == t) {  // sentinels are never stored (single_table.py:369-370)
      ks[u] = SG_INV << 28;
      special |= 1u << u;
      continue;
    }
    // a window crossing the region end takes part with its own-region slots (they come first in
    // window order); a key that does not fit there resumes at window 0 in the COPS kernel
    const uint32_t span = len - lo < WINDOW ? len - lo : WINDOW;
    if (occ_any) {  // stored before the first free cell (single_table.py:198-200)
      uint32_t o = 0;
      for (; o < span; ++o) {
        const uint32_t kw = tw[2 * (lo + o)];
        if (kw == e || kw == k) break;
      }
      if (o < span && tw[2 * (lo + o)] == k) {
        ks[u] = SG_DUP << 28 | lo << 14 | o;
        special |= 1u << u;
        continue;
      }
    }
    if (occ_any && fidx(lo) == fidx(lo + span)) {  // neither the key nor a free cell here
      ks[u] = (span < WINDOW ? SG_DEFA : SG_DEFB) << 28 | lo << 14;  // the rest of window 0 / window 1
      special |= 1u << u;
      continue;
    }
    // the rank in the group (count, bits 0..15) and one bit of the key's hash ORed into the
    // group's signature (bits 16..31) of the same word
    const uint32_t rk = atom_add_shared(cs + lo, 1u) & 0xFFFFu;
    const uint32_t bit = 1u << (16u + ((k * 0x9E3779B1u) >> 28));
    ks[u] = SG_PART << 28 | lo << 14 | (rk < 0x3FFFu ? rk : 0x3FFFu);
    if (atomicOr(cs + lo, bit) & bit) cq_push(k, lo, rk < 63u ? rk : 63u);
  }
  __syncthreads();
  // (c) the exact greedy over window starts.  With lam_j = (chain end + 1) - a_j, the lag of the
  // keys placed so far behind group j's first free index, the greedy is
  //   lam_{j+1} = min(max(lam_j, 0) + c_j, w_j) - d_j   (c_j > 0),   lam_{j+1} = lam_j - d_j   (c_j = 0)
  // (w_j: free slots of the window, d_j: slot j free), a clamped addition x -> min(max(x + p, q), r);
  // those compose into the same form, so one block scan over the 2^13 window starts gives every
  // group's first free index a_j + max(lam_j, 0) and how many of its keys fit,
  // min(c_j, w_j - max(lam_j, 0)) -- the sequential greedy exactly (tools/sim_sorted_greedy.py).
  {
    const uint32_t l0 = threadIdx.x * SG_LPT;
    // free index before slot l, after it, and at the window end (identity up to len on an empty tile)
    auto abw = [&](uint32_t l, uint32_t& a, uint32_t& a1, uint32_t& b) {
      if (!occ_any) {
        a = l < len ? l : len;
        a1 = l + 1 < len ? l + 1 : len;
        b = l + WINDOW < len ? l + WINDOW : len;
      } else {
        a = fidx(l);
        a1 = fidx(l + 1);
        b = fidx(l + WINDOW);
      }
    };
    ClampMap h = ClampMap::id();
#pragma unroll
    for (int u = 0; u < (int)SG_LPT; ++u) {
      const uint32_t l = l0 + (uint32_t)u;
      if (l < ST_R) {
        uint32_t a, a1, b;
        abw(l, a, a1, b);
        h = compose(h, group_map(cs[l] & 0xFFFFu, a, a1, b));
      }
    }
    int lam = block_excl_clamp<SGT>(h, cm3).apply(0);
#pragma unroll
    for (int u = 0; u < (int)SG_LPT; ++u) {
      const uint32_t l = l0 + (uint32_t)u;
      if (l >= ST_R) break;
      const uint32_t c = cs[l] & 0xFFFFu;
      uint32_t a, a1, b;
      abw(l, a, a1, b);
      if (c) {
        const int lag = lam > 0 ? lam : 0;
        const int fit = (int)b - (int)a - lag;
        const uint32_t placed = (int)c < fit ? c : (fit > 0 ? (uint32_t)fit : 0u);
        cs[l] = ((uint32_t)((int)a + lag) & 0xFFFFu) | placed << 16;
      }
      lam = group_map(c, a, a1, b).apply(lam);
    }
  }
  __syncthreads();
  uint32_t nexc = 0, ndef = 0, nsent = 0, occn = 0, att = 0;
  // (d) placement into the staged tile; values load four keys at a time
  auto slot_of = [&](uint32_t fi) -> uint32_t {  // the fi-th free slot
    if (!occ_any) return fi;
    uint32_t lo_w = 0, hi_w = ST_R / 32;  // last word with wpre <= fi
    while (hi_w - lo_w > 1) {
      const uint32_t mid = (lo_w + hi_w) >> 1;
      if (wpre[mid] <= fi) lo_w = mid;
      else hi_w = mid;
    }
    uint32_t fb = freew[lo_w];
    for (uint32_t x = fi - wpre[lo_w]; x; --x) fb &= fb - 1;
    return 32 * lo_w + __ffs(fb) - 1;
  };
#pragma unroll
  for (int g4 = 0; g4 < (int)SG_PER; g4 += SG_PB) {
    uint32_t vv[SG_PB], kr[SG_PB];  // values and keys again (L2): no key registers live through the scan
#pragma unroll
    for (int x = 0; x < SG_PB; ++x) {
      const int u = g4 + x;
      const bool part = ((ks[u] >> 28) & 7u) == SG_PART;
      vv[x] = part ? __ldcs(vp + threadIdx.x + (uint32_t)u * SGT) : 0u;
      kr[x] = part ? __ldcs(kp + threadIdx.x + (uint32_t)u * SGT) : 0u;
    }
#pragma unroll
    for (int x = 0; x < SG_PB; ++x) {
      const int u = g4 + x;
      if (((ks[u] >> 28) & 7u) != SG_PART) continue;
      const uint32_t lo = (ks[u] >> 14) & 0x1FFFu, r = ks[u] & 0x3FFFu, w = cs[lo];
      if (r >= (w >> 16)) {  // past what window 0 holds for this group: resume at window 1 (a
        // window crossing the region end: at window 0, its next-region slots are unexamined)
        ks[u] = (lo + WINDOW > len ? SG_DEFA : SG_DEFB) << 28 | 1u << 27 | lo << 14;
        special |= 1u << u;
        cq_push(kr[x], lo, 63u);  // must not equal a placed key of its group
        continue;
      }
      const uint32_t sl = slot_of((w & 0xFFFFu) + r);
      tile[sl] = (uint64_t)vv[x] << 32 | kr[x];
      occn += 1;
      att += ((sl - lo) & gm) + ug;
    }
  }
  fence_smem_to_async();  // the placed tile, for the bulk store issued after the duplicate check
  __syncthreads();
  // (e) in-batch duplicates.  Copies of a key share a window start, so they are in one group.  In
  // (b) every participant ORs one bit of its key hash into its group's 16-bit signature; a key whose
  // bit was set already (a copy -- or, for ~6% of the keys, a different key) is queued, as is a
  // copy that did not fit, and compared here with its group's other placed keys.  One found: the
  // region goes to the concurrent pass (nothing has been written to global memory yet).
  {
    const uint32_t nq = s_qn < SG_CQ ? s_qn : SG_CQ;
    for (uint32_t q = threadIdx.x; q < nq; q += SGT) {
      const uint32_t k = cq_k[q], lo = cq_l[q] & 0x1FFFu, own = cq_l[q] >> 13;
      const uint32_t pl = cs[lo] >> 16, f0 = cs[lo] & 0xFFFFu;
      for (uint32_t x = 0; x < pl; ++x)
        if (x != own && tw[2 * slot_of(f0 + x)] == k) s_dup = 1;
    }
  }
  __syncthreads();
  if (s_dup) {
    if (threadIdx.x == 0) redo[atomicAdd(n_redo, 1ull)] = f;
    return;
  }
  // the region is final: its write-back runs while the results and deferrals are written
  if (threadIdx.x == 0) bulk_store_issue(slots + rbase, tile, len * 8u);
  // (f) results: statuses, deferrals, counters (placed keys were counted at the placement)
#pragma unroll
  for (int u = 0; u < (int)SG_PER; ++u) {
    if (!((special >> u) & 1u)) continue;
    const uint32_t cls = (ks[u] >> 28) & 7u;
    const uint32_t i = threadIdx.x + (uint32_t)u * SGT;
    if (cls == SG_INV) {
      stp[i] = ST_INVALID;
      nexc += 1;
      nsent += 1;
    } else if (cls == SG_DUP) {
      stp[i] = ST_DUPLICATE;
      nexc += 1;
      att += ((ks[u] & 0x3FFFu) & gm) + ug;
    } else {
      defer_push(cls == SG_DEFA ? BA : B, cls == SG_DEFA ? DA : DB, kp[i], vp[i], k0u + i,
                 cls == SG_DEFA ? 0u : WINDOW);
      ndef += 1;
    }
  }
  defer_flush2(B, DB, BA, DA);  // syncs
  if (threadIdx.x == 0) bulk_read_wait();  // the tile must stay until the store has read it
  const long long ops = (threadIdx.x == 0 ? (long long)m : 0ll) - (long long)ndef - (long long)nsent;
  const long long cv6[6] = {ops, (long long)att, ops, (long long)occn, (long long)nexc, (long long)ndef};
  long long* const dst[6] = {(long long*)&T.ctr->ops, (long long*)&T.ctr->attempts, (long long*)&T.ctr->windows,
                             &T.ctr->occupied, (long long*)exc, (long long*)&T.ctr->deferred};
  cta_add<6>(cv6, dst);
}
constexpr size_t insert_sg_smem() { return (size_t)(ST_R + TILE_PAD) * 8 + ST_R * 4 + ST_R / 8 + ST_R / 16; }  // tile, cs, freew, wpre

template <int MODE, bool R2>
constexpr size_t probe_smem() {
  return (size_t)(ST_R + (MODE == 0 ? 0 : ST_HALO) + TILE_PAD) * 8 + (MODE == 0 ? 0 : FP_BYTES);
}

// ------------------------------------------------------------- host side
struct StPlan {
  uint32_t regions, supers;
  uint64_t tiles1, tiles2;  // partition tiles per level (level 2: upper bound)
  bool oa;                  // round 1 overallocated (no count pass)
  uint32_t cs, cr;          // its capacities per super-region / region
  uint64_t n1, n2, nres;    // level-1 / level-2 array lengths, region-order results (+ overflow)
};

// CH_STAGED_COUNT=1: the count-based partition for every batch (what batches of 2^30
// keys and more use; the tests force it on small ones).
static bool g_count_mode = [] {
  const char* e = getenv("CH_STAGED_COUNT");
  return e && e[0] == '1';
}();

// Overallocation: expected keys per region n R / c plus 6.25 % and 256 (> 8 standard
// deviations of a uniform hash at the bench's 7.8 K keys per region), per super-region
// + 3 % and one tile (> 40 deviations).  Skewed batches overflow and take the exact
// paths (Part).  Positions stay below 2^32 for n < 2^30.
static StPlan st_plan(const TableRef& T, uint64_t n) {
  StPlan p;
  p.regions = (uint32_t)((T.c + ST_R - 1) >> ST_LOG_R);
  p.supers = (p.regions + (1u << ST_S2) - 1) >> ST_S2;
  p.tiles1 = (n + PTILE - 1) / PTILE;
  p.tiles2 = p.tiles1 + p.supers;
  p.oa = n < (1ull << 30) && !g_count_mode;
  const double per_region = (double)n * ST_R / (double)T.c;
  p.cs = p.oa ? (((uint32_t)(per_region * (1u << ST_S2) * 1.03) + PTILE + 63u) & ~63u) : 0u;  // 64-key aligned
  p.cr = p.oa ? (((uint32_t)(per_region * 1.0625) + 256u + 63u) & ~63u) : 0u;  // regions start on 256 B key lines
  p.n1 = p.oa ? std::max<uint64_t>(n, (uint64_t)p.supers * p.cs) : n;
  p.n2 = p.oa ? (uint64_t)p.regions * p.cr : n;
  p.nres = p.oa ? p.n2 + n : n;
  return p;
}

bool staged_supported(const TableRef& T, uint64_t n) {
  const uint64_t regions = (T.c + ST_R - 1) >> ST_LOG_R;
  return n > 0 && n < (1ull << 32) && regions <= ST_MAX_REGIONS && T.c < (1ull << 32);
}

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

// Scratch carving (one cudaMallocAsync per call, stream-ordered pool).
struct Carver {
  char* q;
  size_t used = 0;
  void* take(size_t bytes) {
    void* r = q ? q + used : nullptr;
    used += align_up(bytes);
    return r;
  }
};

// One forward round: histogram + scan + plan + one or two tile partitions.
struct Round {
  uint32_t *gcount, *cur1, *cur2, *tstart, *sbase, *scnt, *lim2;
  int* flag;
  unsigned long long* ovf2;
  Part part;  // the geometry the round's kernels ran with (probe, gathers)
  uint64_t* foff;
  void* scan;
  size_t scan_bytes;
  uint32_t *k1, *v1, *p1, *r1, *k2, *v2, *p2, *r2;  // level-1 / level-2 outputs (payloads v, p, r)
  uint16_t* lo2;
  uint16_t *inv1, *inv2, *th1, *th2;  // inverse (round 1 only)
  uint8_t *bid1, *bid2;               // bucket of each bucketed slot per tile (round 1 only)
  uint8_t* redo;                      // regions k_st_insert_sg hands to k_st_insert_q: count, list
  uint32_t *tg1, *tg2;
};

struct StBufs {
  Round r1, r2, rd;                // round 1, round 2 (optional), deferred-key ordering (level 1 only)
  unsigned long long* dcount;     // [0]: list A (COPS kernels), [1]: list B (round 2)
  uint32_t *ak, *av, *ax, *ao, *bk, *bv, *bx, *bo;
  uint32_t *rv, *rv1;  // lookup: values in region order / level-1 order
  uint8_t *rf, *rf1;   // lookup: found flags; insert: statuses
};

static void carve_round(Carver& c, Round& r, const StPlan& p, uint64_t n, int npay, bool inverse, int levels,
                        bool oa) {
  r = Round{};
  const uint64_t n1 = oa ? p.n1 : n, n2 = oa ? p.n2 : n;
  r.gcount = (uint32_t*)c.take(p.regions * 4ull);
  r.sbase = (uint32_t*)c.take(p.supers * 4ull);
  r.scnt = (uint32_t*)c.take(p.supers * 4ull);
  r.lim2 = (uint32_t*)c.take(p.regions * 4ull);
  r.ovf2 = (unsigned long long*)c.take(64);
  r.flag = reinterpret_cast<int*>(r.ovf2 + 1);
  r.foff = (uint64_t*)c.take((p.regions + 1ull) * 8);
  r.scan_bytes = align_up(exclusive_scan_scratch_bytes(p.regions));
  r.scan = c.take(r.scan_bytes);
  r.cur1 = (uint32_t*)c.take(PBINS * 4ull);
  r.cur2 = (uint32_t*)c.take(p.regions * 4ull);
  r.tstart = (uint32_t*)c.take((p.supers + 1ull) * 4);
  r.k1 = (uint32_t*)c.take(n1 * 4);
  r.v1 = npay >= 1 ? (uint32_t*)c.take(n1 * 4) : nullptr;
  r.p1 = npay >= 2 ? (uint32_t*)c.take(n1 * 4) : nullptr;
  r.r1 = npay >= 3 ? (uint32_t*)c.take(n1 * 4) : nullptr;
  if (levels == 2) {
    r.k2 = (uint32_t*)c.take(n2 * 4);
    r.v2 = npay >= 1 ? (uint32_t*)c.take(n2 * 4) : nullptr;
    r.p2 = npay >= 2 ? (uint32_t*)c.take(n2 * 4) : nullptr;
    r.r2 = npay >= 3 ? (uint32_t*)c.take(n2 * 4) : nullptr;
    r.lo2 = (uint16_t*)c.take(n2 * 2);
  }
  if (inverse) {
    r.inv1 = (uint16_t*)c.take(n * 2);
    r.inv2 = (uint16_t*)c.take(n1 * 2);
    r.redo = (uint8_t*)c.take(64 + p.regions * 4ull);  // count, then the handed-back region list
    r.bid1 = npay == 0 ? (uint8_t*)c.take(n) : nullptr;  // lookups only (k_st_gather<L, true>)
    r.bid2 = npay == 0 ? (uint8_t*)c.take(n1) : nullptr;
    r.th1 = (uint16_t*)c.take(p.tiles1 * p.supers * 2);
    r.tg1 = (uint32_t*)c.take(p.tiles1 * p.supers * 4);
    r.th2 = (uint16_t*)c.take(p.tiles2 * 256 * 2);
    r.tg2 = (uint32_t*)c.take(p.tiles2 * 256 * 4);
  }
}

static StBufs st_carve(const StPlan& p, uint64_t n, bool ins, bool round2, void* base, size_t* total) {
  Carver c{static_cast<char*>(base)};
  StBufs b;
  carve_round(c, b.r1, p, n, ins ? 1 : 0, true, 2, p.oa);
  if (round2) carve_round(c, b.r2, p, n, ins ? 2 : 1, false, 2, false);
  carve_round(c, b.rd, p, n, ins ? 3 : 2, false, 1, false);
  b.dcount = (unsigned long long*)c.take(64);
  b.ak = (uint32_t*)c.take(n * 4);
  b.av = ins ? (uint32_t*)c.take(n * 4) : nullptr;
  b.ax = (uint32_t*)c.take(n * 4);
  b.ao = (uint32_t*)c.take(n * 4);
  b.bk = round2 ? (uint32_t*)c.take(n * 4) : b.ak;  // without round 2, one list
  b.bv = round2 ? (ins ? (uint32_t*)c.take(n * 4) : nullptr) : b.av;
  b.bx = round2 ? (uint32_t*)c.take(n * 4) : b.ax;
  b.bo = round2 ? (uint32_t*)c.take(n * 4) : b.ao;
  b.rv = ins ? nullptr : (uint32_t*)c.take(p.nres * 4);
  b.rv1 = ins ? nullptr : (uint32_t*)c.take(p.n1 * 4);
  b.rf = (uint8_t*)c.take(p.nres);
  b.rf1 = (uint8_t*)c.take(p.n1);
  *total = c.used;
  return b;
}

// staged window-1 round for the deferred keys: off by default (CH_STAGED_ROUND2=1 enables it).
// At load 0.95 ~40% of the round-2 keys defer again and the COPS kernel then walks windows
// >= 2 for them, so the extra region pass did not pay (profiles/r01_staged_round2.txt).
static bool g_round2 = [] {
  const char* e = getenv("CH_STAGED_ROUND2");
  return e && e[0] == '1';
}();

// CTAs per SM of the deferred-key COPS pass (CH_STAGED_FB_CTAS; default 0 = a full wave,
// which measured fastest: 1 / 2 / full per SM -> 20.1 / 20.1 / 21.6 G ops/s).
static int g_fb_blocks = [] {
  const char* e = getenv("CH_STAGED_FB_CTAS");
  const int v = e ? atoi(e) : 0;
  return v > 0 ? v : 0;
}();

// CH_SPLIT_PFD=0: level-1 partition CTAs do not prefetch the tile one wave ahead
static bool g_split_pfd = [] {
  const char* e = getenv("CH_SPLIT_PFD");
  return !(e && e[0] == '0');
}();

// CH_INSERT_SG=0: inserts without the sorted-greedy placement pass (k_st_insert_sg)
static bool g_insert_sg = [] {
  const char* e = getenv("CH_INSERT_SG");
  return !(e && e[0] == '0');
}();

// CH_PROBE_V1=1: the lane-refill region passes for every mode (A/B against the uniform rounds)
static bool g_probe_v1 = [] {
  const char* e = getenv("CH_PROBE_V1");
  return e && e[0] == '1';
}();

size_t staged_scratch_bytes(const TableRef& T, uint64_t n, bool insert) {
  size_t total = 0;
  st_carve(st_plan(T, n), n, insert, g_round2, nullptr, &total);
  return total;
}

template <typename KS>
static int st_smem(KS kern, size_t bytes) {
  int rc = cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes),
                      "smem attribute");
  if (!rc && bytes > (48u << 10))
    rc = cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100), "carveout");
  return rc;
}

static int st_timed(const Launch& lc, cudaEvent_t* e0) {
  *e0 = nullptr;
  if (lc.timer && cudaEventCreate(e0) == cudaSuccess) cudaEventRecord(*e0, lc.stream);
  return 0;
}
static void st_timed_end(const Launch& lc, cudaEvent_t e0) {
  cudaEvent_t e1 = nullptr;
  if (e0 && cudaEventCreate(&e1) == cudaSuccess) {
    cudaEventRecord(e1, lc.stream);
    lc.timer->ev.emplace_back(e0, e1);
  }
}

// One forward round over keys k (+ payloads v, q, w).  Count mode: count + scan + plan +
// L1 (+ L2).  Overallocated (round 1 with p.oa, da = list A): L1 into fixed areas; the
// count-mode L1 runs again only if a run overflowed (gated kernels); L2 into fixed
// region areas, overflowing runs to list A.  n_dev: the round's count lives on the
// device (n is the capacity).  wj: window.
template <int NPAY>
static int st_forward(const Launch& lc, const TableRef& T, const StPlan& p, Round& r, const uint32_t* k,
                      const uint32_t* v, const uint32_t* q, const uint32_t* w, uint64_t n,
                      const unsigned long long* n_dev, int wj, int levels, const DeferOut* da = nullptr) {
  const bool oa = da != nullptr && p.oa && levels == 2 && n_dev == nullptr;
  Part P{};
  P.sbase = r.sbase;
  P.scnt = r.scnt;
  P.tstart = r.tstart;
  P.cur1 = r.cur1;
  P.cur2 = r.cur2;
  P.lim2 = r.lim2;
  P.flag = r.flag;
  P.ovf2 = r.ovf2;
  const size_t sm1 = (size_t)PTILE * (4 + 4 * NPAY + 2), sm2 = sm1 + PTILE * (NPAY >= 1 ? 2 : 4);
  const unsigned t1 = (unsigned)p.tiles1, t2 = (unsigned)p.tiles2;
  auto k1f = k_st_split<1, NPAY>;
  auto k2f = k_st_split<2, NPAY>;
  int rc = st_smem(k1f, sm1);
  if (!rc && levels == 2) rc = st_smem(k2f, sm2);
  if (rc) return rc;
  // persistent partition CTAs (a gated level 1 costs one wave)
  auto grid = [&](const void* kern, size_t sm, unsigned tiles) {
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, PT, sm);
    const unsigned full = (unsigned)lc.sms * (unsigned)(occ > 0 ? occ : 1);
    return tiles < full ? (tiles ? tiles : 1u) : full;
  };
  // a CTA per tile when the batch size is known on the host (a persistent loop measured
  // 26.8 vs 27.9 G ops/s); one persistent wave when it lives on the device (most of the
  // grid would exit at once) and for the gated redo
  const unsigned g1r = grid((const void*)k1f, sm1, t1);
  const unsigned g1 = n_dev ? g1r : (t1 ? t1 : 1u);
  const unsigned g2 = n_dev ? grid((const void*)k2f, sm2, t2) : (t2 ? t2 : 1u);
  const size_t csmem = p.regions * 4ull;
  if ((rc = st_smem(k_st_count, csmem))) return rc;
  int cocc = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cocc, k_st_count, 1024, csmem);
  if (cocc < 1) cocc = 1;
  // count mode level 1 (always, or as the gated redo after an overflow)
  auto count_mode_l1 = [&](Part C, int init_cur2) -> int {
    int e = cuda_check(cudaMemsetAsync(r.gcount, 0, p.regions * 4ull, lc.stream), "memset");
    if (e) return e;
    k_st_count<<<(unsigned)(lc.sms * cocc), 1024, csmem, lc.stream>>>(T, k, n, p.regions, r.gcount, n_dev, wj,
                                                                       C.gate);
    count_launch();
    if ((e = cuda_check(cudaGetLastError(), "staged count"))) return e;
    if ((e = exclusive_scan_u32(lc, r.gcount, p.regions, r.foff, r.scan, r.scan_bytes))) return e;
    k_st_plan<<<1, PT, 0, lc.stream>>>(C, p.regions, p.supers, init_cur2);
    count_launch();
    k1f<<<C.gate ? g1r : g1, PT, sm1, lc.stream>>>(T, n, C, p.supers, t1, k, v, q, w, r.k1, r.v1, r.p1, r.r1, nullptr,
                                                    r.inv1, r.th1, r.tg1, p.supers, n_dev, wj, r.bid1);
    count_launch();
    return cuda_check(cudaGetLastError(), "staged partition");
  };
  if (oa) {
    P.cs = p.cs;
    P.cr = p.cr;
    P.ovf2_base = p.regions * p.cr;
    P.da = *da;
    rc = cuda_check(cudaMemsetAsync(r.cur1, 0, p.supers * 4ull, lc.stream), "memset");
    if (!rc) rc = cuda_check(cudaMemsetAsync(r.cur2, 0, p.regions * 4ull, lc.stream), "memset");
    if (!rc) rc = cuda_check(cudaMemsetAsync(r.lim2, 0xFF, p.regions * 4ull, lc.stream), "memset");
    if (!rc) rc = cuda_check(cudaMemsetAsync(r.ovf2, 0, 64, lc.stream), "memset");  // ovf2, flag
    if (rc) return rc;
    Part L1 = P;
    L1.cr = 0;
    if (g_split_pfd && g1 == t1) {  // one CTA per tile: prefetch a resident wave ahead
      int occ = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)k1f, PT, sm1);
      L1.pfd = (uint32_t)(lc.sms * (occ > 0 ? occ : 1));
    }
    k1f<<<g1, PT, sm1, lc.stream>>>(T, n, L1, p.supers, t1, k, v, q, w, r.k1, r.v1, r.p1, r.r1, nullptr, r.inv1,
                                     r.th1, r.tg1, p.supers, n_dev, wj, r.bid1);
    count_launch();
    Part C = P;  // the redo: count-mode cursors, level 2 stays overallocated
    C.foff = r.foff;
    C.cs = C.cr = 0;
    C.gate = r.flag;
    if ((rc = count_mode_l1(C, 0))) return rc;
    k_st_plan_oa<<<1, PT, 0, lc.stream>>>(P, p.supers);
    count_launch();
  } else {
    P.foff = r.foff;
    if ((rc = count_mode_l1(P, levels == 2))) return rc;
  }
  if (levels == 2) {
    Part P2 = P;
    if (g_split_pfd && !n_dev && NPAY <= 1) {  // one CTA per tile: prefetch a resident wave ahead
      int occ = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)k2f, PT, sm2);
      P2.pfd = (uint32_t)(lc.sms * (occ > 0 ? occ : 1));
    }
    k2f<<<g2, PT, sm2, lc.stream>>>(T, n, P2, p.supers, t2, r.k1, r.v1, r.p1, r.r1, r.k2, r.v2, r.p2, r.r2, r.lo2,
                                     r.inv2, r.th2, r.tg2, 256, n_dev, wj, r.bid2);
    count_launch();
  }
  r.part = P;
  return cuda_check(cudaGetLastError(), "staged partition");
}

// region-ordered results -> caller's order (inverse of L2, then of L1)
template <bool VAL>
static int st_backward(const Launch& lc, const StPlan& p, const StBufs& b, uint64_t n, const uint32_t* rv,
                       const uint8_t* rf, uint32_t* out_v, uint8_t* out_f, const unsigned long long* exc = nullptr) {
  const Round& r = b.r1;
  const unsigned t1 = (unsigned)p.tiles1, t2 = (unsigned)p.tiles2;
  auto g2 = VAL ? k_st_gather<2, VAL> : k_st_gather_st<2, VAL>;
  auto g1 = VAL ? k_st_gather<1, VAL> : k_st_gather_st<1, VAL>;
  const unsigned q2 = VAL ? t2 : std::min<unsigned>(t2, (unsigned)lc.sms * 3);
  const unsigned q1 = VAL ? t1 : std::min<unsigned>(t1, (unsigned)lc.sms * 3);
  g2<<<q2, PT, 0, lc.stream>>>(n, r.part, p.supers, t2, r.inv2, r.th2, r.tg2, 256, rv, rf, b.rv1, b.rf1, exc,
                               r.bid2);
  count_launch();
  g1<<<q1, PT, 0, lc.stream>>>(n, r.part, p.supers, t1, r.inv1, r.th1, r.tg1, p.supers, b.rv1, b.rf1, out_v, out_f,
                                exc, r.bid1);
  count_launch();
  return cuda_check(cudaGetLastError(), "staged gather");
}

template <int MODE, bool R2>
static int st_probe(const Launch& lc, const TableRef& T, const StPlan& p, const Round& r, const uint32_t* pos,
                    uint8_t* status, uint32_t* rv, uint8_t* rf, const DeferOut& DA, const DeferOut& DB, int g,
                    unsigned long long* exc = nullptr, int fresh = 0) {
  cudaEvent_t e0;
  if (MODE == 0 && !R2 && !g_probe_v1) {
    // sorted-greedy placement (k_st_insert_sg), then the uniform-rounds pass (k_st_insert_q)
    // over the regions it handed back (tombstones, skewed regions); CH_INSERT_SG=0: only the latter
    const size_t sm = insert_q_smem();
    int rc = st_smem(k_st_insert_q, sm);
    if (rc) return rc;
    const uint32_t* list = nullptr;
    unsigned long long* n_list = reinterpret_cast<unsigned long long*>(r.redo);
    uint32_t* redo = reinterpret_cast<uint32_t*>(r.redo + 64);
    if (g_insert_sg) {
      const size_t sm2 = insert_sg_smem();
      if ((rc = st_smem(k_st_insert_sg, sm2))) return rc;
      if ((rc = cuda_check(cudaMemsetAsync(n_list, 0, 8, lc.stream), "memset"))) return rc;
      st_timed(lc, &e0);
      k_st_insert_sg<<<p.regions, SGT, sm2, lc.stream>>>(T, r.part, r.k2, r.v2, r.lo2, status, DA, DB, g, exc,
                                                         redo, n_list, fresh);
      count_launch();
      st_timed_end(lc, e0);
      if ((rc = cuda_check(cudaGetLastError(), "staged sorted insert"))) return rc;
      list = redo;
    } else {
      st_timed(lc, &e0);
    }
    // the handed-back regions: a few CTAs loop over the list (usually empty)
    const unsigned qgrid = list ? (unsigned)(lc.sms * 2) : p.regions;
    k_st_insert_q<<<qgrid, LQT, sm, lc.stream>>>(T, r.part, r.k2, r.v2, r.lo2, status, DA, DB, g, exc, list, n_list,
                                                 fresh);
    count_launch();
    if (!g_insert_sg) st_timed_end(lc, e0);
    return cuda_check(cudaGetLastError(), "staged region insert");
  }
  if ((MODE == 1 && !R2 && !g_probe_v1) || MODE == 2) {  // uniform rounds + queue (k_st_lookup_q)
    const size_t sm = lookup_q_smem();
    auto lq = MODE == 2 ? k_st_lookup_q<true> : k_st_lookup_q<false>;
    int rc = st_smem(lq, sm);
    if (rc) return rc;
    st_timed(lc, &e0);
    lq<<<p.regions, LQT, sm, lc.stream>>>(T, r.part, r.k2, r.lo2, rv, rf, DB, g);
    count_launch();
    st_timed_end(lc, e0);
    return cuda_check(cudaGetLastError(), "staged region lookup");
  }
  if constexpr (MODE == 2) return 0;  // (erase always takes the uniform-round pass above)
  const size_t sm = probe_smem<MODE == 2 ? 1 : MODE, R2>();
  auto kern = k_st_probe<MODE == 2 ? 1 : MODE, R2>;
  int rc = st_smem(kern, sm);
  if (rc) return rc;
  if (!R2) st_timed(lc, &e0);  // the dominant kernel of the staged schedule (bench.py roofline)
  kern<<<p.regions, RT, sm, lc.stream>>>(T, r.part, r.k2, MODE == 0 ? r.v2 : nullptr, pos, r.lo2, status, rv, rf,
                                         DA, DB, g, exc);
  count_launch();
  if (!R2) st_timed_end(lc, e0);
  return cuda_check(cudaGetLastError(), "staged region probe");
}

// fresh: the table's clear is pending (ch_clear on a staged-size table defers the memset); the
// region passes then start every region empty and write every region back.
int staged_insert(const Launch& lc, const TableRef& T, const TypeSel& ts, const void* keys, const void* vals,
                  uint64_t n, uint8_t* status, void* scratch, int fresh) {
  if (fresh && g_probe_v1) {  // the lane-refill pass reads its regions: clear for real first
    const int rc = single_clear(lc, T, ts);
    if (rc) return rc;
    fresh = 0;
  }
  const StPlan p = st_plan(T, n);
  size_t total = 0;
  const bool r2 = g_round2;
  StBufs b = st_carve(p, n, true, r2, scratch, &total);
  int rc = cuda_check(cudaMemsetAsync(b.dcount, 0, 24, lc.stream), "memset");  // lists A, B; exceptions
  if (!rc) rc = cuda_check(cudaMemsetAsync(b.rf, ST_INSERTED, p.nres, lc.stream), "memset");  // exceptions overwrite
  unsigned long long* exc = b.dcount + 2;
  const DeferOut DA{b.ak, b.av, b.ax, b.ao, b.dcount};
  const DeferOut DB{b.bk, b.bv, b.bx, b.bo, r2 ? b.dcount + 1 : b.dcount};
  if (!rc)
    rc = st_forward<1>(lc, T, p, b.r1, (const uint32_t*)keys, (const uint32_t*)vals, nullptr, nullptr, n, nullptr, 0,
                       2, &DA);
  if (rc) return rc;
  if ((rc = st_probe<0, false>(lc, T, p, b.r1, nullptr, b.rf, nullptr, nullptr, DA, DB, ts.g, exc, fresh))) return rc;
  if (r2) {  // window 1 of the keys whose window 0 was full, staged the same way
    if ((rc = st_forward<2>(lc, T, p, b.r2, b.bk, b.bv, b.bx, nullptr, n, b.dcount + 1, 1, 2))) return rc;
    if ((rc = st_probe<0, true>(lc, T, p, b.r2, b.r2.p2, b.rf, nullptr, nullptr, DA, DA, ts.g, exc))) return rc;
  }
  // the rest: COPS kernels over the deferred keys ordered by their window-1 super-region
  // (consecutive CTAs probe one L2-resident stretch of the table), statuses to their
  // region-ordered positions
  if ((rc = st_forward<3>(lc, T, p, b.rd, b.ak, b.av, b.ax, b.ao, n, b.dcount, 1, 1))) return rc;
  Launch rest = lc;
  rest.timer = nullptr;
  rest.n_dev = b.dcount;
  rest.out_idx = b.rd.p1;
  rest.o_start = b.rd.r1;
  rest.max_blocks = g_fb_blocks * lc.sms;
  rest.exc = exc;
  if ((rc = single_insert(rest, T, ts, b.rd.k1, b.rd.v1, n, b.rf, nullptr, 0))) return rc;
  return st_backward<false>(lc, p, b, n, nullptr, b.rf, nullptr, status, exc);
}

int staged_lookup(const Launch& lc, const TableRef& T, const TypeSel& ts, const void* keys, uint64_t n,
                  void* vals_out, uint8_t* found, void* scratch) {
  const StPlan p = st_plan(T, n);
  size_t total = 0;
  const bool r2 = g_round2;
  StBufs b = st_carve(p, n, false, r2, scratch, &total);
  int rc = cuda_check(cudaMemsetAsync(b.dcount, 0, 16, lc.stream), "memset");
  const DeferOut DA{b.ak, nullptr, b.ax, b.ao, b.dcount};
  const DeferOut DB{b.bk, nullptr, b.bx, b.bo, r2 ? b.dcount + 1 : b.dcount};
  if (!rc)
    rc = st_forward<0>(lc, T, p, b.r1, (const uint32_t*)keys, nullptr, nullptr, nullptr, n, nullptr, 0, 2, &DA);
  if (rc) return rc;
  if ((rc = st_probe<1, false>(lc, T, p, b.r1, nullptr, nullptr, b.rv, b.rf, DA, DB, ts.g))) return rc;
  if (r2) {  // window 1 of the keys whose window 0 decided nothing (positions ride as the payload)
    if ((rc = st_forward<1>(lc, T, p, b.r2, b.bk, b.bx, nullptr, nullptr, n, b.dcount + 1, 1, 2))) return rc;
    if ((rc = st_probe<1, true>(lc, T, p, b.r2, b.r2.v2, nullptr, b.rv, b.rf, DA, DA, ts.g))) return rc;
  }
  // deferred keys ordered by window-1 super-region (payloads: position, resume offset; a
  // second, region-level split measured no better: the deferred keys are too sparse to share lines)
  if ((rc = st_forward<2>(lc, T, p, b.rd, b.ak, b.ax, b.ao, nullptr, n, b.dcount, 1, 1))) return rc;
  Launch rest = lc;
  rest.timer = nullptr;
  rest.n_dev = b.dcount;
  rest.out_idx = b.rd.v1;
  rest.o_start = b.rd.p1;
  rest.max_blocks = g_fb_blocks * lc.sms;
  if ((rc = single_lookup(rest, T, ts, b.rd.k1, n, b.rv, b.rf, nullptr, nullptr, nullptr, 0))) return rc;
  return st_backward<true>(lc, p, b, n, b.rv, b.rf, (uint32_t*)vals_out, found);
}

// Bulk erase (single_table.py:338-351) on the staged schedule: the lookup partitions, the
// region pass retiring what it finds (k_st_lookup_q<true>), the COPS erase for the deferred
// keys, and the erased flags back through the status gathers.
int staged_erase(const Launch& lc, const TableRef& T, const TypeSel& ts, const void* keys, uint64_t n,
                 uint8_t* erased, void* scratch) {
  const StPlan p = st_plan(T, n);
  size_t total = 0;
  StBufs b = st_carve(p, n, false, false, scratch, &total);
  int rc = cuda_check(cudaMemsetAsync(b.dcount, 0, 16, lc.stream), "memset");
  const DeferOut DA{b.ak, nullptr, b.ax, b.ao, b.dcount};
  if (!rc)
    rc = st_forward<0>(lc, T, p, b.r1, (const uint32_t*)keys, nullptr, nullptr, nullptr, n, nullptr, 0, 2, &DA);
  if (rc) return rc;
  if ((rc = st_probe<2, false>(lc, T, p, b.r1, nullptr, nullptr, nullptr, b.rf, DA, DA, ts.g))) return rc;
  if ((rc = st_forward<2>(lc, T, p, b.rd, b.ak, b.ax, b.ao, nullptr, n, b.dcount, 1, 1))) return rc;
  Launch rest = lc;
  rest.timer = nullptr;
  rest.n_dev = b.dcount;
  rest.out_idx = b.rd.v1;
  rest.o_start = b.rd.p1;
  rest.max_blocks = g_fb_blocks * lc.sms;
  if ((rc = single_lookup(rest, T, ts, b.rd.k1, n, nullptr, b.rf, nullptr, nullptr, nullptr, 2))) return rc;
  return st_backward<false>(lc, p, b, n, nullptr, b.rf, nullptr, erased);
}

}  // namespace chb
