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
// 171-245 / 247-269, shared-memory 64-bit CAS for claims), and writes the region
// back with one bulk copy.  Every table byte crosses HBM once per batch, in 64 KiB
// transfers; keys that window 0 cannot decide (window full, a tombstone before
// the first empty, an insert window crossing the region end) are appended to a
// device-counted list and finished by the unchanged COPS probe kernels
// (single.cu) after the region pass -- a valid linearisation of the concurrent
// batch, since nothing is ever removed from a table during an insert or lookup.
//
// Pipeline (all passes stream; n keys):
//   count   region histogram of the keys                     k_st_count
//   scan    region offsets (+ per-super-region L2 tile map)   prims.cu, k_st_plan
//   L1      tile partition by super-region (256 regions)      k_st_split<1>
//   L2      tile partition by region, per super-region tiles  k_st_split<2>
//   region  shared-memory probe of window 0                   k_st_probe
//   rest    deferred keys through the COPS kernels            single.cu (n_dev, out_idx, o_start)
//   back    results (status / value + found) to the caller's order: the inverse
//           of each tile partition, gathering that tile's runs   k_st_gather<2>, <1>
// A tile partition buckets a 4096-element tile in shared memory, writes whole
// (bucket, tile) runs, and records where each element went (u16 rank inside the
// tile, per-tile run table), so results return by gathering the same runs --
// every pass reads and writes coalesced and no position is carried per key.
#include "dispatch.cuh"

namespace chb {

constexpr int ST_LOG_R = 13;
constexpr uint32_t ST_R = 1u << ST_LOG_R;  // region slots
constexpr uint32_t ST_HALO = WINDOW;       // lookups read window 0 past the region end
constexpr int ST_S2 = 8;                   // regions per super-region = 2^ST_S2
constexpr int PT = 512, PI = 8;            // partition CTA: threads x items
constexpr uint32_t PTILE = (uint32_t)PT * PI;
constexpr uint32_t PBINS = 512;
constexpr int RT = 256;                    // region CTA threads
constexpr uint32_t ST_MAX_REGIONS = 51200; // count histogram in shared memory (200 KiB)

__device__ __forceinline__ uint32_t region_of_key(const TableRef& T, uint32_t key) {
  return (uint32_t)(T.modc.mod(mix64((uint64_t)key)) >> ST_LOG_R);
}

// ------------------------------------------------------------- TMA helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

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
// shared -> global bulk copy; waits until the writes are performed
__device__ __forceinline__ void bulk_store_wait(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_addr(src)),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_smem_to_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// ------------------------------------------------------------- count
// Region histogram of the batch (dynamic shared memory, one counter per region).
__global__ void __launch_bounds__(1024) k_st_count(TableRef T, const uint32_t* __restrict__ keys, uint64_t n,
                                                   uint32_t regions, uint32_t* __restrict__ gcount) {
  extern __shared__ uint32_t s_cnt[];
  for (uint32_t i = threadIdx.x; i < regions; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    uint32_t k[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) k[u] = __ldcs(keys + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) atomicAdd(&s_cnt[region_of_key(T, k[u])], 1u);
  }
  for (; i < n; i += stride) atomicAdd(&s_cnt[region_of_key(T, keys[i])], 1u);
  __syncthreads();
  for (uint32_t r = threadIdx.x; r < regions; r += blockDim.x)
    if (s_cnt[r]) atomicAdd(&gcount[r], s_cnt[r]);
}

// Cursors (region starts, super-region starts) and the L2 tile map: the L2 pass
// cuts every super-region into its own 4096-element tiles, so a tile never
// spans two super-regions (<= 256 buckets).  tstart[b] = first L2 tile of
// super-region b, tstart[supers] = number of L2 tiles.  One CTA of PT threads.
__global__ void __launch_bounds__(PT) k_st_plan(const uint64_t* __restrict__ foff, uint32_t regions,
                                                uint32_t supers, uint32_t* __restrict__ cur1,
                                                uint32_t* __restrict__ cur2, uint32_t* __restrict__ tstart) {
  for (uint32_t i = threadIdx.x; i < regions; i += PT) cur2[i] = (uint32_t)foff[i];
  __shared__ uint32_t wt[PT / 32];
  uint32_t carry = 0;
  for (uint32_t b0 = 0; b0 < supers; b0 += PT) {
    const uint32_t b = b0 + threadIdx.x;
    uint32_t v = 0;
    if (b < supers) {
      const uint64_t s = foff[(uint64_t)b << ST_S2];
      const uint64_t e = foff[((uint64_t)(b + 1) << ST_S2) < regions ? ((uint64_t)(b + 1) << ST_S2) : regions];
      cur1[b] = (uint32_t)s;
      v = (uint32_t)((e - s + PTILE - 1) / PTILE);
    }
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

// Geometry of partition tile `t` of level L.  Level 1 tiles are the input cut in
// PTILE pieces; level 2 tiles are each super-region (input: level-1 order) cut in
// PTILE pieces.  Returns false for CTAs past the last tile.
struct TileGeo {
  uint64_t pos0;   // first element (position in this level's input order)
  uint32_t cnt;    // elements
  uint32_t cbase;  // cursor index of bucket 0 (level 2: first region of the super-region)
};

template <int L>
__device__ __forceinline__ bool tile_geo(uint32_t t, uint64_t n, const uint64_t* __restrict__ foff,
                                         const uint32_t* tstart, uint32_t supers, uint32_t regions,
                                         TileGeo& g) {
  if (L == 1) {
    g.pos0 = (uint64_t)t * PTILE;
    if (g.pos0 >= n) return false;
    g.cnt = (uint32_t)((n - g.pos0) < PTILE ? (n - g.pos0) : PTILE);
    g.cbase = 0;
    return true;
  }
  if (t >= tstart[supers]) return false;
  uint32_t lo = 0, hi = supers;  // last b with tstart[b] <= t (tstart: a shared-memory copy)
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (tstart[mid] <= t) lo = mid;
    else hi = mid;
  }
  const uint64_t r0 = (uint64_t)lo << ST_S2;
  const uint64_t r1 = ((uint64_t)(lo + 1) << ST_S2) < regions ? ((uint64_t)(lo + 1) << ST_S2) : regions;
  const uint64_t s = foff[r0], e = foff[r1];
  g.pos0 = s + (uint64_t)(t - tstart[lo]) * PTILE;
  g.cnt = (uint32_t)((e - g.pos0) < PTILE ? (e - g.pos0) : PTILE);
  g.cbase = (uint32_t)r0;
  return true;
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
  uint32_t before = 0;
  for (int w = 0; w < warp; ++w) before += wt[w];
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
template <int L, bool VALS>
__global__ void __launch_bounds__(PT, 2) k_st_split(TableRef T, uint64_t n, const uint64_t* __restrict__ foff,
                                                    const uint32_t* __restrict__ tstart, uint32_t supers,
                                                    uint32_t regions, uint32_t ntiles,
                                                    const uint32_t* __restrict__ kin,
                                                    const uint32_t* __restrict__ vin, uint32_t* __restrict__ kout,
                                                    uint32_t* __restrict__ vout, uint16_t* __restrict__ lo_out,
                                                    uint16_t* __restrict__ inv, uint16_t* __restrict__ th,
                                                    uint32_t* __restrict__ tg, uint32_t nb,
                                                    uint32_t* __restrict__ cursor) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* sK = reinterpret_cast<uint32_t*>(smem);
  uint32_t* sV = sK + PTILE;
  uint16_t* sD = reinterpret_cast<uint16_t*>(sV + (VALS ? PTILE : 0));
  uint16_t* sL = sD + PTILE;  // level 2 only
  __shared__ uint32_t hist[PBINS], boff[PBINS], gbase[PBINS];
  __shared__ uint32_t wt[PT / 32];
  const uint32_t t = blockIdx.x;
  __shared__ uint32_t s_ts[L == 2 ? PBINS + 1 : 1];
  if (L == 2) {
    for (uint32_t i = threadIdx.x; i <= supers; i += PT) s_ts[i] = tstart[i];
    __syncthreads();
  }
  TileGeo g;
  if (t >= ntiles || !tile_geo<L>(t, n, foff, s_ts, supers, regions, g)) return;
  hist[threadIdx.x] = 0;  // PBINS == PT
  uint32_t k[PI], v[PI], d[PI], r[PI];
#pragma unroll
  for (int it = 0; it < PI; ++it) {  // all loads in flight before any use
    const uint32_t li = (uint32_t)it * PT + threadIdx.x;
    k[it] = li < g.cnt ? __ldcs(kin + g.pos0 + li) : 0u;
    if (VALS) v[it] = li < g.cnt ? __ldcs(vin + g.pos0 + li) : 0u;
  }
  __syncthreads();  // hist zeroed
#pragma unroll
  for (int it = 0; it < PI; ++it) {
    const uint32_t li = (uint32_t)it * PT + threadIdx.x;
    if (li >= g.cnt) continue;
    const uint32_t h = (uint32_t)T.modc.mod(mix64((uint64_t)k[it]));  // c < 2^32
    const uint32_t b = L == 1 ? (h >> ST_LOG_R) >> ST_S2 : (h >> ST_LOG_R) - g.cbase;
    r[it] = atomicAdd(&hist[b], 1u);
    d[it] = b | (L == 2 ? (h & (ST_R - 1)) << 16 : 0u);  // window start rides along (registers)
  }
  __syncthreads();
  const uint32_t hv = hist[threadIdx.x];
  const uint32_t bo = block_excl_scan(hv, wt);
  boff[threadIdx.x] = bo;
  const uint32_t gb = hv ? atomicAdd(&cursor[g.cbase + threadIdx.x], hv) : 0u;
  gbase[threadIdx.x] = gb;
  if (threadIdx.x < nb) {
    th[(uint64_t)t * nb + threadIdx.x] = (uint16_t)hv;
    tg[(uint64_t)t * nb + threadIdx.x] = gb;
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < PI; ++it) {
    const uint32_t li = (uint32_t)it * PT + threadIdx.x;
    if (li >= g.cnt) continue;
    const uint32_t b = d[it] & 0xFFFFu;
    const uint32_t j = boff[b] + r[it];
    sK[j] = k[it];
    if (VALS) sV[j] = v[it];
    sD[j] = (uint16_t)b;
    if (L == 2) sL[j] = (uint16_t)(d[it] >> 16);
    inv[g.pos0 + li] = (uint16_t)j;
  }
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < g.cnt; j += PT) {
    const uint32_t b = sD[j];
    const uint32_t dst = gbase[b] + (j - boff[b]);
    kout[dst] = sK[j];
    if (VALS) vout[dst] = sV[j];
    if (L == 2) lo_out[dst] = sL[j];
  }
}

// Inverse of k_st_split<L>: bring the tile's results back from its runs and
// emit them in the tile's input order.  The tile's bucketed order is rebuilt in
// shared memory (bucket id per slot), every thread then gathers PI slots with
// all loads in flight (consecutive slots of a run are consecutive addresses;
// default caching: a sector is shared by the runs of neighbouring tiles).
// VAL: u32 value + u8 flag, otherwise u8 only (insert status).
template <int L, bool VAL>
__global__ void __launch_bounds__(PT) k_st_gather(uint64_t n, const uint64_t* __restrict__ foff,
                                                  const uint32_t* __restrict__ tstart, uint32_t supers,
                                                  uint32_t regions, uint32_t ntiles,
                                                  const uint16_t* __restrict__ inv,
                                                  const uint16_t* __restrict__ th, const uint32_t* __restrict__ tg,
                                                  uint32_t nb, const uint32_t* __restrict__ src_v,
                                                  const uint8_t* __restrict__ src_f, uint32_t* __restrict__ dst_v,
                                                  uint8_t* __restrict__ dst_f) {
  __shared__ uint32_t sV[VAL ? PTILE : 1];
  __shared__ uint8_t sF[PTILE];
  __shared__ uint16_t sB[PTILE];
  __shared__ uint32_t boff[PBINS], hist[PBINS], gsrc[PBINS];
  __shared__ uint32_t wt[PT / 32];
  const uint32_t t = blockIdx.x;
  __shared__ uint32_t s_ts[L == 2 ? PBINS + 1 : 1];
  if (L == 2) {
    for (uint32_t i = threadIdx.x; i <= supers; i += PT) s_ts[i] = tstart[i];
    __syncthreads();
  }
  TileGeo g;
  if (t >= ntiles || !tile_geo<L>(t, n, foff, s_ts, supers, regions, g)) return;
  const uint32_t hv = threadIdx.x < nb ? th[(uint64_t)t * nb + threadIdx.x] : 0u;
  const uint32_t gs = threadIdx.x < nb ? tg[(uint64_t)t * nb + threadIdx.x] : 0u;
  uint16_t iv[PI];
#pragma unroll
  for (int it = 0; it < PI; ++it) {  // the inverse ranks load alongside the run table
    const uint32_t li = (uint32_t)it * PT + threadIdx.x;
    iv[it] = li < g.cnt ? __ldcs(inv + g.pos0 + li) : (uint16_t)0;
  }
  const uint32_t bo = block_excl_scan(hv, wt);
  hist[threadIdx.x] = hv;
  boff[threadIdx.x] = bo;
  gsrc[threadIdx.x] = gs;
  __syncthreads();
  for (uint32_t x = 0; x < hv; ++x) sB[bo + x] = (uint16_t)threadIdx.x;  // thread b: its run's slots
  __syncthreads();
  uint32_t v[PI];
  uint8_t fl[PI];
#pragma unroll
  for (int it = 0; it < PI; ++it) {
    const uint32_t j = (uint32_t)it * PT + threadIdx.x;
    if (j < g.cnt) {
      const uint32_t b = sB[j];
      const uint32_t src = gsrc[b] + (j - boff[b]);
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
#pragma unroll
  for (int it = 0; it < PI; ++it) {
    const uint32_t li = (uint32_t)it * PT + threadIdx.x;
    if (li < g.cnt) {
      const uint32_t j = iv[it];
      if (VAL) dst_v[g.pos0 + li] = sV[j];
      dst_f[g.pos0 + li] = sF[j];
    }
  }
}

// ------------------------------------------------------------- region pass
// Keys that window 0 cannot decide are buffered in shared memory and appended to
// the device-counted list in batches (one global atomic per flush: a per-warp
// atomic on one counter serialised the whole pass).
constexpr uint32_t DBUF = 256;    // deferred entries buffered per CTA
constexpr uint32_t SEG = 2048;    // keys staged per segment
constexpr uint32_t STEP = 8;      // slots one key examines per round
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

struct DeferOut {
  uint32_t *k, *v, *x;
  uint8_t* o;
  unsigned long long* count;
};

template <bool VALS, uint32_t CAP>
__device__ __forceinline__ void defer_push(DeferBuf<VALS, CAP>& B, const DeferOut& D, uint32_t k, uint32_t v,
                                           uint32_t x, uint32_t o) {
  const uint32_t s = atomicAdd(&B.n, 1u);
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
    D.o[g] = (uint8_t)o;
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

__device__ __forceinline__ uint64_t lds64(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(smem_addr(p)) : "memory");
  return v;
}

// warp-aggregated append of e to a shared-memory queue (all lanes call it)
__device__ __forceinline__ void queue_push(bool push, uint16_t e, uint16_t* q, uint32_t* qn) {
  const unsigned mk = __ballot_sync(0xffffffffu, push);
  if (!mk) return;
  const int lane = threadIdx.x & 31, leader = __ffs(mk) - 1;
  uint32_t b = 0;
  if (lane == leader) b = atomicAdd(qn, (uint32_t)__popc(mk));
  b = __shfl_sync(0xffffffffu, b, leader);
  if (push) q[b + __popc(mk & ((1u << lane) - 1u))] = e;
}

// Region pass.  Results are written at the key's region-ordered position (the
// gather passes return them to the caller's order): MODE 0 insert the status,
// MODE 1 lookup the value and found flag.
//
// The region's keys are staged a segment at a time and resolved in ROUNDS: in
// every round each pending key examines the next STEP slots of window 0 (one
// thread per key, the same work for every lane), and keys that are still open
// -- nothing decisive in those slots, or an insert that lost its CAS to
// another key of the round -- are compacted into the next round's queue.  A
// thread-per-key loop over the whole window ran at ~7 of 32 active lanes (the
// warp waited on its longest probe; profiles/r01_region_v3).
template <int MODE>
__global__ void __launch_bounds__(RT, 2) k_st_probe(TableRef T, const uint64_t* __restrict__ foff,
                                                    const uint32_t* __restrict__ keys,
                                                    const uint32_t* __restrict__ vals,
                                                    const uint16_t* __restrict__ los, uint8_t* __restrict__ status,
                                                    uint32_t* __restrict__ res_val, uint8_t* __restrict__ res_flag,
                                                    DeferOut D, int g) {
  constexpr bool INS = MODE == 0;
  constexpr uint32_t HALO = INS ? 0u : ST_HALO;
  extern __shared__ __align__(128) unsigned char dsm[];
  uint64_t* tile = reinterpret_cast<uint64_t*>(dsm);
  uint32_t* s_key = reinterpret_cast<uint32_t*>(tile + ST_R + HALO + TILE_PAD);
  uint32_t* s_val = s_key + SEG;  // insert only
  uint16_t* s_lo = reinterpret_cast<uint16_t*>(s_val + (INS ? SEG : 0));
  uint16_t* s_q0 = s_lo + SEG;  // two round queues, SEG entries each: i << 5 | o
  __shared__ DeferBuf<INS, DBUF> B;
  __shared__ uint32_t s_qn[2];
  __shared__ __align__(8) uint64_t bar;
  __shared__ int dirty;
  const uint32_t f = blockIdx.x;
  const uint64_t k0 = foff[f], k1 = foff[f + 1];
  if (k0 == k1) return;  // no key starts in this region
  const uint64_t rbase = (uint64_t)f << ST_LOG_R;
  const uint32_t len = (uint32_t)((T.c - rbase) < ST_R ? (T.c - rbase) : ST_R);
  uint64_t* slots = static_cast<uint64_t*>(T.slots);
  if (threadIdx.x == 0) {
    dirty = 0;
    B.n = 0;
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
  long long ops = 0, att = 0, win = 0, occ = 0, ndef = 0;
  bool claimed_any = false, waited = false;

  // one probe step of segment key i from in-window offset o; returns true (and the
  // queue entry) when the key stays open for the next round
  auto step = [&](uint64_t s0, uint32_t i, uint32_t o, uint16_t* pe) -> bool {
    const uint32_t k = s_key[i], lo = s_lo[i];
    uint64_t w[STEP];
#pragma unroll
    for (int u = 0; u < (int)STEP; ++u) w[u] = INS ? lds64(tile + lo + o + u) : tile[lo + o + u];
    uint32_t dec = 0;
#pragma unroll
    for (int u = 0; u < (int)STEP; ++u) {
      const uint32_t c = (uint32_t)w[u];
      const bool d = INS ? ((c == k) | (c == e) | (c == t)) : ((c == k) | (c == e));  // lookups pass tombstones
      dec |= (uint32_t)d << u;
    }
    const uint32_t room = WINDOW - o;
    if (room < STEP) dec &= (1u << room) - 1u;
    if (!dec) {
      o += STEP;
      if (o < WINDOW) {
        *pe = (uint16_t)(i << 5 | o);
        return true;
      }
      // window 0 holds neither the key nor a free cell: resume at window 1
      defer_push(B, D, k, INS ? s_val[i] : 0u, (uint32_t)(s0 + i), WINDOW);
      ndef += 1;
      return false;
    }
    o += (uint32_t)__ffs(dec) - 1u;
    const uint64_t wd = INS ? lds64(tile + lo + o) : tile[lo + o];
    const uint32_t c = (uint32_t)wd;
    if (INS) {
      if (c == k) {  // present before the first free cell (single_table.py:198-200)
        status[s0 + i] = ST_DUPLICATE;
      } else if (c == t) {  // tombstone first: the deferred-claim rule (:201-223), COPS kernel
        defer_push(B, D, k, s_val[i], (uint32_t)(s0 + i), 0);
        ndef += 1;
        return false;
      } else {
        bool won = false;
        if (c == e) {
          const unsigned long long want = ((unsigned long long)s_val[i] << 32) | k;
          won = atomicCAS((unsigned long long*)(tile + lo + o), (unsigned long long)wd, want) == wd;
        }
        if (!won) {  // another key of this round took it: re-read it next round (:232-233)
          att += ug;
          *pe = (uint16_t)(i << 5 | o);
          return true;
        }
        occ += 1;
        claimed_any = true;
        status[s0 + i] = ST_INSERTED;
      }
    } else {
      const bool hit = c == k;
      res_val[s0 + i] = hit ? (uint32_t)(wd >> 32) : 0u;
      res_flag[s0 + i] = (uint8_t)hit;
    }
    ops += 1;
    att += (long long)chunk_end(o, ug);
    win += 1;
    return false;
  };

  for (uint64_t s0 = k0; s0 < k1; s0 += SEG) {
    const uint32_t m = (uint32_t)((k1 - s0) < SEG ? (k1 - s0) : SEG);
    if (threadIdx.x == 0) {
      s_qn[0] = 0;
      s_qn[1] = 0;
    }
    // stage the segment (all loads in flight): keys, window starts (+ values)
    constexpr int PER = SEG / RT;
    uint32_t kk[PER], vv[PER];
    uint16_t ll[PER];
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const uint32_t i = (uint32_t)r * RT + threadIdx.x;
      kk[r] = i < m ? __ldcs(keys + s0 + i) : e;
      ll[r] = i < m ? __ldcs(los + s0 + i) : (uint16_t)0;
      if (INS) vv[r] = i < m ? __ldcs(vals + s0 + i) : 0u;
    }
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const uint32_t i = (uint32_t)r * RT + threadIdx.x;
      s_key[i] = kk[r];
      s_lo[i] = ll[r];
      if (INS) s_val[i] = vv[r];
    }
    if (!waited) {
      mbar_wait(&bar, 0);
      waited = true;
    }
    __syncthreads();
    // round 0 over the staged segment
    for (uint32_t base = 0; base < m; base += RT) {
      const uint32_t i = base + threadIdx.x;
      bool push = false;
      uint16_t pe = 0;
      if (i < m) {
        const uint32_t k = s_key[i];
        if (k == e || k == t) {  // sentinels are never stored (single_table.py:369-370, 391-393)
          if (INS) {
            status[s0 + i] = ST_INVALID;
          } else {
            res_val[s0 + i] = 0;
            res_flag[s0 + i] = 0;
            ops += 1;  // retrieve_bulk counts every query (:403)
          }
        } else if (INS && s_lo[i] + WINDOW > len) {  // window 0 leaves the staged region
          defer_push(B, D, k, s_val[i], (uint32_t)(s0 + i), 0);
          ndef += 1;
        } else {
          push = step(s0, i, 0, &pe);
        }
      }
      queue_push(push, pe, s_q0, &s_qn[0]);
    }
    // later rounds over the compacted queue
    uint32_t cur = 0;
    for (;;) {
      __syncthreads();
      const uint32_t qn = s_qn[cur];
      if (qn == 0) break;
      const uint32_t nxt = cur ^ 1u;
      if (threadIdx.x == 0) s_qn[nxt] = 0;  // nobody pushes to nxt before the barrier below
      __syncthreads();
      const uint16_t* qc = s_q0 + cur * SEG;
      for (uint32_t base = 0; base < qn; base += RT) {
        const uint32_t j = base + threadIdx.x;
        bool push = false;
        uint16_t pe = 0;
        if (j < qn) {
          const uint32_t ent = qc[j];
          push = step(s0, ent >> 5, ent & 31u, &pe);
        }
        queue_push(push, pe, s_q0 + nxt * SEG, &s_qn[nxt]);
      }
      cur = nxt;
    }
    defer_flush(B, D, s0 + SEG >= k1);  // syncs: the segment buffers are free again
  }
  if (INS) {
    if (claimed_any) dirty = 1;
    fence_smem_to_async();
    __syncthreads();
    if (threadIdx.x == 0 && dirty) bulk_store_wait(slots + rbase, tile, len * 8u);
  }
  const long long v[6] = {ops, att, win, occ, 0, ndef};
  long long* const dst[6] = {(long long*)&T.ctr->ops, (long long*)&T.ctr->attempts, (long long*)&T.ctr->windows,
                             &T.ctr->occupied, nullptr, (long long*)&T.ctr->deferred};
  cta_add<6>(v, dst);
}

template <int MODE>
constexpr size_t probe_smem() {
  return (size_t)(ST_R + (MODE == 0 ? 0 : ST_HALO) + TILE_PAD) * 8 + (size_t)SEG * (4 + (MODE == 0 ? 4 : 0) + 2 + 4);
}

// ------------------------------------------------------------- host side
struct StPlan {
  uint32_t regions, supers;
  uint64_t tiles1, tiles2;  // partition tiles per level (level 2: upper bound)
};

static StPlan st_plan(const TableRef& T, uint64_t n) {
  StPlan p;
  p.regions = (uint32_t)((T.c + ST_R - 1) >> ST_LOG_R);
  p.supers = (p.regions + (1u << ST_S2) - 1) >> ST_S2;
  p.tiles1 = (n + PTILE - 1) / PTILE;
  p.tiles2 = p.tiles1 + p.supers;
  return p;
}

bool staged_supported(const TableRef& T, uint64_t n) {
  const uint64_t regions = (T.c + ST_R - 1) >> ST_LOG_R;
  return n > 0 && n < (1ull << 32) && regions <= ST_MAX_REGIONS && T.c < (1ull << 32);
}

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

// Scratch carving (one cudaMallocAsync per call, stream-ordered pool).
struct StBufs {
  uint32_t *gcount, *cur1, *cur2, *tstart;
  uint64_t* foff;
  void* scan;
  size_t scan_bytes;
  unsigned long long* dcount;
  uint16_t *th1, *th2;
  uint32_t *tg1, *tg2;
  uint32_t *k1, *v1, *k2, *v2, *dx, *rv, *rv1;  // element arrays (u32)
  uint16_t *inv1, *inv2, *lo2;                  // (u16)
  uint8_t *rf, *rf1, *dO;                       // (u8)
};

struct Carver {
  char* q;
  size_t used = 0;
  void* take(size_t bytes) {
    void* r = q ? q + used : nullptr;
    used += align_up(bytes);
    return r;
  }
};

static StBufs st_carve(const StPlan& p, uint64_t n, bool vals, void* base, size_t* total) {
  Carver c{static_cast<char*>(base)};
  StBufs b;
  b.gcount = (uint32_t*)c.take(p.regions * 4ull);
  b.foff = (uint64_t*)c.take((p.regions + 1ull) * 8);
  b.scan_bytes = align_up(exclusive_scan_scratch_bytes(p.regions));
  b.scan = c.take(b.scan_bytes);
  b.cur1 = (uint32_t*)c.take(PBINS * 4ull);
  b.cur2 = (uint32_t*)c.take(p.regions * 4ull);
  b.tstart = (uint32_t*)c.take((p.supers + 1ull) * 4);
  b.dcount = (unsigned long long*)c.take(64);
  b.th1 = (uint16_t*)c.take(p.tiles1 * p.supers * 2);
  b.tg1 = (uint32_t*)c.take(p.tiles1 * p.supers * 4);
  b.th2 = (uint16_t*)c.take(p.tiles2 * 256 * 2);
  b.tg2 = (uint32_t*)c.take(p.tiles2 * 256 * 4);
  b.k1 = (uint32_t*)c.take(n * 4);  // later: deferred keys
  b.v1 = vals ? (uint32_t*)c.take(n * 4) : nullptr;  // later: deferred values
  b.k2 = (uint32_t*)c.take(n * 4);
  b.v2 = vals ? (uint32_t*)c.take(n * 4) : nullptr;
  b.dx = (uint32_t*)c.take(n * 4);
  b.rv = vals ? nullptr : (uint32_t*)c.take(n * 4);
  b.rv1 = vals ? nullptr : (uint32_t*)c.take(n * 4);
  b.inv1 = (uint16_t*)c.take(n * 2);
  b.inv2 = (uint16_t*)c.take(n * 2);
  b.lo2 = (uint16_t*)c.take(n * 2);
  b.rf = (uint8_t*)c.take(n);  // insert: status in region order
  b.rf1 = (uint8_t*)c.take(n);
  b.dO = (uint8_t*)c.take(n);
  *total = c.used;
  return b;
}

size_t staged_scratch_bytes(const TableRef& T, uint64_t n, bool insert) {
  size_t total = 0;
  st_carve(st_plan(T, n), n, insert, nullptr, &total);
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

// persistent grid: one wave of CTAs (no more than there are tiles)
template <typename KS>
static unsigned persist_grid(const Launch& lc, KS kern, size_t smem, uint64_t tiles) {
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, PT, smem) != cudaSuccess || occ < 1) occ = 1;
  const uint64_t full = (uint64_t)lc.sms * occ;
  return (unsigned)(tiles < full ? tiles : full);
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

// count + scan + plan + L1 + L2: keys (and values) in region order, window starts
static int st_forward(const Launch& lc, const TableRef& T, const StPlan& p, const StBufs& b, const uint32_t* keys,
                      const uint32_t* vals, uint64_t n) {
  int rc = cuda_check(cudaMemsetAsync(b.gcount, 0, p.regions * 4ull, lc.stream), "memset");
  if (!rc) rc = cuda_check(cudaMemsetAsync(b.dcount, 0, 8, lc.stream), "memset");
  if (rc) return rc;
  const size_t csmem = p.regions * 4ull;
  if ((rc = st_smem(k_st_count, csmem))) return rc;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_st_count, 1024, csmem);
  if (occ < 1) occ = 1;
  k_st_count<<<(unsigned)(lc.sms * occ), 1024, csmem, lc.stream>>>(T, keys, n, p.regions, b.gcount);
  count_launch();
  if ((rc = cuda_check(cudaGetLastError(), "staged count"))) return rc;
  if ((rc = exclusive_scan_u32(lc, b.gcount, p.regions, b.foff, b.scan, b.scan_bytes))) return rc;
  k_st_plan<<<1, PT, 0, lc.stream>>>(b.foff, p.regions, p.supers, b.cur1, b.cur2, b.tstart);
  count_launch();
  const bool V = vals != nullptr;
  // bucketed (k [, v], bucket, level 2: window start)
  const size_t sm1 = (size_t)PTILE * (4 + (V ? 4 : 0) + 2), sm2 = sm1 + PTILE * 2;
  const unsigned t1 = (unsigned)p.tiles1, t2 = (unsigned)p.tiles2;
  if (V) {
    auto k1f = k_st_split<1, true>;
    auto k2f = k_st_split<2, true>;
    if ((rc = st_smem(k1f, sm1)) || (rc = st_smem(k2f, sm2))) return rc;
    k1f<<<t1, PT, sm1, lc.stream>>>(T, n, b.foff, b.tstart, p.supers, p.regions, t1, keys,
                                                                 vals, b.k1, b.v1, nullptr, b.inv1, b.th1, b.tg1,
                                                                 p.supers, b.cur1);
    count_launch();
    k2f<<<t2, PT, sm2, lc.stream>>>(T, n, b.foff, b.tstart, p.supers, p.regions, t2, b.k1,
                                                                 b.v1, b.k2, b.v2, b.lo2, b.inv2, b.th2, b.tg2, 256,
                                                                 b.cur2);
    count_launch();
  } else {
    auto k1f = k_st_split<1, false>;
    auto k2f = k_st_split<2, false>;
    if ((rc = st_smem(k1f, sm1)) || (rc = st_smem(k2f, sm2))) return rc;
    k1f<<<t1, PT, sm1, lc.stream>>>(T, n, b.foff, b.tstart, p.supers, p.regions, t1, keys,
                                                                 nullptr, b.k1, nullptr, nullptr, b.inv1, b.th1,
                                                                 b.tg1, p.supers, b.cur1);
    count_launch();
    k2f<<<t2, PT, sm2, lc.stream>>>(T, n, b.foff, b.tstart, p.supers, p.regions, t2, b.k1,
                                                                 nullptr, b.k2, nullptr, b.lo2, b.inv2, b.th2, b.tg2,
                                                                 256, b.cur2);
    count_launch();
  }
  return cuda_check(cudaGetLastError(), "staged partition");
}

// region-ordered results -> caller's order (inverse of L2, then of L1)
template <bool VAL>
static int st_backward(const Launch& lc, const StPlan& p, const StBufs& b, uint64_t n, const uint32_t* rv,
                       const uint8_t* rf, uint32_t* out_v, uint8_t* out_f) {
  const unsigned t1 = (unsigned)p.tiles1, t2 = (unsigned)p.tiles2;
  auto g2 = k_st_gather<2, VAL>;
  auto g1 = k_st_gather<1, VAL>;
  g2<<<t2, PT, 0, lc.stream>>>(n, b.foff, b.tstart, p.supers, p.regions, t2, b.inv2, b.th2,
                                                         b.tg2, 256, rv, rf, b.rv1, b.rf1);
  count_launch();
  g1<<<t1, PT, 0, lc.stream>>>(n, b.foff, b.tstart, p.supers, p.regions, t1, b.inv1, b.th1,
                                                         b.tg1, p.supers, b.rv1, b.rf1, out_v, out_f);
  count_launch();
  return cuda_check(cudaGetLastError(), "staged gather");
}

int staged_insert(const Launch& lc, const TableRef& T, const TypeSel& ts, const void* keys, const void* vals,
                  uint64_t n, uint8_t* status, void* scratch) {
  const StPlan p = st_plan(T, n);
  size_t total = 0;
  const StBufs b = st_carve(p, n, true, scratch, &total);
  int rc = st_forward(lc, T, p, b, (const uint32_t*)keys, (const uint32_t*)vals, n);
  if (rc) return rc;
  const size_t sm = probe_smem<0>();
  if ((rc = st_smem(k_st_probe<0>, sm))) return rc;
  cudaEvent_t e0;
  st_timed(lc, &e0);
  const DeferOut D{b.k1, b.v1, b.dx, b.dO, b.dcount};  // the deferred list reuses the L1 arrays
  k_st_probe<0><<<p.regions, RT, sm, lc.stream>>>(T, b.foff, b.k2, b.v2, b.lo2, b.rf, nullptr, nullptr, D, ts.g);
  count_launch();
  st_timed_end(lc, e0);
  if ((rc = cuda_check(cudaGetLastError(), "staged region insert"))) return rc;
  Launch rest = lc;  // deferred keys: COPS kernels, statuses at their region-ordered positions
  rest.timer = nullptr;
  rest.n_dev = b.dcount;
  rest.out_idx = b.dx;
  rest.o_start = b.dO;
  if ((rc = single_insert(rest, T, ts, b.k1, b.v1, n, b.rf, nullptr, 0))) return rc;
  // statuses back to the caller's order (u8 only)
  return st_backward<false>(lc, p, b, n, nullptr, b.rf, nullptr, status);
}

int staged_lookup(const Launch& lc, const TableRef& T, const TypeSel& ts, const void* keys, uint64_t n,
                  void* vals_out, uint8_t* found, void* scratch) {
  const StPlan p = st_plan(T, n);
  size_t total = 0;
  const StBufs b = st_carve(p, n, false, scratch, &total);
  int rc = st_forward(lc, T, p, b, (const uint32_t*)keys, nullptr, n);
  if (rc) return rc;
  const size_t sm = probe_smem<1>();
  if ((rc = st_smem(k_st_probe<1>, sm))) return rc;
  cudaEvent_t e0;
  st_timed(lc, &e0);
  const DeferOut D{b.k1, nullptr, b.dx, b.dO, b.dcount};
  k_st_probe<1><<<p.regions, RT, sm, lc.stream>>>(T, b.foff, b.k2, nullptr, b.lo2, nullptr, b.rv, b.rf, D, ts.g);
  count_launch();
  st_timed_end(lc, e0);
  if ((rc = cuda_check(cudaGetLastError(), "staged region lookup"))) return rc;
  Launch rest = lc;
  rest.timer = nullptr;
  rest.n_dev = b.dcount;
  rest.out_idx = b.dx;
  rest.o_start = b.dO;
  if ((rc = single_lookup(rest, T, ts, b.k1, n, b.rv, b.rf, nullptr, nullptr, nullptr, 0))) return rc;
  return st_backward<true>(lc, p, b, n, b.rv, b.rf, (uint32_t*)vals_out, found);
}

}  // namespace chb
