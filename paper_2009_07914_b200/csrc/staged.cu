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
//   count   fine-region histogram of the keys              k_st_count
//   scan    region offsets                                  (prims.cu)
//   L1      tile partition by super-region (256 regions)    k_st_part<0>
//   L2      tile partition by region                        k_st_part<1>
//   region  shared-memory probe of window 0                 k_st_region
//   rest    deferred keys through the COPS kernels          single.cu (n_dev, out_idx)
//   lookup only: results back to the caller's order         k_st_part<2>, k_st_final
// Each tile partition buckets a 4096-element tile in shared memory and writes
// whole (bucket, tile) runs, so every pass reads and writes coalesced.
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

// cursors: super-region starts, region starts, reverse-bin starts
__global__ void k_st_cursors(const uint64_t* __restrict__ foff, uint32_t regions, uint32_t supers,
                             uint32_t* __restrict__ cur1, uint32_t* __restrict__ cur2, uint32_t rbins, int rshift,
                             uint32_t* __restrict__ curr) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (cur2 && i < regions) cur2[i] = (uint32_t)foff[i];
  if (cur1 && i < supers) cur1[i] = (uint32_t)foff[(uint64_t)i << ST_S2];
  if (curr && i < rbins) curr[i] = i << rshift;
}

// ------------------------------------------------------------- tile partition
// MODE 0: bucket = region(a) >> ST_S2           (super-region; cursor = bucket)
// MODE 1: bucket = region(a) - base, base = the first element's super-region
//         start (the input is super-region sorted, so a tile spans <= 2 of them;
//         anything further away takes a per-element cursor); cursor = base + bucket
// MODE 2: bucket = p0 >> shift                  (position bins; cursor = bucket)
// Payload arrays p0/p1 that are null on input carry the element's position.
template <int MODE, int NP, bool FLAG>
__global__ void __launch_bounds__(PT) k_st_part(TableRef T, uint64_t n, int shift, const uint32_t* __restrict__ a_in,
                                                const uint32_t* __restrict__ p0_in,
                                                const uint32_t* __restrict__ p1_in,
                                                const uint8_t* __restrict__ f_in, uint32_t* __restrict__ a_out,
                                                uint32_t* __restrict__ p0_out, uint32_t* __restrict__ p1_out,
                                                uint8_t* __restrict__ f_out, uint32_t* __restrict__ cursor) {
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* sA = reinterpret_cast<uint32_t*>(smem);
  uint32_t* sP0 = sA + PTILE;
  uint32_t* sP1 = sP0 + (NP >= 1 ? PTILE : 0);
  uint16_t* sD = reinterpret_cast<uint16_t*>(sP1 + (NP >= 2 ? PTILE : 0));
  uint8_t* sF = reinterpret_cast<uint8_t*>(sD + PTILE);
  __shared__ uint32_t hist[PBINS], boff[PBINS], gbase[PBINS];
  __shared__ uint32_t s_base;
  __shared__ uint32_t warp_tot[PT / 32];

  const uint64_t base = (uint64_t)blockIdx.x * PTILE;
  const uint32_t cnt = (uint32_t)((n - base) < PTILE ? (n - base) : PTILE);
  for (uint32_t b = threadIdx.x; b < PBINS; b += PT) hist[b] = 0;
  if (MODE == 1 && threadIdx.x == 0) s_base = (region_of_key(T, a_in[base]) >> ST_S2) << ST_S2;

  uint32_t a[PI], p0[PI], p1[PI], d[PI], r[PI];
  uint8_t fl[PI];
#pragma unroll
  for (int it = 0; it < PI; ++it) {  // all loads in flight before any use
    const uint32_t li = (uint32_t)it * PT + threadIdx.x;
    const bool ok = li < cnt;
    const uint64_t gi = base + li;
    a[it] = ok ? __ldcs(a_in + gi) : 0u;
    if (NP >= 1) p0[it] = ok ? (p0_in ? __ldcs(p0_in + gi) : (uint32_t)gi) : 0u;
    if (NP >= 2) p1[it] = ok ? (p1_in ? __ldcs(p1_in + gi) : (uint32_t)gi) : 0u;
    if (FLAG) fl[it] = ok ? __ldcs(f_in + gi) : (uint8_t)0;
  }
  __syncthreads();  // hist zeroed, s_base set
  const uint32_t sb = MODE == 1 ? s_base : 0u;
#pragma unroll
  for (int it = 0; it < PI; ++it) {
    const uint32_t li = (uint32_t)it * PT + threadIdx.x;
    r[it] = 0xFFFFFFFFu;
    if (li >= cnt) continue;
    if (MODE == 0) d[it] = region_of_key(T, a[it]) >> ST_S2;
    else if (MODE == 1) d[it] = region_of_key(T, a[it]) - sb;
    else d[it] = p0[it] >> shift;
    if (d[it] < PBINS) {
      r[it] = atomicAdd(&hist[d[it]], 1u);
    } else {  // far bucket (MODE 1, skewed batches): element-wise cursor
      const uint32_t dst = atomicAdd(&cursor[sb + d[it]], 1u);
      a_out[dst] = a[it];
      if (NP >= 1) p0_out[dst] = p0[it];
      if (NP >= 2) p1_out[dst] = p1[it];
      if (FLAG) f_out[dst] = fl[it];
    }
  }
  __syncthreads();
  // exclusive scan of the PBINS (== PT) bucket counts; claim global runs
  {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t v = hist[threadIdx.x];
    uint32_t x = v;
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, dd);
      if (lane >= dd) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    uint32_t before = 0;
    for (int w = 0; w < warp; ++w) before += warp_tot[w];
    boff[threadIdx.x] = before + x - v;
    gbase[threadIdx.x] = v ? atomicAdd(&cursor[sb + threadIdx.x], v) : 0u;
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < PI; ++it) {
    if (r[it] == 0xFFFFFFFFu) continue;
    const uint32_t j = boff[d[it]] + r[it];
    sA[j] = a[it];
    if (NP >= 1) sP0[j] = p0[it];
    if (NP >= 2) sP1[j] = p1[it];
    if (FLAG) sF[j] = fl[it];
    sD[j] = (uint16_t)d[it];
  }
  __syncthreads();
  const uint32_t placed = boff[PBINS - 1] + hist[PBINS - 1];
  for (uint32_t j = threadIdx.x; j < placed; j += PT) {
    const uint32_t b = sD[j];
    const uint32_t dst = gbase[b] + (j - boff[b]);
    a_out[dst] = sA[j];
    if (NP >= 1) p0_out[dst] = sP0[j];
    if (NP >= 2) p1_out[dst] = sP1[j];
    if (FLAG) f_out[dst] = sF[j];
  }
}

// ------------------------------------------------------------- region pass
// Keys that window 0 cannot decide are buffered in shared memory and appended to
// the device-counted list a few hundred at a time (one global atomic per flush:
// a per-warp atomic on one counter serialised the whole pass).
constexpr uint32_t DBUF_I = 512;      // deferred entries buffered per CTA (insert)
constexpr uint32_t DBUF_L = 256;      // (lookup: 3 CTAs / SM must fit)
constexpr uint32_t SEG_I = 2048;      // insert: keys staged per segment
constexpr uint32_t SEG_L = 1024;      // lookup: keys staged per segment
constexpr uint32_t NBKT = ST_R / 32;  // insert: 32-slot buckets, one per thread
constexpr uint32_t TILE_PAD = 8;      // grouped loads may read up to 3 slots past a window
static_assert(NBKT == (uint32_t)RT, "one bucket per thread");

template <bool VALS, uint32_t DBUF>
struct DeferBuf {
  uint32_t k[DBUF];
  uint32_t v[VALS ? DBUF : 1];
  uint32_t x[DBUF];
  uint8_t o[DBUF];
  uint32_t n;
  unsigned long long gb;
};

struct DeferOut {
  uint32_t *k, *v, *x;
  uint8_t* o;
  unsigned long long* count;
};

template <bool VALS, uint32_t DBUF>
__device__ __forceinline__ void defer_push(DeferBuf<VALS, DBUF>& B, const DeferOut& D, uint32_t k, uint32_t v, uint32_t x,
                                           uint32_t o) {
  const uint32_t s = atomicAdd(&B.n, 1u);
  if (s < DBUF) {
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
template <bool VALS, uint32_t DBUF>
__device__ __forceinline__ void defer_flush(DeferBuf<VALS, DBUF>& B, const DeferOut& D, bool force) {
  __syncthreads();
  const uint32_t dn = B.n < DBUF ? B.n : DBUF;
  __syncthreads();  // everyone has read B.n
  if (!(dn >= DBUF / 2 || (force && dn))) return;
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

// Region CTA prologue: stage slots [rbase, rbase+len) (+ halo) with one TMA bulk copy.
__device__ __forceinline__ void region_load(uint64_t* tile, uint64_t* bar, const TableRef& T, uint64_t rbase,
                                            uint32_t len, uint32_t halo) {
  if (threadIdx.x == 0) {
    const uint64_t* slots = static_cast<const uint64_t*>(T.slots);
    mbar_init(bar, 1);
    mbar_expect_tx(bar, (len + halo) * 8u);
    bulk_load(tile, slots + rbase, len * 8u, bar);
    if (halo) {  // window 0 of the region's last keys runs into the next region (or wraps)
      const uint64_t hb = rbase + len < T.c ? rbase + len : 0;
      bulk_load(tile + len, slots + hb, halo * 8u, bar);
    }
  }
}

// One probe step: examine the 4 slots [lo+o, lo+o+4) of window 0 (independent
// shared-memory loads) and return the offset of the first decisive slot -- the
// key, or a free (empty / tombstone) cell -- or 4 if none (slots past the window
// end never count).  *wd receives that slot's word.
__device__ __forceinline__ uint32_t probe4(const uint64_t* tile, uint32_t lo, uint32_t o, uint32_t k, uint32_t e,
                                           uint32_t t, uint64_t* wd) {
  uint64_t w[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) w[u] = lds64(tile + lo + o + u);
  uint32_t dec = 0;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const uint32_t c = (uint32_t)w[u];
    dec |= (uint32_t)((c == k) | (c == e) | (c == t)) << u;
  }
  const uint32_t room = WINDOW - o;
  if (room < 4) dec &= (1u << room) - 1u;
  const uint32_t u = dec ? (uint32_t)__ffs(dec) - 1u : 4u;
  uint64_t x = w[3];
  x = u == 2 ? w[2] : x;
  x = u == 1 ? w[1] : x;
  x = u == 0 ? w[0] : x;
  *wd = x;
  return u;
}

// Insert.  Status is pre-set to INSERTED; exceptions are written at the key's
// input position.  A segment of keys is bucketed by the 16-slot block of its
// window start; threads take blocks from a scrambled queue and insert each
// block's keys in turn, one 4-slot probe step per loop iteration (a thread that
// resolves a key starts its next one, a thread whose blocks run out takes
// another), so concurrent claims rarely meet (only across block edges: CAS) and
// warps never wait on one long probe.  One thread per key racing at load 0.95
// cost ~7 CAS and ~26 warp-instructions per key (profiles/r01_region_v1).
constexpr uint32_t NBK = 512;                 // 16-slot blocks per region
constexpr uint32_t BK_SHIFT = 4;
static_assert((ST_R >> BK_SHIFT) == NBK, "blocks per region");

__global__ void __launch_bounds__(RT, 2) k_st_insert(TableRef T, const uint64_t* __restrict__ foff,
                                                     const uint32_t* __restrict__ keys,
                                                     const uint32_t* __restrict__ vals,
                                                     const uint32_t* __restrict__ idx, uint8_t* __restrict__ status,
                                                     DeferOut D, int g) {
  extern __shared__ __align__(128) unsigned char dsm[];
  uint64_t* tile = reinterpret_cast<uint64_t*>(dsm);
  uint32_t* s_key = reinterpret_cast<uint32_t*>(tile + ST_R + TILE_PAD);
  uint32_t* s_val = s_key + SEG_I;
  uint16_t* s_lo = reinterpret_cast<uint16_t*>(s_val + SEG_I);
  uint16_t* s_ord = s_lo + SEG_I;
  __shared__ DeferBuf<true, DBUF_I> B;
  __shared__ uint32_t s_cnt[NBK], s_off[NBK];
  __shared__ uint32_t s_next;
  __shared__ __align__(8) uint64_t bar;
  __shared__ int dirty;
  const uint32_t f = blockIdx.x;
  const uint64_t k0 = foff[f], k1 = foff[f + 1];
  if (k0 == k1) return;  // no key starts in this region
  const uint64_t rbase = (uint64_t)f << ST_LOG_R;
  const uint32_t len = (uint32_t)((T.c - rbase) < ST_R ? (T.c - rbase) : ST_R);
  region_load(tile, &bar, T, rbase, len, 0);
  if (threadIdx.x == 0) {
    dirty = 0;
    B.n = 0;
  }
  const uint32_t e = (uint32_t)T.e, t = (uint32_t)T.t;
  const uint32_t ug = (uint32_t)g;
  long long ops = 0, att = 0, win = 0, occ = 0, ndef = 0;
  bool claimed_any = false, waited = false;

  for (uint64_t s0 = k0; s0 < k1; s0 += SEG_I) {
    const uint32_t m = (uint32_t)((k1 - s0) < SEG_I ? (k1 - s0) : SEG_I);
    for (uint32_t b = threadIdx.x; b < NBK; b += RT) s_cnt[b] = 0;
    if (threadIdx.x == 0) s_next = 0;
    __syncthreads();
    // A: stage keys / values, hash, count per block
    constexpr int PER = SEG_I / RT;
    uint32_t kk[PER], vv[PER];
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const uint32_t i = (uint32_t)r * RT + threadIdx.x;
      kk[r] = i < m ? __ldcs(keys + s0 + i) : e;
      vv[r] = i < m ? __ldcs(vals + s0 + i) : 0u;
    }
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const uint32_t i = (uint32_t)r * RT + threadIdx.x;
      if (i >= m) continue;
      const uint32_t k = kk[r];
      s_key[i] = k;
      s_val[i] = vv[r];
      uint16_t lo16 = 0xFFFF;
      if (k == e || k == t) {  // INVALID_KEY, no accounting (single_table.py:369-370)
        status[idx[s0 + i]] = ST_INVALID;
      } else {
        const uint32_t lo = (uint32_t)(T.modc.mod(mix64((uint64_t)k)) - rbase);
        if (lo + WINDOW > len) {  // window 0 leaves the staged region: whole probe in the COPS kernel
          defer_push(B, D, k, vv[r], idx[s0 + i], 0);
          ndef += 1;
        } else {
          lo16 = (uint16_t)lo;
          atomicAdd(&s_cnt[lo >> BK_SHIFT], 1u);
        }
      }
      s_lo[i] = lo16;
    }
    __syncthreads();
    // B: block offsets (2 blocks per thread), then the block-ordered key list
    {
      const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
      const uint32_t c0 = s_cnt[2 * threadIdx.x], c1 = s_cnt[2 * threadIdx.x + 1];
      const uint32_t v = c0 + c1;
      uint32_t x = v;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
        if (lane >= d) x += y;
      }
      __shared__ uint32_t wt[RT / 32];
      if (lane == 31) wt[warp] = x;
      __syncthreads();
      uint32_t before = 0;
      for (int w = 0; w < warp; ++w) before += wt[w];
      s_off[2 * threadIdx.x] = before + x - v;
      s_off[2 * threadIdx.x + 1] = before + x - v + c0;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const uint32_t i = (uint32_t)r * RT + threadIdx.x;
      if (i >= m) continue;
      const uint32_t lo = s_lo[i];
      if (lo == 0xFFFF) continue;
      s_ord[atomicAdd(&s_off[lo >> BK_SHIFT], 1u)] = (uint16_t)i;  // s_off ends as each block's end
    }
    if (!waited) {
      mbar_wait(&bar, 0);
      waited = true;
    }
    __syncthreads();
    // C: flattened per-thread loop, one 4-slot probe step per iteration
    uint32_t q = 0, qend = 0, i = 0, k = 0, lo = 0, o = 0;
    bool active = false;
    for (;;) {
      if (!active) {
        while (q == qend) {  // take the next block (scrambled order: neighbours are far apart in time)
          const uint32_t bq = atomicAdd(&s_next, 1u);
          if (bq >= NBK) break;
          const uint32_t bb = (bq * 167u) & (NBK - 1);
          qend = s_off[bb];
          q = qend - s_cnt[bb];
        }
        if (q == qend) break;
        i = s_ord[q++];
        k = s_key[i];
        lo = s_lo[i];
        o = 0;
        active = true;
      }
      uint64_t wd;
      const uint32_t u = probe4(tile, lo, o, k, e, t, &wd);
      if (u == 4) {
        o += 4;
        if (o < WINDOW) continue;
        defer_push(B, D, k, s_val[i], idx[s0 + i], WINDOW);  // window 0 full: resume at window 1
        ndef += 1;
        active = false;
        continue;
      }
      o += u;
      const uint32_t c = (uint32_t)wd;
      if (c == k) {  // present before the first free cell: duplicate (single_table.py:198-200)
        status[idx[s0 + i]] = ST_DUPLICATE;
      } else if (c == t) {  // tombstone first: the deferred-claim rule (:201-223) in the COPS kernel
        defer_push(B, D, k, s_val[i], idx[s0 + i], 0);
        ndef += 1;
        active = false;
        continue;
      } else {
        const unsigned long long want = ((unsigned long long)s_val[i] << 32) | k;
        const unsigned long long old = atomicCAS((unsigned long long*)(tile + lo + o), (unsigned long long)wd, want);
        if (old != wd) {  // a neighbour's claim: re-read from this slot (single_table.py:232-233)
          att += ug;
          continue;
        }
        occ += 1;
        claimed_any = true;
      }
      ops += 1;
      att += (long long)chunk_end(o, ug);
      win += 1;
      active = false;
    }
    defer_flush(B, D, s0 + SEG_I >= k1);  // syncs: the segment buffers are free again
  }
  if (claimed_any) dirty = 1;
  fence_smem_to_async();
  __syncthreads();
  if (threadIdx.x == 0 && dirty) bulk_store_wait(static_cast<uint64_t*>(T.slots) + rbase, tile, len * 8u);
  const long long v[6] = {ops, att, win, occ, 0, ndef};
  long long* const dst[6] = {(long long*)&T.ctr->ops, (long long*)&T.ctr->attempts, (long long*)&T.ctr->windows,
                             &T.ctr->occupied, nullptr, (long long*)&T.ctr->deferred};
  cta_add<6>(v, dst);
}

// Lookup: value / found written at the region-ordered position.  Same
// flattened loop, keys taken in segment order (reads never conflict).
__global__ void __launch_bounds__(RT, 3) k_st_lookup(TableRef T, const uint64_t* __restrict__ foff,
                                                     const uint32_t* __restrict__ keys, uint32_t* __restrict__ res_val,
                                                     uint8_t* __restrict__ res_flag, DeferOut D, int g) {
  extern __shared__ __align__(128) unsigned char dsm[];
  uint64_t* tile = reinterpret_cast<uint64_t*>(dsm);
  uint32_t* s_key = reinterpret_cast<uint32_t*>(tile + ST_R + ST_HALO + TILE_PAD);
  __shared__ DeferBuf<false, DBUF_L> B;
  __shared__ __align__(8) uint64_t bar;
  const uint32_t f = blockIdx.x;
  const uint64_t k0 = foff[f], k1 = foff[f + 1];
  if (k0 == k1) return;
  const uint64_t rbase = (uint64_t)f << ST_LOG_R;
  const uint32_t len = (uint32_t)((T.c - rbase) < ST_R ? (T.c - rbase) : ST_R);
  region_load(tile, &bar, T, rbase, len, ST_HALO);
  if (threadIdx.x == 0) B.n = 0;
  const uint32_t e = (uint32_t)T.e, t = (uint32_t)T.t;
  const uint32_t ug = (uint32_t)g;
  long long ops = 0, att = 0, win = 0, ndef = 0;
  bool waited = false;
  for (uint64_t s0 = k0; s0 < k1; s0 += SEG_L) {
    const uint32_t m = (uint32_t)((k1 - s0) < SEG_L ? (k1 - s0) : SEG_L);
    constexpr int PER = SEG_L / RT;
    uint32_t kk[PER];
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const uint32_t ii = (uint32_t)r * RT + threadIdx.x;
      kk[r] = ii < m ? __ldcs(keys + s0 + ii) : e;
    }
#pragma unroll
    for (int r = 0; r < PER; ++r) s_key[(uint32_t)r * RT + threadIdx.x] = kk[r];
    if (!waited) {
      mbar_wait(&bar, 0);
      waited = true;
    }
    __syncthreads();
    uint32_t i = threadIdx.x, k = 0, lo = 0, o = 0;
    bool active = false;
    for (;;) {
      if (!active) {
        for (; i < m; i += RT) {
          k = s_key[i];
          if (k != e && k != t) break;
          res_val[s0 + i] = 0;  // a sentinel is never stored: absent, counted (single_table.py:391-393, 403)
          res_flag[s0 + i] = 0;
          ops += 1;
        }
        if (i >= m) break;
        lo = (uint32_t)(T.modc.mod(mix64((uint64_t)k)) - rbase);
        o = 0;
        active = true;
      }
      uint64_t wd;
      uint64_t w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) w[u] = tile[lo + o + u];
      uint32_t dec = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t c = (uint32_t)w[u];
        dec |= (uint32_t)((c == k) | (c == e)) << u;  // tombstones do not stop a lookup
      }
      const uint32_t room = WINDOW - o;
      if (room < 4) dec &= (1u << room) - 1u;
      if (!dec) {
        o += 4;
        if (o < WINDOW) continue;
        defer_push(B, D, k, 0u, (uint32_t)(s0 + i), WINDOW);  // window 0 decided nothing: resume at window 1
        ndef += 1;
        active = false;
        i += RT;
        continue;
      }
      const uint32_t u = (uint32_t)__ffs(dec) - 1u;
      wd = w[3];
      wd = u == 2 ? w[2] : wd;
      wd = u == 1 ? w[1] : wd;
      wd = u == 0 ? w[0] : wd;
      o += u;
      const bool hit = (uint32_t)wd == k;
      res_val[s0 + i] = hit ? (uint32_t)(wd >> 32) : 0u;
      res_flag[s0 + i] = (uint8_t)hit;
      ops += 1;
      att += (long long)chunk_end(o, ug);
      win += 1;
      active = false;
      i += RT;
    }
    defer_flush(B, D, s0 + SEG_L >= k1);
  }
  const long long v[4] = {ops, att, win, ndef};
  long long* const dst[4] = {(long long*)&T.ctr->ops, (long long*)&T.ctr->attempts, (long long*)&T.ctr->windows,
                             (long long*)&T.ctr->deferred};
  cta_add<4>(v, dst);
}

// out[p0[j]] = a[j] (and the flags): the last step back to the caller's order.
// Blocks run in index order, so the bins in flight (2^rshift positions each)
// stay L2-resident and every output line is written back once.
__global__ void __launch_bounds__(256) k_st_final(uint64_t n, const uint32_t* __restrict__ a,
                                                  const uint32_t* __restrict__ pos, const uint8_t* __restrict__ fl,
                                                  uint32_t* __restrict__ out_a, uint8_t* __restrict__ out_f) {
  const uint64_t base = (uint64_t)blockIdx.x * 2048;
#pragma unroll
  for (int it = 0; it < 8; ++it) {
    const uint64_t j = base + (uint64_t)it * 256 + threadIdx.x;
    if (j < n) {
      const uint32_t p = __ldcs(pos + j);
      out_a[p] = __ldcs(a + j);
      out_f[p] = __ldcs(fl + j);
    }
  }
}

// ------------------------------------------------------------- host side
struct StPlan {
  uint32_t regions, supers, rbins;
  int rshift;
};

static StPlan st_plan(const TableRef& T, uint64_t n) {
  StPlan p;
  p.regions = (uint32_t)((T.c + ST_R - 1) >> ST_LOG_R);
  p.supers = (p.regions + (1u << ST_S2) - 1) >> ST_S2;
  p.rshift = 0;
  while (((n + (1ull << p.rshift) - 1) >> p.rshift) > PBINS) ++p.rshift;
  p.rbins = (uint32_t)((n + (1ull << p.rshift) - 1) >> p.rshift);
  return p;
}

bool staged_supported(const TableRef& T, uint64_t n) {
  const uint64_t regions = (T.c + ST_R - 1) >> ST_LOG_R;
  return n > 0 && n < (1ull << 32) && regions <= ST_MAX_REGIONS && T.c < (1ull << 32);
}

// scratch: counts | offsets | scan | cursors | dcount | 6 element arrays (u32)
struct StBufs {
  uint32_t* gcount;
  uint64_t* foff;
  void* scan;
  size_t scan_bytes;
  uint32_t *cur1, *cur2, *curr;
  unsigned long long* dcount;
  uint32_t* arr[7];
};

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

size_t staged_scratch_bytes(const TableRef& T, uint64_t n) {
  const StPlan p = st_plan(T, n);
  size_t b = align_up(p.regions * 4ull) + align_up((p.regions + 1ull) * 8) +
             align_up(exclusive_scan_scratch_bytes(p.regions)) + align_up(PBINS * 4ull) +
             align_up(p.regions * 4ull) + align_up(PBINS * 4ull) + align_up(64);
  b += 7 * align_up(n * 4ull);
  return b;
}

static StBufs st_bufs(const StPlan& p, uint64_t n, void* scratch) {
  StBufs b;
  char* q = static_cast<char*>(scratch);
  auto take = [&](size_t bytes) {
    char* r = q;
    q += align_up(bytes);
    return (void*)r;
  };
  b.gcount = (uint32_t*)take(p.regions * 4ull);
  b.foff = (uint64_t*)take((p.regions + 1ull) * 8);
  b.scan_bytes = align_up(exclusive_scan_scratch_bytes(p.regions));
  b.scan = take(b.scan_bytes);
  b.cur1 = (uint32_t*)take(PBINS * 4ull);
  b.cur2 = (uint32_t*)take(p.regions * 4ull);
  b.curr = (uint32_t*)take(PBINS * 4ull);
  b.dcount = (unsigned long long*)take(64);
  for (int i = 0; i < 7; ++i) b.arr[i] = (uint32_t*)take(n * 4ull);
  return b;
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

// count + scan + L1 + L2: keys (and vals) into region order with their positions
static int st_forward(const Launch& lc, const TableRef& T, const StPlan& p, const StBufs& b, const uint32_t* keys,
                      const uint32_t* vals, uint64_t n, uint32_t* k2, uint32_t* v2, uint32_t* x2, uint32_t* k1,
                      uint32_t* v1, uint32_t* x1) {
  int rc = cuda_check(cudaMemsetAsync(b.gcount, 0, p.regions * 4ull, lc.stream), "memset");
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
  const uint32_t cmax = p.regions > PBINS ? p.regions : PBINS;
  k_st_cursors<<<(cmax + 255) / 256, 256, 0, lc.stream>>>(b.foff, p.regions, p.supers, b.cur1, b.cur2, 0, 0,
                                                          nullptr);
  count_launch();
  const unsigned tiles = (unsigned)((n + PTILE - 1) / PTILE);
  if (vals) {
    const size_t sm = (size_t)PTILE * (4 + 4 + 4 + 2);
    if ((rc = st_smem(k_st_part<0, 2, false>, sm)) || (rc = st_smem(k_st_part<1, 2, false>, sm))) return rc;
    k_st_part<0, 2, false><<<tiles, PT, sm, lc.stream>>>(T, n, 0, keys, vals, nullptr, nullptr, k1, v1, x1, nullptr,
                                                          b.cur1);
    count_launch();
    k_st_part<1, 2, false><<<tiles, PT, sm, lc.stream>>>(T, n, 0, k1, v1, x1, nullptr, k2, v2, x2, nullptr, b.cur2);
    count_launch();
  } else {
    const size_t sm = (size_t)PTILE * (4 + 4 + 2);
    if ((rc = st_smem(k_st_part<0, 1, false>, sm)) || (rc = st_smem(k_st_part<1, 1, false>, sm))) return rc;
    k_st_part<0, 1, false><<<tiles, PT, sm, lc.stream>>>(T, n, 0, keys, nullptr, nullptr, nullptr, k1, x1, nullptr,
                                                          nullptr, b.cur1);
    count_launch();
    k_st_part<1, 1, false><<<tiles, PT, sm, lc.stream>>>(T, n, 0, k1, x1, nullptr, nullptr, k2, x2, nullptr, nullptr,
                                                          b.cur2);
    count_launch();
  }
  return cuda_check(cudaGetLastError(), "staged partition");
}

int staged_insert(const Launch& lc, const TableRef& T, const TypeSel& ts, const void* keys, const void* vals,
                  uint64_t n, uint8_t* status, void* scratch) {
  const StPlan p = st_plan(T, n);
  const StBufs b = st_bufs(p, n, scratch);
  uint32_t *k1 = b.arr[0], *v1 = b.arr[1], *x1 = b.arr[2], *k2 = b.arr[3], *v2 = b.arr[4], *x2 = b.arr[5];
  int rc = cuda_check(cudaMemsetAsync(status, ST_INSERTED, n, lc.stream), "memset");
  if (!rc) rc = cuda_check(cudaMemsetAsync(b.dcount, 0, 8, lc.stream), "memset");
  if (!rc) rc = st_forward(lc, T, p, b, (const uint32_t*)keys, (const uint32_t*)vals, n, k2, v2, x2, k1, v1, x1);
  if (rc) return rc;
  const size_t sm = (size_t)(ST_R + TILE_PAD) * 8 + SEG_I * (4 + 4 + 2 + 2);
  if ((rc = st_smem(k_st_insert, sm))) return rc;
  cudaEvent_t e0;
  st_timed(lc, &e0);
  // the deferred list reuses the L1 arrays
  uint8_t* dO = (uint8_t*)b.arr[6];
  const DeferOut D{k1, v1, x1, dO, b.dcount};
  k_st_insert<<<p.regions, RT, sm, lc.stream>>>(T, b.foff, k2, v2, x2, status, D, ts.g);
  count_launch();
  st_timed_end(lc, e0);
  if ((rc = cuda_check(cudaGetLastError(), "staged region insert"))) return rc;
  Launch rest = lc;
  rest.timer = nullptr;
  rest.n_dev = b.dcount;
  rest.out_idx = x1;
  rest.o_start = dO;
  return single_insert(rest, T, ts, k1, v1, n, status, nullptr, 0);
}

int staged_lookup(const Launch& lc, const TableRef& T, const TypeSel& ts, const void* keys, uint64_t n,
                  void* vals_out, uint8_t* found, void* scratch) {
  const StPlan p = st_plan(T, n);
  const StBufs b = st_bufs(p, n, scratch);
  uint32_t *k1 = b.arr[0], *x1 = b.arr[1], *k2 = b.arr[2], *x2 = b.arr[3], *rv = b.arr[4];
  uint8_t* rf = (uint8_t*)b.arr[5];
  int rc = cuda_check(cudaMemsetAsync(b.dcount, 0, 8, lc.stream), "memset");
  if (!rc) rc = st_forward(lc, T, p, b, (const uint32_t*)keys, nullptr, n, k2, nullptr, x2, k1, nullptr, x1);
  if (rc) return rc;
  const size_t sm = (size_t)(ST_R + ST_HALO + TILE_PAD) * 8 + SEG_L * 4;
  if ((rc = st_smem(k_st_lookup, sm))) return rc;
  cudaEvent_t e0;
  st_timed(lc, &e0);
  uint8_t* dO = (uint8_t*)b.arr[6];
  const DeferOut D{k1, nullptr, x1, dO, b.dcount};
  k_st_lookup<<<p.regions, RT, sm, lc.stream>>>(T, b.foff, k2, rv, rf, D, ts.g);
  count_launch();
  st_timed_end(lc, e0);
  if ((rc = cuda_check(cudaGetLastError(), "staged region lookup"))) return rc;
  Launch rest = lc;
  rest.timer = nullptr;
  rest.n_dev = b.dcount;
  rest.out_idx = x1;
  rest.o_start = dO;
  if ((rc = single_lookup(rest, T, ts, k1, n, rv, rf, nullptr, nullptr, nullptr, 0))) return rc;
  // back to the caller's order: bin by position (k_st_part<2>), then scatter
  // inside L2-resident bins (k_st_final).  k1/x1 and k2 are free again.
  k_st_cursors<<<(PBINS + 255) / 256, 256, 0, lc.stream>>>(b.foff, 0, 0, nullptr, nullptr, p.rbins, p.rshift, b.curr);
  count_launch();
  const size_t psm = (size_t)PTILE * (4 + 4 + 2 + 1);
  if ((rc = st_smem(k_st_part<2, 1, true>, psm))) return rc;
  const unsigned tiles = (unsigned)((n + PTILE - 1) / PTILE);
  uint8_t* rf1 = (uint8_t*)k2;
  k_st_part<2, 1, true><<<tiles, PT, psm, lc.stream>>>(T, n, p.rshift, rv, x2, nullptr, rf, k1, x1, nullptr, rf1,
                                                        b.curr);
  count_launch();
  k_st_final<<<(unsigned)((n + 2047) / 2048), 256, 0, lc.stream>>>(n, k1, x1, rf1, (uint32_t*)vals_out, found);
  count_launch();
  return cuda_check(cudaGetLastError(), "staged unpermute");
}

}  // namespace chb
