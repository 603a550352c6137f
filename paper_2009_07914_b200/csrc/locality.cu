// locality.cu -- region-ordered execution of big bulk operations.
//
// Measured on B200 (profiles/r01_*): a random 64 B probe costs a 128 B L2 line
// fill from HBM, so a probe-per-key kernel over a 2 GiB table reads ~240-290 B
// of DRAM per op.  For a batch that covers the table (n >= c/16), we instead:
//   1. bucket the keys by the super-region their first window starts in
//      (h >> shift, regions of ~8 MiB)            k_loc_count, scan, k_loc_scatter
//   2. run the unchanged probe kernels on the region-ordered batch; their
//      chunked scheduler (sched.cuh) keeps the elements in flight inside one or
//      two regions, which stay L2-resident: each table line is read from (and
//      written back to) HBM about once per batch
//   3. return the per-key results to the caller's order       k_loc_unpermute
// Passes 1 and 3 are streaming.  A tile of LOC_TILE consecutive elements is
// bucketed in shared memory first, so both directions move whole runs per
// (region, tile) with coalesced accesses instead of one scattered 4 B access
// per element.  Semantics are those of the direct kernels (a concurrent batch);
// only the schedule changes.
#include "dispatch.cuh"

namespace chb {

constexpr int LOC_THREADS = 256;
constexpr int LOC_ITEMS = 16;
constexpr uint32_t LOC_TILE = (uint32_t)LOC_THREADS * LOC_ITEMS;
constexpr uint32_t LOC_MAX_REGIONS = 1024;

template <typename K>
__device__ __forceinline__ uint32_t region_of(const TableRef& T, K key, int shift) {
  return (uint32_t)(T.modc.mod_any(mix64((uint64_t)key)) >> shift);
}

// hist[r * tiles + tile] = keys of the tile whose first window starts in region r
template <typename K>
__global__ void __launch_bounds__(LOC_THREADS) k_loc_count(TableRef T, const K* __restrict__ keys, uint64_t n,
                                                          int shift, uint32_t regions, uint32_t* __restrict__ hist) {
  __shared__ uint32_t cnt[LOC_MAX_REGIONS];
  for (uint32_t r = threadIdx.x; r < regions; r += LOC_THREADS) cnt[r] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * LOC_TILE;
  K k[LOC_ITEMS];
#pragma unroll
  for (int it = 0; it < LOC_ITEMS; ++it) {  // all loads in flight before any use
    const uint64_t i = base + (uint64_t)it * LOC_THREADS + threadIdx.x;
    k[it] = i < n ? keys[i] : K{};
  }
#pragma unroll
  for (int it = 0; it < LOC_ITEMS; ++it) {
    const uint64_t i = base + (uint64_t)it * LOC_THREADS + threadIdx.x;
    if (i < n) atomicAdd(&cnt[region_of(T, k[it], shift)], 1u);
  }
  __syncthreads();
  for (uint32_t r = threadIdx.x; r < regions; r += LOC_THREADS) hist[(uint64_t)r * gridDim.x + blockIdx.x] = cnt[r];
}

// Exclusive scan of this tile's per-region counts into loff[] (block-wide).
__device__ __forceinline__ void tile_region_offsets(const uint32_t* __restrict__ hist, uint32_t regions,
                                                    uint32_t* cnt, uint32_t* loff) {
  __shared__ uint32_t warp_tot[LOC_THREADS / 32];
  constexpr int PER = LOC_MAX_REGIONS / LOC_THREADS;
  uint32_t v[PER];
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const uint32_t r = threadIdx.x * PER + k;
    v[k] = r < regions ? hist[(uint64_t)r * gridDim.x + blockIdx.x] : 0;
    s += v[k];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = s;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  uint32_t before = 0;
  for (int w = 0; w < warp; ++w) before += warp_tot[w];
  uint32_t run = before + x - s;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const uint32_t r = threadIdx.x * PER + k;
    if (r < regions) {
      loff[r] = run;
      cnt[r] = v[k];
    }
    run += v[k];
  }
}

// Bucket a tile in shared memory, then write each (region, tile) run with
// consecutive threads.  inv[i] = the element's position inside its tile's
// region-sorted order (what k_loc_unpermute reads back).
template <typename K, typename V>
__global__ void __launch_bounds__(LOC_THREADS) k_loc_scatter(TableRef T, const K* __restrict__ keys,
                                                            const V* __restrict__ vals, uint64_t n, int shift,
                                                            uint32_t regions, const uint32_t* __restrict__ hist,
                                                            const uint64_t* __restrict__ hist_off,
                                                            K* __restrict__ keys_out, V* __restrict__ vals_out,
                                                            uint16_t* __restrict__ inv) {
  extern __shared__ __align__(16) unsigned char smem[];
  K* s_keys = reinterpret_cast<K*>(smem);
  V* s_vals = reinterpret_cast<V*>(s_keys + LOC_TILE);
  uint16_t* s_reg = reinterpret_cast<uint16_t*>(s_vals + LOC_TILE);
  __shared__ uint32_t cnt[LOC_MAX_REGIONS], loff[LOC_MAX_REGIONS], fill[LOC_MAX_REGIONS];
  tile_region_offsets(hist, regions, cnt, loff);
  for (uint32_t r = threadIdx.x; r < regions; r += LOC_THREADS) fill[r] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * LOC_TILE;
  const uint32_t valid = (uint32_t)((n - base) < LOC_TILE ? (n - base) : LOC_TILE);
  K k[LOC_ITEMS];
  V v[LOC_ITEMS];
#pragma unroll
  for (int it = 0; it < LOC_ITEMS; ++it) {  // all loads in flight before any use
    const uint32_t li = (uint32_t)it * LOC_THREADS + threadIdx.x;
    k[it] = li < valid ? keys[base + li] : K{};
    if (vals) v[it] = li < valid ? vals[base + li] : V{};
  }
#pragma unroll
  for (int it = 0; it < LOC_ITEMS; ++it) {
    const uint32_t li = (uint32_t)it * LOC_THREADS + threadIdx.x;
    if (li < valid) {
      const uint32_t r = region_of(T, k[it], shift);
      const uint32_t j = loff[r] + atomicAdd(&fill[r], 1u);
      s_keys[j] = k[it];
      if (vals) s_vals[j] = v[it];
      s_reg[j] = (uint16_t)r;
      inv[base + li] = (uint16_t)j;
    }
  }
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < valid; j += LOC_THREADS) {
    const uint32_t r = s_reg[j];
    const uint64_t pos = hist_off[(uint64_t)r * gridDim.x + blockIdx.x] + (j - loff[r]);
    keys_out[pos] = s_keys[j];
    if (vals) vals_out[pos] = s_vals[j];
  }
}

// Reverse: load the tile's runs (one warp per run, coalesced) into shared
// memory in region order, then emit the results in the caller's order.
template <typename A, typename B>
__global__ void __launch_bounds__(LOC_THREADS) k_loc_unpermute(uint64_t n, uint32_t regions,
                                                              const uint32_t* __restrict__ hist,
                                                              const uint64_t* __restrict__ hist_off,
                                                              const uint16_t* __restrict__ inv,
                                                              const A* __restrict__ pa, A* __restrict__ oa,
                                                              const B* __restrict__ pb, B* __restrict__ ob) {
  extern __shared__ __align__(16) unsigned char smem[];
  A* s_a = reinterpret_cast<A*>(smem);
  B* s_b = reinterpret_cast<B*>(s_a + LOC_TILE);
  __shared__ uint32_t cnt[LOC_MAX_REGIONS], loff[LOC_MAX_REGIONS];
  tile_region_offsets(hist, regions, cnt, loff);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t r = warp; r < regions; r += LOC_THREADS / 32) {
    const uint32_t c = cnt[r];
    if (!c) continue;
    const uint64_t src = hist_off[(uint64_t)r * gridDim.x + blockIdx.x];
    for (uint32_t k = lane; k < c; k += 32) {
      s_a[loff[r] + k] = pa[src + k];
      if (pb) s_b[loff[r] + k] = pb[src + k];
    }
  }
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * LOC_TILE;
  const uint32_t valid = (uint32_t)((n - base) < LOC_TILE ? (n - base) : LOC_TILE);
  for (uint32_t li = threadIdx.x; li < valid; li += LOC_THREADS) {
    const uint32_t j = inv[base + li];
    oa[base + li] = s_a[j];
    if (pb) ob[base + li] = s_b[j];
  }
}

struct LocPlan {
  int shift;
  uint32_t regions;
  uint64_t tiles;
};

LocPlan loc_plan(const TableRef& T, uint64_t n, int bytes_per_slot) {
  // ~8 MiB regions: 2^shift slots x bytes_per_slot
  int shift = 0;
  while ((1ull << (shift + 1)) * (uint64_t)bytes_per_slot <= (8ull << 20)) ++shift;
  while (((T.c - 1) >> shift) + 1 > LOC_MAX_REGIONS) ++shift;
  LocPlan p;
  p.shift = shift;
  p.regions = (uint32_t)(((T.c - 1) >> shift) + 1);
  p.tiles = (n + LOC_TILE - 1) / LOC_TILE;
  return p;
}

// scratch: hist (u32) | hist_off (u64) | scan scratch; inv (u16 per element) separately
size_t loc_scratch_bytes(const LocPlan& p) {
  const uint64_t h = p.tiles * p.regions;
  return h * 4 + 16 + (h + 1) * 8 + 16 + exclusive_scan_scratch_bytes(h) + 64;
}

struct LocBufs {
  uint32_t* hist;
  uint64_t* hist_off;
  void* scan;
  size_t scan_bytes;
};

static LocBufs loc_bufs(const LocPlan& p, void* scratch, size_t scratch_bytes) {
  const uint64_t h = p.tiles * p.regions;
  LocBufs b;
  b.hist = (uint32_t*)scratch;
  b.hist_off = (uint64_t*)(((uintptr_t)(b.hist + h) + 15) & ~(uintptr_t)15);
  b.scan = (void*)(((uintptr_t)(b.hist_off + h + 1) + 15) & ~(uintptr_t)15);
  const size_t used = (size_t)((char*)b.scan - (char*)scratch);
  b.scan_bytes = used <= scratch_bytes ? scratch_bytes - used : 0;
  return b;
}

template <typename KS>
static int set_smem(KS kern, size_t bytes) {
  return cuda_check(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes), "smem attr");
}

template <typename K, typename V>
static int partition_impl(const Launch& lc, const TableRef& T, const LocPlan& p, const K* keys, const V* vals,
                          uint64_t n, K* keys_out, V* vals_out, uint16_t* inv, void* scratch, size_t scratch_bytes) {
  const uint64_t h = p.tiles * p.regions;
  const LocBufs b = loc_bufs(p, scratch, scratch_bytes);
  k_loc_count<K><<<(unsigned)p.tiles, LOC_THREADS, 0, lc.stream>>>(T, keys, n, p.shift, p.regions, b.hist);
  count_launch();
  int rc = cuda_check(cudaGetLastError(), "locality count");
  if (rc) return rc;
  rc = exclusive_scan_u32(lc, b.hist, h, b.hist_off, b.scan, b.scan_bytes);
  if (rc) return rc;
  const size_t smem = (size_t)LOC_TILE * (sizeof(K) + sizeof(V) + sizeof(uint16_t));
  rc = set_smem(k_loc_scatter<K, V>, smem);
  if (rc) return rc;
  k_loc_scatter<K, V><<<(unsigned)p.tiles, LOC_THREADS, smem, lc.stream>>>(T, keys, vals, n, p.shift, p.regions,
                                                                          b.hist, b.hist_off, keys_out, vals_out, inv);
  count_launch();
  return cuda_check(cudaGetLastError(), "locality scatter");
}

int loc_partition(const Launch& lc, const TableRef& T, const LocPlan& p, int kbytes, int vbytes, const void* keys,
                  const void* vals, uint64_t n, void* keys_out, void* vals_out, uint16_t* inv, void* scratch,
                  size_t scratch_bytes) {
#define CHB_LOC(K, V)                                                                                            \
  return partition_impl<K, V>(lc, T, p, (const K*)keys, (const V*)vals, n, (K*)keys_out, (V*)vals_out, inv, \
                              scratch, scratch_bytes);
  if (kbytes == 4 && vbytes == 4) CHB_LOC(uint32_t, uint32_t)
  if (kbytes == 4 && vbytes == 8) CHB_LOC(uint32_t, uint64_t)
  if (kbytes == 8 && vbytes == 4) CHB_LOC(uint64_t, uint32_t)
  if (kbytes == 8 && vbytes == 8) CHB_LOC(uint64_t, uint64_t)
#undef CHB_LOC
  set_error("bad key/value width");
  return -22;
}

// out_a[i] = part_a[pos(i)] (and the same for b when given), pos from the partition
int loc_unpermute(const Launch& lc, const LocPlan& p, uint64_t n, const uint16_t* inv, void* scratch,
                  size_t scratch_bytes, const void* pa, void* oa, int abytes, const void* pb, void* ob, int bbytes) {
  const LocBufs b = loc_bufs(p, scratch, scratch_bytes);
#define CHB_UNP(A, B)                                                                                          \
  {                                                                                                            \
    const size_t smem = (size_t)LOC_TILE * (sizeof(A) + sizeof(B));                                            \
    int rc = set_smem(k_loc_unpermute<A, B>, smem);                                                            \
    if (rc) return rc;                                                                                         \
    k_loc_unpermute<A, B><<<(unsigned)p.tiles, LOC_THREADS, smem, lc.stream>>>(                                \
        n, p.regions, b.hist, b.hist_off, inv, (const A*)pa, (A*)oa, (const B*)pb, (B*)ob);                   \
    count_launch();                                                                                            \
    return cuda_check(cudaGetLastError(), "locality unpermute");                                               \
  }
  if (abytes == 1) CHB_UNP(uint8_t, uint8_t)
  if (abytes == 4 && (bbytes == 1 || !pb)) CHB_UNP(uint32_t, uint8_t)
  if (abytes == 8 && (bbytes == 1 || !pb)) CHB_UNP(uint64_t, uint8_t)
#undef CHB_UNP
  set_error("bad element width");
  return -22;
}

}  // namespace chb
