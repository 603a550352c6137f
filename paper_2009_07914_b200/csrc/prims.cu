// prims.cu -- device primitives around the tables:
//   exclusive prefix sum      (multi_table.py:28-30)       reduce-then-scan, 3 passes
//   mix64 over an array       (probing.py:90-117)
//   route + stable multi-split (distributed.py:44-45,59-69) K10
//   scatter / gather / segmented copy (distributed.py:143-147,163-178,197-203) K11
#include "dispatch.cuh"

namespace chb {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 16;
constexpr uint64_t SCAN_TILE = (uint64_t)SCAN_THREADS * SCAN_ITEMS;

template <typename T>
__device__ __forceinline__ T block_exclusive_sum(T v, T* total) {
  __shared__ T warp_tot[SCAN_THREADS / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    T y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  if (warp == 0) {
    T w = lane < SCAN_THREADS / 32 ? warp_tot[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      T y = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= d) w += y;
    }
    if (lane < SCAN_THREADS / 32) warp_tot[lane] = w;  // inclusive
  }
  __syncthreads();
  const T warp_prefix = warp == 0 ? 0 : warp_tot[warp - 1];
  *total = warp_tot[SCAN_THREADS / 32 - 1];
  __syncthreads();
  return warp_prefix + x - v;
}

template <typename TIn>
__global__ void __launch_bounds__(SCAN_THREADS) k_tile_sums(const TIn* __restrict__ in, uint64_t n,
                                                           uint64_t* __restrict__ sums) {
  const uint64_t base = blockIdx.x * SCAN_TILE;
  uint64_t s = 0;
#pragma unroll 4
  for (int r = 0; r < SCAN_ITEMS; ++r) {
    const uint64_t i = base + (uint64_t)r * SCAN_THREADS + threadIdx.x;
    if (i < n) s += (uint64_t)in[i];
  }
  uint64_t tot;
  block_exclusive_sum<uint64_t>(s, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// out[i] = prefix[tile] + exclusive sum within the tile; out[n] = grand total.  The tile
// goes through shared memory both ways (coalesced loads and stores; each thread scans 16
// consecutive elements there -- a blocked layout straight from global memory put every
// lane of a warp on its own line and measured 0.89 ms for 2^27 counts)
__device__ __forceinline__ uint32_t scan_pad(uint32_t j) { return j + (j >> 4); }
template <typename TIn>
__global__ void __launch_bounds__(SCAN_THREADS) k_tile_scan(const TIn* __restrict__ in, uint64_t n,
                                                           const uint64_t* __restrict__ prefix,
                                                           uint64_t* __restrict__ out) {
  __shared__ uint64_t st[SCAN_TILE + SCAN_TILE / 16];
  const uint64_t tb = (uint64_t)blockIdx.x * SCAN_TILE;
  const uint64_t pre = prefix ? prefix[blockIdx.x] : 0;
#pragma unroll
  for (int r = 0; r < SCAN_ITEMS; ++r) {
    const uint32_t j = (uint32_t)r * SCAN_THREADS + threadIdx.x;
    const uint64_t i = tb + j;
    st[scan_pad(j)] = i < n ? (uint64_t)in[i] : 0;
  }
  __syncthreads();
  uint64_t v[SCAN_ITEMS];
  uint64_t s = 0;
#pragma unroll
  for (int r = 0; r < SCAN_ITEMS; ++r) {
    v[r] = st[scan_pad(threadIdx.x * SCAN_ITEMS + r)];
    s += v[r];
  }
  uint64_t tot;
  uint64_t run = block_exclusive_sum<uint64_t>(s, &tot) + pre;  // syncs
#pragma unroll
  for (int r = 0; r < SCAN_ITEMS; ++r) {
    const uint32_t j = threadIdx.x * SCAN_ITEMS + r;
    st[scan_pad(j)] = run;
    run += v[r];
    if (tb + j == n - 1) out[n] = run;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < SCAN_ITEMS; ++r) {
    const uint32_t j = (uint32_t)r * SCAN_THREADS + threadIdx.x;
    const uint64_t i = tb + j;
    if (i < n) out[i] = st[scan_pad(j)];
  }
}

static size_t scan_words_needed(uint64_t n) {
  size_t w = 0;
  uint64_t m = n;
  while (m > SCAN_TILE) {
    m = (m + SCAN_TILE - 1) / SCAN_TILE;
    w += 2 * (m + 1);
  }
  return w + 8;
}

size_t exclusive_scan_scratch_bytes(uint64_t n) { return scan_words_needed(n) * 8; }

template <typename TIn>
static int scan_impl(const Launch& lc, const TIn* in, uint64_t n, uint64_t* out, uint64_t* scratch,
                     size_t scratch_words) {
  if (n == 0) return cuda_check(cudaMemsetAsync(out, 0, sizeof(uint64_t), lc.stream), "scan memset");
  const uint64_t tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  if (tiles == 1) {
    k_tile_scan<TIn><<<1, SCAN_THREADS, 0, lc.stream>>>(in, n, nullptr, out);
    count_launch();
    return cuda_check(cudaGetLastError(), "scan");
  }
  if (scratch_words < tiles + 1) {
    set_error("scan scratch too small");
    return -22;
  }
  uint64_t* sums = scratch;  // tiles sums, then scanned in place into sums_scan
  uint64_t* sums_scan = scratch + 0;
  k_tile_sums<TIn><<<(unsigned)tiles, SCAN_THREADS, 0, lc.stream>>>(in, n, sums);
  count_launch();
  int rc = cuda_check(cudaGetLastError(), "scan sums");
  if (rc) return rc;
  // scan the tile sums (recursively) into the scratch area that follows them
  uint64_t* next = scratch + tiles + 1;
  rc = scan_impl<uint64_t>(lc, sums, tiles, next, next + tiles + 1, scratch_words - 2 * (tiles + 1));
  if (rc) return rc;
  (void)sums_scan;
  k_tile_scan<TIn><<<(unsigned)tiles, SCAN_THREADS, 0, lc.stream>>>(in, n, next, out);
  count_launch();
  return cuda_check(cudaGetLastError(), "scan tiles");
}

int exclusive_scan_u32(const Launch& lc, const uint32_t* counts, uint64_t n, uint64_t* out, void* scratch,
                       size_t scratch_bytes) {
  if (scratch_bytes / 8 < scan_words_needed(n)) {
    set_error("scan scratch too small");
    return -22;
  }
  return scan_impl<uint32_t>(lc, counts, n, out, (uint64_t*)scratch, scratch_bytes / 8);
}
int exclusive_scan_u64(const Launch& lc, const uint64_t* counts, uint64_t n, uint64_t* out, void* scratch,
                       size_t scratch_bytes) {
  if (scratch_bytes / 8 < scan_words_needed(n)) {
    set_error("scan scratch too small");
    return -22;
  }
  return scan_impl<uint64_t>(lc, counts, n, out, (uint64_t*)scratch, scratch_bytes / 8);
}

// ---------------------------------------------------------------- mix64
__global__ void k_mix64(const uint64_t* __restrict__ in, uint64_t n, uint64_t seed, uint64_t* __restrict__ out) {
  const uint64_t stride = gridDim.x * (uint64_t)blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = mix64(seed ^ in[i]);
}
int mix64_array(const Launch& lc, const uint64_t* in, uint64_t n, uint64_t seed, uint64_t* out) {
  return launch_persistent(lc, (const void*)k_mix64, n, 1,
                           [&](dim3 g, dim3 b) { k_mix64<<<g, b, 0, lc.stream>>>(in, n, seed, out); });
}

// ---------------------------------------------------------- multi-split
constexpr int SPLIT_THREADS = 256;
constexpr int SPLIT_ROUNDS = 8;
constexpr uint64_t SPLIT_TILE = (uint64_t)SPLIT_THREADS * SPLIT_ROUNDS;
constexpr uint32_t SPLIT_MAX_SHARDS = 256;

// key -> shard: ShardRouter.route; DEST_GIVEN: the "key" already is the destination
struct DestGiven {
  uint32_t d;
};
template <typename K>
__device__ __forceinline__ uint32_t route(K key, uint32_t shards) {
  return (uint32_t)((mix64((uint64_t)key) >> 32) % shards);  // ShardRouter.route
}
template <>
__device__ __forceinline__ uint32_t route<DestGiven>(DestGiven key, uint32_t) {
  return key.d;
}

// per-tile destination histogram, dest-major: hist[d * tiles + tile]
template <typename K>
__global__ void __launch_bounds__(SPLIT_THREADS) k_split_count(const K* __restrict__ keys, uint64_t n,
                                                              uint32_t shards, uint32_t* __restrict__ hist) {
  __shared__ uint32_t cnt[SPLIT_MAX_SHARDS];
  for (uint32_t d = threadIdx.x; d < shards; d += SPLIT_THREADS) cnt[d] = 0;
  __syncthreads();
  const uint64_t base = blockIdx.x * SPLIT_TILE;
  const unsigned lane = threadIdx.x & 31u;
  for (int r = 0; r < SPLIT_ROUNDS; ++r) {
    const uint64_t i = base + (uint64_t)r * SPLIT_THREADS + threadIdx.x;
    const uint32_t d = i < n ? route(keys[i], shards) : shards;
    // one shared atomic per destination present in the warp (few shards: 32 lanes on a
    // handful of counters serialised the pass)
    const unsigned m = __match_any_sync(0xffffffffu, d);
    if (d < shards && lane == (unsigned)(__ffs(m) - 1)) atomicAdd(&cnt[d], (uint32_t)__popc(m));
  }
  __syncthreads();
  for (uint32_t d = threadIdx.x; d < shards; d += SPLIT_THREADS) hist[(uint64_t)d * gridDim.x + blockIdx.x] = cnt[d];
}

// stable scatter: rounds in input order, ranks within a round by warp then lane
template <typename K, typename V, typename PI_T, bool INV>
__global__ void __launch_bounds__(SPLIT_THREADS) k_split_scatter(const K* __restrict__ keys,
                                                                const V* __restrict__ vals, uint64_t n,
                                                                uint32_t shards,
                                                                const uint64_t* __restrict__ hist_off,
                                                                PI_T* __restrict__ perm,
                                                                K* __restrict__ keys_out,
                                                                V* __restrict__ vals_out) {
  constexpr int NW = SPLIT_THREADS / 32;
  __shared__ uint64_t run[SPLIT_MAX_SHARDS];
  __shared__ uint32_t wcnt[NW][SPLIT_MAX_SHARDS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t d = threadIdx.x; d < shards; d += SPLIT_THREADS) {
    run[d] = hist_off[(uint64_t)d * gridDim.x + blockIdx.x];
    for (int w = 0; w < NW; ++w) wcnt[w][d] = 0;
  }
  __syncthreads();
  const uint64_t base = blockIdx.x * SPLIT_TILE;
  const unsigned lt = (1u << lane) - 1u;
  for (int r = 0; r < SPLIT_ROUNDS; ++r) {
    const uint64_t i = base + (uint64_t)r * SPLIT_THREADS + threadIdx.x;
    const bool valid = i < n;
    K key = valid ? keys[i] : K{};
    const uint32_t d = valid ? route(key, shards) : shards;  // `shards` = no destination
    const unsigned m = __match_any_sync(0xffffffffu, d);
    const uint32_t rank = __popc(m & lt);
    if (valid && rank == 0) wcnt[warp][d] = __popc(m);
    __syncthreads();
    if (valid) {
      uint64_t pos = run[d] + rank;
      for (int w = 0; w < warp; ++w) pos += wcnt[w][d];
      if (INV) perm[i] = (PI_T)pos;  // source -> split position (coalesced)
      else perm[pos] = (PI_T)i;
      if (keys_out) keys_out[pos] = key;
      if (vals_out) vals_out[pos] = vals[i];
    }
    __syncthreads();
    for (uint32_t dd = threadIdx.x; dd < shards; dd += SPLIT_THREADS) {
      uint64_t add = 0;
      for (int w = 0; w < NW; ++w) {
        add += wcnt[w][dd];
        wcnt[w][dd] = 0;
      }
      run[dd] += add;
    }
    __syncthreads();
  }
}

__global__ void k_split_offsets(const uint64_t* __restrict__ hist_off, uint32_t shards, uint64_t tiles,
                                uint64_t n, uint64_t* __restrict__ offsets) {
  for (uint32_t d = threadIdx.x; d <= shards; d += blockDim.x)
    offsets[d] = d == shards ? n : (hist_off ? hist_off[(uint64_t)d * tiles] : 0);  // n == 0: no tiles
}

size_t split_scratch_bytes(uint64_t n, uint32_t shards) {
  const uint64_t tiles = (n + SPLIT_TILE - 1) / SPLIT_TILE;
  const uint64_t h = tiles * shards;
  return h * 4 + (h + 1) * 8 + scan_words_needed(h) * 8 + 256;
}

template <typename K, typename V, typename PI_T, bool INV = false>
static int split_impl(const Launch& lc, const K* keys, const V* vals, uint64_t n, uint32_t shards,
                      PI_T* perm, uint64_t* offsets, K* keys_out, V* vals_out, void* scratch,
                      size_t scratch_bytes) {
  const uint64_t tiles = (n + SPLIT_TILE - 1) / SPLIT_TILE;
  if (n == 0) {
    k_split_offsets<<<1, 256, 0, lc.stream>>>(nullptr, shards, 0, 0, offsets);
    count_launch();
    return cuda_check(cudaGetLastError(), "split offsets");
  }
  const uint64_t h = tiles * shards;
  uint32_t* hist = (uint32_t*)scratch;
  uint64_t* hist_off = (uint64_t*)(((uintptr_t)(hist + h) + 15) & ~(uintptr_t)15);
  uint64_t* scan_scratch = hist_off + h + 1;
  const size_t used = (size_t)((char*)scan_scratch - (char*)scratch);
  if (used > scratch_bytes) {
    set_error("split scratch too small");
    return -22;
  }
  k_split_count<K><<<(unsigned)tiles, SPLIT_THREADS, 0, lc.stream>>>(keys, n, shards, hist);
  count_launch();
  int rc = cuda_check(cudaGetLastError(), "split count");
  if (rc) return rc;
  rc = exclusive_scan_u32(lc, hist, h, hist_off, scan_scratch, scratch_bytes - used);
  if (rc) return rc;
  k_split_scatter<K, V, PI_T, INV><<<(unsigned)tiles, SPLIT_THREADS, 0, lc.stream>>>(keys, vals, n, shards, hist_off, perm,
                                                                         keys_out, vals_out);
  count_launch();
  rc = cuda_check(cudaGetLastError(), "split scatter");
  if (rc) return rc;
  k_split_offsets<<<1, 256, 0, lc.stream>>>(hist_off, shards, tiles, n, offsets);
  count_launch();
  return cuda_check(cudaGetLastError(), "split offsets");
}

// One-pass route partition (ShardedTable's split, ch_route_part32): a 4096-key tile is
// bucketed by destination shard in shared memory and written as one run per shard at a
// cursor inside that shard's fixed-capacity segment [d cap, d cap + count_d) -- no count
// pass, one read of the batch.  pos[i] = the element's position (the inverse map the results
// return through).  The order inside a segment is not the input order (the table does not
// need it); a segment past its capacity raises *flag and the caller takes the stable split.
constexpr int RP_T = 512, RP_I = 8;
constexpr uint32_t RP_TILE = (uint32_t)RP_T * RP_I;
constexpr uint32_t RP_MAX_SHARDS = 64;

template <bool VALS>
__global__ void __launch_bounds__(RP_T) k_route_part(const uint32_t* __restrict__ keys,
                                                    const uint32_t* __restrict__ vals, uint64_t n, uint32_t shards,
                                                    uint64_t cap, uint32_t* __restrict__ pos,
                                                    unsigned long long* __restrict__ cnt,
                                                    uint32_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                                    int* __restrict__ flag) {
  __shared__ uint32_t sK[RP_TILE];
  __shared__ uint32_t sV[VALS ? RP_TILE : 1];
  __shared__ uint8_t sD[RP_TILE];
  __shared__ uint32_t hist[RP_MAX_SHARDS], boff[RP_MAX_SHARDS];
  __shared__ unsigned long long gb[RP_MAX_SHARDS];
  __shared__ uint8_t ovf[RP_MAX_SHARDS];
  const uint64_t pos0 = (uint64_t)blockIdx.x * RP_TILE;
  const uint32_t cntt = (uint32_t)((n - pos0) < RP_TILE ? (n - pos0) : RP_TILE);
  if (threadIdx.x < shards) hist[threadIdx.x] = 0;
  uint32_t k[RP_I], v[RP_I], d[RP_I];
#pragma unroll
  for (int it = 0; it < RP_I; ++it) {
    const uint32_t li = (uint32_t)it * RP_T + threadIdx.x;
    k[it] = li < cntt ? __ldcs(keys + pos0 + li) : 0u;
    if (VALS) v[it] = li < cntt ? __ldcs(vals + pos0 + li) : 0u;
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < RP_I; ++it) {
    const uint32_t li = (uint32_t)it * RP_T + threadIdx.x;
    if (li >= cntt) continue;
    const uint32_t dd = route(k[it], shards);  // ShardRouter.route (distributed.py:44-45)
    d[it] = dd | atomicAdd(&hist[dd], 1u) << 8;
  }
  __syncthreads();
  if (threadIdx.x < 32) {  // shard runs: global cursor, tile offset
    uint32_t run = 0;
    for (uint32_t b0 = 0; b0 < shards; b0 += 32) {
      const uint32_t b = b0 + threadIdx.x;
      const uint32_t hv = b < shards ? hist[b] : 0u;
      uint32_t inc = hv;
#pragma unroll
      for (int dl = 1; dl < 32; dl <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, dl);
        if ((int)threadIdx.x >= dl) inc += y;
      }
      if (b < shards) {
        boff[b] = run + inc - hv;
        const unsigned long long old = hv ? atomicAdd(cnt + b, (unsigned long long)hv) : 0ull;
        gb[b] = (unsigned long long)b * cap + old;
        ovf[b] = (uint8_t)(old + hv > cap);
        if (old + hv > cap) *flag = 1;
      }
      run += __shfl_sync(0xffffffffu, inc, 31);
    }
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < RP_I; ++it) {
    const uint32_t li = (uint32_t)it * RP_T + threadIdx.x;
    if (li >= cntt) continue;
    const uint32_t dd = d[it] & 0xFFu, r = d[it] >> 8;
    const uint32_t j = boff[dd] + r;
    sK[j] = k[it];
    if (VALS) sV[j] = v[it];
    sD[j] = (uint8_t)dd;
    pos[pos0 + li] = (uint32_t)(gb[dd] + r);
  }
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < cntt; j += RP_T) {  // runs, coalesced
    const uint32_t dd = sD[j];
    if (ovf[dd]) continue;
    const unsigned long long dst = gb[dd] + (j - boff[dd]);
    kout[dst] = sK[j];
    if (VALS) vout[dst] = sV[j];
  }
}

int route_part32(const Launch& lc, const uint32_t* keys, const uint32_t* vals, uint64_t n, uint32_t shards,
                 uint64_t cap, uint32_t* pos, unsigned long long* counts, uint32_t* keys_out, uint32_t* vals_out,
                 int* flag) {
  if (shards < 1 || shards > RP_MAX_SHARDS) {
    set_error("route partition: 1 to 64 shards");
    return -22;
  }
  int rc = cuda_check(cudaMemsetAsync(counts, 0, shards * sizeof(unsigned long long), lc.stream), "memset");
  if (!rc) rc = cuda_check(cudaMemsetAsync(flag, 0, sizeof(int), lc.stream), "memset");
  if (rc || n == 0) return rc;
  const unsigned tiles = (unsigned)((n + RP_TILE - 1) / RP_TILE);
  if (vals)
    k_route_part<true><<<tiles, RP_T, 0, lc.stream>>>(keys, vals, n, shards, cap, pos, counts, keys_out, vals_out,
                                                       flag);
  else
    k_route_part<false><<<tiles, RP_T, 0, lc.stream>>>(keys, nullptr, n, shards, cap, pos, counts, keys_out, nullptr,
                                                        flag);
  count_launch();
  return cuda_check(cudaGetLastError(), "route partition");
}

int multi_split(const Launch& lc, const void* keys, int kbytes, const void* vals, int vbytes, uint64_t n,
                uint32_t shards, void* perm, int perm_bytes, uint64_t* offsets, void* keys_out, void* vals_out,
                void* scratch, size_t scratch_bytes) {
  if (perm_bytes != 4 && perm_bytes != 8 && perm_bytes != -4) {  // -4: u32 inverse (source -> position)
    set_error("perm_bytes must be 4 or 8");
    return -22;
  }
  if (perm_bytes != 8 && n > 0xFFFFFFFFull) {
    set_error("32-bit permutations need n < 2^32");
    return -22;
  }
  if (shards < 1 || shards > SPLIT_MAX_SHARDS) {
    set_error("shards must be in [1, 256]");
    return -22;
  }
  if (!vals) vals_out = nullptr;
#define CHB_SPLIT(K, V)                                                                                  \
  return perm_bytes == -4                                                                                \
             ? split_impl<K, V, uint32_t, true>(lc, (const K*)keys, (const V*)vals, n, shards,              \
                                                (uint32_t*)perm, offsets, (K*)keys_out, (V*)vals_out,       \
                                                scratch, scratch_bytes)                                     \
         : perm_bytes == 4                                                                               \
             ? split_impl<K, V, uint32_t>(lc, (const K*)keys, (const V*)vals, n, shards, (uint32_t*)perm,   \
                                          offsets, (K*)keys_out, (V*)vals_out, scratch, scratch_bytes)     \
             : split_impl<K, V, uint64_t>(lc, (const K*)keys, (const V*)vals, n, shards, (uint64_t*)perm,   \
                                          offsets, (K*)keys_out, (V*)vals_out, scratch, scratch_bytes);
  if (kbytes == 0) CHB_SPLIT(DestGiven, uint32_t)
  if (kbytes == 4 && vbytes == 4) CHB_SPLIT(uint32_t, uint32_t)
  if (kbytes == 4 && vbytes == 8) CHB_SPLIT(uint32_t, uint64_t)
  if (kbytes == 8 && vbytes == 4) CHB_SPLIT(uint64_t, uint32_t)
  if (kbytes == 8 && vbytes == 8) CHB_SPLIT(uint64_t, uint64_t)
#undef CHB_SPLIT
  set_error("key/value bytes must be 4 or 8");
  return -22;
}

// ------------------------------------------------- scatter / gather / copy
template <typename X, bool SCATTER, typename PI_T>
__global__ void k_permute(const X* __restrict__ src, const PI_T* __restrict__ perm, uint64_t n,
                          X* __restrict__ dst) {
  const uint64_t stride = gridDim.x * (uint64_t)blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    if (SCATTER) dst[perm[i]] = src[i];
    else dst[i] = src[perm[i]];
  }
}

template <typename PI_T>
static int permute_impl(const Launch& lc, const void* src, int elem_bytes, const PI_T* perm, uint64_t n, void* dst,
                        bool scatter) {
#define CHB_PERM(X)                                                                                       \
  {                                                                                                       \
    if (scatter) {                                                                                        \
      auto kern = k_permute<X, true, PI_T>;                                                               \
      return launch_persistent(lc, (const void*)kern, n, 1, [&](dim3 g, dim3 b) {                        \
        kern<<<g, b, 0, lc.stream>>>((const X*)src, perm, n, (X*)dst);                                    \
      });                                                                                                 \
    }                                                                                                     \
    auto kern = k_permute<X, false, PI_T>;                                                                \
    return launch_persistent(lc, (const void*)kern, n, 1,                                                 \
                             [&](dim3 g, dim3 b) { kern<<<g, b, 0, lc.stream>>>((const X*)src, perm, n, (X*)dst); }); \
  }
  switch (elem_bytes) {
    case 1: CHB_PERM(uint8_t)
    case 4: CHB_PERM(uint32_t)
    case 8: CHB_PERM(uint64_t)
  }
#undef CHB_PERM
  set_error("elem_bytes must be 1, 4 or 8");
  return -22;
}

int permute(const Launch& lc, const void* src, int elem_bytes, const uint64_t* perm, uint64_t n, void* dst,
            bool scatter) {
  return permute_impl<uint64_t>(lc, src, elem_bytes, perm, n, dst, scatter);
}
int permute32(const Launch& lc, const void* src, int elem_bytes, const uint32_t* perm, uint64_t n, void* dst,
              bool scatter) {
  return permute_impl<uint32_t>(lc, src, elem_bytes, perm, n, dst, scatter);
}

template <typename X>
__global__ void k_segment_copy(const X* __restrict__ src, const uint64_t* __restrict__ src_off,
                               const uint64_t* __restrict__ idx, uint64_t n, const uint64_t* __restrict__ dst_off,
                               X* __restrict__ dst) {
  const uint64_t stride = gridDim.x * (uint64_t)blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t q = idx[i];
    const uint64_t d0 = dst_off[q], len = dst_off[q + 1] - d0, s0 = src_off[i];
    for (uint64_t k = 0; k < len; ++k) dst[d0 + k] = src[s0 + k];
  }
}

int segment_copy(const Launch& lc, const void* src, int elem_bytes, const uint64_t* src_off, const uint64_t* idx,
                 uint64_t n, const uint64_t* dst_off, void* dst) {
#define CHB_SEG(X)                                                                                         \
  {                                                                                                        \
    auto kern = k_segment_copy<X>;                                                                         \
    return launch_persistent(lc, (const void*)kern, n, 1, [&](dim3 g, dim3 b) {                           \
      kern<<<g, b, 0, lc.stream>>>((const X*)src, src_off, idx, n, dst_off, (X*)dst);                      \
    });                                                                                                    \
  }
  switch (elem_bytes) {
    case 4: CHB_SEG(uint32_t)
    case 8: CHB_SEG(uint64_t)
  }
#undef CHB_SEG
  set_error("elem_bytes must be 4 or 8");
  return -22;
}

}  // namespace chb
