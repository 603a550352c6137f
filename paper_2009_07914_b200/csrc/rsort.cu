// rsort.cu -- stable LSD radix sort of (key, payload) pairs, the grouping step of the
// grouped multi-value insert (mgroup.cu).
//
// The grouped insert needs every copy of a key contiguous and the copies in batch order
// (a group claims its cells in sequence order, which must be the order the reference's
// sequential inserts would have filled them, multi_table.py:113-152).  A stable sort by
// key gives both.  8 bits per pass, sizeof(K) passes, onesweep style:
//   k_rs_hist     one read of the keys: the global histogram of every pass's digit,
//                 scanned into digit offsets (k_rs_hist_scan)
//   k_rs_pass     per pass: a tile (4096 pairs) ranked stably in shared memory, its digit
//                 counts published and the counts of all earlier tiles found by decoupled
//                 look-back (tiles are numbered in start order, so every predecessor is
//                 running or done), then written as whole (tile, digit) runs -- coalesced,
//                 like the staged tile partitions.  One read and one write of the pairs.
// Stable ranks without atomics: warp w owns the tile's items [256 w, 256 w + 256) in
// eight rounds of 32; within a round eight ballots group a digit's lanes and the
// lowest of them advances the warp's running count of that digit; after the rounds one
// scan across the 16 warps per digit and one across the digits place every item.
#include <cstdlib>

#include "dispatch.cuh"

namespace chb {

constexpr int RS_T = 512;                     // threads per tile CTA
constexpr int RS_W = RS_T / 32;               // warps
constexpr int RS_I = 8;                       // items per thread
constexpr uint32_t RS_TILE = RS_T * RS_I;     // 4096 items per tile
constexpr uint32_t RS_WI = 32u * RS_I;        // items per warp (contiguous)

template <typename K>
__device__ __forceinline__ uint32_t rs_digit(K k, int shift) {
  return (uint32_t)(k >> shift) & 0xFFu;
}

// the global digit histogram of every pass (hist[pass * 256 + digit])
template <typename K>
__global__ void __launch_bounds__(RS_T) k_rs_hist(const K* __restrict__ keys, uint64_t n,
                                                  uint32_t* __restrict__ hist) {
  constexpr int NP = (int)sizeof(K);
  __shared__ uint32_t h[NP * 256];
  for (uint32_t i = threadIdx.x; i < NP * 256; i += RS_T) h[i] = 0;
  __syncthreads();
  for (uint64_t i = (uint64_t)blockIdx.x * RS_T + threadIdx.x; i < n; i += (uint64_t)gridDim.x * RS_T) {
    const K k = keys[i];
#pragma unroll
    for (int p = 0; p < NP; ++p) atomicAdd(&h[p * 256 + rs_digit(k, 8 * p)], 1u);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < NP * 256; i += RS_T)
    if (h[i]) atomicAdd(&hist[i], h[i]);
}

// lanes of the warp holding the same 8-bit digit (valid lanes only): eight ballots, a fixed
// cost -- __match_any_sync measured 1.5x slower per pass on batches whose warps see 32
// distinct digits (its cost grows with the number of distinct values)
__device__ __forceinline__ unsigned rs_match(uint32_t d, bool ok) {
  unsigned m = __ballot_sync(0xffffffffu, ok);
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const unsigned x = __ballot_sync(0xffffffffu, (d >> b) & 1u);
    m &= ((d >> b) & 1u) ? x : ~x;
  }
  return m;
}

// the histograms -> exclusive digit offsets per pass, in place (one CTA of 256 threads)
__global__ void __launch_bounds__(256) k_rs_hist_scan(uint32_t* __restrict__ hist, int passes) {
  __shared__ uint32_t wt[8];
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  for (int p = 0; p < passes; ++p) {
    const uint32_t v = hist[p * 256 + threadIdx.x];
    uint32_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
      if ((int)lane >= d) x += y;
    }
    if (lane == 31) wt[warp] = x;
    __syncthreads();
    uint32_t before = 0;
    for (uint32_t w = 0; w < warp; ++w) before += wt[w];
    hist[p * 256 + threadIdx.x] = before + x - v;
    __syncthreads();
  }
}

// exclusive scan over the CTA's threads in order (RS_T threads); syncs
__device__ __forceinline__ uint32_t block_scan_rs(uint32_t v, uint32_t* wt) {
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if ((int)lane >= d) x += y;
  }
  if (lane == 31) wt[warp] = x;
  __syncthreads();
  uint32_t y = lane < (uint32_t)RS_W ? wt[lane] : 0u;
#pragma unroll
  for (int d = 1; d < RS_W; d <<= 1) {
    const uint32_t z = __shfl_up_sync(0xffffffffu, y, d);
    if ((int)lane >= d) y += z;
  }
  const uint32_t r = (warp ? __shfl_sync(0xffffffffu, y, (int)warp - 1) : 0u) + x - v;
  __syncthreads();  // wt reusable
  return r;
}

// look-back status of (tile, digit): flag << 62 | count (1: the tile's own count,
// 2: inclusive of every earlier tile)
constexpr uint64_t RS_AGG = 1ull << 62, RS_INC = 2ull << 62, RS_VAL = (1ull << 62) - 1;
constexpr int RS_LB = 4;  // look-back window

template <typename K, typename P, int MINB>
__global__ void __launch_bounds__(RS_T, MINB) k_rs_pass(const K* __restrict__ kin, const P* __restrict__ pin,
                                                     K* __restrict__ kout, P* __restrict__ pout, uint64_t n,
                                                     int shift, const uint32_t* __restrict__ hist,
                                                     unsigned long long* __restrict__ status,
                                                     uint32_t* __restrict__ next_tile) {
  extern __shared__ __align__(16) unsigned char rs_sm[];
  P* sP = reinterpret_cast<P*>(rs_sm);
  K* sK = reinterpret_cast<K*>(sP + RS_TILE);
  uint16_t* wc = reinterpret_cast<uint16_t*>(sK + RS_TILE);  // [warp][digit]: running counts, then prefixes
  uint8_t* sD = reinterpret_cast<uint8_t*>(wc + RS_W * 256);
  __shared__ uint32_t dstart[256];
  __shared__ uint64_t gbase[256];
  __shared__ uint32_t wt[RS_W];
  __shared__ uint32_t s_t;
  if (threadIdx.x == 0) s_t = atomicAdd(next_tile, 1u);  // tiles in start order (look-back)
  for (uint32_t i = threadIdx.x; i < RS_W * 256 / 2; i += RS_T) reinterpret_cast<uint32_t*>(wc)[i] = 0u;
  __syncthreads();  // tile number, wc zeroed
  const uint32_t t = s_t;
  const uint64_t base = (uint64_t)t * RS_TILE;
  const uint32_t cnt = (n - base) < RS_TILE ? (uint32_t)(n - base) : RS_TILE;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  K k[RS_I];
#pragma unroll
  for (int r = 0; r < RS_I; ++r) {  // all key loads in flight before any use
    const uint32_t li = warp * RS_WI + (uint32_t)r * 32u + lane;
    k[r] = li < cnt ? kin[base + li] : (K)0;
  }
  const uint32_t gx = threadIdx.x < 256 ? hist[threadIdx.x] : 0u;  // where this pass's digit starts
  uint16_t* const my = wc + warp * 256;
  const unsigned lt = (1u << lane) - 1u;
  uint32_t rk[RS_I / 2];  // within-warp ranks, two u16 per register
#pragma unroll
  for (int r = 0; r < RS_I; ++r) {  // rounds in item order: the warp's running count per digit
    const uint32_t li = warp * RS_WI + (uint32_t)r * 32u + lane;
    const bool ok = li < cnt;
    const uint32_t d = ok ? rs_digit(k[r], shift) : 256u;
    const unsigned peers = rs_match(d, ok);
    const uint32_t before = ok ? (uint32_t)my[d] : 0u;
    __syncwarp();
    if (ok && (int)lane == __ffs(peers) - 1) my[d] = (uint16_t)(before + (uint32_t)__popc(peers));
    __syncwarp();
    const uint32_t rank = before + (uint32_t)__popc(peers & lt);
    if (r & 1) rk[r / 2] |= rank << 16;
    else rk[r / 2] = rank;
  }
  __syncthreads();
  // per digit: exclusive prefix over the warps (in place) and the tile's total
  uint32_t tot = 0;
  if (threadIdx.x < 256) {
#pragma unroll
    for (int w = 0; w < RS_W; ++w) {
      const uint32_t x = wc[w * 256 + threadIdx.x];
      wc[w * 256 + threadIdx.x] = (uint16_t)tot;
      tot += x;
    }
  }
  // publish the tile's digit counts, then look back for the earlier tiles' (thread d: digit d)
  volatile unsigned long long* const st = status;
  uint64_t before_tiles = 0;
  if (threadIdx.x < 256) {
    st[(uint64_t)t * 256 + threadIdx.x] = (t == 0 ? RS_INC : RS_AGG) | tot;
    // eight predecessors per step (independent loads): consume them nearest first up to an
    // inclusive count; an unpublished one ends the step and is read again
    for (int64_t j = (int64_t)t - 1; j >= 0;) {
      uint64_t sv[RS_LB];
#pragma unroll
      for (int u = 0; u < RS_LB; ++u) sv[u] = j - u >= 0 ? st[(uint64_t)(j - u) * 256 + threadIdx.x] : RS_INC;
      bool done = false;
      int used = 0;
#pragma unroll
      for (int u = 0; u < RS_LB; ++u) {
        if (done || used < u || (sv[u] & ~RS_VAL) == 0) continue;
        before_tiles += sv[u] & RS_VAL;
        used = u + 1;
        if (sv[u] & RS_INC) done = true;
      }
      if (done) break;
      j -= used;
    }
    if (t) st[(uint64_t)t * 256 + threadIdx.x] = RS_INC | (before_tiles + tot);
  }
  // exclusive scan of the tile's digit totals
  const uint32_t ds = block_scan_rs(tot, wt);
  if (threadIdx.x < 256) {
    dstart[threadIdx.x] = ds;
    gbase[threadIdx.x] = (uint64_t)gx + before_tiles - ds;  // run destination minus its tile offset
  }
  __syncthreads();
  uint32_t ps[RS_I / 2];  // bucketed positions, two u16 per register
#pragma unroll
  for (int r = 0; r < RS_I; ++r) {  // keys to bucketed order in shared memory
    const uint32_t li = warp * RS_WI + (uint32_t)r * 32u + lane;
    uint32_t pos = 0;
    if (li < cnt) {
      const uint32_t d = rs_digit(k[r], shift);
      pos = dstart[d] + wc[warp * 256 + d] + ((rk[r / 2] >> (16 * (r & 1))) & 0xFFFFu);
      sK[pos] = k[r];
      sD[pos] = (uint8_t)d;
    }
    if (r & 1) ps[r / 2] |= pos << 16;
    else ps[r / 2] = pos;
  }
  {  // then the payloads (loaded only now: the keys' registers are free)
    P q[RS_I];
#pragma unroll
    for (int r = 0; r < RS_I; ++r) {
      const uint32_t li = warp * RS_WI + (uint32_t)r * 32u + lane;
      q[r] = li < cnt ? pin[base + li] : (P)0;
    }
#pragma unroll
    for (int r = 0; r < RS_I; ++r) {
      const uint32_t li = warp * RS_WI + (uint32_t)r * 32u + lane;
      if (li < cnt) sP[(ps[r / 2] >> (16 * (r & 1))) & 0xFFFFu] = q[r];
    }
  }
  __syncthreads();
  for (uint32_t j = threadIdx.x; j < cnt; j += RS_T) {  // whole runs, consecutive addresses
    const uint64_t dst = gbase[sD[j]] + j;
    kout[dst] = sK[j];
    pout[dst] = sP[j];
  }
}

static uint64_t rs_al(uint64_t x) { return (x + 255) & ~(uint64_t)255; }

size_t radix_sort_scratch_bytes(uint64_t n, int kbytes, int pbytes) {
  const uint64_t tiles = (n + RS_TILE - 1) / RS_TILE;
  return rs_al(n * (uint64_t)kbytes) + rs_al(n * (uint64_t)pbytes) + rs_al(8 * 256 * 4) + rs_al(8 * 4) +
         rs_al(256 * tiles * 8);
}

template <typename K, typename P>
int radix_sort_pairs(const Launch& lc, const K* kin, const P* pin, K* kout, P* pout, uint64_t n, void* scratch,
                     size_t scratch_bytes) {
  if (n == 0) return 0;
  if (n >= (1ull << 31)) {
    set_error("radix sort: batch too large");
    return -22;
  }
  constexpr int passes = (int)sizeof(K);
  const uint32_t tiles = (uint32_t)((n + RS_TILE - 1) / RS_TILE);
  char* q = static_cast<char*>(scratch);
  const auto take = [&](uint64_t bytes) {
    char* r = q;
    q += rs_al(bytes);
    return (void*)r;
  };
  K* kt = (K*)take(n * sizeof(K));
  P* pt = (P*)take(n * sizeof(P));
  uint32_t* hist = (uint32_t*)take(8 * 256 * 4);
  uint32_t* next = (uint32_t*)take(8 * 4);
  unsigned long long* status = (unsigned long long*)take(256ull * tiles * 8);
  if ((size_t)(q - static_cast<char*>(scratch)) > scratch_bytes) {
    set_error("radix sort scratch too small");
    return -22;
  }
  const size_t smem = (size_t)RS_TILE * (sizeof(K) + sizeof(P) + 1) + RS_W * 256 * 2;
  // 3 CTAs per SM (40 registers, a few bytes of spill) measured 1.10 ms per pass at 2^27
  // pairs against 1.34 ms at 2 (64 registers); CH_RS_MINB=2 selects the latter
  static const bool two = [] {
    const char* e = getenv("CH_RS_MINB");
    return e && e[0] == '2';
  }();
  auto kp = two ? k_rs_pass<K, P, 2> : k_rs_pass<K, P, 3>;
  int rc = cuda_check(cudaFuncSetAttribute((const void*)kp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                      "radix sort smem");
  if (!rc) rc = cuda_check(cudaMemsetAsync(hist, 0, 8 * 256 * 4 + 256, lc.stream), "memset");  // + tile counters
  if (rc) return rc;
  k_rs_hist<K><<<(unsigned)(lc.sms * 4), RS_T, 0, lc.stream>>>(kin, n, hist);
  count_launch();
  k_rs_hist_scan<<<1, 256, 0, lc.stream>>>(hist, passes);
  count_launch();
  const K* sk = kin;
  const P* sp = pin;
  for (int p = 0; p < passes; ++p) {
    const bool to_out = ((passes - 1 - p) & 1) == 0;  // the last pass lands in the output
    K* dk = to_out ? kout : kt;
    P* dp = to_out ? pout : pt;
    if ((rc = cuda_check(cudaMemsetAsync(status, 0, 256ull * tiles * 8, lc.stream), "memset"))) return rc;
    kp<<<tiles, RS_T, smem, lc.stream>>>(sk, sp, dk, dp, n, 8 * p, hist + 256 * p, status, next + p);
    count_launch();
    if ((rc = cuda_check(cudaGetLastError(), "radix sort pass"))) return rc;
    sk = dk;
    sp = dp;
  }
  return 0;
}

template int radix_sort_pairs<uint32_t, uint64_t>(const Launch&, const uint32_t*, const uint64_t*, uint32_t*,
                                                  uint64_t*, uint64_t, void*, size_t);
template int radix_sort_pairs<uint32_t, uint32_t>(const Launch&, const uint32_t*, const uint32_t*, uint32_t*,
                                                  uint32_t*, uint64_t, void*, size_t);
template int radix_sort_pairs<uint64_t, uint64_t>(const Launch&, const uint64_t*, const uint64_t*, uint64_t*,
                                                  uint64_t*, uint64_t, void*, size_t);
template int radix_sort_pairs<uint64_t, uint32_t>(const Launch&, const uint64_t*, const uint32_t*, uint64_t*,
                                                  uint32_t*, uint64_t, void*, size_t);

}  // namespace chb
