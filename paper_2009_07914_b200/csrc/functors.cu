// functors.cu -- device-side for_all / for_each (reference
// single_table.py:412-429, multi_table.py:299-339).
//
// The reference calls a host callback per occupied slot (for_all) or per match
// (for_each).  On the device the enumeration itself is the kernel:
//
//   for_all    stable compaction of the live cells (neither empty nor tombstone) in
//              slot order: per-tile live counts -> exclusive scan -> each tile
//              writes its live (key, value, slot) triples at its offset.  Two
//              coalesced passes over the slot array, the output written once.
//   reduce     built-in functors folded over the live cells without materialising
//              them (count, sum of values, xor of keys, min / max value): one pass,
//              per-CTA partials, one atomic per CTA.
//
// The caller applies its own functor to the compacted device arrays (a CUDA tensor
// op, or another kernel); for_each's matches come from the lookup kernels
// (ch_find for single-value, ch_multi_retrieve_slots for multi-value).
#include "dispatch.cuh"

namespace chb {

constexpr int FA_THREADS = 256;
constexpr int FA_ITEMS = 16;
constexpr uint64_t FA_TILE = (uint64_t)FA_THREADS * FA_ITEMS;

template <Layout LAY, typename K, typename V>
struct Cell;
template <>
struct Cell<PACKED, uint32_t, uint32_t> {
  __device__ __forceinline__ static void get(const TableRef& T, uint64_t i, uint32_t& k, uint32_t& v) {
    const uint64_t w = static_cast<const uint64_t*>(T.slots)[i];
    k = (uint32_t)w;
    v = (uint32_t)(w >> 32);
  }
};
template <typename K, typename V>
struct Cell<SOA, K, V> {
  __device__ __forceinline__ static void get(const TableRef& T, uint64_t i, K& k, V& v) {
    k = static_cast<const K*>(T.slots)[i];
    v = static_cast<const V*>(T.vals)[i];
  }
};
template <typename K, typename V>
struct Cell<AOS, K, V> {
  __device__ __forceinline__ static void get(const TableRef& T, uint64_t i, K& k, V& v) {
    const CellT<K, V> c = static_cast<const CellT<K, V>*>(T.slots)[i];
    k = c.k;
    v = c.v;
  }
};

template <typename K>
__device__ __forceinline__ bool live(K k, const TableRef& T) {
  return k != (K)T.e && k != (K)T.t;
}

// pass 1: live cells per tile (slots in [tile * FA_TILE, +FA_TILE), strided by thread)
template <Layout LAY, typename K, typename V>
__global__ void __launch_bounds__(FA_THREADS) k_live_count(TableRef T, uint32_t* __restrict__ tile_counts) {
  const uint64_t base = blockIdx.x * FA_TILE;
  uint32_t c = 0;
#pragma unroll 4
  for (int r = 0; r < FA_ITEMS; ++r) {
    const uint64_t i = base + (uint64_t)r * FA_THREADS + threadIdx.x;
    if (i < T.c) {
      K k;
      V v;
      Cell<LAY, K, V>::get(T, i, k, v);
      c += live(k, T);
    }
  }
  c = warp_sum(c);
  __shared__ uint32_t ws[FA_THREADS / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (int w = 0; w < FA_THREADS / 32; ++w) s += ws[w];
    tile_counts[blockIdx.x] = s;
  }
}

// pass 2: each tile writes its live cells in slot order at tile_off[tile]
template <Layout LAY, typename K, typename V>
__global__ void __launch_bounds__(FA_THREADS) k_live_compact(TableRef T, const uint64_t* __restrict__ tile_off,
                                                            uint64_t cap, K* __restrict__ keys_out,
                                                            V* __restrict__ vals_out,
                                                            int64_t* __restrict__ slots_out) {
  __shared__ uint32_t wsum[FA_THREADS / 32];
  __shared__ uint64_t run;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t base = blockIdx.x * FA_TILE;
  if (threadIdx.x == 0) run = tile_off[blockIdx.x];
  __syncthreads();
  for (int r = 0; r < FA_ITEMS; ++r) {  // rounds in slot order; ranks by warp then lane
    const uint64_t i = base + (uint64_t)r * FA_THREADS + threadIdx.x;
    K k = 0;
    V v = 0;
    bool on = false;
    if (i < T.c) {
      Cell<LAY, K, V>::get(T, i, k, v);
      on = live(k, T);
    }
    const unsigned m = __ballot_sync(0xffffffffu, on);
    if (lane == 0) wsum[warp] = __popc(m);
    __syncthreads();
    uint64_t pos = run + __popc(m & ((1u << lane) - 1u));
    for (int w = 0; w < warp; ++w) pos += wsum[w];
    if (on && pos < cap) {
      if (keys_out) keys_out[pos] = k;
      if (vals_out) vals_out[pos] = v;
      if (slots_out) slots_out[pos] = (int64_t)i;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t add = 0;
      for (int w = 0; w < FA_THREADS / 32; ++w) add += wsum[w];
      run += add;
    }
    __syncthreads();
  }
}

// built-in reductions over the live cells: out[0] count, [1] sum of values (mod 2^64),
// [2] xor of keys, [3] min value, [4] max value
template <Layout LAY, typename K, typename V>
__global__ void __launch_bounds__(FA_THREADS) k_live_reduce(TableRef T, unsigned long long* __restrict__ out) {
  unsigned long long cnt = 0, sum = 0, kx = 0, mn = ~0ull, mx = 0;
  const uint64_t stride = gridDim.x * (uint64_t)FA_THREADS;
  for (uint64_t i = blockIdx.x * (uint64_t)FA_THREADS + threadIdx.x; i < T.c; i += stride) {
    K k;
    V v;
    Cell<LAY, K, V>::get(T, i, k, v);
    if (!live(k, T)) continue;
    cnt += 1;
    sum += (unsigned long long)v;
    kx ^= (unsigned long long)k;
    mn = (unsigned long long)v < mn ? (unsigned long long)v : mn;
    mx = (unsigned long long)v > mx ? (unsigned long long)v : mx;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
    sum += __shfl_xor_sync(0xffffffffu, sum, d);
    kx ^= __shfl_xor_sync(0xffffffffu, kx, d);
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, mn, d), b = __shfl_xor_sync(0xffffffffu, mx, d);
    mn = a < mn ? a : mn;
    mx = b > mx ? b : mx;
  }
  if ((threadIdx.x & 31) == 0 && cnt) {
    atomicAdd(&out[0], cnt);
    atomicAdd(&out[1], sum);
    atomicXor(&out[2], kx);
    atomicMin(&out[3], mn);
    atomicMax(&out[4], mx);
  }
}

template <Layout LAY, typename K, typename V, int G>
struct FunctorKernels {
  static int for_all(const Launch& lc, const TableRef& T, void* keys_out, void* vals_out, int64_t* slots_out,
                     uint64_t cap, uint64_t* d_count, void* scratch, size_t scratch_bytes) {
    const uint64_t tiles = (T.c + FA_TILE - 1) / FA_TILE;
    uint32_t* counts = (uint32_t*)scratch;
    uint64_t* off = (uint64_t*)(((uintptr_t)(counts + tiles) + 15) & ~(uintptr_t)15);
    void* scan = off + tiles + 1;
    const size_t used = (size_t)((char*)scan - (char*)scratch);
    if (used > scratch_bytes) {
      set_error("for_all scratch too small");
      return -22;
    }
    k_live_count<LAY, K, V><<<(unsigned)tiles, FA_THREADS, 0, lc.stream>>>(T, counts);
    count_launch();
    int rc = cuda_check(cudaGetLastError(), "live count");
    if (!rc) rc = exclusive_scan_u32(lc, counts, tiles, off, scan, scratch_bytes - used);
    if (rc) return rc;
    k_live_compact<LAY, K, V><<<(unsigned)tiles, FA_THREADS, 0, lc.stream>>>(T, off, cap, (K*)keys_out,
                                                                             (V*)vals_out, slots_out);
    count_launch();
    if (!(rc = cuda_check(cudaGetLastError(), "live compact")) && d_count)
      rc = cuda_check(cudaMemcpyAsync(d_count, off + tiles, 8, cudaMemcpyDeviceToDevice, lc.stream), "count");
    return rc;
  }
  static int reduce(const Launch& lc, const TableRef& T, unsigned long long* out) {
    int rc = cuda_check(cudaMemsetAsync(out, 0, 5 * 8, lc.stream), "memset");
    if (!rc) rc = cuda_check(cudaMemsetAsync(out + 3, 0xFF, 8, lc.stream), "memset");
    if (rc) return rc;
    auto kern = k_live_reduce<LAY, K, V>;
    return launch_persistent(lc, (const void*)kern, T.c, 1, [&](dim3 g, dim3 b) {
      kern<<<g, b, 0, lc.stream>>>(T, out);
    });
  }
};

size_t for_all_scratch_bytes(uint64_t c) {
  const uint64_t tiles = (c + FA_TILE - 1) / FA_TILE;
  return tiles * 4 + 16 + (tiles + 1) * 8 + exclusive_scan_scratch_bytes(tiles) + 64;
}

int table_for_all(const Launch& lc, const TableRef& T, const TypeSel& ts, void* keys_out, void* vals_out,
                  int64_t* slots_out, uint64_t cap, uint64_t* d_count, void* scratch, size_t scratch_bytes) {
  TypeSel t1 = ts;
  t1.g = 1;
  return dispatch_types<FunctorKernels>(t1, [&](auto tag) {
    return decltype(tag)::type::for_all(lc, T, keys_out, vals_out, slots_out, cap, d_count, scratch, scratch_bytes);
  });
}

int table_reduce(const Launch& lc, const TableRef& T, const TypeSel& ts, unsigned long long* out) {
  TypeSel t1 = ts;
  t1.g = 1;
  return dispatch_types<FunctorKernels>(t1, [&](auto tag) { return decltype(tag)::type::reduce(lc, T, out); });
}

}  // namespace chb
