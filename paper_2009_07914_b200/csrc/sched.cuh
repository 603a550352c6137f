// sched.cuh -- CTA-chunked dynamic scheduling for the probe kernels.
//
// A CTA claims CHUNK consecutive batch elements from a global queue (one
// atomicAdd), stages their keys/values in shared memory with coalesced loads,
// lets its probe groups drain the chunk through a shared-memory counter (a
// group that resolves a key immediately takes the next one), then writes the
// chunk's results back with coalesced stores.  Two properties matter on B200:
//  * the elements in flight across the GPU are always a narrow band of the
//    batch (CTAs claim chunks in order), so a region-ordered batch keeps its
//    table region L2-resident (locality.cu); a static grid-stride let fast and
//    slow CTAs drift across the whole table (profiles/r01_loc_v1: 11-16 % L2 hits);
//  * inputs and outputs move as whole lines instead of per-lane 1-8 B accesses
//    at scattered times.
#pragma once
#include "common.cuh"

namespace chb {

struct ChunkState {
  uint64_t base;
  uint32_t cnt;
  uint32_t next;
};

// Claim the next chunk; returns false (CTA-uniformly) once the batch is done.
template <int CHUNK>
__device__ __forceinline__ bool chunk_begin(ChunkState& cs, unsigned long long* queue, uint64_t n) {
  __syncthreads();  // the previous chunk is fully consumed and written back
  if (threadIdx.x == 0) {
    const uint64_t b = atomicAdd(queue, (unsigned long long)CHUNK);
    cs.base = b;
    cs.cnt = b < n ? (uint32_t)((n - b) < (uint64_t)CHUNK ? (n - b) : (uint64_t)CHUNK) : 0u;
    cs.next = 0;
  }
  __syncthreads();
  return cs.cnt > 0;
}

// Next chunk-local element for a probe group (lane 0 claims, the tile shares it).
template <typename Tile>
__device__ __forceinline__ uint32_t group_claim(ChunkState& cs, const Tile& tile, int lane) {
  uint32_t li = 0;
  if (lane == 0) li = atomicAdd(&cs.next, 1u);
  if constexpr (Tile::num_threads() > 1) li = tile.shfl(li, 0);
  return li;
}

template <typename X>
__device__ __forceinline__ void stage_in(X* dst, const X* __restrict__ src, const ChunkState& cs) {
  for (uint32_t j = threadIdx.x; j < cs.cnt; j += blockDim.x) dst[j] = src[cs.base + j];
}
// Probe starts staged per chunk element: h = 32 hw + ho, step = 32 sw
// (p < 2^32 is enforced at table creation, so hw and sw fit 32 bits).
struct StartSlots {
  uint32_t* hw;
  uint32_t* sw;
  uint8_t* ho;
  __device__ __forceinline__ ProbeStart get(uint32_t j) const {
    ProbeStart ps;
    ps.h = (uint64_t)hw[j] * WINDOW + ho[j];
    ps.step = (uint64_t)sw[j] * WINDOW;
    return ps;
  }
};

// Stage keys and their probe starts (h, step): the hashing runs here, SIMT-
// uniformly over the chunk, instead of inside the divergent per-group loop.
template <typename K>
__device__ __forceinline__ void stage_keys(K* s_keys, const StartSlots& ss, const K* __restrict__ keys,
                                           const ChunkState& cs, const TableRef& T) {
  for (uint32_t j = threadIdx.x; j < cs.cnt; j += blockDim.x) {
    const K k = keys[cs.base + j];
    s_keys[j] = k;
    const ProbeStart ps = probe_start(T, (uint64_t)k);
    ss.hw[j] = (uint32_t)(ps.h / WINDOW);
    ss.ho[j] = (uint8_t)(ps.h % WINDOW);
    ss.sw[j] = (uint32_t)(ps.step / WINDOW);
  }
}

// Chunk size: keep the staged inputs/outputs of one CTA within ~40 KB of
// static shared memory.
template <typename K, typename V>
constexpr int chunk_for() { return (sizeof(K) + sizeof(V)) > 8 ? 1024 : 2048; }

template <typename X>
__device__ __forceinline__ void stage_out(X* __restrict__ dst, const X* src, const ChunkState& cs) {
  for (uint32_t j = threadIdx.x; j < cs.cnt; j += blockDim.x) dst[cs.base + j] = src[j];
}

// Results of a device-counted list (staged.cu) go back to their owners' positions.
template <typename X>
__device__ __forceinline__ void stage_out_ix(X* __restrict__ dst, const X* src, const ChunkState& cs,
                                             const uint32_t* __restrict__ ix) {
  if (!ix) {
    stage_out(dst, src, cs);
    return;
  }
  for (uint32_t j = threadIdx.x; j < cs.cnt; j += blockDim.x) dst[ix[cs.base + j]] = src[j];
}

}  // namespace chb
