// Random-access microbenchmark: the practical DRAM ceiling for hash-table probes
// on B200 (SURVEY.md §8(d) asks for it next to the roofline numbers).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/randbench tools/randbench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint64_t mixr(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull; x ^= x >> 33; x *= 0xff51afd7ed558ccdull;
  x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull; x ^= x >> 33; return x;
}

__device__ __forceinline__ uint4 ldcg16(const void* p) { return __ldcg((const uint4*)p); }
__device__ __forceinline__ uint64_t ldcg8(const void* p) {
  uint64_t r; asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(r) : "l"(p)); return r;
}

// LANES lanes cooperate on one access of LANES*16 bytes (LANES=0: one thread, 8 B).
// ILP independent accesses per group per iteration.
template <int LANES, int ILP>
__global__ void rand_read(const uint8_t* buf, uint64_t nbytes, uint64_t nops, uint64_t* out) {
  constexpr int L = LANES == 0 ? 1 : LANES;
  constexpr int SPAN = LANES == 0 ? 8 : LANES * 16;
  uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t group = tid / L; int lane = tid % L;
  uint64_t ngroups = (gridDim.x * (uint64_t)blockDim.x) / L;
  uint64_t nspans = nbytes / SPAN;
  uint64_t acc = 0;
  for (uint64_t i = group * ILP; i < nops; i += ngroups * ILP) {
    uint64_t v[ILP];
#pragma unroll
    for (int u = 0; u < ILP; ++u) {
      uint64_t idx = mixr(i + u) % nspans;
      const uint8_t* p = buf + idx * SPAN;
      if (LANES == 0) v[u] = ldcg8(p);
      else { uint4 q = ldcg16(p + lane * 16); v[u] = q.x ^ q.y ^ q.z ^ q.w; }
    }
#pragma unroll
    for (int u = 0; u < ILP; ++u) acc ^= v[u];
  }
  if ((uint32_t)acc == 0x12345678u) out[0] = acc;
}

// random 64-bit CAS (mostly succeeds on a fresh all-ones buffer)
template <bool LOAD_FIRST>
__global__ void rand_cas(uint64_t* buf, uint64_t nwords, uint64_t nops, uint64_t* out) {
  uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t n = gridDim.x * (uint64_t)blockDim.x;
  uint64_t acc = 0;
  for (uint64_t i = tid; i < nops; i += n) {
    uint64_t idx = mixr(i) % nwords;
    uint64_t expct = ~0ull;
    if (LOAD_FIRST) expct = ldcg8(buf + idx);
    acc += atomicCAS((unsigned long long*)buf + idx, expct, i);
  }
  if ((uint32_t)acc == 0x12345678u) out[0] = acc;
}

__global__ void rand_store(uint64_t* buf, uint64_t nwords, uint64_t nops) {
  uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t n = gridDim.x * (uint64_t)blockDim.x;
  for (uint64_t i = tid; i < nops; i += n) buf[mixr(i) % nwords] = i;
}

__global__ void seq_copy(const uint4* a, uint4* b, uint64_t n) {
  uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint64_t s = gridDim.x * (uint64_t)blockDim.x;
  for (uint64_t i = tid; i < n; i += s) b[i] = a[i];
}

int main(int argc, char** argv) {
  const uint64_t nbytes = (argc > 1 ? strtoull(argv[1], 0, 10) : 2048ull) << 20;
  printf("buffer %llu MiB\n", (unsigned long long)(nbytes >> 20));
  const uint64_t nops = 1ull << 28;
  uint8_t* buf; uint64_t* out; uint8_t* buf2;
  CK(cudaMalloc(&buf, nbytes)); CK(cudaMalloc(&buf2, nbytes)); CK(cudaMalloc(&out, 64));
  CK(cudaMemset(buf, 0xff, nbytes));
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto launch, double bytes_per_op) {
    launch(); cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    printf("%-28s %9.3f ms  %8.2f Gops/s  %8.1f GB/s(useful)  %s\n", name, best, nops / best / 1e6,
           nops * bytes_per_op / best / 1e6, err == cudaSuccess ? "" : cudaGetErrorString(err));
  };
  int blocks = sms * 8, thr = 256;
#define RR(L, I) timeit("read lanes=" #L " ilp=" #I, [&] { rand_read<L, I><<<blocks, thr>>>(buf, nbytes, nops, out); }, (L == 0 ? 8.0 : L * 16.0))
  RR(0, 1); RR(0, 2); RR(0, 4); RR(0, 8);
  RR(1, 1); RR(1, 4);
  RR(2, 1); RR(2, 2); RR(2, 4);
  RR(4, 1); RR(4, 2); RR(4, 4);
  RR(8, 1); RR(8, 2);
  RR(16, 1);
  timeit("cas 8B (no load)", [&] { cudaMemset(buf, 0xff, nbytes); }, 0);  // memset time reference
  timeit("cas 8B + memset", [&] { cudaMemsetAsync(buf, 0xff, nbytes); rand_cas<false><<<blocks, thr>>>((uint64_t*)buf, nbytes / 8, nops, out); }, 8);
  timeit("load+cas 8B + memset", [&] { cudaMemsetAsync(buf, 0xff, nbytes); rand_cas<true><<<blocks, thr>>>((uint64_t*)buf, nbytes / 8, nops, out); }, 8);
  timeit("rand store 8B", [&] { rand_store<<<blocks, thr>>>((uint64_t*)buf, nbytes / 8, nops); }, 8);
  {
    uint64_t n16 = nbytes / 16;
    cudaEventRecord(e0); seq_copy<<<sms * 8, 512>>>((uint4*)buf, (uint4*)buf2, n16); cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventRecord(e0); seq_copy<<<sms * 8, 512>>>((uint4*)buf, (uint4*)buf2, n16); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("seq copy 2GiB: %.3f ms  %.1f GB/s (r+w)\n", ms, 2.0 * nbytes / ms / 1e6);
  }
  return 0;
}
