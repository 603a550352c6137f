// kmer.cu -- device k-mer sketching for the index demo (reference
// kmer.py:63-137, "device-sided interface").
//
// Input: sequence bytes (ASCII, concatenated) and a window table (byte start, length,
// tag).  One warp per window:
//   1. canonical k-mers: for every position p of the window whose k bases ending at p are
//      all A/C/G/T (either case; anything else resets the roll, kmer.py:63-88), the 2-bit
//      forward and reverse-complement encodings are built from the k bytes and the smaller
//      one kept, with its mix64 hash, in a per-position scratch (positions that end no
//      k-mer are marked invalid);
//   2. bottom-s sketch (kmer.py:91-100): s passes, each a warp-wide minimum of
//      (mix64(kmer), kmer) strictly above the previous pick -- the picks are the distinct
//      k-mers with the s smallest keys, in ascending order, as the reference's sorted()[:s].
// A scan + compaction then packs the (kmer, tag) pairs in window order for a bulk insert
// (build_index) or a bulk lookup (classify).
#include "dispatch.cuh"

namespace chb {

__device__ __forceinline__ int base_code(uint8_t c) {
  switch (c) {
    case 'A': case 'a': return 0;
    case 'C': case 'c': return 1;
    case 'G': case 'g': return 2;
    case 'T': case 't': return 3;
  }
  return -1;
}

// (h, km) < (h2, km2) lexicographically
__device__ __forceinline__ bool key_less(uint64_t h, uint64_t km, uint64_t h2, uint64_t km2) {
  return h < h2 || (h == h2 && km < km2);
}

__global__ void __launch_bounds__(256) k_kmer_sketch(const uint8_t* __restrict__ text,
                                                    const uint64_t* __restrict__ win_start,
                                                    const uint32_t* __restrict__ win_len, uint64_t n_windows,
                                                    int k, uint32_t sketch, uint64_t* __restrict__ sc_km,
                                                    uint64_t* __restrict__ sc_h, uint8_t* __restrict__ sc_ok,
                                                    const uint64_t* __restrict__ sc_off,
                                                    uint64_t* __restrict__ out_km, uint32_t* __restrict__ out_cnt) {
  const int lane = threadIdx.x & 31;
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t mask = k == 32 ? ~0ull : ((1ull << (2 * k)) - 1);
  const int shift = 2 * (k - 1);
  for (uint64_t w = blockIdx.x * (uint64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); w < n_windows; w += warps) {
    const uint8_t* s = text + win_start[w];
    const uint32_t len = win_len[w];
    const uint64_t so = sc_off[w];
    // 1. canonical k-mer ending at every position
    for (uint32_t p = lane; p < len; p += 32) {
      bool ok = p + 1 >= (uint32_t)k;
      uint64_t fwd = 0, rev = 0;
      if (ok) {
        for (int i = 0; i < k; ++i) {  // bases p-k+1 .. p, oldest first
          const int c = base_code(s[p + 1 - k + i]);
          if (c < 0) {
            ok = false;
            break;
          }
          fwd = ((fwd << 2) | (uint64_t)c) & mask;
          rev = (rev >> 2) | ((uint64_t)(3 - c) << shift);
        }
      }
      const uint64_t km = fwd <= rev ? fwd : rev;
      sc_ok[so + p] = ok;
      sc_km[so + p] = km;
      sc_h[so + p] = ok ? mix64(km) : 0;
    }
    __syncwarp();
    // 2. s smallest distinct (mix64(km), km), ascending
    uint64_t last_h = 0, last_k = 0;
    bool have_last = false;
    uint32_t cnt = 0;
    for (; cnt < sketch; ++cnt) {
      uint64_t bh = ~0ull, bk = ~0ull;
      bool found = false;
      for (uint32_t p = lane; p < len; p += 32) {
        if (!sc_ok[so + p]) continue;
        const uint64_t h = sc_h[so + p], km = sc_km[so + p];
        if (have_last && !key_less(last_h, last_k, h, km)) continue;  // not above the last pick
        if (!found || key_less(h, km, bh, bk)) {
          bh = h;
          bk = km;
          found = true;
        }
      }
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) {
        const uint64_t oh = __shfl_xor_sync(0xffffffffu, bh, d), ok2 = __shfl_xor_sync(0xffffffffu, bk, d);
        const int of = __shfl_xor_sync(0xffffffffu, (int)found, d);
        if (of && (!found || key_less(oh, ok2, bh, bk))) {
          bh = oh;
          bk = ok2;
          found = true;
        }
      }
      if (!found) break;  // fewer distinct k-mers than the sketch size
      if (lane == 0) out_km[w * (uint64_t)sketch + cnt] = bk;
      last_h = bh;
      last_k = bk;
      have_last = true;
    }
    if (lane == 0) out_cnt[w] = cnt;
  }
}

// packed[off[w] + j] = (out_km[w * sketch + j], tag[w]) for j < cnt[w]
__global__ void k_kmer_pack(const uint64_t* __restrict__ out_km, const uint32_t* __restrict__ cnt,
                            const uint64_t* __restrict__ off, const uint32_t* __restrict__ tag, uint64_t n_windows,
                            uint32_t sketch, uint64_t* __restrict__ km_dst, uint32_t* __restrict__ tag_dst) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n_windows * sketch; i += stride) {
    const uint64_t w = i / sketch, j = i % sketch;
    if (j >= cnt[w]) continue;
    km_dst[off[w] + j] = out_km[i];
    if (tag_dst) tag_dst[off[w] + j] = tag ? tag[w] : (uint32_t)w;
  }
}

__global__ void k_win_len64(const uint32_t* __restrict__ len, uint64_t n, uint32_t* __restrict__ out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) out[i] = len[i];
}

int kmer_sketch(const Launch& lc, const uint8_t* text, const uint64_t* win_start, const uint32_t* win_len,
                const uint32_t* win_tag, uint64_t n_windows, int k, uint32_t sketch, uint64_t* km_out,
                uint32_t* tag_out, uint64_t* d_count, void* scratch, size_t scratch_bytes, uint64_t total_len) {
  char* q = static_cast<char*>(scratch);
  auto take = [&](size_t b) {
    char* r = q;
    q += (b + 255) & ~(size_t)255;
    return (void*)r;
  };
  uint64_t* sc_off = (uint64_t*)take((n_windows + 1) * 8);
  uint32_t* lens = (uint32_t*)take(n_windows * 4);
  uint64_t* sc_km = (uint64_t*)take(total_len * 8);
  uint64_t* sc_h = (uint64_t*)take(total_len * 8);
  uint8_t* sc_ok = (uint8_t*)take(total_len);
  uint64_t* okm = (uint64_t*)take(n_windows * (uint64_t)sketch * 8);
  uint32_t* cnt = (uint32_t*)take(n_windows * 4);
  uint64_t* off = (uint64_t*)take((n_windows + 1) * 8);
  const size_t scan_b = exclusive_scan_scratch_bytes(n_windows);
  void* scan = take(scan_b);
  if ((size_t)(q - static_cast<char*>(scratch)) > scratch_bytes) {
    set_error("k-mer scratch too small");
    return -22;
  }
  const unsigned grid = (unsigned)(lc.sms * 8);
  k_win_len64<<<grid, 256, 0, lc.stream>>>(win_len, n_windows, lens);
  count_launch();
  int rc = exclusive_scan_u32(lc, lens, n_windows, sc_off, scan, scan_b);  // scratch position of each window
  if (rc) return rc;
  k_kmer_sketch<<<grid, 256, 0, lc.stream>>>(text, win_start, win_len, n_windows, k, sketch, sc_km, sc_h, sc_ok,
                                             sc_off, okm, cnt);
  count_launch();
  if ((rc = cuda_check(cudaGetLastError(), "k-mer sketch"))) return rc;
  if ((rc = exclusive_scan_u32(lc, cnt, n_windows, off, scan, scan_b))) return rc;
  k_kmer_pack<<<grid, 256, 0, lc.stream>>>(okm, cnt, off, win_tag, n_windows, sketch, km_out, tag_out);
  count_launch();
  if ((rc = cuda_check(cudaGetLastError(), "k-mer pack"))) return rc;
  return d_count ? cuda_check(cudaMemcpyAsync(d_count, off + n_windows, 8, cudaMemcpyDeviceToDevice, lc.stream),
                              "count")
                 : 0;
}

size_t kmer_scratch_bytes(uint64_t n_windows, uint32_t sketch, uint64_t total_len) {
  auto a = [](size_t b) { return (b + 255) & ~(size_t)255; };
  return a((n_windows + 1) * 8) + a(n_windows * 4) + 2 * a(total_len * 8) + a(total_len) +
         a(n_windows * (uint64_t)sketch * 8) + a(n_windows * 4) + a((n_windows + 1) * 8) +
         a(exclusive_scan_scratch_bytes(n_windows)) + 256;
}

}  // namespace chb
