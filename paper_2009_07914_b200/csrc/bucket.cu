// bucket.cu -- bucket-list table kernels (bucket_list.py).
//
// The reference appends one value at a time through a CAS state machine on
// the key's 64-bit list handle (state | count | tail, :61-70), growing the
// chain bucket by bucket from a bump arena (:228-294).  A GPU batch instead
// aggregates all appends of one key first, so each key's handle moves ONCE
// per batch with no contention:
//   1. find_or_claim every key in the key store                (single.cu K1 MODE 1)
//   2. rank[i] = atomicAdd(batch_count[slot])                  k_bucket_rank
//   3. the batch's distinct key-store slots (rank 0), compacted in batch order
//      (flag + exclusive scan)                                 k_bucket_touch
//   4. per touched slot: how many values fit, how many arena
//      cells the new buckets need                              k_bucket_need
//   5. exclusive scan of the needs -> contention-free bump offsets (prims.cu)
//   6. per touched slot: carve its buckets, link the headers, publish the
//      new handle (READY, or FULL once the pool/count limit hits) k_bucket_alloc
//      (pool exhaustion falls back to the reference's bucket-by-bucket order in
//      k_bucket_alloc_seq, so OUT_OF_MEMORY stays per key and sticky)
// Every pass is O(batch): steps 3-6 run over the touched-slot list, never over the
// key store's capacity (an element insert into a 2^23-key store is a handful of tiny
// launches, not three sweeps of the store).
//   6. every pair writes its value at the arena cell its index maps to    k_bucket_write
// The chain geometry is a pure function of the growth policy (:11-15), so the
// arena cell of value index v is computed, never searched.
#include "bucket.cuh"
#include "dispatch.cuh"
#include "probe.cuh"

namespace chb {

template <typename K>
__device__ __forceinline__ uint64_t* handle_ptr(const TableRef& T, Layout lay, uint64_t s) {
  if (lay == SOA) return static_cast<uint64_t*>(T.vals) + s;
  return &static_cast<CellT<K, uint64_t>*>(T.slots)[s].v;
}

__global__ void k_bucket_rank(const int64_t* __restrict__ slots, uint64_t n, uint32_t* __restrict__ bcnt,
                              uint32_t* __restrict__ rank) {
  const uint64_t stride = gridDim.x * (uint64_t)blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t s = slots[i];
    if (s >= 0) rank[i] = atomicAdd(bcnt + s, 1u);
  }
}

// touched[pos[i]] = slots[i] for the first element of every slot (rank 0), batch order
__global__ void k_bucket_flag(const int64_t* __restrict__ slots, const uint32_t* __restrict__ rank, uint64_t n,
                              uint32_t* __restrict__ flag) {
  const uint64_t stride = gridDim.x * (uint64_t)blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    flag[i] = (slots[i] >= 0 && rank[i] == 0) ? 1u : 0u;
}
__global__ void k_bucket_touch(const int64_t* __restrict__ slots, const uint32_t* __restrict__ flag,
                               const uint64_t* __restrict__ pos, uint64_t n, uint64_t* __restrict__ touched) {
  const uint64_t stride = gridDim.x * (uint64_t)blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    if (flag[i]) touched[pos[i]] = (uint64_t)slots[i];
}

// need_out[i] for entry i: touched-list entry i < d (*d_touched), 0 up to n (the scan runs
// over n); without a list (touched == nullptr, batches larger than the key store) entry i
// is key-store slot i, i < n = capacity, untouched slots need 0
template <typename K>
__global__ void k_bucket_need(BucketRef B, Layout lay, const uint64_t* __restrict__ touched,
                              const uint64_t* __restrict__ d_touched, uint64_t n, uint64_t* __restrict__ need_out) {
  const uint64_t d = touched ? *d_touched : n;
  const uint64_t stride = gridDim.x * (uint64_t)blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    uint64_t need = 0;
    const uint64_t s = touched ? (i < d ? touched[i] : 0) : i;
    const uint32_t m = i < d ? B.bcnt[s] : 0u;
    if (m) {
      const uint64_t h = *handle_ptr<K>(B.T, lay, s);
      const uint64_t state = h >> (COUNT_BITS + TAIL_BITS), count = (h >> TAIL_BITS) & COUNT_MAX,
                     tail = h & TAIL_MAX;
      BucketInfo in;
      in.region = 0;
      in.tail_old = tail;
      in.c0 = state == H_UNINIT ? 0 : (uint32_t)count;
      in.overflow = 0;
      in.pad = 0;
      if (state == H_FULL) {  // sticky (:245-246)
        in.fit = 0;
        in.new_count = count;
      } else {
        uint64_t fit = m;
        if (in.c0 + fit > COUNT_MAX) {  // count >= COUNT_MAX -> FULL (:261-264)
          fit = COUNT_MAX - in.c0;
          in.overflow = 1;
        }
        in.fit = (uint32_t)fit;
        in.new_count = in.c0 + fit;
        const uint64_t have = B.gr.before(B.gr.buckets_for(in.c0));  // capacity of the current chain
        if (in.new_count > have) {
          const uint64_t b0 = B.gr.buckets_for(in.c0);  // first new bucket
          const uint64_t b1 = B.gr.buckets_for(in.new_count) - 1;
          need = B.gr.cells(b0, b1);
        }
      }
      in.need = need;
      B.info[s] = in;
    }
    need_out[i] = need;
  }
}

// Carve the new buckets of slot s starting at arena offset `region`, link the
// headers, return the tail.  b0..b1 are the new bucket indices.
__device__ __forceinline__ uint64_t link_buckets(const BucketRef& B, uint64_t region, uint64_t b0, uint64_t b1,
                                                 uint64_t prev_tail, int vbytes) {
  uint64_t base = region, prev = prev_tail;
  for (uint64_t b = b0; b <= b1; ++b) {
    if (b > 0) {  // leading cell references the previous bucket (:288)
      if (vbytes == 8) static_cast<uint64_t*>(B.arena)[base] = prev;
      else static_cast<uint32_t*>(B.arena)[base] = (uint32_t)prev;
    }
    prev = base;
    base += B.gr.size(b) + (b > 0 ? 1 : 0);
  }
  return prev;
}

template <typename K>
__global__ void k_bucket_alloc(BucketRef B, Layout lay, const uint64_t* __restrict__ touched,
                               const uint64_t* __restrict__ d_touched, const uint64_t* __restrict__ alloc_off,
                               int vbytes) {
  const uint64_t d = touched ? *d_touched : B.T.c;
  const uint64_t stride = gridDim.x * (uint64_t)blockDim.x;
  const unsigned long long bump0 = *B.bump;
  long long values = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < d; i += stride) {
    const uint64_t s = touched ? touched[i] : i;
    if (!touched && !B.bcnt[s]) continue;
    BucketInfo in = B.info[s];
    uint64_t* hp = handle_ptr<K>(B.T, lay, s);
    const uint64_t h = *hp;
    if ((h >> (COUNT_BITS + TAIL_BITS)) == H_FULL) {  // sticky FULL: nothing fits
      B.winfo[s] = make_ulonglong2(in.region | ((uint64_t)in.c0 << TAIL_BITS), in.tail_old);
      continue;
    }
    uint64_t tail = in.tail_old;
    if (in.need) {
      const uint64_t off = bump0 + alloc_off[i];
      if (off + in.need > B.pool_cap) {  // pool exhausted from here on: sequential fallback
        B.info[s].fit = FIT_DEFERRED;
        atomicMin(B.first_fail, (unsigned long long)i);
        continue;
      }
      const uint64_t b0 = B.gr.buckets_for(in.c0);
      const uint64_t b1 = B.gr.buckets_for(in.new_count) - 1;
      tail = link_buckets(B, off, b0, b1, in.tail_old, vbytes);
      B.info[s].region = off;
      in.region = off;
    }
    B.winfo[s] = make_ulonglong2(in.region | ((uint64_t)in.c0 << TAIL_BITS),
                                 in.tail_old | ((uint64_t)in.fit << TAIL_BITS));
    *hp = pack_handle(in.overflow ? H_FULL : H_READY, in.new_count, tail);
    values += in.fit;
  }
  const long long v[1] = {values};
  long long* const dst[1] = {&B.T.ctr->total_values};
  cta_add<1>(v, dst);
}

// Pool exhausted: from the first failing touched slot on (batch order of the keys' first
// values), allocate bucket by bucket exactly like the reference's sequential appends
// (:252-255, :283-287).
template <typename K>
__global__ void k_bucket_alloc_seq(BucketRef B, Layout lay, const uint64_t* __restrict__ touched,
                                   const uint64_t* __restrict__ d_touched, uint64_t n,
                                   const uint64_t* __restrict__ alloc_off, int vbytes) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const unsigned long long ff = *B.first_fail;
  const unsigned long long bump0 = *B.bump;
  const uint64_t d = touched ? *d_touched : B.T.c;
  if (ff == ~0ull) {  // everything fit: advance the bump by the total
    *B.bump = bump0 + alloc_off[n];
    B.T.ctr->pool_used += alloc_off[n];
    return;
  }
  uint64_t cursor = bump0 + alloc_off[ff];
  long long values = 0;
  for (uint64_t i = ff; i < d; ++i) {
    const uint64_t s = touched ? touched[i] : i;
    if ((!touched && !B.bcnt[s]) || B.info[s].fit != FIT_DEFERRED) continue;
    BucketInfo in = B.info[s];
    uint64_t* hp = handle_ptr<K>(B.T, lay, s);
    const uint64_t b0 = B.gr.buckets_for(in.c0);
    const uint64_t b1 = B.gr.buckets_for(in.new_count) - 1;
    uint64_t prev = in.tail_old, cap = B.gr.before(b0), region = cursor;
    bool failed = false;
    for (uint64_t b = b0; b <= b1; ++b) {
      const uint64_t cells = B.gr.size(b) + (b > 0 ? 1 : 0);
      if (cursor + cells > B.pool_cap) { failed = true; break; }
      if (b > 0) {
        if (vbytes == 8) static_cast<uint64_t*>(B.arena)[cursor] = prev;
        else static_cast<uint32_t*>(B.arena)[cursor] = (uint32_t)prev;
      }
      prev = cursor;
      cursor += cells;
      cap += B.gr.size(b);
    }
    const uint64_t fit = failed ? (cap > in.c0 ? cap - in.c0 : 0) : in.fit;
    const uint64_t count = in.c0 + (fit < in.fit ? fit : in.fit);
    B.info[s].fit = (uint32_t)(fit < in.fit ? fit : in.fit);
    B.info[s].region = region;
    B.winfo[s] = make_ulonglong2(region | ((uint64_t)in.c0 << TAIL_BITS),
                                 in.tail_old | ((uint64_t)(fit < in.fit ? fit : in.fit) << TAIL_BITS));
    const bool full = failed || in.overflow;
    // an UNINITIALIZED key whose first bucket does not fit becomes FULL(0, 0) (:254)
    *hp = pack_handle(full ? H_FULL : H_READY, count, count == 0 ? 0 : prev);
    values += B.info[s].fit;
  }
  B.T.ctr->pool_used += cursor - bump0;
  B.T.ctr->total_values += values;
  *B.bump = cursor;
}

template <typename V>
__global__ void k_bucket_write(BucketRef B, const int64_t* __restrict__ slots, const uint32_t* __restrict__ rank,
                               const V* __restrict__ vals, uint64_t n, uint8_t* __restrict__ status) {
  // growth prefix sums in shared memory when the table is short (a binary search per
  // value over global memory dominated this pass)
  constexpr uint32_t SM_SUMS = 2048;
  __shared__ uint64_t s_sums[SM_SUMS];
  Growth gr = B.gr;
  if (gr.m <= SM_SUMS) {
    for (uint32_t i = threadIdx.x; i < gr.m; i += blockDim.x) s_sums[i] = __ldg(B.gr.sums + i);
    __syncthreads();
    gr.sums = s_sums;
  }
  const uint64_t stride = gridDim.x * (uint64_t)blockDim.x;
  V* arena = static_cast<V*>(B.arena);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t s = slots[i];
    if (s < 0) continue;  // INVALID_KEY / TABLE_FULL from the key store stay
    const ulonglong2 wi = B.winfo[s];  // 16 B: region | c0, tail_old | fit
    const uint64_t region = wi.x & TAIL_MAX, tail_old = wi.y & TAIL_MAX;
    const uint32_t c0 = (uint32_t)(wi.x >> TAIL_BITS), fit = (uint32_t)(wi.y >> TAIL_BITS);
    const uint32_t r = rank[i];
    if (r >= fit) {
      status[i] = ST_OOM;
      continue;
    }
    const uint64_t v = (uint64_t)c0 + r;  // value index in the key's chain
    const uint64_t b = gr.buckets_for_gen(v + 1) - 1;
    const uint64_t within = v - gr.before_gen(b);
    uint64_t base;
    const uint64_t b_new0 = gr.buckets_for_gen(c0);
    if (c0 > 0 && b + 1 == b_new0) {
      base = tail_old;  // room left in the old tail bucket (:266-276)
    } else {
      base = region + (gr.before_gen(b) - gr.before_gen(b_new0)) + (b - b_new0) - ((b_new0 == 0 && b > 0) ? 1 : 0);
    }
    arena[base + (b > 0 ? 1 : 0) + within] = ld_stream(vals + i);
    status[i] = ST_INSERTED;
  }
}

__global__ void k_bucket_reset(const int64_t* __restrict__ slots, const uint32_t* __restrict__ rank, uint64_t n,
                               uint32_t* __restrict__ bcnt) {
  const uint64_t stride = gridDim.x * (uint64_t)blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t s = slots[i];
    if (s >= 0 && rank[i] == 0) bcnt[s] = 0;
  }
}

// counts from handles (:320-326): the lookup wrote handle 0 for absent keys
__global__ void k_handle_counts(const uint64_t* __restrict__ handles, uint64_t n, uint32_t* __restrict__ counts) {
  const uint64_t stride = gridDim.x * (uint64_t)blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    counts[i] = (uint32_t)((handles[i] >> TAIL_BITS) & COUNT_MAX);
}

// chain walk, tail -> head through the prev links, values emitted head first (:328-355)
template <typename V>
__global__ void k_bucket_walk(BucketRef B, const uint64_t* __restrict__ handles, uint64_t n,
                              const uint64_t* __restrict__ offsets, V* __restrict__ out) {
  const uint64_t stride = gridDim.x * (uint64_t)blockDim.x;
  const V* arena = static_cast<const V*>(B.arena);
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t want = offsets[i + 1] - offsets[i];
    if (!want) continue;
    const uint64_t h = handles[i];
    if ((h >> 62) == 1) {
      // BLOCKED (bucket_list.py:300-318): batches are stream-ordered, so no insert of this
      // library is ever in flight here -- the handle was left blocked from outside and
      // would never become ready.  The reference raises ContentionTimeout after its retry
      // budget; the sticky device error bit 0 makes the host raise the same.
      atomicOr(&B.T.ctr->error, 1ull);
      continue;
    }
    const uint64_t count = (h >> TAIL_BITS) & COUNT_MAX;
    const uint64_t take_all = count < want ? count : want;  // raced writer: keep the segment length
    uint64_t base = h & TAIL_MAX;
    const uint64_t m = B.gr.buckets_for(count);
    for (uint64_t bb = m; bb-- > 0;) {
      if (base >= B.pool_cap) {  // a chain reference outside the arena: corrupt handle / header
        atomicOr(&B.T.ctr->error, 2ull);
        break;
      }
      const uint64_t first = B.gr.before(bb);
      if (first < take_all) {
        const uint64_t sz = B.gr.size(bb);
        const uint64_t take = (take_all - first) < sz ? (take_all - first) : sz;
        const uint64_t src = base + (bb > 0 ? 1 : 0);
        for (uint64_t k = 0; k < take && src + k < B.pool_cap; ++k) out[offsets[i] + first + k] = arena[src + k];
      }
      if (bb > 0) base = (uint64_t)arena[base];
    }
  }
}

// ------------------------------------------------------------ host side
size_t bucket_insert_scratch_bytes(uint64_t n, uint64_t c) {
  auto a = [](size_t b) { return (b + 255) & ~(size_t)255; };
  const uint64_t m = n < c ? n : c;
  return a(n * 8) + a(n * 4) + a(n * 4) + a((n + 1) * 8) + a(n * 8) + a(m * 8) + a((m + 1) * 8) +
         a(exclusive_scan_scratch_bytes((n > m ? n : m) + 1)) + 256;
}

int bucket_insert(const Launch& lc, const BucketRef& B, const TypeSel& ts, const void* keys, const void* vals,
                  uint64_t n, uint8_t* status, void* scratch, size_t scratch_bytes) {
  char* q = static_cast<char*>(scratch);
  auto take = [&](size_t b) {
    char* r = q;
    q += (b + 255) & ~(size_t)255;
    return (void*)r;
  };
  // small batches work over the list of the slots they touch; batches of at least the
  // key store's capacity sweep the slots instead (O(min(n, c)) either way)
  const bool use_list = n < B.T.c;
  const uint64_t m = use_list ? n : B.T.c;  // entries of the need / scan / alloc passes
  int64_t* slots = (int64_t*)take(n * 8);
  uint32_t* rank = (uint32_t*)take(n * 4);
  uint32_t* flag = (uint32_t*)take(use_list ? n * 4 : 4);
  uint64_t* pos = (uint64_t*)take(use_list ? (n + 1) * 8 : 8);  // pos[n] = touched slots
  uint64_t* touched = (uint64_t*)take(use_list ? n * 8 : 8);
  uint64_t* need = (uint64_t*)take(m * 8);
  uint64_t* alloc_off = (uint64_t*)take((m + 1) * 8);
  const size_t scan_bytes = exclusive_scan_scratch_bytes((n > m ? n : m) + 1);
  void* scan_scratch = take(scan_bytes);
  if ((size_t)(q - static_cast<char*>(scratch)) > scratch_bytes) {
    set_error("bucket insert scratch too small");
    return -22;
  }
  const Layout lay = (Layout)ts.layout;
  TypeSel kts = ts;
  kts.vbytes = 8;  // key store values are 64-bit handles
  int rc = single_insert(lc, B.T, kts, keys, nullptr, n, status, slots, 1);
  if (rc) return rc;
  rc = launch_persistent(lc, (const void*)k_bucket_rank, n, 1, [&](dim3 g, dim3 b) {
    k_bucket_rank<<<g, b, 0, lc.stream>>>(slots, n, B.bcnt, rank);
  });
  if (use_list) {
    if (!rc) rc = launch_persistent(lc, (const void*)k_bucket_flag, n, 1, [&](dim3 g, dim3 b) {
      k_bucket_flag<<<g, b, 0, lc.stream>>>(slots, rank, n, flag);
    });
    if (!rc) rc = exclusive_scan_u32(lc, flag, n, pos, scan_scratch, scan_bytes);
    if (!rc) rc = launch_persistent(lc, (const void*)k_bucket_touch, n, 1, [&](dim3 g, dim3 b) {
      k_bucket_touch<<<g, b, 0, lc.stream>>>(slots, flag, pos, n, touched);
    });
  }
  if (rc) return rc;
  const uint64_t* d_touched = use_list ? pos + n : nullptr;
  if (!use_list) touched = nullptr;
  const bool k4 = ts.kbytes == 4;
  auto need_k = k4 ? (const void*)k_bucket_need<uint32_t> : (const void*)k_bucket_need<uint64_t>;
  rc = launch_persistent(lc, need_k, m, 1, [&](dim3 g, dim3 b) {
    if (k4) k_bucket_need<uint32_t><<<g, b, 0, lc.stream>>>(B, lay, touched, d_touched, m, need);
    else k_bucket_need<uint64_t><<<g, b, 0, lc.stream>>>(B, lay, touched, d_touched, m, need);
  });
  if (rc) return rc;
  rc = exclusive_scan_u64(lc, need, m, alloc_off, scan_scratch, scan_bytes);
  if (rc) return rc;
  rc = cuda_check(cudaMemsetAsync(B.first_fail, 0xff, sizeof(unsigned long long), lc.stream), "memset");
  if (rc) return rc;
  auto alloc_k = k4 ? (const void*)k_bucket_alloc<uint32_t> : (const void*)k_bucket_alloc<uint64_t>;
  rc = launch_persistent(lc, alloc_k, m, 1, [&](dim3 g, dim3 b) {
    if (k4) k_bucket_alloc<uint32_t><<<g, b, 0, lc.stream>>>(B, lay, touched, d_touched, alloc_off, ts.vbytes);
    else k_bucket_alloc<uint64_t><<<g, b, 0, lc.stream>>>(B, lay, touched, d_touched, alloc_off, ts.vbytes);
  });
  if (rc) return rc;
  if (k4) k_bucket_alloc_seq<uint32_t><<<1, 32, 0, lc.stream>>>(B, lay, touched, d_touched, m, alloc_off, ts.vbytes);
  else k_bucket_alloc_seq<uint64_t><<<1, 32, 0, lc.stream>>>(B, lay, touched, d_touched, m, alloc_off, ts.vbytes);
  count_launch();
  rc = cuda_check(cudaGetLastError(), "bucket alloc seq");
  if (rc) return rc;
  if (ts.vbytes == 8) {
    rc = launch_persistent(lc, (const void*)k_bucket_write<uint64_t>, n, 1, [&](dim3 g, dim3 b) {
      k_bucket_write<uint64_t><<<g, b, 0, lc.stream>>>(B, slots, rank, (const uint64_t*)vals, n, status);
    });
  } else {
    rc = launch_persistent(lc, (const void*)k_bucket_write<uint32_t>, n, 1, [&](dim3 g, dim3 b) {
      k_bucket_write<uint32_t><<<g, b, 0, lc.stream>>>(B, slots, rank, (const uint32_t*)vals, n, status);
    });
  }
  if (rc) return rc;
  return launch_persistent(lc, (const void*)k_bucket_reset, n, 1, [&](dim3 g, dim3 b) {
    k_bucket_reset<<<g, b, 0, lc.stream>>>(slots, rank, n, B.bcnt);
  });
}

int bucket_counts(const Launch& lc, const uint64_t* handles, uint64_t n, uint32_t* counts) {
  return launch_persistent(lc, (const void*)k_handle_counts, n, 1, [&](dim3 g, dim3 b) {
    k_handle_counts<<<g, b, 0, lc.stream>>>(handles, n, counts);
  });
}

int bucket_walk(const Launch& lc, const BucketRef& B, int vbytes, const uint64_t* handles, uint64_t n,
                const uint64_t* offsets, void* out) {
  if (vbytes == 8)
    return launch_persistent(lc, (const void*)k_bucket_walk<uint64_t>, n, 1, [&](dim3 g, dim3 b) {
      k_bucket_walk<uint64_t><<<g, b, 0, lc.stream>>>(B, handles, n, offsets, (uint64_t*)out);
    });
  return launch_persistent(lc, (const void*)k_bucket_walk<uint32_t>, n, 1, [&](dim3 g, dim3 b) {
    k_bucket_walk<uint32_t><<<g, b, 0, lc.stream>>>(B, handles, n, offsets, (uint32_t*)out);
  });
}

}  // namespace chb
