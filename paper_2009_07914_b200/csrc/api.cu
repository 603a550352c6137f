// api.cu -- the extern "C" boundary (include/coophash_b200.h).
//
// Owns table memory (cudaMalloc), orders every operation on a table after the
// previous one (a per-table event), validates configurations the way the
// reference constructors do, and turns CUDA errors into negative codes with a
// thread-local message.  No exception crosses the ABI.
#include <atomic>
#include <cerrno>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/coophash_b200.h"
#include "bucket.cuh"
#include "dispatch.cuh"

namespace chb {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
static std::atomic<uint64_t> g_launches{0};
void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// prims.cu / bucket.cu entry points
int mix64_array(const Launch& lc, const uint64_t* in, uint64_t n, uint64_t seed, uint64_t* out);
int route_part32(const Launch& lc, const uint32_t* keys, const uint32_t* vals, uint64_t n, uint32_t shards,
                 uint64_t cap, uint32_t* pos, unsigned long long* counts, uint32_t* keys_out, uint32_t* vals_out,
                 int* flag);
int multi_split(const Launch& lc, const void* keys, int kbytes, const void* vals, int vbytes, uint64_t n,
                uint32_t shards, void* perm, int perm_bytes, uint64_t* offsets, void* keys_out, void* vals_out,
                void* scratch, size_t scratch_bytes);
int permute32(const Launch& lc, const void* src, int elem_bytes, const uint32_t* perm, uint64_t n, void* dst,
              bool scatter);
size_t split_scratch_bytes(uint64_t n, uint32_t shards);
int permute(const Launch& lc, const void* src, int elem_bytes, const uint64_t* perm, uint64_t n, void* dst,
            bool scatter);
int segment_copy(const Launch& lc, const void* src, int elem_bytes, const uint64_t* src_off, const uint64_t* idx,
                 uint64_t n, const uint64_t* dst_off, void* dst);

int bucket_insert(const Launch& lc, const BucketRef& B, const TypeSel& ts, const void* keys, const void* vals,
                  uint64_t n, uint8_t* status, void* scratch, size_t scratch_bytes);
size_t bucket_insert_scratch_bytes(uint64_t n, uint64_t c);
int bucket_counts(const Launch& lc, const uint64_t* handles, uint64_t n, uint32_t* counts);
struct LocPlan {
  int shift;
  uint32_t regions;
  uint64_t tiles;
};
LocPlan loc_plan(const TableRef& T, uint64_t n, int bytes_per_slot);
size_t loc_scratch_bytes(const LocPlan& p);
int loc_partition(const Launch& lc, const TableRef& T, const LocPlan& p, int kbytes, int vbytes, const void* keys,
                  const void* vals, uint64_t n, void* keys_out, void* vals_out, uint16_t* inv, void* scratch,
                  size_t scratch_bytes);
int loc_unpermute(const Launch& lc, const LocPlan& p, uint64_t n, const uint16_t* inv, void* scratch,
                  size_t scratch_bytes, const void* pa, void* oa, int abytes, const void* pb, void* ob, int bbytes);
bool staged_supported(const TableRef& T, uint64_t n);
size_t staged_scratch_bytes(const TableRef& T, uint64_t n, bool insert);
int staged_insert(const Launch& lc, const TableRef& T, const TypeSel& ts, const void* keys, const void* vals,
                  uint64_t n, uint8_t* status, void* scratch, int fresh);
int staged_erase(const Launch& lc, const TableRef& T, const TypeSel& ts, const void* keys, uint64_t n,
                 uint8_t* erased, void* scratch);
int staged_lookup(const Launch& lc, const TableRef& T, const TypeSel& ts, const void* keys, uint64_t n,
                  void* vals_out, uint8_t* found, void* scratch);
size_t mgroup_scratch_bytes(uint64_t n, int kbytes, int vbytes);
int multi_insert_grouped(const Launch& lc, const TableRef& T, const TypeSel& ts, const void* keys, const void* vals,
                         uint64_t n, uint8_t* status, void* scratch, size_t scratch_bytes);
int bucket_walk(const Launch& lc, const BucketRef& B, int vbytes, const uint64_t* handles, uint64_t n,
                const uint64_t* offsets, void* out);
int kmer_sketch(const Launch& lc, const uint8_t* text, const uint64_t* win_start, const uint32_t* win_len,
                const uint32_t* win_tag, uint64_t n_windows, int k, uint32_t sketch, uint64_t* km_out,
                uint32_t* tag_out, uint64_t* d_count, void* scratch, size_t scratch_bytes, uint64_t total_len);
size_t kmer_scratch_bytes(uint64_t n_windows, uint32_t sketch, uint64_t total_len);

}  // namespace chb

using namespace chb;

namespace {
// CH_STAGED_ERASE=0: bulk erases of staged-size batches through the direct COPS kernel
const bool g_staged_erase = [] {
  const char* e = getenv("CH_STAGED_ERASE");
  return !(e && e[0] == '0');
}();
constexpr uint32_t kStashS = 64;  // values stashed per query by the multi-value count pass
// CH_MULTI_STASH=0: the retrieve pass always walks again
const bool g_multi_stash = [] {
  const char* e = getenv("CH_MULTI_STASH");
  return !(e && e[0] == '0');
}();
}  // namespace

struct ch_table {
  ch_config cfg;
  TypeSel ts;          // storage types of the slot array
  TableRef T;
  int kbytes, vbytes;  // user-visible value width (bucket: arena value width)
  size_t slot_bytes = 0, val_bytes = 0;
  DevCounters* ctr = nullptr;
  uint64_t host_ops = 0;  // ops accounted on the host (count passes)
  // bucket list
  void* arena = nullptr;
  unsigned long long* bump = nullptr;  // also holds first_fail at [1]
  uint32_t* bcnt = nullptr;
  BucketInfo* info = nullptr;
  ulonglong2* winfo = nullptr;
  uint64_t* gsizes = nullptr;
  uint64_t* gsums = nullptr;
  uint64_t gm = 0;
  cudaEvent_t last = nullptr;
  std::mutex mu;
  int sms = 148;
  // big-batch schedule: 0 auto, 1 direct, 2 L2 region order (locality.cu),
  // 3 shared-memory staged regions (staged.cu, packed 32|32 tables)
  int loc_mode = 0;
  int group_mode = 0;  // multi-value bulk insert: 0 grouped for n >= 4096, 1 per pair
  bool timing = false;
  KernelTimer timer;
  // ch_clear of a packed table that bulk inserts stage (>= 256 MiB) defers the memset: the next
  // staged insert starts every region empty and writes every region (staged.cu, fresh); any other
  // operation performs the clear first (Ordered, ch_read_slot_range).  CH_LAZY_CLEAR=0: always eager.
  bool pending_clear = false;
  // multi-value count -> retrieve: the count pass stashes the first kStashS values of every short
  // chain (multi.cu, MultiStashMeta); the next call, if it is ch_multi_retrieve of the same keys
  // buffer and count, copies them instead of walking again.  Any other call invalidates it.
  void* stash = nullptr;
  size_t stash_cap = 0;
  bool stash_valid = false;
  const void* stash_keys = nullptr;
  uint64_t stash_n = 0;
};

namespace {

struct DeviceGuard {
  int prev = -1;
  bool ok = true;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) ok = cudaSetDevice(dev) == cudaSuccess;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

int check(cudaError_t e, const char* what) { return cuda_check(e, what); }

// Every op on a table runs after the previous one, on the caller's stream.
struct Ordered {
  ch_table* t;
  cudaStream_t s;
  Launch lc;
  std::lock_guard<std::mutex> lock;
  DeviceGuard dev;
  int pre = 0;  // a deferred clear that failed to run
  // lazy_ok: the operation handles a pending clear itself (a staged insert)
  Ordered(ch_table* t_, void* stream, bool lazy_ok = false)
      : t(t_), s((cudaStream_t)stream), lock(t_->mu), dev(t_->cfg.device) {
    lc.stream = s;
    lc.device = t->cfg.device;
    lc.sms = t->sms;
    lc.timer = t->timing ? &t->timer : nullptr;
    t->stash_valid = false;  // consumed or invalidated by every operation (ch_multi_retrieve)
    cudaStreamWaitEvent(s, t->last, 0);
    if (t->pending_clear && !lazy_ok) {
      Launch c = lc;
      c.timer = nullptr;
      pre = single_clear(c, t->T, t->ts);
      t->pending_clear = false;
    }
  }
  int done(int rc) {
    cudaError_t e = cudaEventRecord(t->last, s);
    if (pre) return pre;
    if (rc) return rc;
    return check(e, "event record");
  }
};

struct Scratch {  // stream-ordered transient device memory
  cudaStream_t s;
  std::vector<void*> bufs;
  explicit Scratch(cudaStream_t s_) : s(s_) {}
  void* get(size_t bytes) {
    void* p = nullptr;
    if (cudaMallocAsync(&p, bytes ? bytes : 8, s) != cudaSuccess) return nullptr;
    bufs.push_back(p);
    return p;
  }
  ~Scratch() {
    for (void* p : bufs) cudaFreeAsync(p, s);
  }
};

bool pow2_group(int g) { return g == 1 || g == 2 || g == 4 || g == 8 || g == 16 || g == 32; }

// exact growth sizes: s_i = ceil(num/den * s_{i-1}) until the sums cover COUNT_MAX
bool growth_table(uint64_t s0, uint64_t num, uint64_t den, std::vector<uint64_t>& sizes, std::vector<uint64_t>& sums) {
  const uint64_t count_max = (1ull << 20) - 1;
  uint64_t s = s0, acc = 0;
  while (acc < count_max) {
    sizes.push_back(s);
    acc += s;
    sums.push_back(acc);
    unsigned __int128 nx = ((unsigned __int128)s * num + den - 1) / den;
    if (nx > ((unsigned __int128)1 << 62)) nx = (unsigned __int128)1 << 62;
    s = (uint64_t)nx;
  }
  return true;
}

BucketRef bucket_ref(ch_table* t) {
  BucketRef B;
  B.T = t->T;
  B.arena = t->arena;
  B.pool_cap = t->cfg.pool_capacity;
  B.bump = t->bump;
  B.bcnt = t->bcnt;
  B.info = t->info;
  B.winfo = t->winfo;
  B.first_fail = t->bump + 1;
  B.gr.sizes = t->gsizes;
  B.gr.sums = t->gsums;
  B.gr.m = t->gm;
  return B;
}

int slot_bytes_of(const ch_table* t) {
  if (t->cfg.layout == CH_PACKED) return 8;
  const int kb = t->ts.kbytes, vb = t->ts.vbytes;
  if (t->cfg.layout == CH_SOA) return kb + vb;
  return (kb == 8 || vb == 8) ? 16 : 8;
}

// Region-ordered execution pays off once the table outgrows L2 and the batch
// touches most of its lines (locality.cu).  Positions travel as uint32.
bool use_staged(const ch_table* t, uint64_t n) {
  if (t->cfg.layout != CH_PACKED || !staged_supported(t->T, n)) return false;
  if (t->loc_mode == 3) return true;
  if (t->loc_mode != 0) return false;
  const uint64_t bytes = t->T.c * 8ull;  // a table larger than L2, a batch covering it
  return bytes >= (256ull << 20) && n * 16 >= t->T.c;
}

bool use_locality(const ch_table* t, uint64_t n) {
  if (n == 0 || n >= (1ull << 32) || t->loc_mode == 1 || t->loc_mode == 3) return false;
  if (t->loc_mode == 2) return true;
  const uint64_t bytes = t->T.c * (uint64_t)slot_bytes_of(t);
  return bytes >= (256ull << 20) && n * 32 >= t->T.c;
}

void keep_pool_memory(int device) {
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
}

__global__ void k_zero_counters(DevCounters* c) { *c = DevCounters{}; }

__global__ void k_reset_probe(DevCounters* c) {
  c->ops = 0;
  c->attempts = 0;
  c->windows = 0;
  c->deferred = 0;
}

// element transitions of layout.py:140-243 on one slot
template <typename K, typename V>
__global__ void k_slot_op(TableRef T, int layout, int op, uint64_t slot, uint64_t expected, uint64_t desired,
                          uint64_t value, unsigned long long* out) {
  const K e = (K)T.e, t = (K)T.t;
  int w = 0;
  uint64_t seen_k = 0, seen_v = 0;
  if (layout == PACKED) {
    unsigned long long* p = static_cast<unsigned long long*>(T.slots) + slot;
    unsigned long long cur = *p;
    for (;;) {
      const uint32_t k = (uint32_t)cur;
      unsigned long long nxt = cur;
      bool apply = false;
      if (op == 0) { apply = k == (uint32_t)expected; nxt = (cur & ~0xFFFFFFFFull) | (uint32_t)desired; }
      else if (op == 1) { apply = k == (uint32_t)e || k == (uint32_t)t; nxt = (value << 32) | (uint32_t)desired; }
      else if (op == 3) { apply = k == (uint32_t)expected; nxt = (value << 32) | (uint32_t)t; }
      else if (op == 4) { apply = true; nxt = (value << 32) | k; }
      seen_k = k;
      seen_v = cur >> 32;
      if (!apply) break;
      const unsigned long long prev = atomicCAS(p, cur, nxt);
      if (prev == cur) { w = 1; break; }
      cur = prev;
    }
  } else {
    K* kp;
    V* vp;
    if (layout == SOA) { kp = static_cast<K*>(T.slots) + slot; vp = static_cast<V*>(T.vals) + slot; }
    else { auto* c = static_cast<CellT<K, V>*>(T.slots) + slot; kp = &c->k; vp = &c->v; }
    seen_k = *(volatile K*)kp;
    seen_v = *(volatile V*)vp;
    if (op == 0 || op == 3) {
      const K des = op == 0 ? (K)desired : t;
      const K prev = atomic_cas(kp, (K)expected, des);
      w = prev == (K)expected;
      seen_k = prev;
    } else if (op == 2) {
      const V prev = atomic_cas(vp, (V)expected, (V)desired);
      w = prev == (V)expected;
      seen_v = prev;
    } else if (op == 4) {
      *vp = (V)value;
      w = 1;
    } else if (op == 5) {
      w = 1;
    }
  }
  out[0] = (unsigned long long)w;
  out[1] = seen_k;
  out[2] = seen_v;
}

}  // namespace

extern "C" {

const char* ch_last_error(void) { return g_err.c_str(); }
uint64_t ch_kernel_launches(void) { return g_launches.load(); }
int ch_version(void) { return 1; }

int ch_create(ch_table** out, const ch_config* cfg) {
  if (!out || !cfg) return fail(CH_EINVAL, "null argument");
  *out = nullptr;
  const ch_config& c = *cfg;
  if (c.kind < CH_SINGLE || c.kind > CH_BUCKET) return fail(CH_EINVAL, "bad table kind");
  if (c.layout < CH_SOA || c.layout > CH_PACKED) return fail(CH_EINVAL, "bad layout");
  if (c.key_bits < 1 || c.key_bits > 64 || c.value_bits < 1 || c.value_bits > 64)
    return fail(CH_EINVAL, "key_bits / value_bits must be in [1, 64]");
  if (c.layout == CH_PACKED && (c.key_bits > 32 || c.value_bits > 32))
    return fail(CH_EINVAL, "packed layout needs 32-bit keys and values");
  if (c.kind == CH_BUCKET && c.layout == CH_PACKED)
    return fail(CH_EINVAL, "list handles need 64-bit value cells; use the soa or aos layout");
  if (!pow2_group(c.group_width)) return fail(CH_EINVAL, "group_width must be one of (1, 2, 4, 8, 16, 32)");
  if (c.p < 2) return fail(CH_EINVAL, "window count p must be a prime >= 2");
  if (c.p >= (1ull << 32)) return fail(CH_EINVAL, "window count p must be < 2^32 (capacity < 2^37 slots)");
  const uint64_t maxw = c.max_outer_attempts ? c.max_outer_attempts : c.p;
  if (maxw < 1 || maxw > c.p) return fail(CH_EINVAL, "max_outer_attempts must be in [1, p]");
  if (c.empty_key == c.tombstone_key) return fail(CH_EINVAL, "empty and tombstone sentinels must differ");
  const int kbytes = c.key_bits <= 32 ? 4 : 8;
  const int vbytes = c.value_bits <= 32 ? 4 : 8;
  if (kbytes == 4 && (c.empty_key > 0xFFFFFFFFull || c.tombstone_key > 0xFFFFFFFFull))
    return fail(CH_EINVAL, "sentinels do not fit the key width");
  if (c.kind == CH_BUCKET) {
    if (c.pool_capacity == 0) return fail(CH_EINVAL, "pool capacity must be positive");
    if (c.growth_s0 < 1) return fail(CH_EINVAL, "initial bucket size must be >= 1");
    if (c.growth_den == 0 || c.growth_num < c.growth_den) return fail(CH_EINVAL, "growth factor must be >= 1");
    if (vbytes == 4 && c.pool_capacity > 0xFFFFFFFFull)
      return fail(CH_EINVAL, "32-bit value arenas hold at most 2^32-1 cells");
    if (c.pool_capacity > (1ull << 42) - 1) return fail(CH_EINVAL, "pool capacity exceeds the 42-bit tail");
  }
  DeviceGuard dev(c.device);
  if (!dev.ok) return fail(CH_EINVAL, "bad device ordinal");

  ch_table* t = new (std::nothrow) ch_table();
  if (!t) return fail(CH_ENOMEM, "host allocation failed");
  t->cfg = c;
  t->cfg.max_outer_attempts = maxw;
  t->kbytes = kbytes;
  t->vbytes = vbytes;
  t->ts.layout = c.layout;
  t->ts.kbytes = kbytes;
  t->ts.vbytes = c.kind == CH_BUCKET ? 8 : vbytes;
  t->ts.g = c.group_width;
  cudaDeviceGetAttribute(&t->sms, cudaDevAttrMultiProcessorCount, c.device);

  const uint64_t cap = 32 * c.p;
  TableRef& T = t->T;
  T.c = cap;
  T.p = c.p;
  T.max_windows = maxw;
  T.e = c.empty_key;
  T.t = c.tombstone_key;
  T.modc = FastMod::make(cap);
  T.modpm1 = FastMod::make(c.p - 1);
  T.slots = T.vals = nullptr;

  auto cleanup = [&](int code, const std::string& msg) {
    ch_destroy(t);
    return fail(code, msg);
  };
  if (cudaEventCreateWithFlags(&t->last, cudaEventDisableTiming) != cudaSuccess)
    return cleanup(CH_EIO, "event create failed");
  const int sv = t->ts.vbytes;
  if (c.layout == CH_PACKED) t->slot_bytes = cap * 8;
  else if (c.layout == CH_SOA) { t->slot_bytes = cap * kbytes; t->val_bytes = cap * sv; }
  else t->slot_bytes = cap * (size_t)(kbytes == 8 || sv == 8 ? 16 : 8);
  if (cudaMalloc(&T.slots, t->slot_bytes) != cudaSuccess) return cleanup(CH_ENOMEM, "slot array allocation failed");
  if (t->val_bytes && cudaMalloc(&T.vals, t->val_bytes) != cudaSuccess)
    return cleanup(CH_ENOMEM, "value array allocation failed");
  if (cudaMalloc(&t->ctr, sizeof(DevCounters) + 64) != cudaSuccess) return cleanup(CH_ENOMEM, "counter allocation failed");
  T.ctr = t->ctr;
  T.work = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(t->ctr) + sizeof(DevCounters));

  if (c.kind == CH_BUCKET) {
    std::vector<uint64_t> sizes, sums;
    growth_table(c.growth_s0, c.growth_num, c.growth_den, sizes, sums);
    t->gm = sizes.size();
    if (cudaMalloc(&t->arena, c.pool_capacity * vbytes) != cudaSuccess) return cleanup(CH_ENOMEM, "arena allocation failed");
    if (cudaMalloc(&t->bump, 2 * sizeof(unsigned long long)) != cudaSuccess) return cleanup(CH_ENOMEM, "bump alloc");
    if (cudaMalloc(&t->bcnt, cap * sizeof(uint32_t)) != cudaSuccess) return cleanup(CH_ENOMEM, "batch count alloc");
    if (cudaMalloc(&t->info, cap * sizeof(BucketInfo)) != cudaSuccess) return cleanup(CH_ENOMEM, "bucket info alloc");
    if (cudaMalloc(&t->winfo, cap * sizeof(ulonglong2)) != cudaSuccess) return cleanup(CH_ENOMEM, "bucket info alloc");
    if (cudaMalloc(&t->gsizes, t->gm * 8) != cudaSuccess || cudaMalloc(&t->gsums, t->gm * 8) != cudaSuccess)
      return cleanup(CH_ENOMEM, "growth table alloc");
    if (cudaMemcpy(t->gsizes, sizes.data(), t->gm * 8, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(t->gsums, sums.data(), t->gm * 8, cudaMemcpyHostToDevice) != cudaSuccess)
      return cleanup(CH_EIO, "growth table upload failed");
  }
  keep_pool_memory(c.device);
  int rc = ch_clear(t, nullptr);
  if (rc) {
    std::string m = g_err;
    return cleanup(rc, m);
  }
  if (cudaDeviceSynchronize() != cudaSuccess) return cleanup(CH_EIO, "table init failed");
  *out = t;
  return CH_OK;
}

int ch_destroy(ch_table* t) {
  if (!t) return CH_OK;
  DeviceGuard dev(t->cfg.device);
  if (t->last) cudaEventSynchronize(t->last);
  cudaFree(t->T.slots);
  cudaFree(t->T.vals);
  cudaFree(t->ctr);
  cudaFree(t->arena);
  cudaFree(t->bump);
  cudaFree(t->bcnt);
  cudaFree(t->info);
  cudaFree(t->winfo);
  cudaFree(t->gsizes);
  cudaFree(t->gsums);
  cudaFree(t->stash);
  if (t->last) cudaEventDestroy(t->last);
  delete t;
  return CH_OK;
}

static bool g_lazy_clear = [] {
  const char* e = getenv("CH_LAZY_CLEAR");
  return !(e && e[0] == '0');
}();

int ch_clear(ch_table* t, void* stream) {
  if (!t) return fail(CH_EINVAL, "null table");
  Ordered o(t, stream, true);
  const bool lazy = g_lazy_clear && t->cfg.kind == CH_SINGLE && t->cfg.layout == CH_PACKED &&
                    t->T.c * 8ull >= (256ull << 20);
  int rc = 0;
  if (lazy) t->pending_clear = true;  // counters reset now, the slots by the next operation
  else {
    t->pending_clear = false;
    rc = single_clear(o.lc, t->T, t->ts);
  }
  if (!rc) {
    k_zero_counters<<<1, 1, 0, o.s>>>(t->ctr);
    count_launch();
    rc = check(cudaGetLastError(), "zero counters");
  }
  if (!rc && t->cfg.kind == CH_BUCKET) {
    rc = check(cudaMemsetAsync(t->bump, 0, 2 * sizeof(unsigned long long), o.s), "bump reset");
    if (!rc) rc = check(cudaMemsetAsync(t->bcnt, 0, t->T.c * sizeof(uint32_t), o.s), "batch count reset");
    if (!rc) rc = check(cudaMemsetAsync(t->arena, 0, t->cfg.pool_capacity * t->vbytes, o.s), "arena reset");
  }
  t->host_ops = 0;
  return o.done(rc);
}

int ch_kernel_timing(ch_table* t, int enable) {
  if (!t) return fail(CH_EINVAL, "null table");
  std::lock_guard<std::mutex> lock(t->mu);
  t->timing = enable != 0;
  return CH_OK;
}

int ch_kernel_time(ch_table* t, double* ms, uint64_t cap, uint64_t* launches) {
  if (!t || !launches) return fail(CH_EINVAL, "null argument");
  std::lock_guard<std::mutex> lock(t->mu);
  DeviceGuard dev(t->cfg.device);
  int rc = check(cudaEventSynchronize(t->last), "synchronize");
  uint64_t i = 0;
  for (auto& p : t->timer.ev) {
    float x = 0;
    if (!rc && cudaEventElapsedTime(&x, p.first, p.second) != cudaSuccess) x = -1;
    if (ms && i < cap) ms[i] = x;
    ++i;
    cudaEventDestroy(p.first);
    cudaEventDestroy(p.second);
  }
  *launches = t->timer.ev.size();
  t->timer.ev.clear();
  return rc;
}

int ch_set_locality(ch_table* t, int mode) {
  if (!t || mode < 0 || mode > 3)
    return fail(CH_EINVAL, "schedule must be 0 (auto), 1 (direct), 2 (L2 region order) or 3 (staged regions)");
  std::lock_guard<std::mutex> lock(t->mu);
  t->loc_mode = mode;
  return CH_OK;
}

int ch_set_multi_grouping(ch_table* t, int on) {
  if (!t) return fail(CH_EINVAL, "null table");
  std::lock_guard<std::mutex> lock(t->mu);
  t->group_mode = on ? 0 : 1;
  return CH_OK;
}

int ch_batch_schedule(ch_table* t, uint64_t n) {
  if (!t) return fail(CH_EINVAL, "null table");
  std::lock_guard<std::mutex> lock(t->mu);
  if (t->cfg.kind != CH_SINGLE) return 1;
  if (use_staged(t, n)) return 3;
  return use_locality(t, n) ? 2 : 1;
}

int ch_synchronize(ch_table* t) {
  if (!t) return fail(CH_EINVAL, "null table");
  DeviceGuard dev(t->cfg.device);
  return check(cudaEventSynchronize(t->last), "synchronize");
}

int ch_get_stats(ch_table* t, ch_stats* out) {
  if (!t || !out) return fail(CH_EINVAL, "null argument");
  std::lock_guard<std::mutex> lock(t->mu);
  DeviceGuard dev(t->cfg.device);
  int rc = check(cudaEventSynchronize(t->last), "synchronize");
  if (rc) return rc;
  DevCounters c;
  rc = check(cudaMemcpy(&c, t->ctr, sizeof(c), cudaMemcpyDeviceToHost), "read counters");
  if (rc) return rc;
  out->capacity = t->T.c;
  out->occupied = c.occupied;
  out->tombstones = c.tombstones;
  out->ops = c.ops + t->host_ops;
  out->attempts = c.attempts;
  out->windows = c.windows;
  out->total_values = c.total_values;
  out->pool_allocated = c.pool_used;
  out->device_error = c.error;
  out->deferred = c.deferred;
  return CH_OK;
}

int ch_get_config(ch_table* t, ch_config* out) {
  if (!t || !out) return fail(CH_EINVAL, "null argument");
  *out = t->cfg;
  return CH_OK;
}

int ch_reset_probe_counters(ch_table* t, void* stream) {
  if (!t) return fail(CH_EINVAL, "null table");
  Ordered o(t, stream);
  k_reset_probe<<<1, 1, 0, o.s>>>(t->ctr);
  count_launch();
  t->host_ops = 0;
  return o.done(check(cudaGetLastError(), "reset counters"));
}

int ch_insert(ch_table* t, const void* keys, const void* vals, uint64_t n, uint8_t* status, void* stream) {
  if (!t) return fail(CH_EINVAL, "null table");
  if (t->cfg.kind != CH_SINGLE) return fail(CH_EINVAL, "ch_insert needs a single-value table");
  if (n && (!keys || !vals || !status)) return fail(CH_EINVAL, "null buffer");
  const bool staged = use_staged(t, n);
  Ordered o(t, stream, staged);
  if (staged) {
    Scratch sc(o.s);
    void* p = sc.get(staged_scratch_bytes(t->T, n, true));
    if (!p) return o.done(fail(CH_ENOMEM, "scratch allocation failed"));
    const int fresh = t->pending_clear ? 1 : 0;
    t->pending_clear = false;
    return o.done(staged_insert(o.lc, t->T, t->ts, keys, vals, n, status, p, fresh));
  }
  if (!use_locality(t, n)) return o.done(single_insert(o.lc, t->T, t->ts, keys, vals, n, status, nullptr, 0));
  const LocPlan p = loc_plan(t->T, n, slot_bytes_of(t));
  Scratch sc(o.s);
  const int kb = t->ts.kbytes, vb = t->ts.vbytes;
  void* kp = sc.get(n * kb);
  void* vp = sc.get(n * vb);
  uint16_t* inv = (uint16_t*)sc.get(n * 2);
  uint8_t* sp = (uint8_t*)sc.get(n);
  const size_t lb = loc_scratch_bytes(p);
  void* ls = sc.get(lb);
  if (!kp || !vp || !inv || !sp || !ls) return o.done(fail(CH_ENOMEM, "scratch allocation failed"));
  int rc = loc_partition(o.lc, t->T, p, kb, vb, keys, vals, n, kp, vp, inv, ls, lb);
  if (!rc) rc = single_insert(o.lc, t->T, t->ts, kp, vp, n, sp, nullptr, 0);
  if (!rc) rc = loc_unpermute(o.lc, p, n, inv, ls, lb, sp, status, 1, nullptr, nullptr, 0);
  return o.done(rc);
}

int ch_find_or_claim(ch_table* t, const void* keys, uint64_t n, uint8_t* status, int64_t* slots, void* stream) {
  if (!t) return fail(CH_EINVAL, "null table");
  if (t->cfg.kind == CH_MULTI) return fail(CH_EINVAL, "find_or_claim needs a single-value or bucket table");
  if (n && (!keys || !status || !slots)) return fail(CH_EINVAL, "null buffer");
  Ordered o(t, stream);
  return o.done(single_insert(o.lc, t->T, t->ts, keys, nullptr, n, status, slots, 1));
}

int ch_retrieve(ch_table* t, const void* keys, uint64_t n, void* vals_out, uint8_t* found, void* stream) {
  if (!t) return fail(CH_EINVAL, "null table");
  if (t->cfg.kind != CH_SINGLE) return fail(CH_EINVAL, "ch_retrieve needs a single-value table");
  if (n && (!keys || !vals_out || !found)) return fail(CH_EINVAL, "null buffer");
  Ordered o(t, stream);
  if (use_staged(t, n)) {
    Scratch sc(o.s);
    void* p = sc.get(staged_scratch_bytes(t->T, n, false));
    if (!p) return o.done(fail(CH_ENOMEM, "scratch allocation failed"));
    return o.done(staged_lookup(o.lc, t->T, t->ts, keys, n, vals_out, found, p));
  }
  if (!use_locality(t, n))
    return o.done(single_lookup(o.lc, t->T, t->ts, keys, n, vals_out, found, nullptr, nullptr, nullptr, 0));
  const LocPlan p = loc_plan(t->T, n, slot_bytes_of(t));
  Scratch sc(o.s);
  const int kb = t->ts.kbytes, vb = t->ts.vbytes;
  void* kp = sc.get(n * kb);
  uint16_t* inv = (uint16_t*)sc.get(n * 2);
  void* vp = sc.get(n * vb);
  uint8_t* fp = (uint8_t*)sc.get(n);
  const size_t lb = loc_scratch_bytes(p);
  void* ls = sc.get(lb);
  if (!kp || !vp || !inv || !fp || !ls) return o.done(fail(CH_ENOMEM, "scratch allocation failed"));
  int rc = loc_partition(o.lc, t->T, p, kb, vb, keys, nullptr, n, kp, nullptr, inv, ls, lb);
  if (!rc) rc = single_lookup(o.lc, t->T, t->ts, kp, n, vp, fp, nullptr, nullptr, nullptr, 0);
  if (!rc) rc = loc_unpermute(o.lc, p, n, inv, ls, lb, vp, vals_out, vb, fp, found, 1);
  return o.done(rc);
}

int ch_erase(ch_table* t, const void* keys, uint64_t n, uint8_t* erased, void* stream) {
  if (!t) return fail(CH_EINVAL, "null table");
  if (t->cfg.kind != CH_SINGLE) return fail(CH_EINVAL, "erase is only defined for single-value tables");
  if (n && (!keys || !erased)) return fail(CH_EINVAL, "null buffer");
  Ordered o(t, stream);
  if (use_staged(t, n) && g_staged_erase) {
    Scratch sc(o.s);
    void* p = sc.get(staged_scratch_bytes(t->T, n, false));
    if (!p) return o.done(fail(CH_ENOMEM, "scratch allocation failed"));
    return o.done(staged_erase(o.lc, t->T, t->ts, keys, n, erased, p));
  }
  return o.done(single_lookup(o.lc, t->T, t->ts, keys, n, nullptr, erased, nullptr, nullptr, nullptr, 2));
}

int ch_find(ch_table* t, const void* keys, uint64_t n, int64_t* slots, uint32_t* attempts, uint32_t* windows,
            void* vals_out, void* stream) {
  if (!t) return fail(CH_EINVAL, "null table");
  if (n && (!keys || !slots)) return fail(CH_EINVAL, "null buffer");
  Ordered o(t, stream);
  return o.done(single_lookup(o.lc, t->T, t->ts, keys, n, vals_out, nullptr, slots, attempts, windows, 1));
}

int ch_multi_insert(ch_table* t, const void* keys, const void* vals, uint64_t n, uint8_t* status, void* stream) {
  if (!t) return fail(CH_EINVAL, "null table");
  if (t->cfg.kind != CH_MULTI) return fail(CH_EINVAL, "ch_multi_insert needs a multi-value table");
  if (n && (!keys || !vals || !status)) return fail(CH_EINVAL, "null buffer");
  Ordered o(t, stream);
  if (n >= 4096 && n < (1ull << 31) && t->group_mode != 1) {  // grouped: one walk per distinct key (mgroup.cu)
    Scratch sc(o.s);
    const size_t bytes = mgroup_scratch_bytes(n, t->ts.kbytes, t->ts.vbytes);
    void* p = sc.get(bytes);
    if (!p) return o.done(fail(CH_ENOMEM, "scratch allocation failed"));
    return o.done(multi_insert_grouped(o.lc, t->T, t->ts, keys, vals, n, status, p, bytes));
  }
  return o.done(multi_insert(o.lc, t->T, t->ts, keys, vals, n, status));
}

int ch_multi_count(ch_table* t, const void* keys, uint64_t n, uint32_t* counts, uint64_t* offsets, void* stream) {
  if (!t) return fail(CH_EINVAL, "null table");
  if (t->cfg.kind != CH_MULTI) return fail(CH_EINVAL, "ch_multi_count needs a multi-value table");
  if (!offsets || (n && (!keys || !counts))) return fail(CH_EINVAL, "null buffer");
  Ordered o(t, stream);
  Scratch sc(o.s);
  uint32_t* ll = (uint32_t*)sc.get(n * 4 + 16);
  unsigned long long* lc2 = (unsigned long long*)sc.get(multi_scan_counter_bytes());
  if (!ll || !lc2) return o.done(fail(CH_ENOMEM, "scratch allocation failed"));
  // the stash for the retrieve pass that usually follows (batches of >= 4096 queries, <= 4 GiB)
  void* stash = nullptr;
  void* meta = nullptr;
  const size_t sv = (size_t)n * kStashS * (size_t)t->vbytes, need = sv + (size_t)n * sizeof(MultiStashMeta) + 256;
  if (g_multi_stash && n >= 4096 && need <= (4ull << 30)) {
    if (t->stash_cap < need) {  // stream-ordered: the pool keeps the memory between calls
      if (t->stash) cudaFreeAsync(t->stash, o.s);
      t->stash = nullptr;
      t->stash_cap = 0;
      if (cudaMallocAsync(&t->stash, need, o.s) == cudaSuccess) t->stash_cap = need;
      else cudaGetLastError();  // no stash: the retrieve walks again
    }
    if (t->stash) {
      stash = t->stash;
      meta = (char*)t->stash + ((sv + 255) & ~(size_t)255);
    }
  }
  int rc = multi_scan(o.lc, t->T, t->ts, keys, n, counts, nullptr, nullptr, 0, ll, lc2, nullptr, stash, meta,
                      stash ? kStashS : 0u);
  if (!rc) {
    const size_t sb = exclusive_scan_scratch_bytes(n);
    void* p = sc.get(sb);
    rc = p ? exclusive_scan_u32(o.lc, counts, n, offsets, p, sb) : fail(CH_ENOMEM, "scratch allocation failed");
  }
  t->host_ops += n;
  if (!rc && stash) {
    t->stash_valid = true;
    t->stash_keys = keys;
    t->stash_n = n;
  }
  return o.done(rc);
}

int ch_multi_retrieve(ch_table* t, const void* keys, uint64_t n, const uint64_t* offsets, void* vals_out,
                      void* stream) {
  if (!t) return fail(CH_EINVAL, "null table");
  if (t->cfg.kind != CH_MULTI) return fail(CH_EINVAL, "ch_multi_retrieve needs a multi-value table");
  if (n && (!keys || !offsets)) return fail(CH_EINVAL, "null buffer");
  // the stash of the count pass just before, over the same keys buffer (the copy kernel also
  // checks every query's key and count against it)
  std::unique_lock<std::mutex> peek(t->mu);
  const bool use = t->stash_valid && t->stash && t->stash_keys == keys && t->stash_n == n && vals_out;
  peek.unlock();
  Ordered o(t, stream);
  t->host_ops += n;
  Scratch sc(o.s);
  uint32_t* ll = (uint32_t*)sc.get(n * 4 + 16);
  unsigned long long* lc2 = (unsigned long long*)sc.get(multi_scan_counter_bytes());
  if (!ll || !lc2) return o.done(fail(CH_ENOMEM, "scratch allocation failed"));
  const size_t sv = (size_t)n * kStashS * (size_t)t->vbytes;
  const int rc = multi_scan(o.lc, t->T, t->ts, keys, n, nullptr, offsets, vals_out, 1, ll, lc2, nullptr,
                            use ? t->stash : nullptr, use ? (char*)t->stash + ((sv + 255) & ~(size_t)255) : nullptr,
                            use ? kStashS : 0u);
  if (t->stash) {  // back to the pool once read (the next count pass takes it again)
    cudaFreeAsync(t->stash, o.s);
    t->stash = nullptr;
    t->stash_cap = 0;
  }
  return o.done(rc);
}

int ch_multi_retrieve_slots(ch_table* t, const void* keys, uint64_t n, const uint64_t* offsets, void* vals_out,
                            int64_t* slots_out, void* stream) {
  if (!t) return fail(CH_EINVAL, "null table");
  if (t->cfg.kind != CH_MULTI) return fail(CH_EINVAL, "ch_multi_retrieve_slots needs a multi-value table");
  if (n && (!keys || !offsets || !vals_out || !slots_out)) return fail(CH_EINVAL, "null buffer");
  Ordered o(t, stream);
  t->host_ops += n;
  Scratch sc(o.s);
  uint32_t* ll = (uint32_t*)sc.get(n * 4 + 16);
  unsigned long long* lc2 = (unsigned long long*)sc.get(multi_scan_counter_bytes());
  if (!ll || !lc2) return o.done(fail(CH_ENOMEM, "scratch allocation failed"));
  return o.done(multi_scan(o.lc, t->T, t->ts, keys, n, nullptr, offsets, vals_out, 1, ll, lc2, slots_out));
}

int ch_for_all(ch_table* t, void* keys_out, void* vals_out, int64_t* slots_out, uint64_t cap, uint64_t* d_count,
               void* stream) {
  if (!t) return fail(CH_EINVAL, "null table");
  Ordered o(t, stream);
  Scratch sc(o.s);
  const size_t sb = for_all_scratch_bytes(t->T.c);
  void* p = sc.get(sb);
  if (!p) return o.done(fail(CH_ENOMEM, "scratch allocation failed"));
  return o.done(table_for_all(o.lc, t->T, t->ts, keys_out, vals_out, slots_out, cap, d_count, p, sb));
}

int ch_reduce_live(ch_table* t, uint64_t* d_out, void* stream) {
  if (!t || !d_out) return fail(CH_EINVAL, "null argument");
  Ordered o(t, stream);
  return o.done(table_reduce(o.lc, t->T, t->ts, (unsigned long long*)d_out));
}

int ch_bucket_insert(ch_table* t, const void* keys, const void* vals, uint64_t n, uint8_t* status, void* stream) {
  if (!t) return fail(CH_EINVAL, "null table");
  if (t->cfg.kind != CH_BUCKET) return fail(CH_EINVAL, "ch_bucket_insert needs a bucket-list table");
  if (n && (!keys || !vals || !status)) return fail(CH_EINVAL, "null buffer");
  if (n == 0) return CH_OK;
  Ordered o(t, stream);
  Scratch sc(o.s);
  const size_t sb = bucket_insert_scratch_bytes(n, t->T.c);  // O(min(batch, key store))
  void* p = sc.get(sb);
  if (!p) return o.done(fail(CH_ENOMEM, "scratch allocation failed"));
  TypeSel ts = t->ts;
  ts.vbytes = t->vbytes;  // arena value width for the write pass
  return o.done(bucket_insert(o.lc, bucket_ref(t), ts, keys, vals, n, status, p, sb));
}

int ch_bucket_count(ch_table* t, const void* keys, uint64_t n, uint32_t* counts, uint64_t* offsets,
                    uint64_t* handles, void* stream) {
  if (!t) return fail(CH_EINVAL, "null table");
  if (t->cfg.kind != CH_BUCKET) return fail(CH_EINVAL, "ch_bucket_count needs a bucket-list table");
  if (!offsets || (n && (!keys || !counts || !handles))) return fail(CH_EINVAL, "null buffer");
  Ordered o(t, stream);
  Scratch sc(o.s);
  uint8_t* found = (uint8_t*)sc.get(n);
  const size_t sb = exclusive_scan_scratch_bytes(n);
  void* scan = sc.get(sb);
  if (!found || !scan) return o.done(fail(CH_ENOMEM, "scratch allocation failed"));
  int rc = single_lookup(o.lc, t->T, t->ts, keys, n, handles, found, nullptr, nullptr, nullptr, 0);
  if (!rc) rc = bucket_counts(o.lc, handles, n, counts);
  if (!rc) rc = exclusive_scan_u32(o.lc, counts, n, offsets, scan, sb);
  return o.done(rc);
}

int ch_bucket_retrieve(ch_table* t, const uint64_t* handles, uint64_t n, const uint64_t* offsets, void* vals_out,
                       void* stream) {
  if (!t) return fail(CH_EINVAL, "null table");
  if (t->cfg.kind != CH_BUCKET) return fail(CH_EINVAL, "ch_bucket_retrieve needs a bucket-list table");
  if (n && (!handles || !offsets)) return fail(CH_EINVAL, "null buffer");
  Ordered o(t, stream);
  return o.done(bucket_walk(o.lc, bucket_ref(t), t->vbytes, handles, n, offsets, vals_out));
}

int ch_read_slot_range(ch_table* t, uint64_t start, uint64_t count, void* h_keys, void* h_vals) {
  if (!t) return fail(CH_EINVAL, "null table");
  if (start > t->T.c || count > t->T.c - start) return fail(CH_EINVAL, "slot range out of bounds");
  std::lock_guard<std::mutex> lock(t->mu);
  DeviceGuard dev(t->cfg.device);
  int rc = check(cudaEventSynchronize(t->last), "synchronize");
  if (!rc && t->pending_clear) {  // a deferred clear: run it before reading
    Launch c;
    c.stream = nullptr;
    c.device = t->cfg.device;
    c.sms = t->sms;
    rc = single_clear(c, t->T, t->ts);
    if (!rc) rc = check(cudaDeviceSynchronize(), "clear");
    t->pending_clear = false;
  }
  if (rc || count == 0) return rc;
  const int kb = t->ts.kbytes, vb = t->ts.vbytes;
  if (t->cfg.layout == CH_SOA) {
    if (h_keys)
      rc = check(cudaMemcpy(h_keys, (const char*)t->T.slots + start * kb, count * kb, cudaMemcpyDeviceToHost),
                 "read keys");
    if (!rc && h_vals)
      rc = check(cudaMemcpy(h_vals, (const char*)t->T.vals + start * vb, count * vb, cudaMemcpyDeviceToHost),
                 "read values");
    return rc;
  }
  const size_t cell = t->cfg.layout == CH_PACKED ? 8 : (kb == 8 || vb == 8 ? 16 : 8);
  std::vector<unsigned char> buf;
  try {
    buf.resize(count * cell);
  } catch (...) {
    return fail(CH_ENOMEM, "host buffer");
  }
  rc = check(cudaMemcpy(buf.data(), (const char*)t->T.slots + start * cell, count * cell, cudaMemcpyDeviceToHost),
             "read cells");
  if (rc) return rc;
  const size_t voff = t->cfg.layout == CH_PACKED ? 4 : (cell == 16 ? 8 : 4);
  for (uint64_t i = 0; i < count; ++i) {
    const unsigned char* p = buf.data() + i * cell;
    if (h_keys) memcpy((char*)h_keys + i * kb, p, kb);
    if (h_vals) memcpy((char*)h_vals + i * vb, p + voff, vb);
  }
  return CH_OK;
}

int ch_read_slots(ch_table* t, void* h_keys, void* h_vals) {
  if (!t) return fail(CH_EINVAL, "null table");
  return ch_read_slot_range(t, 0, t->T.c, h_keys, h_vals);
}

int ch_write_slots(ch_table* t, const void* h_keys, const void* h_vals) {
  if (!t || !h_keys || !h_vals) return fail(CH_EINVAL, "null argument");
  std::lock_guard<std::mutex> lock(t->mu);
  DeviceGuard dev(t->cfg.device);
  int rc = check(cudaEventSynchronize(t->last), "synchronize");
  if (rc) return rc;
  t->pending_clear = false;  // every cell is written below
  const uint64_t c = t->T.c;
  const int kb = t->ts.kbytes, vb = t->ts.vbytes;
  if (t->cfg.layout == CH_SOA) {
    rc = check(cudaMemcpy(t->T.slots, h_keys, c * kb, cudaMemcpyHostToDevice), "write keys");
    if (!rc) rc = check(cudaMemcpy(t->T.vals, h_vals, c * vb, cudaMemcpyHostToDevice), "write values");
    return rc;
  }
  const size_t cell = t->cfg.layout == CH_PACKED ? 8 : (kb == 8 || vb == 8 ? 16 : 8);
  const size_t voff = t->cfg.layout == CH_PACKED ? 4 : (cell == 16 ? 8 : 4);
  std::vector<unsigned char> buf(c * cell, 0);
  for (uint64_t i = 0; i < c; ++i) {
    memcpy(buf.data() + i * cell, (const char*)h_keys + i * kb, kb);
    memcpy(buf.data() + i * cell + voff, (const char*)h_vals + i * vb, vb);
  }
  return check(cudaMemcpy(t->T.slots, buf.data(), c * cell, cudaMemcpyHostToDevice), "write cells");
}

int ch_read_arena(ch_table* t, void* h_arena, uint64_t count) {
  if (!t || !h_arena) return fail(CH_EINVAL, "null argument");
  if (t->cfg.kind != CH_BUCKET) return fail(CH_EINVAL, "not a bucket-list table");
  if (count > t->cfg.pool_capacity) count = t->cfg.pool_capacity;
  std::lock_guard<std::mutex> lock(t->mu);
  DeviceGuard dev(t->cfg.device);
  int rc = check(cudaEventSynchronize(t->last), "synchronize");
  if (rc) return rc;
  return check(cudaMemcpy(h_arena, t->arena, count * t->vbytes, cudaMemcpyDeviceToHost), "read arena");
}

int ch_slot_op(ch_table* t, int op, uint64_t slot, uint64_t expected, uint64_t desired, uint64_t value, int* h_won,
               uint64_t* h_key, uint64_t* h_val) {
  if (!t || !h_won || !h_key || !h_val) return fail(CH_EINVAL, "null argument");
  if (slot >= t->T.c) return fail(CH_EINVAL, "slot out of range");
  if (op < 0 || op > 5) return fail(CH_EINVAL, "bad slot op");
  if (t->cfg.layout == CH_PACKED && op == 2) return fail(CH_EINVAL, "value CAS is not available on packed cells");
  if (t->cfg.layout != CH_PACKED && op == 1) return fail(CH_EINVAL, "pair claim requires the packed layout");
  Ordered o(t, nullptr);
  Scratch sc(o.s);
  unsigned long long* d = (unsigned long long*)sc.get(24);
  if (!d) return o.done(fail(CH_ENOMEM, "scratch"));
  const int kb = t->ts.kbytes, vb = t->ts.vbytes;
  if (kb == 4 && vb == 4) k_slot_op<uint32_t, uint32_t><<<1, 1, 0, o.s>>>(t->T, t->cfg.layout, op, slot, expected, desired, value, d);
  else if (kb == 4) k_slot_op<uint32_t, uint64_t><<<1, 1, 0, o.s>>>(t->T, t->cfg.layout, op, slot, expected, desired, value, d);
  else if (vb == 4) k_slot_op<uint64_t, uint32_t><<<1, 1, 0, o.s>>>(t->T, t->cfg.layout, op, slot, expected, desired, value, d);
  else k_slot_op<uint64_t, uint64_t><<<1, 1, 0, o.s>>>(t->T, t->cfg.layout, op, slot, expected, desired, value, d);
  count_launch();
  int rc = check(cudaGetLastError(), "slot op");
  unsigned long long hbuf[3] = {0, 0, 0};
  if (!rc) rc = check(cudaMemcpyAsync(hbuf, d, 24, cudaMemcpyDeviceToHost, o.s), "slot op read");
  if (!rc) rc = check(cudaStreamSynchronize(o.s), "slot op sync");
  *h_won = (int)hbuf[0];
  *h_key = hbuf[1];
  *h_val = hbuf[2];
  return o.done(rc);
}

// ---- device primitives ----
static Launch plain_launch(int device, void* stream) {
  Launch lc;
  lc.stream = (cudaStream_t)stream;
  lc.device = device;
  lc.sms = 148;
  cudaDeviceGetAttribute(&lc.sms, cudaDevAttrMultiProcessorCount, device);
  return lc;
}

int ch_exclusive_scan_u32(const uint32_t* counts, uint64_t n, uint64_t* out, int device, void* stream) {
  if (!out || (n && !counts)) return fail(CH_EINVAL, "null buffer");
  DeviceGuard dev(device);
  Launch lc = plain_launch(device, stream);
  Scratch sc(lc.stream);
  const size_t sb = exclusive_scan_scratch_bytes(n);
  void* p = sc.get(sb);
  if (!p) return fail(CH_ENOMEM, "scratch allocation failed");
  return exclusive_scan_u32(lc, counts, n, out, p, sb);
}

int ch_mix64(const uint64_t* keys, uint64_t n, uint64_t seed, uint64_t* out, int device, void* stream) {
  if (n && (!keys || !out)) return fail(CH_EINVAL, "null buffer");
  DeviceGuard dev(device);
  return mix64_array(plain_launch(device, stream), keys, n, seed, out);
}

int ch_multi_split(const void* keys, int key_bytes, const void* vals, int val_bytes, uint64_t n, uint32_t shards,
                   uint64_t* perm, uint64_t* offsets, void* keys_out, void* vals_out, int device, void* stream) {
  if (!offsets || (n && (!keys || !perm))) return fail(CH_EINVAL, "null buffer");
  if (key_bytes != 4 && key_bytes != 8) return fail(CH_EINVAL, "key_bytes must be 4 or 8");
  if (vals && val_bytes != 4 && val_bytes != 8) return fail(CH_EINVAL, "val_bytes must be 4 or 8");
  DeviceGuard dev(device);
  Launch lc = plain_launch(device, stream);
  Scratch sc(lc.stream);
  const size_t sb = split_scratch_bytes(n, shards);
  void* p = sc.get(sb);
  if (!p) return fail(CH_ENOMEM, "scratch allocation failed");
  return multi_split(lc, keys, key_bytes, vals, vals ? val_bytes : 4, n, shards, perm, 8, offsets, keys_out,
                     vals_out, p, sb);
}

int ch_partition(const uint32_t* dest, uint64_t n, uint32_t shards, uint64_t* perm, uint64_t* offsets, int device,
                 void* stream) {
  if (!offsets || (n && (!dest || !perm))) return fail(CH_EINVAL, "null buffer");
  DeviceGuard dev(device);
  Launch lc = plain_launch(device, stream);
  Scratch sc(lc.stream);
  const size_t sb = split_scratch_bytes(n, shards);
  void* p = sc.get(sb);
  if (!p) return fail(CH_ENOMEM, "scratch allocation failed");
  return multi_split(lc, dest, 0, nullptr, 4, n, shards, perm, 8, offsets, nullptr, nullptr, p, sb);
}

int ch_multi_split32(const void* keys, int key_bytes, const void* vals, int val_bytes, uint64_t n, uint32_t shards,
                     uint32_t* perm, uint64_t* offsets, void* keys_out, void* vals_out, int device, void* stream) {
  if (!offsets || (n && (!keys || !perm))) return fail(CH_EINVAL, "null buffer");
  if (key_bytes != 4 && key_bytes != 8) return fail(CH_EINVAL, "key_bytes must be 4 or 8");
  if (vals && val_bytes != 4 && val_bytes != 8) return fail(CH_EINVAL, "val_bytes must be 4 or 8");
  DeviceGuard dev(device);
  Launch lc = plain_launch(device, stream);
  Scratch sc(lc.stream);
  const size_t sb = split_scratch_bytes(n, shards);
  void* p = sc.get(sb);
  if (!p) return fail(CH_ENOMEM, "scratch allocation failed");
  return multi_split(lc, keys, key_bytes, vals, vals ? val_bytes : 4, n, shards, perm, 4, offsets, keys_out,
                     vals_out, p, sb);
}

int ch_route_split32(const void* keys, int key_bytes, const void* vals, int val_bytes, uint64_t n, uint32_t shards,
                     uint32_t* pos, uint64_t* offsets, void* keys_out, void* vals_out, int device, void* stream) {
  if (!offsets || (n && (!keys || !pos))) return fail(CH_EINVAL, "null buffer");
  if (key_bytes != 4 && key_bytes != 8) return fail(CH_EINVAL, "key_bytes must be 4 or 8");
  if (vals && val_bytes != 4 && val_bytes != 8) return fail(CH_EINVAL, "val_bytes must be 4 or 8");
  DeviceGuard dev(device);
  Launch lc = plain_launch(device, stream);
  Scratch sc(lc.stream);
  const size_t sb = split_scratch_bytes(n, shards);
  void* p = sc.get(sb);
  if (!p) return fail(CH_ENOMEM, "scratch allocation failed");
  return multi_split(lc, keys, key_bytes, vals, vals ? val_bytes : 4, n, shards, pos, -4, offsets, keys_out,
                     vals_out, p, sb);
}

int ch_route_part32(const uint32_t* keys, const uint32_t* vals, uint64_t n, uint32_t shards, uint64_t cap,
                    uint32_t* pos, uint64_t* counts, uint32_t* keys_out, uint32_t* vals_out, int* flag, int device,
                    void* stream) {
  if (!counts || !flag || (n && (!keys || !pos || !keys_out))) return fail(CH_EINVAL, "null buffer");
  if (vals && !vals_out) return fail(CH_EINVAL, "null buffer");
  if (n >= (1ull << 32) || (uint64_t)shards * cap >= (1ull << 32)) return fail(CH_EINVAL, "positions must fit 32 bits");
  DeviceGuard dev(device);
  Launch lc = plain_launch(device, stream);
  return route_part32(lc, keys, vals, n, shards, cap, pos, reinterpret_cast<unsigned long long*>(counts), keys_out,
                      vals_out, flag);
}

int ch_scatter32(const void* src, int elem_bytes, const uint32_t* perm, uint64_t n, void* dst, int device,
                 void* stream) {
  if (n && (!src || !perm || !dst)) return fail(CH_EINVAL, "null buffer");
  DeviceGuard dev(device);
  return permute32(plain_launch(device, stream), src, elem_bytes, perm, n, dst, true);
}

int ch_gather32(const void* src, int elem_bytes, const uint32_t* perm, uint64_t n, void* dst, int device,
                void* stream) {
  if (n && (!src || !perm || !dst)) return fail(CH_EINVAL, "null buffer");
  DeviceGuard dev(device);
  return permute32(plain_launch(device, stream), src, elem_bytes, perm, n, dst, false);
}

int ch_scatter(const void* src, int elem_bytes, const uint64_t* perm, uint64_t n, void* dst, int device,
               void* stream) {
  if (n && (!src || !perm || !dst)) return fail(CH_EINVAL, "null buffer");
  DeviceGuard dev(device);
  return permute(plain_launch(device, stream), src, elem_bytes, perm, n, dst, true);
}

int ch_gather(const void* src, int elem_bytes, const uint64_t* perm, uint64_t n, void* dst, int device,
              void* stream) {
  if (n && (!src || !perm || !dst)) return fail(CH_EINVAL, "null buffer");
  DeviceGuard dev(device);
  return permute(plain_launch(device, stream), src, elem_bytes, perm, n, dst, false);
}

int ch_kmer_sketch(const uint8_t* text, const uint64_t* win_start, const uint32_t* win_len, const uint32_t* win_tag,
                   uint64_t n_windows, uint64_t total_len, int k, uint32_t sketch, uint64_t* kmers_out,
                   uint32_t* tags_out, uint64_t* d_count, int device, void* stream) {
  if (k < 1 || k > 32) return fail(CH_EINVAL, "k must lie in [1, 32] (2 bits per base)");
  if (sketch < 1) return fail(CH_EINVAL, "sketch_size must be >= 1");
  if (n_windows == 0) {
    if (d_count) {
      DeviceGuard dev(device);
      return check(cudaMemsetAsync(d_count, 0, 8, (cudaStream_t)stream), "count");
    }
    return CH_OK;
  }
  if (!text || !win_start || !win_len || !kmers_out) return fail(CH_EINVAL, "null buffer");
  DeviceGuard dev(device);
  Launch lc = plain_launch(device, stream);
  Scratch sc(lc.stream);
  const size_t sb = kmer_scratch_bytes(n_windows, sketch, total_len);
  void* p = sc.get(sb);
  if (!p) return fail(CH_ENOMEM, "scratch allocation failed");
  return kmer_sketch(lc, text, win_start, win_len, win_tag, n_windows, k, sketch, kmers_out, tags_out, d_count, p, sb,
                     total_len);
}

int ch_segment_copy(const void* src, int elem_bytes, const uint64_t* src_off, const uint64_t* idx, uint64_t n,
                    const uint64_t* dst_off, void* dst, int device, void* stream) {
  if (n && (!src_off || !idx || !dst_off)) return fail(CH_EINVAL, "null buffer");
  DeviceGuard dev(device);
  return segment_copy(plain_launch(device, stream), src, elem_bytes, src_off, idx, n, dst_off, dst);
}

}  // extern "C"
