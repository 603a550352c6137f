// dist.cu -- ch_dist_*: one hash-partitioned single-value table over several
// devices of one process (reference distributed.py:84-178).
//
// Every shard is an ordinary ch_table on its own device.  Key k lives on shard
// (mix64(k) >> 32) mod S (ShardRouter.route, distributed.py:44-45).  A bulk call
// takes one batch per source device and runs, per source and per shard:
//
//   split      route + stable multi-split on the source device (K10, prims.cu):
//              keys / values grouped by destination, u32 split position per source element
//   counts     segment sizes to the host (the only host synchronisation of a call)
//   exchange   every (source, shard) segment to its shard: NCCL grouped
//              ncclSend / ncclRecv over NVLink (one group for keys + values), or
//              the copy engines (cudaMemcpyPeerAsync) when shards share a device
//              or NCCL is not loadable
//   local      ch_insert / ch_retrieve on each shard's own stream (staged regions
//              when the received batch covers the shard)
//   back       statuses / (value, found) back to the sources, same transport
//   back-map   gather through the split's inverse map into the caller's order (K11)
//
// NCCL is dlopen'ed on first use ("libnccl.so.2": the copy torch already loaded,
// else the system one), so single-GPU users of the library never need it.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/coophash_b200.h"
#include "dispatch.cuh"

namespace chb {
int multi_split(const Launch& lc, const void* keys, int kbytes, const void* vals, int vbytes, uint64_t n,
                uint32_t shards, void* perm, int perm_bytes, uint64_t* offsets, void* keys_out, void* vals_out,
                void* scratch, size_t scratch_bytes);
size_t split_scratch_bytes(uint64_t n, uint32_t shards);
int permute32(const Launch& lc, const void* src, int elem_bytes, const uint32_t* perm, uint64_t n, void* dst,
              bool scatter);
}  // namespace chb

using namespace chb;

namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  decltype(&ncclCommInitAll) init_all = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGetErrorString) err = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = std::string("libnccl not loadable: ") + dlerror();
      return;
    }
#define CHB_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
    CHB_SYM(init_all, "ncclCommInitAll");
    CHB_SYM(destroy, "ncclCommDestroy");
    CHB_SYM(group_start, "ncclGroupStart");
    CHB_SYM(group_end, "ncclGroupEnd");
    CHB_SYM(send, "ncclSend");
    CHB_SYM(recv, "ncclRecv");
    CHB_SYM(err, "ncclGetErrorString");
#undef CHB_SYM
    api.ok = api.init_all && api.destroy && api.group_start && api.group_end && api.send && api.recv && api.err;
    if (!api.ok) api.why = "libnccl lacks a required symbol";
  });
  return api;
}

int nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return 0;
  set_error(std::string(what) + ": " + nccl().err(r));
  return CH_EIO;
}

struct DevGuard {
  int prev = -1;
  explicit DevGuard(int d) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != d) cudaSetDevice(d);
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

Launch launch_on(int device, cudaStream_t s) {
  Launch lc;
  lc.stream = s;
  lc.device = device;
  lc.sms = 148;
  cudaDeviceGetAttribute(&lc.sms, cudaDevAttrMultiProcessorCount, device);
  return lc;
}

// stream-ordered scratch that is freed on its own stream at the end of a call
struct Buf {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  int dev = 0;
};

}  // namespace

struct ch_dist {
  int S = 0;
  std::vector<ch_table*> shards;
  std::vector<int> dev;
  int kbytes = 4, vbytes = 4;
  int transport = CH_DIST_COPY;
  std::vector<ncclComm_t> comms;
  std::vector<cudaEvent_t> ev;  // per shard: cross-stream ordering of the copy transport
  uint64_t* h_off = nullptr;    // pinned: S x (S+1) split offsets
  std::mutex mu;
};

namespace {

int fail(int code, const std::string& m) {
  set_error(m);
  return code;
}

// exchange: dst[t] + roff(t, s) <- src[s] + off(s, t) for every (s, t), `w` bytes per element.
// fwd: counts cnt(s, t) = segment of source s for shard t.  Back direction swaps roles.
struct Plan {
  int S;
  std::vector<uint64_t> cnt;   // S x S: cnt[s * S + t]
  std::vector<uint64_t> off;   // S x S: offset of (s -> t) in source s's split order
  std::vector<uint64_t> roff;  // S x S: offset of (s -> t) in shard t's received order
  std::vector<uint64_t> rtot;  // S
  uint64_t c(int s, int t) const { return cnt[(size_t)s * S + t]; }
};

int exchange(ch_dist* D, const Plan& P, const std::vector<const void*>& src, const std::vector<void*>& dst, int w,
             const std::vector<cudaStream_t>& ss, bool forward) {
  const int S = D->S;
  // forward: source s sends cnt(s,t) elements from src[s] + off(s,t) to dst[t] + roff(s,t)
  // back:    shard t sends cnt(s,t) elements from src[t] + roff(s,t) to dst[s] + off(s,t)
  auto sender_of = [&](int s, int t) { return forward ? s : t; };
  auto receiver_of = [&](int s, int t) { return forward ? t : s; };
  auto src_off = [&](int s, int t) { return forward ? P.off[(size_t)s * S + t] : P.roff[(size_t)s * S + t]; };
  auto dst_off = [&](int s, int t) { return forward ? P.roff[(size_t)s * S + t] : P.off[(size_t)s * S + t]; };
  if (D->transport == CH_DIST_NCCL) {
    NcclApi& api = nccl();
    int rc = nccl_check(api.group_start(), "ncclGroupStart");
    if (rc) return rc;
    for (int s = 0; s < S && !rc; ++s)
      for (int t = 0; t < S && !rc; ++t) {
        const uint64_t n = P.c(s, t);
        if (!n) continue;
        const int a = sender_of(s, t), b = receiver_of(s, t);
        rc = nccl_check(api.send((const char*)src[a] + src_off(s, t) * w, n * w, ncclUint8, b, D->comms[a], ss[a]),
                        "ncclSend");
        if (!rc)
          rc = nccl_check(api.recv((char*)dst[b] + dst_off(s, t) * w, n * w, ncclUint8, a, D->comms[b], ss[b]),
                          "ncclRecv");
      }
    const int rc2 = nccl_check(api.group_end(), "ncclGroupEnd");
    return rc ? rc : rc2;
  }
  // copy engines: every sender waits until every receiver's buffers exist, copies on its
  // own stream, and every receiver waits for every sender
  for (int r = 0; r < S; ++r) {
    DevGuard g(D->dev[r]);
    if (int rc = cuda_check(cudaEventRecord(D->ev[r], ss[r]), "event record")) return rc;
  }
  for (int a = 0; a < S; ++a) {
    DevGuard g(D->dev[a]);
    for (int r = 0; r < S; ++r)
      if (r != a && cudaStreamWaitEvent(ss[a], D->ev[r], 0) != cudaSuccess) return cuda_check(cudaGetLastError(), "wait");
  }
  for (int s = 0; s < S; ++s)
    for (int t = 0; t < S; ++t) {
      const uint64_t n = P.c(s, t);
      if (!n) continue;
      const int a = sender_of(s, t), b = receiver_of(s, t);
      DevGuard g(D->dev[a]);
      const cudaError_t e =
          D->dev[a] == D->dev[b]
              ? cudaMemcpyAsync((char*)dst[b] + dst_off(s, t) * w, (const char*)src[a] + src_off(s, t) * w, n * w,
                                cudaMemcpyDeviceToDevice, ss[a])
              : cudaMemcpyPeerAsync((char*)dst[b] + dst_off(s, t) * w, D->dev[b],
                                    (const char*)src[a] + src_off(s, t) * w, D->dev[a], n * w, ss[a]);
      if (int rc = cuda_check(e, "exchange copy")) return rc;
    }
  for (int a = 0; a < S; ++a) {
    DevGuard g(D->dev[a]);
    if (int rc = cuda_check(cudaEventRecord(D->ev[a], ss[a]), "event record")) return rc;
  }
  for (int r = 0; r < S; ++r) {
    DevGuard g(D->dev[r]);
    for (int a = 0; a < S; ++a)
      if (a != r && cudaStreamWaitEvent(ss[r], D->ev[a], 0) != cudaSuccess) return cuda_check(cudaGetLastError(), "wait");
  }
  return 0;
}

// one bulk call; insert when d_vals / d_status are given, retrieve otherwise
int dist_op(ch_dist* D, bool insert, const void* const* keys, const void* const* vals, const uint64_t* n,
            uint8_t* const* status, void* const* vals_out, uint8_t* const* found, void* const* streams) {
  const int S = D->S;
  const int kb = D->kbytes, vb = D->vbytes;
  std::lock_guard<std::mutex> lock(D->mu);
  std::vector<cudaStream_t> ss(S);
  for (int s = 0; s < S; ++s) {
    ss[s] = streams ? (cudaStream_t)streams[s] : nullptr;
    if (n[s] && (!keys[s] || (insert ? (!vals[s] || !status[s]) : (!vals_out[s] || !found[s]))))
      return fail(CH_EINVAL, "null buffer");
    if (n[s] > 0xFFFFFFFFull) return fail(CH_EINVAL, "batches are limited to 2^32 - 1 keys per source");
  }
  std::vector<Buf> bufs;
  auto get = [&](int s, size_t bytes) -> void* {
    DevGuard g(D->dev[s]);
    void* p = nullptr;
    if (cudaMallocAsync(&p, bytes ? bytes : 8, ss[s]) != cudaSuccess) return nullptr;
    bufs.push_back({p, ss[s], D->dev[s]});
    return p;
  };
  auto release = [&](int rc) {
    for (auto& b : bufs) {
      DevGuard g(b.dev);
      cudaFreeAsync(b.p, b.s);
    }
    return rc;
  };
  // ---- split (K10) on every source
  std::vector<uint32_t*> perm(S);
  std::vector<void*> kout(S), vout(S);
  std::vector<uint64_t*> doff(S);
  for (int s = 0; s < S; ++s) {
    perm[s] = (uint32_t*)get(s, n[s] * 4);
    kout[s] = get(s, n[s] * kb);
    vout[s] = insert ? get(s, n[s] * vb) : nullptr;
    doff[s] = (uint64_t*)get(s, (S + 1) * 8);
    const size_t sb = split_scratch_bytes(n[s], S);
    void* scr = get(s, sb);
    if (!perm[s] || !kout[s] || (insert && !vout[s]) || !doff[s] || !scr)
      return release(fail(CH_ENOMEM, "split scratch allocation failed"));
    DevGuard g(D->dev[s]);
    int rc = multi_split(launch_on(D->dev[s], ss[s]), keys[s], kb, insert ? vals[s] : nullptr, vb, n[s], S, perm[s],
                         -4, doff[s], kout[s], vout[s], scr, sb);  // perm[s][i] = split position of i
    if (!rc)
      rc = cuda_check(cudaMemcpyAsync(D->h_off + (size_t)s * (S + 1), doff[s], (S + 1) * 8, cudaMemcpyDeviceToHost,
                                      ss[s]),
                      "offsets to host");
    if (rc) return release(rc);
  }
  for (int s = 0; s < S; ++s) {
    DevGuard g(D->dev[s]);
    if (int rc = cuda_check(cudaStreamSynchronize(ss[s]), "split")) return release(rc);
  }
  Plan P;
  P.S = S;
  P.cnt.assign((size_t)S * S, 0);
  P.off.assign((size_t)S * S, 0);
  P.roff.assign((size_t)S * S, 0);
  P.rtot.assign(S, 0);
  for (int s = 0; s < S; ++s)
    for (int t = 0; t < S; ++t) {
      const uint64_t* o = D->h_off + (size_t)s * (S + 1);
      P.cnt[(size_t)s * S + t] = o[t + 1] - o[t];
      P.off[(size_t)s * S + t] = o[t];
    }
  for (int t = 0; t < S; ++t)
    for (int s = 0; s < S; ++s) {
      P.roff[(size_t)s * S + t] = P.rtot[t];
      P.rtot[t] += P.c(s, t);
    }
  // ---- receive buffers, exchange of keys (+ values)
  std::vector<void*> rk(S), rv(S), rres(S), rflag(S);
  for (int t = 0; t < S; ++t) {
    rk[t] = get(t, P.rtot[t] * kb);
    rv[t] = get(t, P.rtot[t] * vb);  // insert: received values; retrieve: looked-up values
    rflag[t] = get(t, P.rtot[t]);    // insert: statuses; retrieve: found flags
    if (!rk[t] || !rv[t] || !rflag[t]) return release(fail(CH_ENOMEM, "receive buffer allocation failed"));
  }
  std::vector<void*> back_v(S), back_f(S);
  for (int s = 0; s < S; ++s) {
    back_f[s] = get(s, n[s]);
    back_v[s] = insert ? nullptr : get(s, n[s] * vb);
    if (!back_f[s] || (!insert && !back_v[s])) return release(fail(CH_ENOMEM, "result buffer allocation failed"));
  }
  std::vector<const void*> ck(kout.begin(), kout.end()), cv(vout.begin(), vout.end());
  int rc = 0;
  if (insert && D->transport == CH_DIST_NCCL) {
    // keys and values of a pair travel in the same NCCL group
    NcclApi& api = nccl();
    rc = nccl_check(api.group_start(), "ncclGroupStart");
    for (int s = 0; s < S && !rc; ++s)
      for (int t = 0; t < S && !rc; ++t) {
        const uint64_t c = P.c(s, t);
        if (!c) continue;
        const uint64_t o = P.off[(size_t)s * S + t], ro = P.roff[(size_t)s * S + t];
        rc = nccl_check(api.send((const char*)kout[s] + o * kb, c * kb, ncclUint8, t, D->comms[s], ss[s]), "ncclSend");
        if (!rc) rc = nccl_check(api.send((const char*)vout[s] + o * vb, c * vb, ncclUint8, t, D->comms[s], ss[s]), "ncclSend");
        if (!rc) rc = nccl_check(api.recv((char*)rk[t] + ro * kb, c * kb, ncclUint8, s, D->comms[t], ss[t]), "ncclRecv");
        if (!rc) rc = nccl_check(api.recv((char*)rv[t] + ro * vb, c * vb, ncclUint8, s, D->comms[t], ss[t]), "ncclRecv");
      }
    const int rc2 = nccl_check(api.group_end(), "ncclGroupEnd");
    if (!rc) rc = rc2;
  } else {
    rc = exchange(D, P, ck, rk, kb, ss, true);
    if (!rc && insert) rc = exchange(D, P, cv, rv, vb, ss, true);
  }
  if (rc) return release(rc);
  // ---- local op on every shard
  for (int t = 0; t < S && !rc; ++t)
    rc = insert ? ch_insert(D->shards[t], rk[t], rv[t], P.rtot[t], (uint8_t*)rflag[t], ss[t])
                : ch_retrieve(D->shards[t], rk[t], P.rtot[t], rv[t], (uint8_t*)rflag[t], ss[t]);
  if (rc) return release(rc);
  // ---- results back, inverse permutation
  std::vector<const void*> cf(rflag.begin(), rflag.end()), cvv(rv.begin(), rv.end());
  rc = exchange(D, P, cf, back_f, 1, ss, false);
  if (!rc && !insert) rc = exchange(D, P, cvv, back_v, vb, ss, false);
  for (int s = 0; s < S && !rc; ++s) {
    DevGuard g(D->dev[s]);
    const Launch lc = launch_on(D->dev[s], ss[s]);
    if (insert) {  // gathers: coalesced writes in the source's order
      rc = permute32(lc, back_f[s], 1, perm[s], n[s], status[s], false);
    } else {
      rc = permute32(lc, back_v[s], vb, perm[s], n[s], vals_out[s], false);
      if (!rc) rc = permute32(lc, back_f[s], 1, perm[s], n[s], found[s], false);
    }
  }
  return release(rc);
}

}  // namespace

extern "C" {

int ch_get_config(ch_table* t, ch_config* out);

int ch_dist_create(ch_dist** out, ch_table* const* shards, int num_shards, int transport) {
  if (!out || !shards) return fail(CH_EINVAL, "null argument");
  *out = nullptr;
  if (num_shards < 1 || num_shards > 256) return fail(CH_EINVAL, "num_shards must be in [1, 256]");
  if (transport < CH_DIST_AUTO || transport > CH_DIST_COPY) return fail(CH_EINVAL, "bad transport");
  ch_dist* D = new (std::nothrow) ch_dist();
  if (!D) return fail(CH_ENOMEM, "host allocation failed");
  D->S = num_shards;
  bool distinct = true;
  for (int s = 0; s < num_shards; ++s) {
    ch_config c;
    if (!shards[s] || ch_get_config(shards[s], &c)) {
      delete D;
      return fail(CH_EINVAL, "bad shard table");
    }
    if (c.kind != CH_SINGLE) {
      delete D;
      return fail(CH_EINVAL, "distributed tables shard single-value tables");
    }
    const int kb = c.key_bits <= 32 ? 4 : 8, vb = c.value_bits <= 32 ? 4 : 8;
    if (s == 0) {
      D->kbytes = kb;
      D->vbytes = vb;
    } else if (kb != D->kbytes || vb != D->vbytes) {
      delete D;
      return fail(CH_EINVAL, "shards must share key and value widths");
    }
    for (int d : D->dev)
      if (d == c.device) distinct = false;
    D->shards.push_back(shards[s]);
    D->dev.push_back(c.device);
  }
  if (transport == CH_DIST_NCCL && !distinct) {
    delete D;
    return fail(CH_EINVAL, "the NCCL transport needs one shard per device");
  }
  if (transport == CH_DIST_NCCL && !nccl().ok) {
    delete D;
    return fail(CH_EINVAL, nccl().why);
  }
  D->transport = transport == CH_DIST_AUTO ? (distinct && num_shards > 1 && nccl().ok ? CH_DIST_NCCL : CH_DIST_COPY)
                                           : transport;
  if (D->transport == CH_DIST_NCCL) {
    D->comms.resize(num_shards);
    const int rc = nccl_check(nccl().init_all(D->comms.data(), num_shards, D->dev.data()), "ncclCommInitAll");
    if (rc) {
      D->comms.clear();
      delete D;
      return rc;
    }
  } else {
    for (int s = 0; s < num_shards; ++s)  // peer access where the devices allow it (NVLink)
      for (int t = 0; t < num_shards; ++t) {
        int can = 0;
        if (D->dev[s] != D->dev[t] && cudaDeviceCanAccessPeer(&can, D->dev[s], D->dev[t]) == cudaSuccess && can) {
          DevGuard g(D->dev[s]);
          cudaDeviceEnablePeerAccess(D->dev[t], 0);
          cudaGetLastError();  // already enabled is fine
        }
      }
  }
  D->ev.resize(num_shards, nullptr);
  for (int s = 0; s < num_shards; ++s) {
    DevGuard g(D->dev[s]);
    if (cudaEventCreateWithFlags(&D->ev[s], cudaEventDisableTiming) != cudaSuccess) {
      ch_dist_destroy(D);
      return fail(CH_EIO, "event create failed");
    }
  }
  if (cudaMallocHost(&D->h_off, (size_t)num_shards * (num_shards + 1) * 8) != cudaSuccess) {
    ch_dist_destroy(D);
    return fail(CH_ENOMEM, "pinned offsets allocation failed");
  }
  *out = D;
  return CH_OK;
}

int ch_dist_destroy(ch_dist* D) {
  if (!D) return CH_OK;
  for (auto c : D->comms)
    if (c) nccl().destroy(c);
  for (size_t s = 0; s < D->ev.size(); ++s)
    if (D->ev[s]) {
      DevGuard g(D->dev[s]);
      cudaEventDestroy(D->ev[s]);
    }
  if (D->h_off) cudaFreeHost(D->h_off);
  delete D;
  return CH_OK;
}

int ch_dist_info(ch_dist* D, int* num_shards, int* transport) {
  if (!D) return fail(CH_EINVAL, "null argument");
  if (num_shards) *num_shards = D->S;
  if (transport) *transport = D->transport;
  return CH_OK;
}

int ch_dist_insert(ch_dist* D, const void* const* d_keys, const void* const* d_vals, const uint64_t* n,
                   uint8_t* const* d_status, void* const* streams) {
  if (!D || !d_keys || !d_vals || !n || !d_status) return fail(CH_EINVAL, "null argument");
  return dist_op(D, true, d_keys, d_vals, n, d_status, nullptr, nullptr, streams);
}

int ch_dist_retrieve(ch_dist* D, const void* const* d_keys, const uint64_t* n, void* const* d_vals_out,
                     uint8_t* const* d_found, void* const* streams) {
  if (!D || !d_keys || !n || !d_vals_out || !d_found) return fail(CH_EINVAL, "null argument");
  return dist_op(D, false, d_keys, nullptr, n, nullptr, d_vals_out, d_found, streams);
}

}  // extern "C"
