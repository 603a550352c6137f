/*
 * coophash_b200.h -- C ABI of the B200-native COPS hash tables.
 *
 * This is the drop-in boundary for the reference package's table API
 * (coophash, /root/reference/pkg/src/coophash).  The Python classes in
 * paper_2009_07914_b200/ bind exactly these symbols with ctypes; any other
 * host language (cgo, JNI, N-API) binds the same ones.
 *
 * Conventions
 *   - All entry points return 0 on success or a negative errno-style code
 *     (CH_EINVAL, CH_ENOMEM, CH_EIO); ch_last_error() holds the message
 *     (thread-local).  Nothing throws across the ABI.
 *   - d_* pointers are device pointers on the table's device; h_* are host.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default).
 *     Bulk operations are asynchronous and stream-ordered.  Operations on one
 *     table are additionally ordered after the previous operation on that
 *     table, whatever stream it used (the table keeps an event), which is the
 *     B200 equivalent of the reference's "concurrent bulk calls serialize".
 *   - Keys/values use the table's storage widths: 4 bytes when
 *     key_bits/value_bits <= 32, else 8 bytes.
 *   - Per-element status codes are the InsertStatus order of the reference
 *     (single_table.py:48-53).
 */
#ifndef COOPHASH_B200_H
#define COOPHASH_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CH_OK 0
#define CH_EINVAL (-22)
#define CH_ENOMEM (-12)
#define CH_EIO (-5)
#define CH_ETIMEDOUT (-110) /* bucket-list contention timeout (bucket_list.py:50,294) */

/* table kinds and layouts (layout.py:29-32) */
enum { CH_SINGLE = 0, CH_MULTI = 1, CH_BUCKET = 2 };
enum { CH_SOA = 0, CH_AOS = 1, CH_PACKED = 2 };
/* InsertStatus (single_table.py:48-53) */
enum { CH_INSERTED = 0, CH_DUPLICATE_KEY = 1, CH_TABLE_FULL = 2, CH_INVALID_KEY = 3, CH_OUT_OF_MEMORY = 4 };

typedef struct ch_table ch_table;

typedef struct ch_config {
  int kind;                    /* CH_SINGLE / CH_MULTI / CH_BUCKET */
  int layout;                  /* CH_SOA / CH_AOS / CH_PACKED */
  int key_bits;                /* 1..64 ; storage 4 B if <= 32 else 8 B */
  int value_bits;              /* 1..64 ; bucket tables store 64-bit handles */
  int group_width;             /* 1,2,4,8,16,32 (probing.py:65) */
  uint64_t p;                  /* prime window count; capacity = 32 p (probing.py:153-176) */
  uint64_t max_outer_attempts; /* 0 => p (probing.py:214-217) */
  uint64_t empty_key;          /* sentinels (layout.py:35-53) */
  uint64_t tombstone_key;
  /* bucket list only (bucket_list.py:73-153) */
  uint64_t pool_capacity;      /* value cells in the arena */
  uint64_t growth_s0;          /* initial bucket size */
  uint64_t growth_num;         /* growth factor lambda = num / den, exact */
  uint64_t growth_den;
  int device;                  /* CUDA ordinal */
} ch_config;

typedef struct ch_stats {
  uint64_t capacity;
  int64_t occupied;     /* single_table.py:122-128 */
  int64_t tombstones;
  uint64_t ops, attempts, windows; /* ProbeCounters (single_table.py:63-72) */
  int64_t total_values; /* bucket list (bucket_list.py:200-202) */
  uint64_t pool_allocated; /* BucketPool.allocated (bucket_list.py:151-153) */
  uint64_t device_error;   /* sticky device error bits */
  uint64_t deferred;       /* staged-region keys finished by the COPS probe kernels (csrc/staged.cu) */
} ch_stats;

const char* ch_last_error(void);
int ch_version(void);
/* number of CUDA kernels this library has launched (process-wide counter) */
uint64_t ch_kernel_launches(void);

/* ---- lifetime ---- replaces SingleValueHashTable/MultiValueHashTable/BucketListHashTable
 * construction (single_table.py:91-114, multi_table.py:36-58, bucket_list.py:167-188).
 * The caller resolves the capacity plan (choose_capacity) and passes p. */
int ch_create(ch_table** out, const ch_config* cfg);
int ch_destroy(ch_table* t);
int ch_clear(ch_table* t, void* stream);               /* K0: every cell empty, counters 0 */
int ch_get_stats(ch_table* t, ch_stats* out);          /* synchronizes the table's work */
int ch_get_config(ch_table* t, ch_config* out);        /* the resolved configuration (max_outer_attempts set) */
int ch_reset_probe_counters(ch_table* t, void* stream); /* single_table.py:136-138 */
int ch_synchronize(ch_table* t);
/* schedule of big bulk insert / retrieve batches: 0 auto (table > 256 MiB and n >= c/16:
 * staged regions for packed tables, L2 region order otherwise), 1 direct probes, 2 L2 region
 * order (csrc/locality.cu), 3 shared-memory staged regions (csrc/staged.cu; packed only, other
 * layouts run direct).  Result semantics are identical; only the schedule changes. */
int ch_set_locality(ch_table* t, int mode);
/* the schedule a single-value bulk insert / retrieve of n keys takes: 1 direct probes,
 * 2 L2 region order, 3 shared-memory staged regions (bench.py reports it) */
int ch_batch_schedule(ch_table* t, uint64_t n);
/* multi-value bulk insert: 1 (default) groups the batch by key and walks each distinct key's
 * sequence once (csrc/mgroup.cu, batches >= 4096 pairs); 0 inserts pair by pair */
int ch_set_multi_grouping(ch_table* t, int on);
/* CUDA-event timing of the table's probe kernels (insert / lookup / multi passes):
 * enable, then read each launch's device time in launch order (up to cap entries) and
 * the number of launches timed (synchronizes, resets) */
int ch_kernel_timing(ch_table* t, int enable);
int ch_kernel_time(ch_table* t, double* ms, uint64_t cap, uint64_t* launches);

/* ---- single-value (and bucket key store) ---- */
/* insert_bulk (single_table.py:355-374): d_status[n] */
int ch_insert(ch_table* t, const void* d_keys, const void* d_vals, uint64_t n, uint8_t* d_status,
              void* stream);
/* find_or_claim (single_table.py:292-311): claim the key's slot without writing the value
 * cell; d_status[n] (INSERTED = newly claimed, DUPLICATE_KEY = already present), d_slots[n] */
int ch_find_or_claim(ch_table* t, const void* d_keys, uint64_t n, uint8_t* d_status, int64_t* d_slots,
                     void* stream);
/* retrieve_bulk (single_table.py:376-408): d_vals_out[n], d_found[n] */
int ch_retrieve(ch_table* t, const void* d_keys, uint64_t n, void* d_vals_out, uint8_t* d_found,
                void* stream);
/* erase (single_table.py:338-351) applied to a batch: d_erased[n] */
int ch_erase(ch_table* t, const void* d_keys, uint64_t n, uint8_t* d_erased, void* stream);
/* slot_of / retrieve_with_stats (single_table.py:317-336): slot or -1 per key; optional
 * per-key probe attempts / windows (reference g-slot units) and the value cell of the
 * found slot (for_each, single_table.py:412-424).  Works for every kind (bucket: the
 * value cell is the list handle). */
int ch_find(ch_table* t, const void* d_keys, uint64_t n, int64_t* d_slots, uint32_t* d_attempts,
            uint32_t* d_windows, void* d_vals_out, void* stream);

/* ---- multi-value (multi_table.py) ---- */
int ch_multi_insert(ch_table* t, const void* d_keys, const void* d_vals, uint64_t n,
                    uint8_t* d_status, void* stream);              /* :113-152 */
/* count_bulk + exclusive_prefix_sum (:28-30, :228-254): d_offsets[n+1] */
int ch_multi_count(ch_table* t, const void* d_keys, uint64_t n, uint32_t* d_counts,
                   uint64_t* d_offsets, void* stream);
/* second pass of retrieve_bulk (:256-295): values in probe order at d_offsets */
int ch_multi_retrieve(ch_table* t, const void* d_keys, uint64_t n, const uint64_t* d_offsets,
                      void* d_vals_out, void* stream);

/* for_each on a multi-value table (multi_table.py:299-328): ch_multi_retrieve plus the slot
 * index of every value (d_slots_out at the same positions) */
int ch_multi_retrieve_slots(ch_table* t, const void* d_keys, uint64_t n, const uint64_t* d_offsets,
                            void* d_vals_out, int64_t* d_slots_out, void* stream);

/* ---- device functors: for_all (single_table.py:425-429, multi_table.py:330-339) ----
 * the live cells (neither empty nor tombstone) in slot order, compacted on the device:
 * keys / values (storage widths; bucket tables: the list handles) / slot indices, any of
 * them NULL; at most cap written; *d_count (device u64, may be NULL) = live cells */
int ch_for_all(ch_table* t, void* d_keys_out, void* d_vals_out, int64_t* d_slots_out, uint64_t cap,
               uint64_t* d_count, void* stream);
/* built-in reductions over the live cells, one pass: d_out[5] = count, sum of values
 * (mod 2^64), xor of keys, min value, max value (min = 2^64-1 when empty) */
int ch_reduce_live(ch_table* t, uint64_t* d_out, void* stream);

/* ---- bucket list (bucket_list.py) ---- */
int ch_bucket_insert(ch_table* t, const void* d_keys, const void* d_vals, uint64_t n,
                     uint8_t* d_status, void* stream);             /* :228-294, :367-378 */
/* counts read from the handles (:320-326, :380-381) + prefix sum; also keeps the
 * handles for ch_bucket_retrieve in the caller-provided d_handles[n] */
int ch_bucket_count(ch_table* t, const void* d_keys, uint64_t n, uint32_t* d_counts,
                    uint64_t* d_offsets, uint64_t* d_handles, void* stream);
/* chain walk (:300-355, :383-397), values head-first at d_offsets */
int ch_bucket_retrieve(ch_table* t, const uint64_t* d_handles, uint64_t n,
                       const uint64_t* d_offsets, void* d_vals_out, void* stream);

/* ---- raw state (host-materialised views: layout.py SlotArray, bucket pool) ---- */
/* copy the slot arrays to host: keys[c] and values[c] in storage widths
 * (packed tables return key / value halves split) */
int ch_read_slots(ch_table* t, void* h_keys, void* h_vals);
/* cells [start, start + count) only (single-cell reads of the SlotArray view) */
int ch_read_slot_range(ch_table* t, uint64_t start, uint64_t count, void* h_keys, void* h_vals);
int ch_write_slots(ch_table* t, const void* h_keys, const void* h_vals); /* test fixtures */
int ch_read_arena(ch_table* t, void* h_arena, uint64_t count);
/* element transitions on one slot (layout.py:140-243), for SlotArray parity:
 * op 0 try_claim_key(expected, desired), 1 try_claim_pair_packed(desired = key, value),
 * 2 cas_value(expected, desired), 3 retire_key(expected, value = tombstone value),
 * 4 store_value(value), 5 load_pair.  *h_won = 1 when the transition applied; the cell's
 * key and value as observed before the op go to *h_key / *h_val. */
int ch_slot_op(ch_table* t, int op, uint64_t slot, uint64_t expected, uint64_t desired,
               uint64_t value, int* h_won, uint64_t* h_key, uint64_t* h_val);

/* ---- device primitives shared with the distribution layer ---- */
/* exclusive_prefix_sum (multi_table.py:28-30): d_out[n+1] from u32 counts */
int ch_exclusive_scan_u32(const uint32_t* d_counts, uint64_t n, uint64_t* d_out, int device,
                          void* stream);
/* mix64 / HashFn.values (probing.py:90-117) over 8-byte keys */
int ch_mix64(const uint64_t* d_keys, uint64_t n, uint64_t seed, uint64_t* d_out, int device,
             void* stream);
/* ShardRouter.route + multi_split (distributed.py:44-45,59-69): stable partition of
 * n keys (key_bytes 4 or 8) over `shards` destinations.  d_perm[n] = source index of
 * each output position, d_offsets[shards+1].  Optional payload gathers in the same
 * pass: d_keys_out / d_vals_out (val_bytes 4 or 8) may be NULL. */
int ch_multi_split(const void* d_keys, int key_bytes, const void* d_vals, int val_bytes,
                   uint64_t n, uint32_t shards, uint64_t* d_perm, uint64_t* d_offsets,
                   void* d_keys_out, void* d_vals_out, int device, void* stream);
/* stable partition by precomputed destinations (custom routers): d_dest[n] < shards */
int ch_partition(const uint32_t* d_dest, uint64_t n, uint32_t shards, uint64_t* d_perm,
                 uint64_t* d_offsets, int device, void* stream);
/* inverse-permutation scatter (distributed.py:143-147,168-172): d_dst[perm[i]] = d_src[i] */
int ch_scatter(const void* d_src, int elem_bytes, const uint64_t* d_perm, uint64_t n, void* d_dst,
               int device, void* stream);
/* gather: d_dst[i] = d_src[perm[i]] */
int ch_gather(const void* d_src, int elem_bytes, const uint64_t* d_perm, uint64_t n, void* d_dst,
              int device, void* stream);
/* segmented copy (distributed.py:173-178,197-203): for i < n, copy
 * src[src_off[i] .. src_off[i] + len) to dst[dst_off[idx[i]] ..), len = dst_off[idx[i]+1]-dst_off[idx[i]] */
int ch_segment_copy(const void* d_src, int elem_bytes, const uint64_t* d_src_off,
                    const uint64_t* d_idx, uint64_t n, const uint64_t* d_dst_off, void* d_dst,
                    int device, void* stream);

/* ---- distributed single-value table over the devices of one process ----
 * replaces DistributedTable(num_shards, shard_factory, mode=DISTRIBUTED) with
 * single-value shards (distributed.py:84-178): key k lives on shard
 * (mix64(k) >> 32) mod S (distributed.py:44-45).  The shards are ordinary tables
 * made by ch_create (one per device for NCCL; several may share a device with the
 * copy transport); the handle does not own them.  A bulk call takes one batch per
 * source s (device of shards[s], stream streams[s]; n[s] may be 0): route + stable
 * split on the source, segments to their shards (NCCL grouped send/recv over NVLink,
 * or the copy engines), the shard's ch_insert / ch_retrieve, results back, inverse
 * permutation into the source's order.  One host synchronisation per call (the
 * segment sizes); everything else is stream-ordered on streams[]. */
typedef struct ch_dist ch_dist;
enum { CH_DIST_AUTO = 0, CH_DIST_NCCL = 1, CH_DIST_COPY = 2 };
int ch_dist_create(ch_dist** out, ch_table* const* shards, int num_shards, int transport);
int ch_dist_destroy(ch_dist* d);
int ch_dist_info(ch_dist* d, int* num_shards, int* transport);
/* insert_bulk (distributed.py:131-147): d_status[s][n[s]] InsertStatus codes */
int ch_dist_insert(ch_dist* d, const void* const* d_keys, const void* const* d_vals, const uint64_t* n,
                   uint8_t* const* d_status, void* const* streams);
/* retrieve_bulk, distributed mode (distributed.py:151-178): values + found flags */
int ch_dist_retrieve(ch_dist* d, const void* const* d_keys, const uint64_t* n, void* const* d_vals_out,
                     uint8_t* const* d_found, void* const* streams);

/* ---- k-mer sketching for the index demo (kmer.py:63-137) ----
 * d_text: sequence bytes (ASCII); n_windows windows, window w = d_text[d_win_start[w] ..
 * + d_win_len[w]) tagged d_win_tag[w] (NULL: the window number); total_len = sum of the
 * lengths.  Per window: the canonical 2-bit k-mers (k <= 32; bases other than A/C/G/T in
 * either case reset the roll) reduced to the `sketch` distinct ones with the smallest
 * (mix64(kmer), kmer), ascending.  Output packed in window order: d_kmers_out / d_tags_out
 * (capacity n_windows * sketch), *d_count (device u64) = pairs written. */
int ch_kmer_sketch(const uint8_t* d_text, const uint64_t* d_win_start, const uint32_t* d_win_len,
                   const uint32_t* d_win_tag, uint64_t n_windows, uint64_t total_len, int k, uint32_t sketch,
                   uint64_t* d_kmers_out, uint32_t* d_tags_out, uint64_t* d_count, int device, void* stream);

/* ---- u32-permutation variants (batches < 2^32): half the index traffic of the u64 forms ---- */
int ch_multi_split32(const void* d_keys, int key_bytes, const void* d_vals, int val_bytes, uint64_t n,
                     uint32_t shards, uint32_t* d_perm, uint64_t* d_offsets, void* d_keys_out, void* d_vals_out,
                     int device, void* stream);
/* route + stable split returning the INVERSE map: d_pos[i] = split position of source
 * element i (written in source order, coalesced), so results come back with a coalesced
 * ch_gather32(results, d_pos) instead of a scatter's partial-line writes */
int ch_route_split32(const void* d_keys, int key_bytes, const void* d_vals, int val_bytes, uint64_t n,
                     uint32_t shards, uint32_t* d_pos, uint64_t* d_offsets, void* d_keys_out, void* d_vals_out,
                     int device, void* stream);
/* one-pass route partition (the hash-partitioned table's split; replaces the stable
 * ch_route_split32 where the order inside a destination does not matter): segment d of
 * d_keys_out / d_vals_out is [d cap, d cap + d_counts[d]); d_pos[i] = the position of source
 * element i; *d_flag != 0 when a segment passed cap (the outputs are then invalid).  32-bit
 * keys and values, shards <= 64, shards * cap < 2^32. */
int ch_route_part32(const uint32_t* d_keys, const uint32_t* d_vals, uint64_t n, uint32_t shards, uint64_t cap,
                    uint32_t* d_pos, uint64_t* d_counts, uint32_t* d_keys_out, uint32_t* d_vals_out, int* d_flag,
                    int device, void* stream);
int ch_scatter32(const void* d_src, int elem_bytes, const uint32_t* d_perm, uint64_t n, void* d_dst, int device,
                 void* stream);
int ch_gather32(const void* d_src, int elem_bytes, const uint32_t* d_perm, uint64_t n, void* d_dst, int device,
                void* stream);

#ifdef __cplusplus
}
#endif
#endif /* COOPHASH_B200_H */
