/* warpspeed.h -- C ABI of the B200-native WarpSpeed hash-table hot path.
 *
 * libwarpspeed.so (built from paper_2509_16407_b200/csrc/) exports exactly the
 * functions below.  Signatures use plain pointers and sizes only; pointers may
 * be device memory (e.g. torch CUDA tensors' data_ptr) or host memory (pinned
 * or pageable).  Host buffers are staged through the table's device buffers
 * with the copies pipelined against the kernels, so an FFI caller with plain
 * host arrays (ctypes / cgo / JNI) can use the table directly.
 *
 * The reference (warpbench, pure Python) has no FFI; each entry point replaces
 * the Python surface named beside it (paths under /root/reference/pkg/src/warpbench):
 *
 *   ws_create / ws_destroy    make_table(TableConfig)          tables/__init__.py:30-35
 *                             HashTable.__init__               tables/base.py:57-73
 *   ws_clear                  (new) make_table() again without reallocating
 *   ws_upsert                 HashTable.upsert(key, value, merge)  tables/base.py:115-124
 *   ws_query                  HashTable.query(key)             tables/base.py:126-129
 *   ws_erase                  HashTable.erase(key)             tables/base.py:131-134
 *   ws_mixed                  concurrent mixed phase (aging mixed_worker)  bench/runners.py:282-295
 *   ws_locate                 HashTable.slot_of(key)           tables/base.py:136-143
 *   ws_probe_counts           upsert/query/erase(..., probe=ProbeRecorder)  instrument.py:26-85
 *   ws_export_items           HashTable.items()                tables/base.py:147-149
 *   ws_occupied               HashTable.occupied_count()       tables/base.py:158-162
 *   ws_duplicate_scan         HashTable.duplicate_scan()       tables/base.py:151-156
 *   ws_checksum               (new) size-independent content digest for parity at 2^28+
 *   ws_export_raw             slots.key_at / tags.get / arena words (test introspection)
 *   ws_read_range             slots.snapshot / find_free / used_count / tags.get over a
 *                             bucket range (sync.py:279-288, 184-207, 426-473) without a
 *                             whole-table copy
 *   ws_info                   storage_report / arena.next_node / _tombstones_ever
 *   ws_tune                   (new) performance knobs, no semantic effect
 *   ws_partition/ws_unpermute (new) owner routing of the hash-sharded multi-GPU table
 *                             (the reference has no multi-GPU layer)
 *   ws_strerror               exception messages (InvalidKeyError / ConfigError)
 *
 * Semantics: a batch is a set of operations that execute concurrently on the
 * device; every op is linearizable.  Ops on the same key inside one batch are
 * serialised by the key's primary-bucket lock in an unspecified order, so a
 * batch's outcome is deterministic whenever its merges commute (ADD / MAX /
 * MIN) and erase / upsert / query roles are key-disjoint.  A batch holding any
 * sentinel key (0, 2^64-1, 2^64-2) is rejected as a whole before any mutation
 * (reference core.py:103-117).
 */
#ifndef WARPSPEED_H
#define WARPSPEED_H
#include <stdint.h>

#if defined(__GNUC__)
#define WS_API __attribute__((visibility("default")))
#else
#define WS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* return codes */
#define WS_OK 0
#define WS_ERR_INVALID_KEY (-1) /* sentinel key in batch; table untouched */
#define WS_ERR_CONFIG (-2)
#define WS_ERR_CUDA (-3)
#define WS_ERR_ALLOC (-4)
#define WS_ERR_ARG (-5)
#define WS_ERR_INVALID_OP (-6)
#define WS_ERR_TIMEOUT (-7)     /* a peer rank never arrived at a device barrier */

/* designs (same order as reference core.py:40-50 DESIGNS) */
enum {
  WS_DESIGN_DOUBLE = 0, WS_DESIGN_DOUBLE_MD, WS_DESIGN_P2, WS_DESIGN_P2_MD,
  WS_DESIGN_ICEBERG, WS_DESIGN_ICEBERG_MD, WS_DESIGN_CUCKOO, WS_DESIGN_CHAINING,
  WS_DESIGN_UNSAFE_REFERENCE
};
/* merge callbacks as a device enum (reference merge(existing, new) callables) */
enum { WS_MERGE_REPLACE = 0, WS_MERGE_KEEP, WS_MERGE_ADD, WS_MERGE_MAX, WS_MERGE_MIN };
/* upsert status (reference UpsertStatus, tables/base.py:42-45) */
enum { WS_INSERTED = 0, WS_UPDATED = 1, WS_FULL = 2 };
/* mixed-op byte: kind | merge << 4 */
enum { WS_OP_UPSERT = 0, WS_OP_ERASE = 1, WS_OP_QUERY = 2 };

/* call flags */
#define WS_F_SYNC_CHECK 1u  /* validate keys synchronously, return WS_ERR_INVALID_KEY */
#define WS_F_NO_CHECK 2u    /* caller guarantees no sentinels */
#define WS_F_SERIAL 4u      /* one device thread runs the batch in index order:
                               exactly the reference's sequential semantics */
#define WS_F_COMBINE 8u     /* fold same-key upserts of the batch before applying them
                               (hot-key / Zipf batches); statuses as if applied in some order */
#define WS_F_INTERLEAVED 16u /* mixed batch: keep every op kind in ONE interleaved launch (race tests);
                               default: large mixed batches run as per-kind segments */
#define WS_F_CONCURRENT_KINDS 32u /* mixed batch: run the per-kind segments CONCURRENTLY (erases,
                               queries and upserts on three streams forked from the caller's,
                               joined before return) with the tuned kernels, so erases race
                               inserts and queries as in the reference's threaded aging */

/* All derived integers are computed by the host layer exactly as the
 * reference computes them (core.py:209-211, openaddr.py:45-47,351-352,505-507). */
typedef struct ws_config {
  int32_t design;
  int32_t bucket_size;
  uint64_t capacity_slots;
  uint64_t front_buckets;   /* iceberg: round(nb * fraction), clamped */
  uint64_t seeds[8];        /* HashFamily(seed).seeds */
  int32_t n_seeds;
  int32_t shortcut_slots;   /* int(shortcut_threshold * bucket_size) */
  int32_t zero_count_cap;   /* max(1, bucket_size - shortcut_slots + 1) */
  int32_t probe_cap;
  int32_t ways;             /* cuckoo_ways */
  int32_t path_depth;       /* cuckoo_path_depth */
  int32_t phased;           /* mode == "phased": no locks, weak loads */
  int32_t line_bytes;
  int32_t multi_stream;     /* launches may run concurrently on several streams */
  uint64_t chain_pool_nodes;/* chaining: initial physical node pool (0 = default) */
} ws_config;

typedef struct ws_info_t {
  uint64_t capacity_slots, num_buckets, primary_buckets;
  uint64_t slot_bytes, tag_bytes, lock_bytes, node_bytes; /* device allocation */
  uint64_t next_node, pool_nodes;                         /* chaining */
  int32_t tombstones_ever;
  int32_t device;
} ws_info_t;

typedef struct ws_table ws_table;

WS_API int ws_create(const ws_config *cfg, int device, ws_table **out);
WS_API int ws_destroy(ws_table *t);
/* reset to the freshly-created state (all slots EMPTY, flags cleared) */
WS_API int ws_clear(ws_table *t, void *stream);

WS_API int ws_upsert(ws_table *t, const uint64_t *keys, const uint64_t *vals, uint64_t n,
              uint32_t merge, uint8_t *status, void *stream, uint32_t flags);
WS_API int ws_query(ws_table *t, const uint64_t *keys, uint64_t n, uint64_t *vals_out,
             uint8_t *found, void *stream, uint32_t flags);
WS_API int ws_erase(ws_table *t, const uint64_t *keys, uint64_t n, uint8_t *found,
             void *stream, uint32_t flags);
WS_API int ws_mixed(ws_table *t, const uint8_t *ops, const uint64_t *keys, const uint64_t *vals,
             uint64_t n, uint8_t *status, uint64_t *vals_out, void *stream, uint32_t flags);

/* slot index of each key (-1 if absent); chaining: node*bucket_size + pair */
WS_API int ws_locate(ws_table *t, const uint64_t *keys, uint64_t n, int64_t *slot_out, void *stream);

/* instrumented mixed batch: probes[i] = distinct line regions op i touched,
 * *lock_touches = total lock-word touches (reference ProbeRecorder semantics) */
WS_API int ws_probe_counts(ws_table *t, const uint8_t *ops, const uint64_t *keys,
                    const uint64_t *vals, uint64_t n, uint8_t *status, uint64_t *vals_out,
                    uint32_t *probes, uint64_t *lock_touches, void *stream, uint32_t flags);

/* quiescent introspection (synchronous) */
WS_API int ws_occupied(ws_table *t, uint64_t *count_out, void *stream);
WS_API int ws_export_items(ws_table *t, uint64_t *keys, uint64_t *vals, uint64_t cap,
                    uint64_t *n_out, void *stream);
WS_API int ws_duplicate_scan(ws_table *t, uint64_t *dup_keys, uint64_t *dup_counts, uint64_t cap,
                      uint64_t *n_dup_out, void *stream);
/* out[0]=occupied, [1]=sum keys, [2]=sum values, [3]=xor of mix64(k ^ mix64(v)) */
WS_API int ws_checksum(ws_table *t, uint64_t out[4], void *stream);
WS_API int ws_export_raw(ws_table *t, uint64_t *words, uint64_t nwords, uint16_t *tags,
                  void *stream);
/* words [first_word, first_word + nwords) of the cell array (2 per slot, or the
 * chaining node arena) and tags [first_tag, first_tag + ntags) into host or
 * device buffers; WS_ERR_ARG when a range runs past the table */
WS_API int ws_read_range(ws_table *t, uint64_t first_word, uint64_t nwords, uint64_t *words,
                  uint64_t first_tag, uint64_t ntags, uint16_t *tags, void *stream);
WS_API int ws_info(ws_table *t, ws_info_t *info);

/* performance knobs (no semantic effect) */
#define WS_TUNE_QUERY_ILP 1 /* query kernel: > 0 = the per-design tuned kernels (P2-MD: one thread per
                               op with pair-cooperative tag fetches; default 5), 0 = generic kernel
                               (the round-1 variants 1-4/8 -- several lookups per thread, lane-pair
                               tiles -- measured slower and were removed; their values now select
                               the default kernel) */
#define WS_TUNE_L2_POLICY 2 /* 2: 64-byte L2 fills for tag blocks and cells (default); 0/1: 128-byte fills */
#define WS_TUNE_UPSERT 3    /* upsert kernel: 0 = generic one thread per op; P2-MD 2 = warp-synchronous
                               lock rounds, 3 = rounds + 64-byte L2 fills,
                               4 = 3 + full-sector cell writes when the partner cell is EMPTY (default);
                               1 / 5 (lane-pair tiles, deferred lock release: removed) act as 4;
                               cuckoo: 4 = lock rounds + cooperative 8-lane eviction launch (default),
                               6 = lock rounds + one-thread-per-op eviction launch */
#define WS_TUNE_OCCUPANCY 4 /* retired: forcing 4-8 CTAs/SM measured slower; accepted, no effect */
/* race-window widening for the adversarial duplicate-key test (reference
 * bench/adversarial.py:40-93 DelayProfile): at the hook stages pre_reserve,
 * pre_publish, pre_tombstone, pre_scan the generic kernels sleep up to
 * DELAY_NS with probability DELAY_P16/65536.  Off (0) by default. */
#define WS_TUNE_DELAY_NS 5
#define WS_TUNE_DELAY_P16 6
#define WS_TUNE_DELAY_SEED 7
#define WS_TUNE_PREFETCH 10  /* retired: L2 prefetch of a later op's tag block measured slower
                               (profiles/prefetch_r02.log); accepted, no effect */
#define WS_TUNE_KERNEL_EVENTS 11 /* 1: bracket every table-kernel launch with CUDA events on its stream
                                    (benchmark instrumentation; read with ws_kernel_times) */
WS_API int ws_tune(ws_table *t, int knob, int value);
/* elapsed ms of each table-kernel launch recorded since the last call (in
 * launch order; waits for them), *count = how many; clears the record.
 * Benchmark instrumentation for the kernel-level roofline (bench.py). */
WS_API int ws_kernel_times(ws_table *t, float *ms_out, uint64_t cap, uint64_t *count);

/* hash-sharded multi-GPU routing (device pointers): split a batch into
 * 2^log2_parts per-owner contiguous segments, owner = top log2_parts bits of
 * mix64(key ^ seed0); perm[j] = source index of output j; counts[p] = segment
 * sizes.  vals / ops / out_vals / out_ops may be NULL.  n < 2^32. */
WS_API int ws_partition(const uint64_t *keys, const uint64_t *vals, const uint8_t *ops, uint64_t n,
                        uint64_t seed0, int log2_parts, uint64_t *out_keys, uint64_t *out_vals,
                        uint8_t *out_ops, uint32_t *perm, uint64_t *counts, void *stream);
/* out[perm[j]] = in[j] for elements of 1, 4 or 8 bytes (device pointers) */
WS_API int ws_unpermute(const void *in, const uint32_t *perm, uint64_t n, int elem_bytes, void *out,
                        void *stream);

/* fused routing over NVLink peer memory (CUDA IPC): the routing kernel stores
 * each op straight into its owner's inbox, owners apply it with the table
 * kernels and store results straight back into the source's reply buffer.
 * Collective: every rank calls ws_xchg_run with the same `rounds`
 * (= ceil(max batch over ranks / chunk_ops)).  Device pointers only. */
typedef struct ws_xchg ws_xchg;
WS_API int ws_xchg_create(int world, int rank, uint64_t chunk_ops, int device, ws_xchg **out);
WS_API int ws_xchg_handle(ws_xchg *x, void *handle_out /* 64 bytes */);
WS_API int ws_xchg_open(ws_xchg *x, const void *handles /* world x 64 bytes, rank order */);
WS_API int ws_xchg_run(ws_xchg *x, ws_table *local, const uint8_t *ops, uint8_t uop,
                       const uint64_t *keys, const uint64_t *vals, uint64_t n, uint64_t rounds,
                       uint64_t seed0, uint8_t *status, uint64_t *vals_out, void *stream,
                       uint32_t flags);
WS_API int ws_xchg_destroy(ws_xchg *x);

WS_API const char *ws_strerror(int code);

#ifdef __cplusplus
}
#endif
#endif
