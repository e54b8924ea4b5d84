/* ws_oracle.h -- CPU oracle for the WarpSpeed hash-table hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is a sequential C restatement of the
 * reference package's table algorithms (warpbench, pure Python), used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg as the *checker* and the CPU baseline.  The product path
 * (paper_2509_16407_b200/, libwarpspeed.so) never links or calls it.
 *
 * Parity is pinned: tests/golden/ holds fixtures produced by running the
 * reference itself (tests/golden/make_golden.py); tests/test_oracle.py checks
 * this oracle against every one of them (slot positions, statuses, values,
 * probe counts).
 *
 * Semantics follow, per design (paths relative to /root/reference/pkg/src/warpbench):
 *   bucket scan / claim / publish / tombstone  tables/openaddr.py:59-204
 *   double hashing                              tables/openaddr.py:207-318
 *   power-of-two choice (+ unsafe variant)      tables/openaddr.py:326-483
 *   iceberg                                     tables/openaddr.py:486-631
 *   bucketed cuckoo + BFS eviction              tables/cuckoo.py:32-222
 *   chaining over line-sized nodes              tables/chaining.py:32-226
 *   probe accounting                            instrument.py:26-85, tables/base.py:38-39,80-92
 */
#ifndef WS_ORACLE_H
#define WS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_DOUBLE, ORC_DOUBLE_MD, ORC_P2, ORC_P2_MD, ORC_ICEBERG, ORC_ICEBERG_MD,
       ORC_CUCKOO, ORC_CHAINING, ORC_UNSAFE };
enum { ORC_REPLACE = 0, ORC_KEEP = 1, ORC_ADD = 2, ORC_MAX = 3, ORC_MIN = 4 };
enum { ORC_INSERTED = 0, ORC_UPDATED = 1, ORC_FULL = 2 };
enum { ORC_OP_UPSERT = 0, ORC_OP_ERASE = 1, ORC_OP_QUERY = 2 };

typedef struct orc_params {
  int32_t design;
  int32_t bucket_size;
  uint64_t capacity_slots;
  uint64_t front_buckets;     /* iceberg only, precomputed in Python */
  uint64_t seeds[8];
  int32_t n_seeds;
  int32_t shortcut_slots;
  int32_t zero_count_cap;
  int32_t probe_cap;
  int32_t ways;
  int32_t path_depth;
  int32_t phased;
  int32_t line_bytes;
} orc_params;

typedef struct orc_table orc_table;

orc_table *orc_create(const orc_params *p);
void orc_destroy(orc_table *t);

/* single ops (sequential semantics of the reference) */
int orc_upsert(orc_table *t, uint64_t key, uint64_t val, int merge);
int orc_query(orc_table *t, uint64_t key, uint64_t *val_out);
int orc_erase(orc_table *t, uint64_t key);
int64_t orc_slot_of(orc_table *t, uint64_t key);
uint64_t orc_primary_bucket(orc_table *t, uint64_t key);

/* batch drivers: ops applied in index order.  op byte = kind | merge << 4. */
void orc_upsert_n(orc_table *t, const uint64_t *keys, const uint64_t *vals, uint64_t n,
                  int merge, uint8_t *status);
void orc_query_n(orc_table *t, const uint64_t *keys, uint64_t n, uint64_t *vals, uint8_t *found);
void orc_erase_n(orc_table *t, const uint64_t *keys, uint64_t n, uint8_t *found);
void orc_mixed_n(orc_table *t, const uint8_t *ops, const uint64_t *keys, const uint64_t *vals,
                 uint64_t n, uint8_t *status, uint64_t *vals_out);

/* probe accounting: when enabled every op's distinct-line count is written to
 * probes[i] of the next batch call (pass NULL to disable). */
void orc_set_probe_sink(orc_table *t, uint32_t *probes, uint64_t n);
uint64_t orc_lock_touches(orc_table *t);
int orc_probe_saturated(orc_table *t);

/* quiescent introspection */
uint64_t orc_items(orc_table *t, uint64_t *keys, uint64_t *vals, uint64_t cap);
uint64_t orc_occupied(orc_table *t);
uint64_t orc_data_words(orc_table *t);           /* slot / arena words in use */
void orc_export_words(orc_table *t, uint64_t *out); /* raw slot (or arena) words */
void orc_export_tags(orc_table *t, uint16_t *out);
uint64_t orc_next_node(orc_table *t);
uint64_t orc_arena_capacity(orc_table *t);
int orc_tombstones_ever(orc_table *t);

#ifdef __cplusplus
}
#endif
#endif
