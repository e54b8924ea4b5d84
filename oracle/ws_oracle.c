/* ws_oracle.c -- sequential CPU restatement of the reference table algorithms.
 *
 * TEST INFRASTRUCTURE ONLY (see ws_oracle.h).  Every function below cites the
 * reference lines it restates (paths under /root/reference/pkg/src/warpbench).
 * Because it is single-threaded it reproduces the reference's deterministic
 * sequential behaviour exactly: the same slot for every key, the same FULL
 * decisions, the same probe counts.  Locks are not needed; their *probe*
 * accounting (tables/base.py:80-92) is reproduced.
 */
#include "ws_oracle.h"

#include <stdlib.h>
#include <string.h>

#define EMPTY 0ull
#define TOMB 0xFFFFFFFFFFFFFFFFull
#define RESV 0xFFFFFFFFFFFFFFFEull
#define TAG_BASE (1ull << 44) /* tables/base.py:38 */
#define LOCK_BASE (1ull << 45) /* tables/base.py:39 */
#define SCRATCH_CAP 8192u      /* instrument.py:23 */
#define CUCKOO_RETRIES 16      /* cuckoo.py:26 */
#define BFS_BUDGET 4096        /* cuckoo.py:29 */

typedef uint64_t u64;
typedef int64_t i64;

struct orc_table {
  orc_params p;
  int md, bs;
  u64 cap, nb, front, back;
  u64 *w;        /* slots: key,value pairs; chaining: arena words */
  uint16_t *tags;
  int tomb_ever; /* tables/base.py:73,94-98 */
  /* chaining arena (chaining.py:32-59) */
  int pairs, wpn;
  u64 arena_cap, next_node;
  /* probe recorder (instrument.py:26-85) */
  uint32_t *sink;
  u64 sink_n, sink_i;
  u64 *pkey;
  uint32_t *pgen;
  uint32_t gen, pcount, pmask;
  int saturated;
  u64 lock_touches;
};

/* ------------------------------------------------------------------ hashing */

static u64 mix64(u64 x) { /* core.py:120-129 */
  x ^= x >> 30;
  x *= 0xBF58476D1CE4E5B9ull;
  x ^= x >> 27;
  x *= 0x94D049BB133111EBull;
  x ^= x >> 31;
  return x;
}

static u64 hb(const orc_table *t, int i, u64 key, u64 nb) { /* core.py:157-161 */
  return (mix64(key ^ t->p.seeds[i]) >> 16) % nb;
}

/* fingerprint of an md design, 0 for plain designs (core.py:171-182, openaddr.py:373) */
static uint16_t md_tag(const orc_table *t, u64 h0) {
  if (!t->md) return 0;
  return (h0 & 0xFFFF) ? (uint16_t)(h0 & 0xFFFF) : 1;
}

static u64 merge_apply(int m, u64 old, u64 nv) {
  switch (m) {
  case ORC_KEEP: return old;
  case ORC_ADD: return old + nv; /* & MASK64 implicit, openaddr.py:200 */
  case ORC_MAX: return old > nv ? old : nv;
  case ORC_MIN: return old < nv ? old : nv;
  default: return nv;
  }
}

/* ------------------------------------------------------------------- probes */

static int probing(const orc_table *t) { return t->sink != NULL; }

static void ptouch_line(orc_table *t, u64 line) {
  uint32_t h = (uint32_t)(mix64(line) & t->pmask);
  for (;;) {
    if (t->pgen[h] != t->gen) break;
    if (t->pkey[h] == line) return; /* duplicate within the op is free */
    h = (h + 1) & t->pmask;
  }
  t->pgen[h] = t->gen;
  t->pkey[h] = line;
  t->pcount++;
}

static void touch(orc_table *t, u64 off) { /* instrument.py:42-49 */
  if (!probing(t)) return;
  if (t->pcount < SCRATCH_CAP) ptouch_line(t, off / (u64)t->p.line_bytes);
  else t->saturated = 1;
}

static void touch_range(orc_table *t, u64 off, u64 nbytes) { /* instrument.py:51-63 */
  if (!probing(t)) return;
  u64 lb = (u64)t->p.line_bytes, first = off / lb, last = (off + nbytes - 1) / lb;
  if (t->pcount + (last - first + 1) <= SCRATCH_CAP) {
    for (u64 l = first; l <= last; l++) ptouch_line(t, l);
  } else {
    t->saturated = 1;
  }
}

static void touch_lock_bucket(orc_table *t, u64 b) { /* base.py:80-86 */
  if (!probing(t) || t->p.phased) return;
  t->lock_touches++;
  touch(t, LOCK_BASE + (b >> 3));
}

static void finish_op(orc_table *t) { /* instrument.py:65-78 */
  if (!probing(t)) return;
  if (t->sink_i < t->sink_n) t->sink[t->sink_i] = t->pcount;
  t->sink_i++;
  t->pcount = 0;
  if (++t->gen == 0) { /* wrap: reset stamps */
    memset(t->pgen, 0, sizeof(uint32_t) * (t->pmask + 1));
    t->gen = 1;
  }
}

/* ----------------------------------------------------------- slot primitives */

static inline u64 K(const orc_table *t, u64 i) { return t->w[2 * i]; }
static inline u64 V(const orc_table *t, u64 i) { return t->w[2 * i + 1]; }
static inline void PUB(orc_table *t, u64 i, u64 k, u64 v) { t->w[2 * i + 1] = v; t->w[2 * i] = k; }
static inline int FREEK(u64 k) { return k == EMPTY || k == TOMB; }

typedef struct { i64 match, free; int saw_empty, used; } prange_t;

/* sync.py:184-228: one pass that stops at the first EMPTY cell */
static prange_t probe_range(orc_table *t, u64 lo, u64 hi, u64 key) {
  prange_t r = {-1, -1, 0, 0};
  for (u64 j = lo; j < hi; j++) {
    touch(t, 16 * j);
    u64 k = K(t, j);
    if (k == key) { r.match = (i64)j; return r; }
    if (k == EMPTY) {
      if (r.free < 0) r.free = (i64)j;
      r.saw_empty = 1;
      return r;
    }
    if (k == TOMB) {
      if (r.free < 0) r.free = (i64)j;
    } else {
      r.used++;
    }
  }
  return r;
}

static i64 find_free(const orc_table *t, u64 lo, u64 hi) { /* sync.py:230-239 */
  for (u64 j = lo; j < hi; j++)
    if (FREEK(K(t, j))) return (i64)j;
  return -1;
}

static int used_count(const orc_table *t, u64 lo, u64 hi) { /* sync.py:249-257 */
  int n = 0;
  for (u64 j = lo; j < hi; j++) n += !FREEK(K(t, j));
  return n;
}

static i64 next_zero(const orc_table *t, u64 from, u64 hi) { /* sync.py:444-453 */
  for (u64 j = from; j < hi; j++)
    if (t->tags[j] == 0) return (i64)j;
  return -1;
}

static int count_zeros(const orc_table *t, u64 lo, u64 hi, int cap) { /* sync.py:455-473 */
  int n = 0;
  for (u64 j = lo; j < hi; j++)
    if (t->tags[j] == 0 && ++n >= cap) return n;
  return n;
}

/* ---------------------------------------------------- bucket machinery */

typedef struct { i64 idx; u64 val; int saw_empty, used; i64 hint; } find_t;

/* openaddr.py:59-116 */
static find_t find_in_bucket(orc_table *t, u64 b, u64 key, uint16_t tag, int classify) {
  u64 bs = (u64)t->bs, lo = b * bs, hi = lo + bs;
  find_t r = {-1, 0, 0, 0, -1};
  if (!t->md) {
    prange_t pr = probe_range(t, lo, hi, key);
    if (pr.match >= 0) {
      r.idx = pr.match; r.val = V(t, (u64)pr.match); r.used = -1;
      return r;
    }
    r.saw_empty = pr.saw_empty; r.used = pr.used; r.hint = pr.free;
    return r;
  }
  touch_range(t, TAG_BASE + 2 * lo, 2 * bs);
  for (u64 m = lo; m < hi; m++) {
    if (t->tags[m] != tag) continue;
    touch(t, 16 * m);
    if (K(t, m) == key) {
      r.idx = (i64)m; r.val = V(t, m); r.used = -1;
      return r;
    }
  }
  i64 fz = next_zero(t, lo, hi);
  if (fz < 0) { r.used = (int)bs; return r; }
  r.used = (int)bs - count_zeros(t, lo, hi, t->p.zero_count_cap);
  r.hint = fz;
  if (!t->tomb_ever) { r.saw_empty = 1; return r; }
  if (classify) {
    for (i64 z = fz; z >= 0; z = next_zero(t, (u64)z + 1, hi)) {
      touch(t, 16 * (u64)z);
      if (K(t, (u64)z) == EMPTY) { r.saw_empty = 1; return r; }
    }
  }
  return r;
}

/* openaddr.py:118-130 */
static void used_and_free(orc_table *t, u64 b, int *used, int *has_free) {
  u64 bs = (u64)t->bs, lo = b * bs;
  if (t->md) {
    touch_range(t, TAG_BASE + 2 * lo, 2 * bs);
    int z = count_zeros(t, lo, lo + bs, t->p.zero_count_cap);
    *used = (int)bs - z; *has_free = z > 0;
    return;
  }
  touch_range(t, 16 * lo, 16 * bs);
  *used = used_count(t, lo, lo + bs);
  *has_free = *used < (int)bs;
}

/* openaddr.py:132-174 (sequentially every claim attempt succeeds at once) */
static i64 claim_in_bucket(orc_table *t, u64 b, i64 hint) {
  u64 bs = (u64)t->bs, lo = b * bs, hi = lo + bs;
  if (!t->md) {
    if (hint < 0) hint = find_free(t, lo, hi);
    if (hint < 0) return -1;
    touch(t, 16 * (u64)hint);
    t->w[2 * (u64)hint] = RESV;
    return hint;
  }
  i64 z = hint >= 0 ? hint : next_zero(t, lo, hi);
  for (; z >= 0; z = next_zero(t, (u64)z + 1, hi)) {
    touch(t, 16 * (u64)z);
    if (FREEK(K(t, (u64)z))) { t->w[2 * (u64)z] = RESV; return z; }
  }
  return -1;
}

static void publish(orc_table *t, u64 idx, u64 key, u64 val, uint16_t tag) { /* openaddr.py:176-185 */
  if (t->md) { t->tags[idx] = tag; touch(t, TAG_BASE + 2 * idx); }
  PUB(t, idx, key, val);
  touch(t, 16 * idx);
}

static void tombstone(orc_table *t, u64 idx) { /* openaddr.py:187-197 */
  t->tomb_ever = 1;
  t->w[2 * idx] = TOMB;
  t->w[2 * idx + 1] = 0;
  touch(t, 16 * idx);
  if (t->md) { t->tags[idx] = 0; touch(t, TAG_BASE + 2 * idx); }
}

static int apply_update(orc_table *t, u64 idx, u64 old, u64 val, int merge) { /* openaddr.py:199-204 */
  t->w[2 * idx + 1] = merge_apply(merge, old, val);
  touch(t, 16 * idx);
  return ORC_UPDATED;
}

/* ------------------------------------------------------------ double hashing */

static u64 dbl_step_mod(const orc_table *t, u64 key) { /* openaddr.py:220-230 */
  u64 step = mix64(key ^ t->p.seeds[1]) | 1;
  return step % t->nb; /* (b + step) % nb == (b + step % nb) % nb, no 2^64 wrap */
}

static u64 dbl_next(const orc_table *t, u64 b, u64 sm) {
  u64 x = b + sm;
  return x >= t->nb ? x - t->nb : x;
}

static u64 dbl_walk_len(const orc_table *t) {
  return (u64)t->p.probe_cap < t->nb ? (u64)t->p.probe_cap : t->nb;
}

static int dbl_upsert(orc_table *t, u64 key, u64 val, int merge) { /* openaddr.py:232-264 */
  u64 h0 = mix64(key ^ t->p.seeds[0]), b0 = (h0 >> 16) % t->nb;
  uint16_t tag = md_tag(t, h0);
  u64 sm = dbl_step_mod(t, key), walk = dbl_walk_len(t);
  touch_lock_bucket(t, b0);
  for (;;) {
    i64 fb = -1, fh = -1;
    u64 b = b0;
    for (u64 i = 0; i < walk; i++) {
      find_t r = find_in_bucket(t, b, key, tag, 1);
      if (r.idx >= 0) return apply_update(t, (u64)r.idx, r.val, val, merge);
      if (fb < 0 && r.hint >= 0) { fb = (i64)b; fh = r.hint; }
      if (r.saw_empty) break;
      b = dbl_next(t, b, sm);
    }
    if (fb < 0) return ORC_FULL;
    i64 idx = claim_in_bucket(t, (u64)fb, fh);
    if (idx < 0) continue;
    publish(t, (u64)idx, key, val, tag);
    return ORC_INSERTED;
  }
}

static i64 dbl_find(orc_table *t, u64 key, u64 *val) { /* openaddr.py:266-296 */
  u64 h0 = mix64(key ^ t->p.seeds[0]), b = (h0 >> 16) % t->nb;
  uint16_t tag = md_tag(t, h0);
  u64 sm = dbl_step_mod(t, key), walk = dbl_walk_len(t);
  for (u64 i = 0; i < walk; i++) {
    find_t r = find_in_bucket(t, b, key, tag, 1);
    if (r.idx >= 0) { if (val) *val = r.val; return r.idx; }
    if (r.saw_empty) return -1;
    b = dbl_next(t, b, sm);
  }
  return -1;
}

static int dbl_erase(orc_table *t, u64 key) { /* openaddr.py:298-318 */
  u64 h0 = mix64(key ^ t->p.seeds[0]);
  touch_lock_bucket(t, (h0 >> 16) % t->nb);
  i64 idx = dbl_find(t, key, NULL);
  if (idx < 0) return 0;
  tombstone(t, (u64)idx);
  return 1;
}

/* ------------------------------------------------------- power of two choice */

static int p2_upsert(orc_table *t, u64 key, u64 val, int merge) { /* openaddr.py:370-418 */
  u64 h0 = mix64(key ^ t->p.seeds[0]), b0 = (h0 >> 16) % t->nb;
  uint16_t tag = md_tag(t, h0);
  if (t->p.design != ORC_UNSAFE) touch_lock_bucket(t, b0);
  for (;;) {
    find_t r0 = find_in_bucket(t, b0, key, tag, 0);
    if (r0.idx >= 0) return apply_update(t, (u64)r0.idx, r0.val, val, merge);
    int shortcut = !t->tomb_ever && r0.used < t->p.shortcut_slots;
    i64 b1 = -1, hint1 = -1;
    int used1 = 0;
    if (!shortcut) {
      b1 = (i64)hb(t, 1, key, t->nb);
      if ((u64)b1 != b0) {
        find_t r1 = find_in_bucket(t, (u64)b1, key, tag, 0);
        if (r1.idx >= 0) return apply_update(t, (u64)r1.idx, r1.val, val, merge);
        used1 = r1.used; hint1 = r1.hint;
      } else {
        b1 = -1;
      }
    }
    i64 idx;
    if (shortcut || b1 < 0) {
      idx = claim_in_bucket(t, b0, r0.hint);
      if (idx < 0) {
        if (shortcut) continue;
        return ORC_FULL;
      }
    } else {
      u64 first = b0, second = (u64)b1;
      i64 h_first = r0.hint, h_second = hint1;
      if (r0.used > used1) { first = (u64)b1; second = b0; h_first = hint1; h_second = r0.hint; }
      idx = claim_in_bucket(t, first, h_first);
      if (idx < 0) idx = claim_in_bucket(t, second, h_second);
      if (idx < 0) return ORC_FULL;
    }
    publish(t, (u64)idx, key, val, tag);
    return ORC_INSERTED;
  }
}

static i64 p2_find(orc_table *t, u64 key, u64 *val, int early_exit) { /* openaddr.py:420-447 */
  u64 h0 = mix64(key ^ t->p.seeds[0]), b0 = (h0 >> 16) % t->nb;
  uint16_t tag = md_tag(t, h0);
  find_t r0 = find_in_bucket(t, b0, key, tag, 0);
  if (r0.idx >= 0) { if (val) *val = r0.val; return r0.idx; }
  if (early_exit && r0.saw_empty && !t->tomb_ever && r0.used < t->p.shortcut_slots) return -1;
  u64 b1 = hb(t, 1, key, t->nb);
  if (b1 == b0) return -1;
  find_t r1 = find_in_bucket(t, b1, key, tag, 0);
  if (r1.idx >= 0) { if (val) *val = r1.val; return r1.idx; }
  return -1;
}

static int p2_erase(orc_table *t, u64 key) { /* openaddr.py:449-473 */
  u64 h0 = mix64(key ^ t->p.seeds[0]);
  if (t->p.design != ORC_UNSAFE) touch_lock_bucket(t, (h0 >> 16) % t->nb);
  i64 idx = p2_find(t, key, NULL, 1);
  if (idx < 0) return 0;
  tombstone(t, (u64)idx);
  return 1;
}

/* ------------------------------------------------------------------ iceberg */

static void ice_backs(const orc_table *t, u64 key, u64 *b1, u64 *b2) { /* openaddr.py:517-521 */
  *b1 = t->front + hb(t, 1, key, t->back);
  *b2 = t->front + hb(t, 2, key, t->back);
}

static int ice_upsert(orc_table *t, u64 key, u64 val, int merge) { /* openaddr.py:540-578 */
  u64 h0 = mix64(key ^ t->p.seeds[0]), b0 = (h0 >> 16) % t->front;
  uint16_t tag = md_tag(t, h0);
  touch_lock_bucket(t, b0);
  for (;;) {
    find_t r0 = find_in_bucket(t, b0, key, tag, 0);
    if (r0.idx >= 0) return apply_update(t, (u64)r0.idx, r0.val, val, merge);
    u64 bk[2];
    int nbk = 0;
    if (!r0.saw_empty) {
      ice_backs(t, key, &bk[0], &bk[1]);
      nbk = bk[1] == bk[0] ? 1 : 2;
      for (int i = 0; i < nbk; i++) {
        find_t r = find_in_bucket(t, bk[i], key, tag, 0);
        if (r.idx >= 0) return apply_update(t, (u64)r.idx, r.val, val, merge);
      }
    }
    i64 idx = claim_in_bucket(t, b0, r0.hint);
    if (idx < 0) {
      if (!nbk) continue;
      int u[2], f[2], nc = 0;
      u64 cb[2];
      int cu[2];
      for (int i = 0; i < nbk; i++) {
        used_and_free(t, bk[i], &u[i], &f[i]);
        if (f[i]) { cu[nc] = u[i]; cb[nc] = bk[i]; nc++; }
      }
      /* sorted((used, bucket)) */
      if (nc == 2 && (cu[1] < cu[0] || (cu[1] == cu[0] && cb[1] < cb[0]))) {
        u64 tb = cb[0]; cb[0] = cb[1]; cb[1] = tb;
      }
      for (int i = 0; i < nc && idx < 0; i++) idx = claim_in_bucket(t, cb[i], -1);
      if (idx < 0) return ORC_FULL;
    }
    publish(t, (u64)idx, key, val, tag);
    return ORC_INSERTED;
  }
}

static i64 ice_find(orc_table *t, u64 key, u64 *val, int early_exit) { /* openaddr.py:580-610 */
  u64 h0 = mix64(key ^ t->p.seeds[0]), b0 = (h0 >> 16) % t->front;
  uint16_t tag = md_tag(t, h0);
  find_t r0 = find_in_bucket(t, b0, key, tag, 0);
  if (r0.idx >= 0) { if (val) *val = r0.val; return r0.idx; }
  if (early_exit && r0.saw_empty) return -1;
  u64 b1, b2;
  ice_backs(t, key, &b1, &b2);
  find_t r = find_in_bucket(t, b1, key, tag, 0);
  if (r.idx >= 0) { if (val) *val = r.val; return r.idx; }
  if (b2 != b1 || !early_exit) {
    r = find_in_bucket(t, b2, key, tag, 0);
    if (r.idx >= 0) { if (val) *val = r.val; return r.idx; }
  }
  return -1;
}

static int ice_erase(orc_table *t, u64 key) { /* openaddr.py:612-631 */
  u64 h0 = mix64(key ^ t->p.seeds[0]);
  touch_lock_bucket(t, (h0 >> 16) % t->front);
  i64 idx = ice_find(t, key, NULL, 1);
  if (idx < 0) return 0;
  tombstone(t, (u64)idx);
  return 1;
}

/* ------------------------------------------------------------------- cuckoo */

static int ck_buckets(const orc_table *t, u64 key, u64 *all, u64 *uniq) { /* cuckoo.py:54-56 + dict.fromkeys */
  int nu = 0;
  for (int i = 0; i < t->p.ways; i++) {
    u64 b = hb(t, i, key, t->nb);
    all[i] = b;
    int dup = 0;
    for (int j = 0; j < nu; j++) dup |= uniq[j] == b;
    if (!dup) uniq[nu++] = b;
  }
  return nu;
}

static void ck_lock_touch(orc_table *t, const u64 *uniq, int nu) { /* base.py:88-92 */
  for (int i = 0; i < nu; i++) touch_lock_bucket(t, uniq[i]);
}

/* growable bucket set + visit list for the BFS (cuckoo.py:107-156) */
typedef struct { u64 bucket; i64 parent; u64 slot, key; int depth; } visit_t;
typedef struct { u64 *keys; uint8_t *used; u64 mask, n; } bset_t;

static void bset_init(bset_t *s) {
  s->mask = 1023; s->n = 0;
  s->keys = (u64 *)malloc(sizeof(u64) * 1024);
  s->used = (uint8_t *)calloc(1024, 1);
}
static int bset_has(const bset_t *s, u64 k) {
  for (u64 h = mix64(k) & s->mask;; h = (h + 1) & s->mask) {
    if (!s->used[h]) return 0;
    if (s->keys[h] == k) return 1;
  }
}
static void bset_add(bset_t *s, u64 k);
static void bset_grow(bset_t *s) {
  bset_t o = *s;
  u64 cap = (o.mask + 1) * 2;
  s->mask = cap - 1; s->n = 0;
  s->keys = (u64 *)malloc(sizeof(u64) * cap);
  s->used = (uint8_t *)calloc(cap, 1);
  for (u64 i = 0; i <= o.mask; i++)
    if (o.used[i]) bset_add(s, o.keys[i]);
  free(o.keys); free(o.used);
}
static void bset_add(bset_t *s, u64 k) {
  if (2 * (s->n + 1) > s->mask + 1) bset_grow(s);
  for (u64 h = mix64(k) & s->mask;; h = (h + 1) & s->mask) {
    if (!s->used[h]) { s->used[h] = 1; s->keys[h] = k; s->n++; return; }
    if (s->keys[h] == k) return;
  }
}

typedef struct { u64 src_bucket, src_slot, key, dst_bucket; } move_t;

static int ck_find_path(orc_table *t, const u64 *uniq, int nu, move_t **moves_out) {
  u64 bs = (u64)t->bs;
  u64 vcap = 64, vn = 0;
  visit_t *v = (visit_t *)malloc(sizeof(visit_t) * vcap);
  bset_t seen;
  bset_init(&seen);
  for (int i = 0; i < nu; i++) {
    v[vn++] = (visit_t){uniq[i], -1, 0, 0, 0};
    bset_add(&seen, uniq[i]);
  }
  u64 head = 0;
  int expanded = 0, nmoves = -1;
  while (head < vn && expanded < BFS_BUDGET) {
    u64 vi = head++;
    u64 bucket = v[vi].bucket;
    int depth = v[vi].depth;
    if (depth >= t->p.path_depth) continue;
    expanded++;
    for (u64 j = bucket * bs; j < bucket * bs + bs; j++) {
      u64 k = K(t, j);
      if (k == EMPTY || k >= RESV) continue;
      for (int s = 0; s < t->p.ways; s++) {
        u64 alt = hb(t, s, k, t->nb);
        if (alt == bucket || bset_has(&seen, alt)) continue;
        i64 fr = find_free(t, alt * bs, alt * bs + bs);
        if (fr >= 0) {
          /* unwind parent edges: the new entry first, then its ancestors */
          int len = 1;
          for (i64 c = (i64)vi; v[c].parent >= 0; c = v[c].parent) len++;
          move_t *mv = (move_t *)malloc(sizeof(move_t) * (size_t)len);
          int pos = len - 1;
          mv[pos--] = (move_t){bucket, j, k, alt};
          for (i64 c = (i64)vi; v[c].parent >= 0; c = v[c].parent)
            mv[pos--] = (move_t){v[v[c].parent].bucket, v[c].slot, v[c].key, v[c].bucket};
          *moves_out = mv;
          nmoves = len;
          goto done;
        }
        if (vn == vcap) { vcap *= 2; v = (visit_t *)realloc(v, sizeof(visit_t) * vcap); }
        v[vn++] = (visit_t){alt, (i64)vi, j, k, depth + 1};
        bset_add(&seen, alt);
      }
    }
  }
done:
  free(v);
  free(seen.keys);
  free(seen.used);
  return nmoves;
}

static int ck_execute(orc_table *t, const move_t *mv, int n) { /* cuckoo.py:158-183 */
  u64 bs = (u64)t->bs;
  for (int i = n - 1; i >= 0; i--) {
    touch_lock_bucket(t, mv[i].src_bucket);
    if (mv[i].dst_bucket != mv[i].src_bucket) touch_lock_bucket(t, mv[i].dst_bucket);
    if (K(t, mv[i].src_slot) != mv[i].key) return 0;
    i64 d = find_free(t, mv[i].dst_bucket * bs, mv[i].dst_bucket * bs + bs);
    if (d < 0) return 0;
    PUB(t, (u64)d, mv[i].key, V(t, mv[i].src_slot));
    t->tomb_ever = 1;
    t->w[2 * mv[i].src_slot] = TOMB;
    t->w[2 * mv[i].src_slot + 1] = 0;
    touch(t, 16 * mv[i].src_slot);
    touch(t, 16 * (u64)d);
  }
  return 1;
}

static int ck_upsert(orc_table *t, u64 key, u64 val, int merge) { /* cuckoo.py:68-105 */
  u64 all[8], uq[8];
  u64 bs = (u64)t->bs;
  for (int attempt = 0; attempt < CUCKOO_RETRIES; attempt++) {
    int nu = ck_buckets(t, key, all, uq);
    ck_lock_touch(t, uq, nu);
    i64 free_at = -1;
    for (int i = 0; i < nu; i++) {
      prange_t r = probe_range(t, uq[i] * bs, uq[i] * bs + bs, key);
      if (r.match >= 0) {
        u64 m = (u64)r.match;
        t->w[2 * m + 1] = merge_apply(merge, V(t, m), val);
        touch(t, 16 * m);
        return ORC_UPDATED;
      }
      if (free_at < 0 && r.free >= 0) free_at = r.free;
    }
    if (free_at >= 0) {
      PUB(t, (u64)free_at, key, val);
      touch(t, 16 * (u64)free_at);
      return ORC_INSERTED;
    }
    move_t *mv = NULL;
    int n = ck_find_path(t, uq, nu, &mv);
    if (n < 0) return ORC_FULL;
    int ok = ck_execute(t, mv, n);
    free(mv);
    if (!ok) continue;
  }
  return ORC_FULL;
}

static i64 ck_find(orc_table *t, u64 key, u64 *val, int lock_touch) { /* cuckoo.py:185-204 */
  u64 all[8], uq[8];
  u64 bs = (u64)t->bs;
  int nu = ck_buckets(t, key, all, uq);
  if (lock_touch) ck_lock_touch(t, uq, nu);
  for (int i = 0; i < nu; i++) {
    prange_t r = probe_range(t, uq[i] * bs, uq[i] * bs + bs, key);
    if (r.match >= 0) { if (val) *val = V(t, (u64)r.match); return r.match; }
  }
  return -1;
}

static int ck_erase(orc_table *t, u64 key) { /* cuckoo.py:206-222 */
  i64 idx = ck_find(t, key, NULL, 1);
  if (idx < 0) return 0;
  t->tomb_ever = 1;
  t->w[2 * (u64)idx] = TOMB;
  t->w[2 * (u64)idx + 1] = 0;
  touch(t, 16 * (u64)idx);
  return 1;
}

/* ----------------------------------------------------------------- chaining */

static inline u64 *NODE(orc_table *t, u64 m) { return t->w + (u64)t->wpn * m; }

static u64 ch_alloc(orc_table *t) { /* chaining.py:51-59: grow 1.5x, min 64 */
  if (t->next_node >= t->arena_cap) {
    u64 grow = t->arena_cap >> 1;
    if (grow < 64) grow = 64;
    u64 ncap = t->arena_cap + grow;
    t->w = (u64 *)realloc(t->w, sizeof(u64) * (u64)t->wpn * ncap);
    memset(t->w + (u64)t->wpn * t->arena_cap, 0, sizeof(u64) * (u64)t->wpn * grow);
    t->arena_cap = ncap;
  }
  return t->next_node++;
}

typedef struct { i64 m, j; u64 val; u64 tail; i64 fm, fj; } walk_t;

static walk_t ch_walk(orc_table *t, u64 key) { /* chaining.py:137-171 */
  walk_t r = {-1, -1, 0, 0, -1, -1};
  u64 m = hb(t, 0, key, t->nb) + 1;
  for (;;) {
    touch(t, (u64)t->p.line_bytes * m);
    u64 *nd = NODE(t, m);
    for (int j = 0; j < t->pairs; j++) {
      u64 k = nd[2 * j];
      if (k == key) { r.m = (i64)m; r.j = j; r.val = nd[2 * j + 1]; r.tail = m; return r; }
      if (k == EMPTY) {
        if (r.fm < 0) { r.fm = (i64)m; r.fj = j; }
        r.tail = m;
        return r;
      }
      if (k == TOMB && r.fm < 0) { r.fm = (i64)m; r.fj = j; }
    }
    u64 nxt = nd[2 * t->pairs];
    if (!nxt) { r.tail = m; return r; }
    m = nxt;
  }
}

static int ch_upsert(orc_table *t, u64 key, u64 val, int merge) { /* chaining.py:173-203 */
  touch_lock_bucket(t, hb(t, 0, key, t->nb));
  walk_t w = ch_walk(t, key);
  if (w.m >= 0) {
    u64 *nd = NODE(t, (u64)w.m);
    nd[2 * w.j + 1] = merge_apply(merge, w.val, val);
    return ORC_UPDATED;
  }
  if (w.fm < 0) {
    u64 node = ch_alloc(t);
    touch(t, (u64)t->p.line_bytes * node);
    u64 *nd = NODE(t, node);
    nd[1] = val; nd[0] = key;
    NODE(t, w.tail)[2 * t->pairs] = node;
    return ORC_INSERTED;
  }
  u64 *nd = NODE(t, (u64)w.fm);
  nd[2 * w.fj + 1] = val;
  nd[2 * w.fj] = key;
  return ORC_INSERTED;
}

static int ch_erase(orc_table *t, u64 key) { /* chaining.py:213-226 */
  touch_lock_bucket(t, hb(t, 0, key, t->nb));
  walk_t w = ch_walk(t, key);
  if (w.m < 0) return 0;
  t->tomb_ever = 1;
  NODE(t, (u64)w.m)[2 * w.j] = TOMB;
  return 1;
}

/* ------------------------------------------------------------------- public */

orc_table *orc_create(const orc_params *p) {
  orc_table *t = (orc_table *)calloc(1, sizeof(orc_table));
  t->p = *p;
  t->bs = p->bucket_size;
  t->cap = p->capacity_slots;
  t->nb = t->cap / (u64)t->bs;
  t->md = p->design == ORC_DOUBLE_MD || p->design == ORC_P2_MD || p->design == ORC_ICEBERG_MD;
  t->front = t->nb;
  if (p->design == ORC_ICEBERG || p->design == ORC_ICEBERG_MD) {
    t->front = p->front_buckets;
    t->back = t->nb - t->front;
  }
  if (p->design == ORC_CHAINING) {
    t->pairs = t->bs;
    t->wpn = 2 * t->bs + 2;
    t->arena_cap = t->nb + 1;
    t->next_node = t->nb + 1;
    t->w = (u64 *)calloc((size_t)(t->wpn * t->arena_cap), sizeof(u64));
  } else {
    t->w = (u64 *)calloc((size_t)(2 * t->cap), sizeof(u64));
  }
  if (t->md) t->tags = (uint16_t *)calloc((size_t)t->cap, sizeof(uint16_t));
  t->pmask = 32767;
  t->pkey = (u64 *)calloc(t->pmask + 1, sizeof(u64));
  t->pgen = (uint32_t *)calloc(t->pmask + 1, sizeof(uint32_t));
  t->gen = 1;
  return t;
}

void orc_destroy(orc_table *t) {
  if (!t) return;
  free(t->w); free(t->tags); free(t->pkey); free(t->pgen);
  free(t);
}

static int is_sentinel(u64 k) { return k == EMPTY || k >= RESV; }

int orc_upsert(orc_table *t, u64 key, u64 val, int merge) {
  if (is_sentinel(key)) return -1;
  switch (t->p.design) {
  case ORC_DOUBLE: case ORC_DOUBLE_MD: return dbl_upsert(t, key, val, merge);
  case ORC_P2: case ORC_P2_MD: case ORC_UNSAFE: return p2_upsert(t, key, val, merge);
  case ORC_ICEBERG: case ORC_ICEBERG_MD: return ice_upsert(t, key, val, merge);
  case ORC_CUCKOO: return ck_upsert(t, key, val, merge);
  default: return ch_upsert(t, key, val, merge);
  }
}

int orc_query(orc_table *t, u64 key, u64 *val_out) {
  u64 v = 0;
  i64 idx;
  if (is_sentinel(key)) return -1;
  switch (t->p.design) {
  case ORC_DOUBLE: case ORC_DOUBLE_MD: idx = dbl_find(t, key, &v); break;
  case ORC_P2: case ORC_P2_MD: case ORC_UNSAFE: idx = p2_find(t, key, &v, 1); break;
  case ORC_ICEBERG: case ORC_ICEBERG_MD: idx = ice_find(t, key, &v, 1); break;
  case ORC_CUCKOO: idx = ck_find(t, key, &v, 1); break;
  default: { walk_t w = ch_walk(t, key); idx = w.m; v = w.val; }
  }
  if (val_out) *val_out = idx >= 0 ? v : 0;
  return idx >= 0;
}

int orc_erase(orc_table *t, u64 key) {
  if (is_sentinel(key)) return -1;
  switch (t->p.design) {
  case ORC_DOUBLE: case ORC_DOUBLE_MD: return dbl_erase(t, key);
  case ORC_P2: case ORC_P2_MD: case ORC_UNSAFE: return p2_erase(t, key);
  case ORC_ICEBERG: case ORC_ICEBERG_MD: return ice_erase(t, key);
  case ORC_CUCKOO: return ck_erase(t, key);
  default: return ch_erase(t, key);
  }
}

int64_t orc_slot_of(orc_table *t, u64 key) { /* the _locate of each design */
  uint32_t *sink = t->sink;
  t->sink = NULL;
  i64 idx;
  switch (t->p.design) {
  case ORC_DOUBLE: case ORC_DOUBLE_MD: idx = dbl_find(t, key, NULL); break;
  case ORC_P2: case ORC_P2_MD: case ORC_UNSAFE: idx = p2_find(t, key, NULL, 0); break;
  case ORC_ICEBERG: case ORC_ICEBERG_MD: idx = ice_find(t, key, NULL, 0); break;
  case ORC_CUCKOO: idx = ck_find(t, key, NULL, 0); break;
  default: {
    walk_t w = ch_walk(t, key);
    idx = w.m >= 0 ? w.m * t->bs + w.j : -1;
  }
  }
  t->sink = sink;
  return idx;
}

uint64_t orc_primary_bucket(orc_table *t, u64 key) {
  if (t->p.design == ORC_ICEBERG || t->p.design == ORC_ICEBERG_MD) return hb(t, 0, key, t->front);
  return hb(t, 0, key, t->nb);
}

void orc_upsert_n(orc_table *t, const u64 *keys, const u64 *vals, u64 n, int merge, uint8_t *status) {
  t->sink_i = 0;
  for (u64 i = 0; i < n; i++) {
    int s = orc_upsert(t, keys[i], vals[i], merge);
    finish_op(t);
    if (status) status[i] = (uint8_t)s;
  }
}

void orc_query_n(orc_table *t, const u64 *keys, u64 n, u64 *vals, uint8_t *found) {
  t->sink_i = 0;
  for (u64 i = 0; i < n; i++) {
    u64 v = 0;
    int f = orc_query(t, keys[i], &v);
    finish_op(t);
    if (vals) vals[i] = v;
    if (found) found[i] = (uint8_t)f;
  }
}

void orc_erase_n(orc_table *t, const u64 *keys, u64 n, uint8_t *found) {
  t->sink_i = 0;
  for (u64 i = 0; i < n; i++) {
    int f = orc_erase(t, keys[i]);
    finish_op(t);
    if (found) found[i] = (uint8_t)f;
  }
}

void orc_mixed_n(orc_table *t, const uint8_t *ops, const u64 *keys, const u64 *vals, u64 n,
                 uint8_t *status, u64 *vals_out) {
  t->sink_i = 0;
  for (u64 i = 0; i < n; i++) {
    int kind = ops[i] & 15, merge = ops[i] >> 4, s;
    u64 v = 0;
    if (kind == ORC_OP_UPSERT) s = orc_upsert(t, keys[i], vals[i], merge);
    else if (kind == ORC_OP_ERASE) s = orc_erase(t, keys[i]);
    else s = orc_query(t, keys[i], &v);
    finish_op(t);
    if (status) status[i] = (uint8_t)s;
    if (vals_out) vals_out[i] = v;
  }
}

void orc_set_probe_sink(orc_table *t, uint32_t *probes, uint64_t n) {
  t->sink = probes;
  t->sink_n = n;
  t->sink_i = 0;
  t->pcount = 0;
  if (!probes) return; /* detaching keeps the counters readable */
  t->lock_touches = 0;
  t->saturated = 0;
  if (++t->gen == 0) { memset(t->pgen, 0, sizeof(uint32_t) * (t->pmask + 1)); t->gen = 1; }
}

uint64_t orc_lock_touches(orc_table *t) { return t->lock_touches; }
int orc_probe_saturated(orc_table *t) { return t->saturated; }

uint64_t orc_items(orc_table *t, u64 *keys, u64 *vals, u64 cap) {
  u64 n = 0;
  if (t->p.design == ORC_CHAINING) {
    for (u64 m = 1; m < t->next_node; m++) {
      u64 *nd = NODE(t, m);
      for (int j = 0; j < t->pairs; j++) {
        u64 k = nd[2 * j];
        if (is_sentinel(k)) continue;
        if (n < cap) { if (keys) keys[n] = k; if (vals) vals[n] = nd[2 * j + 1]; }
        n++;
      }
    }
    return n;
  }
  for (u64 i = 0; i < t->cap; i++) {
    u64 k = K(t, i);
    if (is_sentinel(k)) continue;
    if (n < cap) { if (keys) keys[n] = k; if (vals) vals[n] = V(t, i); }
    n++;
  }
  return n;
}

uint64_t orc_occupied(orc_table *t) { return orc_items(t, NULL, NULL, 0); }

uint64_t orc_data_words(orc_table *t) {
  if (t->p.design == ORC_CHAINING) return (u64)t->wpn * t->next_node;
  return 2 * t->cap;
}

void orc_export_words(orc_table *t, u64 *out) {
  memcpy(out, t->w, sizeof(u64) * orc_data_words(t));
}

void orc_export_tags(orc_table *t, uint16_t *out) {
  if (t->tags) memcpy(out, t->tags, sizeof(uint16_t) * t->cap);
  else memset(out, 0, sizeof(uint16_t) * t->cap);
}

uint64_t orc_next_node(orc_table *t) { return t->next_node; }
uint64_t orc_arena_capacity(orc_table *t) { return t->arena_cap; }
int orc_tombstones_ever(orc_table *t) { return t->tomb_ever; }
