/*
 * kvcache_oracle.c — TEST INFRASTRUCTURE ONLY (the CPU checker).
 *
 * Plain-C restatement of the reference's prefix-indexed KV block cache and
 * its hashing, used by tests/ (and bench.py's cpu_baseline leg) as the parity
 * oracle for the CUDA product path.  Nothing in paper_2601_12967_b200/ may
 * link or call this file.
 *
 * Parity is pinned: tests/test_oracle_golden.py checks this restatement
 * against golden op logs produced by the reference itself (oracle/_ref,
 * built from /root/reference by oracle/Makefile; see tests/golden/README).
 *
 * Reference (paths relative to /root/reference/proj):
 *   splitmix64 / hash_combine     include/agentsim/common.hpp:136-145
 *   kv_root_hash / kv_chain_hash  src/kv_cache.cpp:35-41
 *   eviction_tier                 src/kv_cache.cpp:23-33
 *   lookup_prefix                 src/kv_cache.cpp:85-101
 *   insert (+rollback)            src/kv_cache.cpp:103-175
 *   evict                         src/kv_cache.cpp:177-197
 *   set_reuse_priority / set_tag  src/kv_cache.cpp:209-226
 *   release / touch               src/kv_cache.cpp:228-240
 *   audit / dump                  src/kv_cache.cpp:242-281
 *   materialize_tokens            src/trace.cpp:50-78
 *   decode_token                  src/trace.cpp:80-83
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* status codes: same numbering as include/sutradhara_b200.h */
#define OC_OK 0
#define OC_CACHE_FULL 1
#define OC_UNKNOWN_BLOCK 2
#define OC_ZERO_REF 3
#define OC_CACHE_ERR 4
#define OC_CONFIG 5

/* ------------------------------------------------------------------ hashing */
uint64_t oc_splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

uint64_t oc_hash_combine(uint64_t seed, uint64_t value) {
  uint64_t mixed = value + 0x9e3779b97f4a7c15ULL + (seed << 6) + (seed >> 2);
  return oc_splitmix64(seed ^ mixed);
}

uint64_t oc_root_hash(void) { return 0x6b76726f6f740001ULL; }

uint64_t oc_chain_hash(uint64_t parent, const uint64_t* tok, int64_t n) {
  uint64_t h = parent;
  for (int64_t i = 0; i < n; ++i) h = oc_hash_combine(h, tok[i]);
  return h;
}

/* SectionTag order: 0 system, 1 user, 2 tool_output, 3 history */
static uint64_t section_salt(int tag) {
  static const uint64_t salts[4] = {0x53595354454d5052ULL, 0x555345525155455aULL,
                                    0x544f4f4c4f555450ULL, 0x48495354f52590aaULL};
  return (tag >= 0 && tag < 4) ? salts[tag] : 0;
}

void oc_materialize(int tag, int64_t len, uint64_t key, int32_t src_iter, uint64_t* out) {
  uint64_t seed = oc_splitmix64(key ^ section_salt(tag));
  if (tag == 2) seed = oc_hash_combine(seed, (uint64_t)(int64_t)src_iter);
  for (int64_t i = 0; i < len; ++i) out[i] = oc_splitmix64(seed + (uint64_t)i);
}

uint64_t oc_decode_token(uint64_t stream_key, int64_t index) {
  return oc_splitmix64(oc_splitmix64(stream_key ^ 0xdec0de0000000001ULL) + (uint64_t)index);
}

/* Tier table indexed by tag: RESPONSE 0, TOOL_OUTPUT 1, USER_QUERY 2,
 * SYSTEM_PROMPT 3, PARTIAL_PREFILL 4, HISTORY 2. */
int oc_tier(int tag) {
  static const int tiers[6] = {0, 1, 2, 3, 4, 2};
  return (tag >= 0 && tag < 6) ? tiers[tag] : 0;
}

/* ------------------------------------------------------------- cache state */
typedef struct {
  int resident;
  uint64_t chain, parent;
  int tag, tier, ref, pinned;
  int64_t last;
  int ntok;
} oc_block;

typedef struct {
  int64_t bs, cap;
  int policy; /* 0 lru, 1 tiered */
  oc_block* blk;
  uint64_t* tok;   /* cap * bs */
  int64_t n_res;
  uint64_t evicted;
  /* chain-hash multimap: open addressing, value = block id, -1 empty, -2 tomb */
  int64_t tcap, ntomb;
  uint64_t* tkey;
  int32_t* tval;
} oc_cache;

static uint64_t slot_of(const oc_cache* c, uint64_t h) { return oc_splitmix64(h) & (uint64_t)(c->tcap - 1); }

static void index_add(oc_cache* c, uint64_t h, int32_t id) {
  uint64_t s = slot_of(c, h);
  while (c->tval[s] >= 0) s = (s + 1) & (uint64_t)(c->tcap - 1);
  c->tkey[s] = h;
  c->tval[s] = id;
}

static void index_rebuild(oc_cache* c);

static void index_del(oc_cache* c, uint64_t h, int32_t id) {
  uint64_t s = slot_of(c, h);
  while (c->tval[s] != -1) {
    if (c->tval[s] == id && c->tkey[s] == h) {
      c->tval[s] = -2;
      if (++c->ntomb > c->tcap / 4) index_rebuild(c);
      return;
    }
    s = (s + 1) & (uint64_t)(c->tcap - 1);
  }
}

oc_cache* oc_create(int64_t bs, int64_t cap, int policy) {
  if (bs < 1 || cap < 1) return NULL;
  oc_cache* c = (oc_cache*)calloc(1, sizeof(oc_cache));
  c->bs = bs;
  c->cap = cap;
  c->policy = policy;
  c->blk = (oc_block*)calloc((size_t)cap, sizeof(oc_block));
  c->tok = (uint64_t*)calloc((size_t)(cap * bs), sizeof(uint64_t));
  c->tcap = 16;
  while (c->tcap < 4 * cap) c->tcap <<= 1;
  c->tkey = (uint64_t*)calloc((size_t)c->tcap, sizeof(uint64_t));
  c->tval = (int32_t*)malloc((size_t)c->tcap * sizeof(int32_t));
  for (int64_t i = 0; i < c->tcap; ++i) c->tval[i] = -1;
  return c;
}

void oc_destroy(oc_cache* c) {
  if (!c) return;
  free(c->blk);
  free(c->tok);
  free(c->tkey);
  free(c->tval);
  free(c);
}

/* Finds a resident block with this (chain, parent, tokens); -1 if none. */
/* drops tombstones: re-adds every resident block (the index is only a
 * lookup accelerator; its probe order never affects results because no two
 * resident blocks share (chain, parent, tokens)). */
static void index_rebuild(oc_cache* c) {
  for (int64_t i = 0; i < c->tcap; ++i) c->tval[i] = -1;
  c->ntomb = 0;
  for (int64_t i = 0; i < c->cap; ++i)
    if (c->blk[i].resident) index_add(c, c->blk[i].chain, (int32_t)i);
}

static int32_t find_block(const oc_cache* c, uint64_t h, uint64_t parent, const uint64_t* t, int64_t n) {
  uint64_t s = slot_of(c, h);
  while (c->tval[s] != -1) {
    int32_t id = c->tval[s];
    if (id >= 0 && c->tkey[s] == h) {
      const oc_block* b = &c->blk[id];
      if (b->resident && b->parent == parent && b->ntok == n &&
          memcmp(&c->tok[(int64_t)id * c->bs], t, (size_t)n * sizeof(uint64_t)) == 0)
        return id;
    }
    s = (s + 1) & (uint64_t)(c->tcap - 1);
  }
  return -1;
}

static void drop_block(oc_cache* c, int32_t id) {
  oc_block* b = &c->blk[id];
  if (!b->resident) return;
  b->resident = 0; /* before index_del: a rebuild there re-adds residents only */
  index_del(c, b->chain, id);
  c->n_res--;
}

static int32_t lowest_free(const oc_cache* c) {
  for (int64_t i = 0; i < c->cap; ++i)
    if (!c->blk[i].resident) return (int32_t)i;
  return -1;
}

int64_t oc_lookup_prefix(oc_cache* c, const uint64_t* t, int64_t n, int64_t now) {
  uint64_t parent = oc_root_hash();
  int64_t nblk = 0;
  int32_t* hit = (int32_t*)malloc((size_t)(n / c->bs + 1) * sizeof(int32_t));
  for (int64_t pos = 0; pos + c->bs <= n; pos += c->bs) {
    uint64_t h = oc_chain_hash(parent, t + pos, c->bs);
    int32_t id = find_block(c, h, parent, t + pos, c->bs);
    if (id < 0) break;
    hit[nblk++] = id;
    parent = h;
  }
  for (int64_t i = 0; i < nblk; ++i) c->blk[hit[i]].last = now;
  free(hit);
  return nblk * c->bs;
}

/* ordering of eviction candidates */
static const oc_cache* g_sort_cache;
static int cmp_victim(const void* pa, const void* pb) {
  const oc_cache* c = g_sort_cache;
  const oc_block* a = &c->blk[*(const int32_t*)pa];
  const oc_block* b = &c->blk[*(const int32_t*)pb];
  if (c->policy == 1 && a->tier != b->tier) return a->tier < b->tier ? -1 : 1;
  if (a->last != b->last) return a->last < b->last ? -1 : 1;
  int32_t ia = *(const int32_t*)pa, ib = *(const int32_t*)pb;
  return ia < ib ? -1 : (ia > ib ? 1 : 0);
}

int64_t oc_evict(oc_cache* c, int64_t needed, int32_t* out) {
  int32_t* cand = (int32_t*)malloc((size_t)c->cap * sizeof(int32_t));
  int64_t nc = 0;
  for (int64_t i = 0; i < c->cap; ++i) {
    const oc_block* b = &c->blk[i];
    if (b->resident && !b->pinned && b->ref == 0) cand[nc++] = (int32_t)i;
  }
  g_sort_cache = c;
  qsort(cand, (size_t)nc, sizeof(int32_t), cmp_victim);
  int64_t take = needed < nc ? needed : nc;
  if (take < 0) take = 0;
  for (int64_t i = 0; i < take; ++i) {
    if (out) out[i] = cand[i];
    drop_block(c, cand[i]);
  }
  c->evicted += (uint64_t)take;
  free(cand);
  return take;
}

/* tags: array of (begin, end, tag) triples flattened as int64 */
int oc_insert(oc_cache* c, const uint64_t* t, int64_t n, const int64_t* tags, int64_t ntags,
              int64_t now, int32_t* out, int64_t* nout) {
  int64_t covered = 0;
  *nout = 0;
  for (int64_t r = 0; r < ntags; ++r) {
    if (tags[3 * r] != covered || tags[3 * r + 1] < tags[3 * r]) return OC_CACHE_ERR;
    covered = tags[3 * r + 1];
  }
  if (covered != n) return OC_CACHE_ERR;
  if (n == 0) return OC_OK;
  int64_t nblocks = (n + c->bs - 1) / c->bs;
  int32_t* chain = (int32_t*)malloc((size_t)nblocks * sizeof(int32_t));
  unsigned char* fresh = (unsigned char*)calloc((size_t)nblocks, 1);
  uint64_t parent = oc_root_hash();
  int64_t k = 0;
  for (int64_t pos = 0; pos < n; pos += c->bs, ++k) {
    int64_t len = (n - pos) < c->bs ? (n - pos) : c->bs;
    uint64_t h = oc_chain_hash(parent, t + pos, len);
    int32_t id = find_block(c, h, parent, t + pos, len);
    if (id >= 0) {
      c->blk[id].ref += 1;
      c->blk[id].last = now;
    } else {
      if (c->n_res >= c->cap) {
        oc_evict(c, 1, NULL);
        if (c->n_res >= c->cap) {
          /* undo: drop this insert's references, free its new blocks */
          for (int64_t j = 0; j < k; ++j) c->blk[chain[j]].ref -= 1;
          for (int64_t j = 0; j < k; ++j)
            if (fresh[j]) drop_block(c, chain[j]);
          free(chain);
          free(fresh);
          return OC_CACHE_FULL;
        }
      }
      id = lowest_free(c);
      int tag = 0;
      int found = 0;
      for (int64_t r = 0; r < ntags; ++r)
        if (pos >= tags[3 * r] && pos < tags[3 * r + 1]) {
          tag = (int)tags[3 * r + 2];
          found = 1;
          break;
        }
      if (!found) tag = ntags ? (int)tags[3 * (ntags - 1) + 2] : 0;
      oc_block* b = &c->blk[id];
      b->resident = 1;
      b->chain = h;
      b->parent = parent;
      b->tag = tag;
      b->tier = oc_tier(tag);
      b->ref = 1;
      b->last = now;
      b->pinned = 0;
      b->ntok = (int)len;
      memcpy(&c->tok[(int64_t)id * c->bs], t + pos, (size_t)len * sizeof(uint64_t));
      index_add(c, h, id);
      c->n_res++;
      fresh[k] = 1;
    }
    chain[k] = id;
    parent = h;
  }
  memcpy(out, chain, (size_t)nblocks * sizeof(int32_t));
  *nout = nblocks;
  free(chain);
  free(fresh);
  return OC_OK;
}

int oc_set_priority(oc_cache* c, const int32_t* ids, int64_t n, int pinned, int tier_override) {
  for (int64_t i = 0; i < n; ++i)
    if (ids[i] < 0 || ids[i] >= c->cap || !c->blk[ids[i]].resident) return OC_UNKNOWN_BLOCK;
  for (int64_t i = 0; i < n; ++i) {
    oc_block* b = &c->blk[ids[i]];
    if (pinned >= 0) b->pinned = pinned;
    if (tier_override >= 0) {
      b->tag = tier_override;
      b->tier = oc_tier(tier_override);
    }
  }
  return OC_OK;
}

int oc_set_tag(oc_cache* c, int32_t id, int tag) {
  if (id < 0 || id >= c->cap || !c->blk[id].resident) return OC_UNKNOWN_BLOCK;
  c->blk[id].tag = tag;
  c->blk[id].tier = oc_tier(tag);
  return OC_OK;
}

int oc_release(oc_cache* c, const int32_t* ids, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    if (ids[i] < 0 || ids[i] >= c->cap || !c->blk[ids[i]].resident) return OC_UNKNOWN_BLOCK;
    if (c->blk[ids[i]].ref < 1) return OC_ZERO_REF;
  }
  for (int64_t i = 0; i < n; ++i) c->blk[ids[i]].ref -= 1;
  return OC_OK;
}

int oc_touch(oc_cache* c, const int32_t* ids, int64_t n, int64_t now) {
  for (int64_t i = 0; i < n; ++i) {
    if (ids[i] < 0 || ids[i] >= c->cap || !c->blk[ids[i]].resident) return OC_UNKNOWN_BLOCK;
    c->blk[ids[i]].last = now;
  }
  return OC_OK;
}

int64_t oc_resident(const oc_cache* c) { return c->n_res; }
uint64_t oc_total_evicted(const oc_cache* c) { return c->evicted; }
int oc_contains(const oc_cache* c, int32_t id) { return id >= 0 && id < c->cap && c->blk[id].resident; }

/* fields: tag, tier, ref, pinned, ntok, last, chain, parent */
int oc_block_info(const oc_cache* c, int32_t id, int64_t* f, uint64_t* h, uint64_t* tokens) {
  if (!oc_contains(c, id)) return OC_UNKNOWN_BLOCK;
  const oc_block* b = &c->blk[id];
  f[0] = b->tag;
  f[1] = b->tier;
  f[2] = b->ref;
  f[3] = b->pinned;
  f[4] = b->ntok;
  f[5] = b->last;
  h[0] = b->chain;
  h[1] = b->parent;
  if (tokens) memcpy(tokens, &c->tok[(int64_t)id * c->bs], (size_t)b->ntok * sizeof(uint64_t));
  return OC_OK;
}

static const char* tag_name(int tag) {
  static const char* names[6] = {"response", "tool_output", "user_query",
                                 "system_prompt", "partial_prefill", "history"};
  return (tag >= 0 && tag < 6) ? names[tag] : "unknown";
}

/* Writes the audit dump (same format as the reference) into buf; returns the
 * full length. */
int64_t oc_dump(const oc_cache* c, char* buf, int64_t cap) {
  int64_t len = 0;
  char line[256];
  for (int64_t i = 0; i < c->cap; ++i) {
    const oc_block* b = &c->blk[i];
    if (!b->resident) continue;
    int m = snprintf(line, sizeof line, "block=%lld tag=%s tier=%d ref=%d pinned=%d last_used=%lld tokens=%d\n",
                     (long long)i, tag_name(b->tag), b->tier, b->ref, b->pinned ? 1 : 0,
                     (long long)b->last, b->ntok);
    if (buf && len + m < cap) memcpy(buf + len, line, (size_t)m);
    len += m;
  }
  if (buf && len < cap) buf[len] = 0;
  return len;
}

int oc_audit(const oc_cache* c) {
  int64_t res = 0;
  for (int64_t i = 0; i < c->cap; ++i) {
    const oc_block* b = &c->blk[i];
    if (!b->resident) continue;
    ++res;
    if (b->ref < 0) return OC_CACHE_ERR;
    if (b->ntok < 1 || b->ntok > c->bs) return OC_CACHE_ERR;
  }
  return res == c->n_res && res <= c->cap ? OC_OK : OC_CACHE_ERR;
}

/* FNV-1a 64 of a byte string (digest used by the golden op logs). */
uint64_t oc_fnv1a(const char* s, int64_t n) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (int64_t i = 0; i < n; ++i) {
    h ^= (unsigned char)s[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}
