// ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
//
// C-ABI shim over the UNMODIFIED reference KvCache and hashing
// (/root/reference/proj/src/kv_cache.cpp, include/agentsim/common.hpp,
// src/trace.cpp), compiled by oracle/Makefile into oracle/_ref/.  Used by the
// golden-vector generator (oracle/gen_golden.py), the parity tests and
// bench.py's reference arm.  Never linked into the product.
//
// The file is compiled twice: once as-is (symbols REF_PREFIX = ref_) and
// once with -Dagentsim=agentsim_ref -DREF_PREFIX=refns_ so that the recording
// KvCache in ref_kvlog.cpp can forward to a renamed copy of the reference
// cache while the reference engine links against the recorder.
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "agentsim/kv_cache.hpp"
#include "agentsim/trace.hpp"

#ifndef REF_PREFIX
#define REF_PREFIX ref_
#endif
#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)
#define F(name) CAT(REF_PREFIX, name)

using namespace agentsim;

namespace {
int status_of(const std::exception& e) {
  if (dynamic_cast<const CacheFull*>(&e)) return 1;
  if (dynamic_cast<const UnknownBlock*>(&e)) return 2;
  if (dynamic_cast<const ZeroRefRelease*>(&e)) return 3;
  if (dynamic_cast<const CacheError*>(&e)) return 4;
  if (dynamic_cast<const ConfigError*>(&e)) return 5;
  return 9;
}
thread_local std::string g_err;
}  // namespace

#define GUARD_BEGIN try {
#define GUARD_END                  \
  }                                \
  catch (const std::exception& e) { \
    g_err = e.what();              \
    return status_of(e);           \
  }                                \
  return 0;

extern "C" {

const char* F(last_error)() { return g_err.c_str(); }

uint64_t F(root_hash)() { return kv_root_hash(); }

uint64_t F(chain_hash)(uint64_t parent, const uint64_t* t, int64_t n) {
  return kv_chain_hash(parent, std::span<const TokenId>(t, static_cast<size_t>(n)));
}

void F(materialize)(int32_t tag, int64_t len, uint64_t key, int32_t src_iter, uint64_t* out) {
  PromptSection s{static_cast<SectionTag>(tag), len, key, src_iter};
  std::vector<TokenId> v = materialize_tokens(s);
  if (!v.empty()) std::memcpy(out, v.data(), v.size() * sizeof(uint64_t));
}

uint64_t F(decode_token)(uint64_t key, int64_t idx) { return decode_token(key, idx); }

int F(kv_create)(int64_t bs, int64_t cap, int32_t policy, void** out) {
  GUARD_BEGIN
  CacheConfig cfg;
  cfg.block_size = bs;
  cfg.capacity_blocks = cap;
  cfg.policy = policy ? EvictionPolicy::kTiered : EvictionPolicy::kLru;
  *out = new KvCache(cfg);
  GUARD_END
}

void F(kv_destroy)(void* c) { delete static_cast<KvCache*>(c); }

int F(kv_lookup)(void* c, const uint64_t* t, int64_t n, int64_t now, int64_t* hit) {
  GUARD_BEGIN
  *hit = static_cast<KvCache*>(c)->lookup_prefix(std::span<const TokenId>(t, size_t(n)), now);
  GUARD_END
}

int F(kv_insert)(void* c, const uint64_t* t, int64_t n, const int64_t* tags, int64_t ntags,
                 int64_t now, int32_t* out, int64_t* nout) {
  *nout = 0;
  GUARD_BEGIN
  std::vector<TagRange> tr;
  for (int64_t i = 0; i < ntags; ++i)
    tr.push_back(TagRange{tags[3 * i], tags[3 * i + 1], static_cast<KvTag>(tags[3 * i + 2])});
  auto ids = static_cast<KvCache*>(c)->insert(std::span<const TokenId>(t, size_t(n)), tr, now);
  for (size_t i = 0; i < ids.size(); ++i) out[i] = ids[i];
  *nout = static_cast<int64_t>(ids.size());
  GUARD_END
}

int F(kv_evict)(void* c, int64_t needed, int32_t* out, int64_t* nout) {
  GUARD_BEGIN
  auto ids = static_cast<KvCache*>(c)->evict(static_cast<size_t>(needed));
  for (size_t i = 0; i < ids.size(); ++i) out[i] = ids[i];
  *nout = static_cast<int64_t>(ids.size());
  GUARD_END
}

int F(kv_set_priority)(void* c, const int32_t* ids, int64_t n, int32_t pinned, int32_t tier) {
  GUARD_BEGIN
  PriorityUpdate u;
  if (pinned >= 0) u.pinned = pinned != 0;
  if (tier >= 0) u.tier_override = static_cast<KvTag>(tier);
  static_cast<KvCache*>(c)->set_reuse_priority(std::span<const int32_t>(ids, size_t(n)), u);
  GUARD_END
}

int F(kv_set_tag)(void* c, int32_t id, int32_t tag) {
  GUARD_BEGIN
  static_cast<KvCache*>(c)->set_tag(id, static_cast<KvTag>(tag));
  GUARD_END
}

int F(kv_release)(void* c, const int32_t* ids, int64_t n) {
  GUARD_BEGIN
  static_cast<KvCache*>(c)->release(std::span<const int32_t>(ids, size_t(n)));
  GUARD_END
}

int F(kv_touch)(void* c, const int32_t* ids, int64_t n, int64_t now) {
  GUARD_BEGIN
  static_cast<KvCache*>(c)->touch(std::span<const int32_t>(ids, size_t(n)), now);
  GUARD_END
}

int64_t F(kv_resident)(void* c) { return static_cast<int64_t>(static_cast<KvCache*>(c)->resident_blocks()); }
uint64_t F(kv_total_evicted)(void* c) { return static_cast<KvCache*>(c)->total_evicted(); }
int F(kv_contains)(void* c, int32_t id) { return static_cast<KvCache*>(c)->contains(id) ? 1 : 0; }

// f: tag, tier, ref, pinned, ntok, last ; h: chain, parent
int F(kv_block)(void* c, int32_t id, int64_t* f, uint64_t* h, uint64_t* tokens) {
  GUARD_BEGIN
  const KvBlock& b = static_cast<KvCache*>(c)->block(id);
  f[0] = static_cast<int64_t>(b.tag);
  f[1] = b.tier;
  f[2] = b.ref_count;
  f[3] = b.pinned ? 1 : 0;
  f[4] = static_cast<int64_t>(b.tokens.size());
  f[5] = b.last_used;
  h[0] = b.chain_hash;
  h[1] = b.parent_hash;
  if (tokens) std::memcpy(tokens, b.tokens.data(), b.tokens.size() * sizeof(uint64_t));
  GUARD_END
}

int64_t F(kv_dump)(void* c, char* buf, int64_t cap) {
  std::string s = static_cast<KvCache*>(c)->dump();
  if (buf && cap > 0) {
    size_t m = std::min<size_t>(s.size(), static_cast<size_t>(cap - 1));
    std::memcpy(buf, s.data(), m);
    buf[m] = 0;
  }
  return static_cast<int64_t>(s.size());
}

int F(kv_audit)(void* c) {
  GUARD_BEGIN
  static_cast<KvCache*>(c)->audit();
  GUARD_END
}

}  // extern "C"
