// agentsim_kvcache_b200.cpp — the reference-side binding a maintainer adds to
// the reference (agentsim) to run its UNMODIFIED engine/orchestrator on the
// B200 block pool: this file replaces src/kv_cache.cpp at link time and
// implements every non-inline member of agentsim::KvCache
// (include/agentsim/kv_cache.hpp:70-128) through the C-ABI of
// include/sutradhara_b200.h.  Exceptions are re-raised with the reference's
// own types (common.hpp:72-90).
//
// The header's inline accessors (resident_blocks, contains, free_blocks,
// total_evicted) read the private members `blocks_` and `total_evicted_`, so
// the binding keeps them mirrored after every call that changes residency
// (insert / evict), from the change itself: the ids the call evicted
// (sb_kv_last_evicted) and the chain it returned — O(change), no O(capacity)
// read-back.  The pool's device comes from SB_DEVICE / LOCAL_RANK.
//
// Build (see oracle/Makefile target `b200`): compile with the reference's
// include/ on the include path and link against libsutradhara_b200.so.
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "agentsim/kv_cache.hpp"
#include "sutradhara_b200.h"

namespace {

std::map<const agentsim::KvCache*, sb_kv_cache*> g_pools;

sb_kv_cache* pool(const agentsim::KvCache* c) { return g_pools.at(c); }

[[noreturn]] void raise(int st) {
  std::string msg = sb_last_error();
  switch (st) {
    case SB_ERR_CACHE_FULL: throw agentsim::CacheFull(msg);
    case SB_ERR_UNKNOWN_BLOCK: throw agentsim::UnknownBlock(msg);
    case SB_ERR_ZERO_REF_RELEASE: throw agentsim::ZeroRefRelease(msg);
    case SB_ERR_CONFIG: throw agentsim::ConfigError(msg);
    default: throw agentsim::CacheError(msg);
  }
}

void check(int st) {
  if (st != SB_OK) raise(st);
}

}  // namespace

namespace agentsim {

const char* to_string(KvTag tag) {
  static const char* n[6] = {"response", "tool_output", "user_query", "system_prompt", "partial_prefill", "history"};
  return n[static_cast<int>(tag)];
}

int eviction_tier(KvTag tag) {
  static const int t[6] = {0, 1, 2, 3, 4, 2};
  return t[static_cast<int>(tag)];
}

std::uint64_t kv_root_hash() { return sb_kv_root_hash(); }

std::uint64_t kv_chain_hash(std::uint64_t parent, std::span<const TokenId> t) {
  return sb_kv_chain_hash_host(parent, t.data(), static_cast<int64_t>(t.size()));
}

// Mirrors the residency change of one insert / evict into the
// header-visible members, in O(change): the ids the device evicted
// (sb_kv_last_evicted) leave blocks_, the chain an insert returned is
// resident (new blocks, including evicted-and-reused ids, get fresh records).
static void apply_delta(sb_kv_cache* p, std::unordered_map<std::int32_t, KvBlock>& blocks,
                        const std::vector<std::int32_t>& chain, std::uint64_t& total_evicted) {
  int64_t n = 0;
  check(sb_kv_last_evicted(p, nullptr, 0, &n));
  std::vector<int32_t> ev(static_cast<size_t>(n));
  if (n) check(sb_kv_last_evicted(p, ev.data(), n, &n));
  for (int32_t id : ev) blocks.erase(id);
  for (int32_t id : chain) {
    auto it = blocks.find(id);
    if (it == blocks.end()) blocks[id].block_id = id;
  }
  total_evicted += static_cast<std::uint64_t>(n);
}

// The device this pool lives on: SB_DEVICE, else the torchrun LOCAL_RANK,
// else 0 — one pool per GPU when each rank runs its own engine.
static int pool_device() {
  for (const char* v : {"SB_DEVICE", "LOCAL_RANK"})
    if (const char* e = std::getenv(v)) return std::atoi(e);
  return 0;
}

KvCache::KvCache(const CacheConfig& config) : config_(config) {
  if (config_.block_size < 1) throw ConfigError("cache block_size must be >= 1");
  if (config_.capacity_blocks < 1) throw ConfigError("cache capacity_blocks must be >= 1");
  sb_kv_cache* p = nullptr;
  check(sb_kv_create(config.block_size, config.capacity_blocks,
                     config.policy == EvictionPolicy::kTiered ? SB_POLICY_TIERED : SB_POLICY_LRU, pool_device(),
                     &p));
  auto old = g_pools.find(this);
  if (old != g_pools.end()) sb_kv_destroy(old->second);
  g_pools[this] = p;
  total_evicted_ = 0;
}

std::int64_t KvCache::lookup_prefix(std::span<const TokenId> tokens, SimTime now) {
  int64_t hit = 0;
  check(sb_kv_lookup_prefix(pool(this), tokens.data(), static_cast<int64_t>(tokens.size()), now, &hit));
  return hit;
}

std::vector<std::int32_t> KvCache::insert(std::span<const TokenId> tokens, std::span<const TagRange> tags,
                                          SimTime now) {
  std::vector<sb_tag_range> tr(tags.size());
  for (size_t i = 0; i < tags.size(); ++i) tr[i] = sb_tag_range{tags[i].begin, tags[i].end, int32_t(tags[i].tag), 0};
  const size_t bs = static_cast<size_t>(config_.block_size);
  std::vector<std::int32_t> out((tokens.size() + bs - 1) / bs + 1);
  int64_t n = 0;
  int st = sb_kv_insert(pool(this), tokens.data(), static_cast<int64_t>(tokens.size()), tr.data(),
                        static_cast<int64_t>(tr.size()), now, out.data(), &n);
  out.resize(st == SB_OK ? static_cast<size_t>(n) : 0);
  apply_delta(pool(this), blocks_, out, total_evicted_);
  if (st != SB_OK) raise(st);
  return out;
}

std::vector<std::int32_t> KvCache::evict(std::size_t needed) {
  std::vector<std::int32_t> out(needed + 1);
  int64_t n = 0;
  check(sb_kv_evict(pool(this), static_cast<int64_t>(needed), out.data(), &n));
  apply_delta(pool(this), blocks_, {}, total_evicted_);
  out.resize(static_cast<size_t>(n));
  return out;
}

void KvCache::set_reuse_priority(std::span<const std::int32_t> ids, const PriorityUpdate& u) {
  check(sb_kv_set_reuse_priority(pool(this), ids.data(), static_cast<int64_t>(ids.size()),
                                 u.pinned ? (*u.pinned ? 1 : 0) : -1,
                                 u.tier_override ? static_cast<int32_t>(*u.tier_override) : -1));
}

void KvCache::set_tag(std::int32_t id, KvTag tag) { check(sb_kv_set_tag(pool(this), id, static_cast<int32_t>(tag))); }

void KvCache::release(std::span<const std::int32_t> ids) {
  check(sb_kv_release(pool(this), ids.data(), static_cast<int64_t>(ids.size())));
}

void KvCache::touch(std::span<const std::int32_t> ids, SimTime now) {
  check(sb_kv_touch(pool(this), ids.data(), static_cast<int64_t>(ids.size()), now));
}

const KvBlock& KvCache::block(std::int32_t id) const {
  sb_block_info info{};
  std::vector<uint64_t> toks(static_cast<size_t>(config_.block_size));
  check(sb_kv_block(pool(this), id, &info, toks.data()));
  auto& self = const_cast<KvCache*>(this)->blocks_;
  KvBlock& b = self[id];
  b.block_id = id;
  b.chain_hash = info.chain_hash;
  b.parent_hash = info.parent_hash;
  b.tag = static_cast<KvTag>(info.tag);
  b.tier = info.tier;
  b.ref_count = info.ref_count;
  b.last_used = info.last_used;
  b.pinned = info.pinned != 0;
  toks.resize(static_cast<size_t>(info.n_tokens));
  b.tokens = std::move(toks);
  return b;
}

void KvCache::audit() const { check(sb_kv_audit(pool(this))); }

std::string KvCache::dump() const {
  int64_t n = 0;
  check(sb_kv_dump(pool(this), nullptr, 0, &n));
  std::string s(static_cast<size_t>(n) + 1, '\0');
  check(sb_kv_dump(pool(this), s.data(), n + 1, &n));
  s.resize(static_cast<size_t>(n));
  return s;
}

}  // namespace agentsim
