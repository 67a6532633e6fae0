// ref_kvlog.cpp — TEST INFRASTRUCTURE ONLY.
//
// A recording implementation of agentsim::KvCache (reference header
// /root/reference/proj/include/agentsim/kv_cache.hpp) that forwards every call
// to the reference's own KvCache (compiled under the renamed namespace
// agentsim_ref, exposed through ref_capi.cpp as refns_*) and appends one JSON
// line per operation (inputs, outputs, status, and an FNV digest of the
// resulting audit dump) to an in-memory op log.  Linking the UNMODIFIED
// reference engine/orchestrator against this recorder yields golden op logs
// of real engine runs: exactly the call sequence a drop-in block pool sees.
#include <cstdint>
#include <cstring>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "agentsim/kv_cache.hpp"

extern "C" {
const char* refns_last_error();
uint64_t refns_root_hash();
uint64_t refns_chain_hash(uint64_t, const uint64_t*, int64_t);
int refns_kv_create(int64_t, int64_t, int32_t, void**);
int refns_kv_lookup(void*, const uint64_t*, int64_t, int64_t, int64_t*);
int refns_kv_insert(void*, const uint64_t*, int64_t, const int64_t*, int64_t, int64_t, int32_t*,
                    int64_t*);
int refns_kv_evict(void*, int64_t, int32_t*, int64_t*);
int refns_kv_set_priority(void*, const int32_t*, int64_t, int32_t, int32_t);
int refns_kv_set_tag(void*, int32_t, int32_t);
int refns_kv_release(void*, const int32_t*, int64_t);
int refns_kv_touch(void*, const int32_t*, int64_t, int64_t);
uint64_t refns_kv_total_evicted(void*);
int refns_kv_contains(void*, int32_t);
int refns_kv_block(void*, int32_t, int64_t*, uint64_t*, uint64_t*);
int64_t refns_kv_dump(void*, char*, int64_t);
int refns_kv_audit(void*);
}

namespace {

std::map<const agentsim::KvCache*, void*> g_impl;
std::string g_log;
bool g_enabled = true;

void* impl(const agentsim::KvCache* c) { return g_impl.at(c); }

const char kB64[] = "ABCDEFGHIJKLMNOPQRSTUVWXYZabcdefghijklmnopqrstuvwxyz0123456789+/";
std::string b64(const void* data, size_t n) {
  const auto* p = static_cast<const unsigned char*>(data);
  std::string out;
  out.reserve((n + 2) / 3 * 4);
  for (size_t i = 0; i < n; i += 3) {
    uint32_t v = p[i] << 16;
    if (i + 1 < n) v |= p[i + 1] << 8;
    if (i + 2 < n) v |= p[i + 2];
    out += kB64[(v >> 18) & 63];
    out += kB64[(v >> 12) & 63];
    out += i + 1 < n ? kB64[(v >> 6) & 63] : '=';
    out += i + 2 < n ? kB64[v & 63] : '=';
  }
  return out;
}

std::string ids_json(const int32_t* ids, size_t n) {
  std::string s = "[";
  for (size_t i = 0; i < n; ++i) {
    if (i) s += ',';
    s += std::to_string(ids[i]);
  }
  return s + "]";
}

uint64_t dump_fnv(void* c) {
  int64_t len = refns_kv_dump(c, nullptr, 0);
  std::string buf(static_cast<size_t>(len) + 1, '\0');
  refns_kv_dump(c, buf.data(), len + 1);
  uint64_t h = 0xcbf29ce484222325ULL;
  for (int64_t i = 0; i < len; ++i) {
    h ^= static_cast<unsigned char>(buf[static_cast<size_t>(i)]);
    h *= 0x100000001b3ULL;
  }
  return h;
}

void emit(const std::string& line) {
  if (g_enabled) {
    g_log += line;
    g_log += '\n';
  }
}

[[noreturn]] void rethrow(int st) {
  std::string msg = refns_last_error();
  switch (st) {
    case 1: throw agentsim::CacheFull(msg);
    case 2: throw agentsim::UnknownBlock(msg);
    case 3: throw agentsim::ZeroRefRelease(msg);
    case 5: throw agentsim::ConfigError(msg);
    default: throw agentsim::CacheError(msg);
  }
}

}  // namespace

extern "C" {
// Returns the op log accumulated so far and clears it.
int64_t kvlog_take(char* buf, int64_t cap) {
  int64_t n = static_cast<int64_t>(g_log.size());
  if (buf && cap > n) {
    std::memcpy(buf, g_log.data(), g_log.size());
    buf[n] = 0;
    g_log.clear();
  }
  return n;
}
void kvlog_enable(int on) { g_enabled = on != 0; }
}

namespace agentsim {

const char* to_string(KvTag tag) {
  switch (tag) {
    case KvTag::kResponse: return "response";
    case KvTag::kToolOutput: return "tool_output";
    case KvTag::kUserQuery: return "user_query";
    case KvTag::kSystemPrompt: return "system_prompt";
    case KvTag::kPartialPrefill: return "partial_prefill";
    case KvTag::kHistory: return "history";
  }
  return "unknown";
}

int eviction_tier(KvTag tag) {
  static const int tiers[6] = {0, 1, 2, 3, 4, 2};
  return tiers[static_cast<int>(tag)];
}

std::uint64_t kv_root_hash() { return refns_root_hash(); }
std::uint64_t kv_chain_hash(std::uint64_t parent, std::span<const TokenId> t) {
  return refns_chain_hash(parent, t.data(), static_cast<int64_t>(t.size()));
}

// Mirror residency + eviction count so the header's inline accessors
// (resident_blocks, contains, total_evicted, free_blocks) stay truthful.
static void resync(KvCache* self, void* c, std::unordered_map<int32_t, KvBlock>& blocks,
                   std::set<int32_t>& free_ids, std::uint64_t& total_evicted, int64_t cap) {
  (void)self;
  blocks.clear();
  free_ids.clear();
  for (int32_t id = 0; id < cap; ++id) {
    if (refns_kv_contains(c, id)) {
      blocks[id].block_id = id;
    } else {
      free_ids.insert(id);
    }
  }
  total_evicted = refns_kv_total_evicted(c);
}

KvCache::KvCache(const CacheConfig& config) : config_(config) {
  void* c = nullptr;
  int st = refns_kv_create(config.block_size, config.capacity_blocks,
                           config.policy == EvictionPolicy::kTiered ? 1 : 0, &c);
  if (st) rethrow(st);
  g_impl[this] = c;
  resync(this, c, blocks_, free_ids_, total_evicted_, config_.capacity_blocks);
  std::ostringstream o;
  o << "{\"op\":\"create\",\"block_size\":" << config.block_size
    << ",\"capacity\":" << config.capacity_blocks
    << ",\"policy\":" << (config.policy == EvictionPolicy::kTiered ? 1 : 0) << "}";
  emit(o.str());
}

std::int64_t KvCache::lookup_prefix(std::span<const TokenId> tokens, SimTime now) {
  void* c = impl(this);
  int64_t hit = 0;
  int st = refns_kv_lookup(c, tokens.data(), static_cast<int64_t>(tokens.size()), now, &hit);
  std::ostringstream o;
  o << "{\"op\":\"lookup\",\"now\":" << now << ",\"tokens\":\""
    << b64(tokens.data(), tokens.size() * 8) << "\",\"ret\":" << hit << ",\"status\":" << st
    << ",\"dump_fnv\":\"" << dump_fnv(c) << "\"}";
  emit(o.str());
  if (st) rethrow(st);
  return hit;
}

std::vector<std::int32_t> KvCache::insert(std::span<const TokenId> tokens,
                                          std::span<const TagRange> tags, SimTime now) {
  void* c = impl(this);
  std::vector<int64_t> tr;
  std::string tj = "[";
  for (size_t i = 0; i < tags.size(); ++i) {
    tr.push_back(tags[i].begin);
    tr.push_back(tags[i].end);
    tr.push_back(static_cast<int64_t>(tags[i].tag));
    if (i) tj += ',';
    tj += "[" + std::to_string(tags[i].begin) + "," + std::to_string(tags[i].end) + "," +
          std::to_string(static_cast<int>(tags[i].tag)) + "]";
  }
  tj += "]";
  const size_t bs = static_cast<size_t>(config_.block_size);
  std::vector<int32_t> out((tokens.size() + bs - 1) / bs + 1);
  int64_t nout = 0;
  uint64_t ev0 = refns_kv_total_evicted(c);
  int st = refns_kv_insert(c, tokens.data(), static_cast<int64_t>(tokens.size()), tr.data(),
                           static_cast<int64_t>(tags.size()), now, out.data(), &nout);
  out.resize(static_cast<size_t>(nout));
  resync(this, c, blocks_, free_ids_, total_evicted_, config_.capacity_blocks);
  std::ostringstream o;
  o << "{\"op\":\"insert\",\"now\":" << now << ",\"tokens\":\""
    << b64(tokens.data(), tokens.size() * 8) << "\",\"tags\":" << tj << ",\"status\":" << st
    << ",\"ids\":" << ids_json(out.data(), out.size())
    << ",\"evicted\":" << (refns_kv_total_evicted(c) - ev0) << ",\"dump_fnv\":\"" << dump_fnv(c)
    << "\"}";
  emit(o.str());
  if (st) rethrow(st);
  return out;
}

std::vector<std::int32_t> KvCache::evict(std::size_t needed) {
  void* c = impl(this);
  std::vector<int32_t> out(needed + 1);
  int64_t n = 0;
  int st = refns_kv_evict(c, static_cast<int64_t>(needed), out.data(), &n);
  out.resize(static_cast<size_t>(n));
  resync(this, c, blocks_, free_ids_, total_evicted_, config_.capacity_blocks);
  std::ostringstream o;
  o << "{\"op\":\"evict\",\"needed\":" << needed << ",\"ret\":" << ids_json(out.data(), out.size())
    << ",\"status\":" << st << ",\"dump_fnv\":\"" << dump_fnv(c) << "\"}";
  emit(o.str());
  if (st) rethrow(st);
  return out;
}

void KvCache::set_reuse_priority(std::span<const std::int32_t> ids, const PriorityUpdate& u) {
  void* c = impl(this);
  int32_t pin = u.pinned ? (*u.pinned ? 1 : 0) : -1;
  int32_t tier = u.tier_override ? static_cast<int32_t>(*u.tier_override) : -1;
  int st = refns_kv_set_priority(c, ids.data(), static_cast<int64_t>(ids.size()), pin, tier);
  std::ostringstream o;
  o << "{\"op\":\"set_priority\",\"ids\":" << ids_json(ids.data(), ids.size())
    << ",\"pinned\":" << pin << ",\"tier\":" << tier << ",\"status\":" << st
    << ",\"dump_fnv\":\"" << dump_fnv(c) << "\"}";
  emit(o.str());
  if (st) rethrow(st);
}

void KvCache::set_tag(std::int32_t id, KvTag tag) {
  void* c = impl(this);
  int st = refns_kv_set_tag(c, id, static_cast<int32_t>(tag));
  std::ostringstream o;
  o << "{\"op\":\"set_tag\",\"id\":" << id << ",\"tag\":" << static_cast<int>(tag)
    << ",\"status\":" << st << ",\"dump_fnv\":\"" << dump_fnv(c) << "\"}";
  emit(o.str());
  if (st) rethrow(st);
}

void KvCache::release(std::span<const std::int32_t> ids) {
  void* c = impl(this);
  int st = refns_kv_release(c, ids.data(), static_cast<int64_t>(ids.size()));
  std::ostringstream o;
  o << "{\"op\":\"release\",\"ids\":" << ids_json(ids.data(), ids.size()) << ",\"status\":" << st
    << ",\"dump_fnv\":\"" << dump_fnv(c) << "\"}";
  emit(o.str());
  if (st) rethrow(st);
}

void KvCache::touch(std::span<const std::int32_t> ids, SimTime now) {
  void* c = impl(this);
  int st = refns_kv_touch(c, ids.data(), static_cast<int64_t>(ids.size()), now);
  std::ostringstream o;
  o << "{\"op\":\"touch\",\"ids\":" << ids_json(ids.data(), ids.size()) << ",\"now\":" << now
    << ",\"status\":" << st << ",\"dump_fnv\":\"" << dump_fnv(c) << "\"}";
  emit(o.str());
  if (st) rethrow(st);
}

const KvBlock& KvCache::block(std::int32_t id) const {
  void* c = impl(this);
  int64_t f[6];
  uint64_t h[2];
  std::vector<uint64_t> toks(static_cast<size_t>(config_.block_size));
  int st = refns_kv_block(c, id, f, h, toks.data());
  std::ostringstream o;
  o << "{\"op\":\"block\",\"id\":" << id << ",\"status\":" << st;
  if (!st)
    o << ",\"tag\":" << f[0] << ",\"tier\":" << f[1] << ",\"ref\":" << f[2]
      << ",\"pinned\":" << f[3] << ",\"ntok\":" << f[4] << ",\"last\":" << f[5]
      << ",\"chain\":\"" << h[0] << "\",\"parent\":\"" << h[1] << "\"";
  o << "}";
  emit(o.str());
  if (st) rethrow(st);
  auto& self = const_cast<KvCache*>(this)->blocks_;
  KvBlock& b = self[id];
  b.block_id = id;
  b.tag = static_cast<KvTag>(f[0]);
  b.tier = static_cast<int>(f[1]);
  b.ref_count = static_cast<int>(f[2]);
  b.pinned = f[3] != 0;
  toks.resize(static_cast<size_t>(f[4]));
  b.tokens = toks;
  b.last_used = f[5];
  b.chain_hash = h[0];
  b.parent_hash = h[1];
  return b;
}

void KvCache::audit() const {
  int st = refns_kv_audit(impl(this));
  emit(std::string("{\"op\":\"audit\",\"status\":") + std::to_string(st) + "}");
  if (st) rethrow(st);
}

std::string KvCache::dump() const {
  void* c = impl(this);
  int64_t len = refns_kv_dump(c, nullptr, 0);
  std::string buf(static_cast<size_t>(len) + 1, '\0');
  refns_kv_dump(c, buf.data(), len + 1);
  buf.resize(static_cast<size_t>(len));
  return buf;
}

}  // namespace agentsim
