// replay.cu — host C++ replay of agentic traces on the B200 block pool.
//
// A restatement (not a port) of the reference simulator's behaviour for the
// quantities the hot path decides: every KV-cache decision goes to the device
// pool through the C-ABI, while virtual time follows the reference's rules so
// that per-request FTR, end-to-end time, hit tokens and the eviction total
// equal the reference's on the same trace (tests/test_replay_gpu.py).
//
// Reference behaviour restated (paths under /root/reference/proj/src):
//   trace generator              trace_gen.cpp:96-193 (+ Rng, common.hpp:161-197)
//   token materialisation         trace.cpp:50-83
//   event loop ordering           sim.cpp:28-43 ((time, sequence) order)
//   engine: admission, chunked prefill + decode steps, scheduler policies,
//           partial prefill pins, extension, completion inserts/releases
//                                 engine.cpp:35-475
//   orchestrator: prompt splitting, streaming / batch tool dispatch, tool
//           latency scaling, iteration advance
//                                 orchestrator.cpp:13-461
//   presets                       runner.cpp:120-153
//   nearest-rank percentiles      metrics.cpp:136-151
// Differences in mechanics only: block tags of a pinned prefix are read and
// updated with one batched pool call instead of one call per block.  The
// engine's step-event rules are kept exactly, including a wake() issued from
// inside a step's completions starting a second step chain (token callbacks
// then repeat, and the streaming parser sees repeated chunks).
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <queue>
#include <random>
#include <set>
#include <string>
#include <vector>

#include "common.h"
#include "hash.cuh"

namespace sb {
namespace rp {

using Time = int64_t;
// SB_REPLAY_TRACE=1 prints an orchestrator timeline (same wording as the
// reference's, orchestrator.cpp:173-177) to stderr for debugging.
static const bool g_trace = [] {
  const char* v = std::getenv("SB_REPLAY_TRACE");
  return v && v[0] == '1';
}();

// ------------------------------------------------------------ randomness
struct Rng {
  std::mt19937_64 e;
  explicit Rng(uint64_t seed) : e(seed) {}
  uint64_t next() { return e(); }
  double uniform01() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  uint64_t below(uint64_t n) { return next() % n; }
  double exponential(double rate) { return -std::log1p(-uniform01()) / rate; }
  double normal() {
    double u1 = uniform01();
    const double u2 = uniform01();
    while (u1 <= 0.0) u1 = uniform01();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * M_PI * u2);
  }
  double lognormal(double log_median, double sigma) { return std::exp(log_median + sigma * normal()); }
  int64_t truncated_geometric(double p, int64_t max_value) {
    const double u = uniform01();
    int64_t k = static_cast<int64_t>(1 + std::floor(std::log1p(-u) / std::log1p(-p)));
    if (k < 1) k = 1;
    return std::min(k, max_value);
  }
};

uint64_t fnv1a(const std::string& s) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (unsigned char c : s) {
    h ^= c;
    h *= 0x100000001b3ULL;
  }
  return h;
}

// ---------------------------------------------------------------- trace
enum SecTag { kSys = 0, kUser = 1, kTool = 2, kHist = 3 };
struct Section {
  int tag;
  int64_t len;
  uint64_t key;
  int32_t src;
};
struct Tool {
  std::string name;
  double ratio;       // < 0: fixed latency
  Time fixed_ms;
  Section out;
  int64_t emit;
};
struct Iter {
  std::vector<Section> sections;
  int64_t decode_len;
  std::vector<Tool> tools;
  bool final;
};
struct Request {
  std::string id;
  Time arrival;
  std::vector<Iter> iters;
};

struct GenConfig {
  int num_requests = 60;
  double qps = 0.05, depth_p = 0.4;
  int64_t depth_max = 7;
  double fanout_p = 0.4;
  int64_t fanout_max = 20;
  double prompt_base_median = 16000.0, prompt_sigma = 0.30, system_frac = 0.62, user_frac = 0.22;
  int system_variants = 2;
  double tool_out_median = 1200.0, tool_out_sigma = 0.5;
  double decode_inter_median = 150.0, decode_final_median = 750.0, decode_sigma = 0.35;
  std::vector<std::pair<std::string, double>> tools = {{"search", 1.2},   {"code_exec", 1.8}, {"kb_lookup", 0.8},
                                                        {"web_fetch", 1.5}, {"calendar", 0.4},  {"email", 0.5},
                                                        {"file_io", 0.7}};
  double ratio_scale = 0.8, ratio_sigma = 0.85;
};

int64_t clamped_len(double v, int64_t lo) { return std::max<int64_t>(std::llround(v), lo); }

std::vector<Request> generate(const GenConfig& c, uint64_t seed) {
  std::vector<Request> trace;
  Rng arrivals(splitmix64(seed ^ 0xa221a221a221a221ULL));
  Time clock = 0;
  for (int r = 0; r < c.num_requests; ++r) {
    clock += static_cast<Time>(std::llround(arrivals.exponential(c.qps) * 1000.0));
    Rng rng(splitmix64(seed ^ (static_cast<uint64_t>(r) * 0x9e3779b97f4a7c15ULL + 1)));
    Request req;
    char buf[16];
    std::snprintf(buf, sizeof(buf), "r%05d", r);
    req.id = buf;
    req.arrival = clock;
    const auto depth = static_cast<size_t>(rng.truncated_geometric(c.depth_p, c.depth_max));
    const double base = rng.lognormal(std::log(c.prompt_base_median), c.prompt_sigma);
    const double hist_frac = 1.0 - c.system_frac - c.user_frac;
    const int64_t user_len = clamped_len(base * c.user_frac, 16), hist_len = clamped_len(base * hist_frac, 16);
    const uint64_t user_key = splitmix64(seed ^ (static_cast<uint64_t>(r) * 31 + 7));
    const uint64_t hist_key = splitmix64(seed ^ (static_cast<uint64_t>(r) * 31 + 11));
    std::set<std::string> prev_tools;
    std::vector<Section> outputs;
    for (size_t i = 0; i < depth; ++i) {
      Iter it;
      it.final = (i + 1 == depth);
      std::string pool_key = it.final ? "final|" : "inter|";
      for (const auto& t : prev_tools) pool_key += t + ",";
      const uint64_t variant = rng.below(static_cast<uint64_t>(c.system_variants));
      const uint64_t sys_key = splitmix64(seed ^ fnv1a(pool_key) ^ (variant * 0x51ed2701b7b5a0dULL + 3));
      Rng pool_rng(sys_key);
      const int64_t sys_len =
          clamped_len(pool_rng.lognormal(std::log(c.prompt_base_median * c.system_frac), c.prompt_sigma), 64);
      it.sections = {{kSys, sys_len, sys_key, -1}, {kUser, user_len, user_key, -1}, {kHist, hist_len, hist_key, -1}};
      for (const auto& o : outputs) it.sections.push_back(o);
      if (it.final) {
        it.decode_len = clamped_len(rng.lognormal(std::log(c.decode_final_median), c.decode_sigma), 16);
      } else {
        const int64_t fan = rng.truncated_geometric(c.fanout_p, c.fanout_max);
        it.decode_len = clamped_len(rng.lognormal(std::log(c.decode_inter_median), c.decode_sigma),
                                    std::max<int64_t>(8, 3 * (fan + 1)));
        std::set<std::string> names;
        for (int64_t j = 0; j < fan; ++j) {
          const auto& prof = c.tools[rng.below(c.tools.size())];
          Tool t;
          t.name = prof.first;
          t.ratio = std::clamp(rng.lognormal(std::log(prof.second * c.ratio_scale), c.ratio_sigma), 0.05, 50.0);
          t.fixed_ms = -1;
          t.out.tag = kTool;
          t.out.src = static_cast<int32_t>(i);
          t.out.len = clamped_len(rng.lognormal(std::log(c.tool_out_median), c.tool_out_sigma), 16);
          t.out.key = splitmix64(seed ^ (static_cast<uint64_t>(r) * 1009 + static_cast<uint64_t>(i) * 131 +
                                         static_cast<uint64_t>(j) * 17 + 13));
          t.emit = (j + 1) * it.decode_len / (fan + 1);
          it.tools.push_back(t);
          names.insert(t.name);
        }
        for (const auto& t : it.tools) outputs.push_back(t.out);
        prev_tools = std::move(names);
      }
      req.iters.push_back(std::move(it));
    }
    trace.push_back(std::move(req));
  }
  return trace;
}

int kv_tag_of(int sec) { return sec == kSys ? SB_TAG_SYSTEM_PROMPT : sec == kUser ? SB_TAG_USER_QUERY : sec == kTool ? SB_TAG_TOOL_OUTPUT : SB_TAG_HISTORY; }

void append_section(std::vector<uint64_t>& toks, std::vector<sb_tag_range>& tags, const Section& s) {
  if (s.len <= 0) return;
  const uint64_t seed = section_seed(s.tag, s.key, s.src);
  const int64_t b = static_cast<int64_t>(toks.size());
  for (int64_t i = 0; i < s.len; ++i) toks.push_back(splitmix64(seed + static_cast<uint64_t>(i)));
  tags.push_back(sb_tag_range{b, b + s.len, kv_tag_of(s.tag), 0});
}


// ------------------------------------------------- tool-call transcript
// Decode transcript of an intermediate iteration and its per-token character
// spans (orchestrator.cpp:38-91): tool j's closing brace lands in decode token
// emit_j.  Fed to the streaming parser token by token, so repeated token
// callbacks (the engine can run two step chains, engine.cpp:119-123 +
// 379-383) reach the parser exactly as in the reference.
struct Transcript {
  std::string text;
  std::vector<std::pair<size_t, size_t>> spans;
};

Transcript make_transcript(const Iter& it, const std::string& rid, size_t iter) {
  Transcript t;
  std::vector<int64_t> close;
  t.text = "[";
  for (size_t j = 0; j < it.tools.size(); ++j) {
    if (j) t.text += ", ";
    t.text += "{\"tool\": \"" + it.tools[j].name + "\", \"query\": \"" + rid + "/" + std::to_string(iter) + "/" +
              std::to_string(j) + "\", \"call\": " + std::to_string(j) + "}";
    close.push_back(static_cast<int64_t>(t.text.size()) - 1);
  }
  t.text += "]";
  const int64_t n = it.decode_len;
  std::vector<int64_t> cnt(static_cast<size_t>(n), 0);
  int64_t pt = -1, pc = -1;
  auto spread = [&](int64_t first, int64_t toks, int64_t chars) {
    for (int64_t k = 0; k < toks; ++k) cnt[static_cast<size_t>(first + k)] = (k + 1) * chars / toks - k * chars / toks;
  };
  for (size_t j = 0; j < close.size(); ++j) {
    spread(pt + 1, it.tools[j].emit - pt, close[j] - pc);
    pt = it.tools[j].emit;
    pc = close[j];
  }
  const int64_t rem_chars = static_cast<int64_t>(t.text.size()) - 1 - pc, rem_toks = n - 1 - pt;
  if (rem_toks <= 0) {
    if (pt >= 0) cnt[static_cast<size_t>(pt)] += rem_chars;
  } else {
    spread(pt + 1, rem_toks, rem_chars);
  }
  size_t pos = 0;
  for (int64_t i = 0; i < n; ++i) {
    t.spans.emplace_back(pos, pos + static_cast<size_t>(cnt[static_cast<size_t>(i)]));
    pos += static_cast<size_t>(cnt[static_cast<size_t>(i)]);
  }
  return t;
}

// Incremental tool-call parser with the reference's acceptance rules
// (streaming_parser.cpp): flat array of objects, string / raw / one-level
// nested values, sink state on malformed input.  Only what dispatch needs is
// kept: the emitted tool names and their close token.
struct ToolParser {
  enum Ph { kBefore, kFirst, kObj, kAfterVal, kFirstKey, kKey, kKeyStr, kColon, kVal, kStr, kRaw, kNested, kObjAfter,
            kAfterArr, kSink };
  Ph ph = kBefore;
  bool esc = false, n_str = false, n_esc = false;
  int nested = 0;
  std::string key, val;
  std::map<std::string, std::string> params;

  static bool ws(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\r'; }
  void esc_append(std::string& o, char c) {
    switch (c) {
      case '"': o += '"'; break;
      case '\\': o += '\\'; break;
      case '/': o += '/'; break;
      case 'b': o += '\b'; break;
      case 'f': o += '\f'; break;
      case 'n': o += '\n'; break;
      case 'r': o += '\r'; break;
      case 't': o += '\t'; break;
      default: o += '\\'; o += c; break;  // includes \u: the hex digits follow verbatim
    }
  }
  void finish_value() {
    params[key] = val;
    key.clear();
    val.clear();
  }
  void close(std::vector<std::string>& out) {
    auto it = params.find("tool");
    if (it == params.end() || it->second.empty()) {
      ph = kSink;
      return;
    }
    out.push_back(it->second);
    params.clear();
    ph = kAfterVal;
  }
  // returns false when c must be re-processed (end of a raw value)
  bool step(char c, std::vector<std::string>& out) {
    switch (ph) {
      case kBefore:
        if (c == '[') ph = kFirst;
        return true;
      case kFirst:
      case kObj:
        if (ws(c)) return true;
        if (c == '{') {
          params.clear();
          ph = kFirstKey;
        } else if (c == ']' && ph == kFirst) {
          ph = kAfterArr;
        } else {
          ph = kSink;
        }
        return true;
      case kAfterVal:
        if (ws(c)) return true;
        ph = c == ',' ? kObj : c == ']' ? kAfterArr : kSink;
        return true;
      case kFirstKey:
      case kKey:
        if (ws(c)) return true;
        if (c == '"') {
          key.clear();
          ph = kKeyStr;
        } else if (c == '}' && ph == kFirstKey) {
          close(out);
        } else {
          ph = kSink;
        }
        return true;
      case kKeyStr:
        if (esc) {
          esc_append(key, c);
          esc = false;
        } else if (c == '\\') {
          esc = true;
        } else if (c == '"') {
          ph = kColon;
        } else {
          key += c;
        }
        return true;
      case kColon:
        if (ws(c)) return true;
        ph = c == ':' ? kVal : kSink;
        return true;
      case kVal:
        if (ws(c)) return true;
        if (c == '"') {
          val.clear();
          ph = kStr;
        } else if (c == '{' || c == '[') {
          val.assign(1, c);
          nested = 1;
          n_str = n_esc = false;
          ph = kNested;
        } else if (c == '}' || c == ']' || c == ',') {
          ph = kSink;
        } else {
          val.assign(1, c);
          ph = kRaw;
        }
        return true;
      case kStr:
        if (esc) {
          esc_append(val, c);
          esc = false;
        } else if (c == '\\') {
          esc = true;
        } else if (c == '"') {
          finish_value();
          ph = kObjAfter;
        } else {
          val += c;
        }
        return true;
      case kRaw:
        if (ws(c) || c == ',' || c == '}') {
          finish_value();
          ph = kObjAfter;
          return ws(c);
        }
        if (c == ']' || c == '{' || c == '[') ph = kSink;
        else val += c;
        return true;
      case kNested:
        val += c;
        if (n_str) {
          if (n_esc) n_esc = false;
          else if (c == '\\') n_esc = true;
          else if (c == '"') n_str = false;
        } else if (c == '"') {
          n_str = true;
        } else if (c == '{' || c == '[') {
          ++nested;
        } else if ((c == '}' || c == ']') && --nested == 0) {
          finish_value();
          ph = kObjAfter;
        }
        return true;
      case kObjAfter:
        if (ws(c)) return true;
        if (c == ',') ph = kKey;
        else if (c == '}') close(out);
        else ph = kSink;
        return true;
      case kAfterArr:
      case kSink:
        return true;
    }
    return true;
  }
  std::vector<std::string> feed(const char* s, size_t n) {
    std::vector<std::string> out;
    if (ph == kSink) return out;
    for (size_t i = 0; i < n; ++i) {
      while (!step(s[i], out))
        if (ph == kSink) break;
      if (ph == kSink) break;
    }
    return out;
  }
  bool malformed() const { return ph == kSink; }
};

// ------------------------------------------------------------- sim core
struct Loop {
  struct Ev {
    Time t;
    uint64_t seq;
    std::function<void()> fn;
  };
  struct Later {
    bool operator()(const Ev& a, const Ev& b) const { return a.t != b.t ? a.t > b.t : a.seq > b.seq; }
  };
  std::priority_queue<Ev, std::vector<Ev>, Later> q;
  Time now = 0;
  uint64_t seq = 0;
  void at(Time t, std::function<void()> fn) { q.push(Ev{t, seq++, std::move(fn)}); }
  void run() {
    while (!q.empty()) {
      Ev e = q.top();
      q.pop();
      now = e.t;
      e.fn();
    }
  }
};

struct Cost {
  double prefill_ms_per_token = 0.05, decode_ms_per_token = 20.0, overhead_ms = 2.0;
  int64_t chunk = 256;
  Time chunk_ms(int64_t tokens) const {
    if (tokens <= 0) return 1;
    return std::max<Time>(static_cast<Time>(std::ceil(static_cast<double>(tokens) * prefill_ms_per_token)), 1);
  }
  Time decode_step_ms() const { return static_cast<Time>(std::ceil(decode_ms_per_token + overhead_ms)); }
};

struct Interval {
  Time b, e;
};
void add_interval(std::vector<Interval>& v, Time b, Time e) {
  if (e <= b) return;
  if (!v.empty() && v.back().e == b) v.back().e = e;
  else v.push_back({b, e});
}
Time busy(const std::vector<Interval>& v) {
  Time t = 0;
  for (const auto& i : v) t += i.e - i.b;
  return t;
}

enum State { kQueued, kPrefilling, kAwaiting, kDecoding, kDone, kAborted };

struct Call {
  int64_t id = 0;
  Time agentic_arrival = 0, arrival_at_engine = 0;
  int32_t iteration = 0;
  State state = kQueued;
  bool partial = false, extended = false;
  int64_t prompt_tokens = 0, cached_prefix = 0, charged_total = 0, charged_done = 0, decode_len = 0, emitted = 0;
  Time first_token = -1, decode_complete = -1;
  std::vector<Interval> prefill_iv, decode_iv;
  std::vector<uint64_t> prompt;
  std::vector<sb_tag_range> tags;
  uint64_t stream_key = 0;
  std::function<void(int64_t, Time)> on_token;
  std::function<void(Time)> on_decoded, on_pin_failed;
  std::vector<int32_t> chain_refs, pinned_ids;
};

struct Pool {
  sb_kv_cache* c;
  static void ok(int st) {
    if (st != SB_OK) throw Error(st, sb_last_error());
  }
  int64_t lookup(const std::vector<uint64_t>& t, Time now) {
    int64_t hit = 0;
    ok(sb_kv_lookup_prefix(c, t.data(), static_cast<int64_t>(t.size()), now, &hit));
    return hit;
  }
  // returns false on CacheFull
  bool insert(const std::vector<uint64_t>& t, const std::vector<sb_tag_range>& tags, Time now, std::vector<int32_t>& ids) {
    ids.assign((t.size() + 15) / 16 + 1, 0);
    int64_t n = 0;
    const int st = sb_kv_insert(c, t.data(), static_cast<int64_t>(t.size()), tags.data(),
                                static_cast<int64_t>(tags.size()), now, ids.data(), &n);
    if (st == SB_ERR_CACHE_FULL) {
      ids.clear();
      return false;
    }
    ok(st);
    ids.resize(static_cast<size_t>(n));
    return true;
  }
  void release(const std::vector<int32_t>& ids) {
    if (!ids.empty()) ok(sb_kv_release(c, ids.data(), static_cast<int64_t>(ids.size())));
  }
};

struct Sim {
  Loop loop;
  Pool pool;
  Cost cost;
  bool request_aware = false, splitting = false, streaming = false;
  int64_t bs = 16;
  std::map<int64_t, Call> calls;
  int64_t next_id = 1;
  bool inflight = false, pending = false;
  struct Step {
    Time start, end, chunk_ms;
    int64_t chunk_call, chunk_tokens;
    std::vector<int64_t> decoding;
  } step{};
  std::map<int32_t, int> pin_count;
  std::map<int32_t, int32_t> real_tag;

  void wake() {
    if (inflight || pending) return;
    pending = true;
    loop.at(loop.now, [this] { on_step(); });
  }
  int64_t submit(Call c) {
    c.id = next_id++;
    c.arrival_at_engine = loop.now;
    c.prompt_tokens = static_cast<int64_t>(c.prompt.size());
    c.cached_prefix = pool.lookup(c.prompt, loop.now);
    c.charged_total = c.prompt_tokens - c.cached_prefix;
    const int64_t id = c.id;
    calls.emplace(id, std::move(c));
    wake();
    return id;
  }
  void extend(int64_t id, const std::vector<uint64_t>& sfx, const std::vector<sb_tag_range>& sfx_tags,
              int64_t decode_len, std::function<void(Time)> done) {
    Call& c = calls.at(id);
    const int64_t pl = static_cast<int64_t>(c.prompt.size());
    c.extended = true;
    c.prompt.insert(c.prompt.end(), sfx.begin(), sfx.end());
    for (auto r : sfx_tags) c.tags.push_back(sb_tag_range{r.begin + pl, r.end + pl, r.tag, 0});
    c.prompt_tokens += static_cast<int64_t>(sfx.size());
    c.charged_total += static_cast<int64_t>(sfx.size());
    c.decode_len = decode_len;
    c.on_decoded = std::move(done);
    if (c.state == kAwaiting) {
      if (c.charged_done >= c.charged_total) complete_prefill(c);
      else c.state = kPrefilling;
    }
    wake();
  }
  void abandon(int64_t id) {
    Call& c = calls.at(id);
    release_pins(c);
    pool.release(c.chain_refs);
    c.chain_refs.clear();
    c.state = kAborted;
  }
  int tag_at(const Call& c, int64_t pos) const {
    for (const auto& r : c.tags)
      if (pos >= r.begin && pos < r.end) return r.tag;
    return SB_TAG_USER_QUERY;
  }
  void pin_partial(Call& c) {
    std::vector<sb_tag_range> whole{sb_tag_range{0, c.prompt_tokens, SB_TAG_PARTIAL_PREFILL, 0}};
    std::vector<int32_t> ids;
    if (!pool.insert(c.prompt, whole, loop.now, ids)) {
      c.state = kAborted;
      if (c.on_pin_failed) c.on_pin_failed(loop.now);
      return;
    }
    c.chain_refs = ids;
    // first pins remember the block's real tag (one batched read-back)
    std::vector<int32_t> first;
    std::vector<size_t> pos;
    for (size_t i = 0; i < ids.size(); ++i)
      if (pin_count[ids[i]]++ == 0) {
        first.push_back(ids[i]);
        pos.push_back(i);
      }
    std::vector<sb_block_info> info(first.size());
    if (!first.empty())
      Pool::ok(sb_kv_blocks(pool.c, first.data(), static_cast<int64_t>(first.size()), info.data()));
    for (size_t k = 0; k < first.size(); ++k) {
      if (info[k].n_tokens == 0) throw Error(SB_ERR_UNKNOWN_BLOCK, "pinned block not resident");
      real_tag[first[k]] =
          info[k].tag != SB_TAG_PARTIAL_PREFILL ? info[k].tag : tag_at(c, static_cast<int64_t>(pos[k]) * bs);
    }
    Pool::ok(sb_kv_set_reuse_priority(pool.c, ids.data(), static_cast<int64_t>(ids.size()), 1,
                                      SB_TAG_PARTIAL_PREFILL));
    c.pinned_ids = ids;
    c.state = kAwaiting;
  }
  void release_pins(Call& c) {
    std::vector<int32_t> last, unpin;
    std::map<int32_t, std::vector<int32_t>> by_tag;
    for (int32_t id : c.pinned_ids) {
      auto it = pin_count.find(id);
      if (it == pin_count.end() || --it->second > 0) continue;
      pin_count.erase(it);
      last.push_back(id);
    }
    // residency of the blocks whose last pin goes (one batched read-back)
    std::vector<sb_block_info> info(last.size());
    if (!last.empty()) Pool::ok(sb_kv_blocks(pool.c, last.data(), static_cast<int64_t>(last.size()), info.data()));
    for (size_t k = 0; k < last.size(); ++k) {
      const int32_t id = last[k];
      if (info[k].n_tokens > 0) {
        unpin.push_back(id);
        auto t = real_tag.find(id);
        if (t != real_tag.end()) by_tag[t->second].push_back(id);
      }
      real_tag.erase(id);
    }
    if (!unpin.empty())
      Pool::ok(sb_kv_set_reuse_priority(pool.c, unpin.data(), static_cast<int64_t>(unpin.size()), 0, -1));
    for (auto& [tag, ids] : by_tag)
      Pool::ok(sb_kv_set_reuse_priority(pool.c, ids.data(), static_cast<int64_t>(ids.size()), -1, tag));
    c.pinned_ids.clear();
  }
  void complete_prefill(Call& c) {
    if (c.partial && !c.extended) {
      pin_partial(c);
      return;
    }
    std::vector<int32_t> old = std::move(c.chain_refs);
    c.chain_refs.clear();
    std::vector<int32_t> ids;
    if (pool.insert(c.prompt, c.tags, loop.now, ids)) c.chain_refs = ids;
    if (!c.pinned_ids.empty()) release_pins(c);
    pool.release(old);
    c.state = kDecoding;
  }
  void finish_decode(Call& c) {
    c.state = kDone;
    c.decode_complete = loop.now;
    std::vector<uint64_t> full = c.prompt;
    for (int64_t i = 0; i < c.emitted; ++i) full.push_back(decode_token(c.stream_key, i));
    std::vector<sb_tag_range> tags = c.tags;
    tags.push_back(sb_tag_range{c.prompt_tokens, c.prompt_tokens + c.emitted, SB_TAG_RESPONSE, 0});
    std::vector<int32_t> ids;
    if (pool.insert(full, tags, loop.now, ids)) pool.release(ids);
    pool.release(c.chain_refs);
    c.chain_refs.clear();
    if (c.on_decoded) c.on_decoded(loop.now);
  }
  int64_t head() const {
    int64_t best = 0;
    std::tuple<Time, int64_t, Time, int64_t> bk{};
    for (const auto& [id, c] : calls) {
      if (!(c.state == kQueued || (c.state == kPrefilling && c.charged_done < c.charged_total))) continue;
      auto k = request_aware ? std::make_tuple(c.agentic_arrival, static_cast<int64_t>(c.iteration), c.arrival_at_engine, id)
                             : std::make_tuple(c.arrival_at_engine, int64_t{0}, Time{0}, id);
      if (best == 0 || k < bk) {
        best = id;
        bk = k;
      }
    }
    return best;
  }
  void on_step() {
    pending = false;
    const Time now = loop.now;
    if (inflight && step.end == now) {
      Step s = step;
      inflight = false;
      if (s.chunk_call) {
        auto it = calls.find(s.chunk_call);
        if (it != calls.end() && it->second.state == kPrefilling) {
          Call& c = it->second;
          c.charged_done += s.chunk_tokens;
          add_interval(c.prefill_iv, s.start, s.start + s.chunk_ms);
          if (c.charged_done >= c.charged_total) complete_prefill(c);
        }
      }
      const Time dbeg = s.start + s.chunk_ms;
      std::vector<int64_t> completed;
      for (int64_t id : s.decoding) {
        Call& c = calls.at(id);
        c.emitted += 1;
        add_interval(c.decode_iv, dbeg, s.end);
        if (c.emitted >= c.decode_len) completed.push_back(id);
      }
      for (int64_t id : completed) finish_decode(calls.at(id));
    }
    // start the next step
    const int64_t h = head();
    std::vector<int64_t> decoding;
    for (const auto& [id, c] : calls)
      if (c.state == kDecoding) decoding.push_back(id);
    if (h == 0 && decoding.empty()) return;
    Step s{};
    s.start = now;
    if (h) {
      Call& c = calls.at(h);
      s.chunk_call = h;
      s.chunk_tokens = std::min<int64_t>(cost.chunk, c.charged_total - c.charged_done);
      s.chunk_ms = cost.chunk_ms(s.chunk_tokens);
      if (c.state == kQueued) c.state = kPrefilling;
    }
    s.decoding = decoding;
    s.end = now + s.chunk_ms + (decoding.empty() ? 0 : cost.decode_step_ms());
    for (int64_t id : decoding) {
      const int64_t tok = calls.at(id).emitted;
      loop.at(s.end, [this, id, tok] {
        Call& c = calls.at(id);
        if (tok == 0 && c.first_token < 0) c.first_token = loop.now;
        if (c.on_token) c.on_token(tok, loop.now);
      });
    }
    loop.at(s.end, [this] { on_step(); });
    step = s;
    inflight = true;
  }
  Time projected(int64_t id, int64_t emitted_tokens) const {
    const Call& c = calls.at(id);
    const int64_t rem = std::max<int64_t>(c.decode_len - emitted_tokens, 0);
    return busy(c.prefill_iv) + busy(c.decode_iv) + rem * cost.decode_step_ms();
  }
  Time actual(int64_t id) const {
    const Call& c = calls.at(id);
    return busy(c.prefill_iv) + busy(c.decode_iv);
  }
};

struct Orchestrator {
  Sim& sim;
  const std::vector<Request>& trace;
  struct ToolRt {
    Time dispatched = -1;
    bool done = false;
  };
  struct IterRt {
    int64_t call = 0;
    std::vector<ToolRt> tools;
    size_t pending = 0, next_dispatch = 0;
    bool decoded = false, advanced = false, fallback = false;
    Transcript transcript;
    std::unique_ptr<ToolParser> parser;
  };
  struct ReqRt {
    std::optional<int64_t> continuation;
    size_t continuation_for = 0;
    std::vector<IterRt> iters;
    bool done = false;
  };
  std::vector<ReqRt> reqs;

  Orchestrator(Sim& s, const std::vector<Request>& t) : sim(s), trace(t) {}
  void note(size_t r, const std::string& what) const {
    if (g_trace) std::fprintf(stderr, "t=%lld request=%s %s\n", static_cast<long long>(sim.loop.now), trace[r].id.c_str(), what.c_str());
  }

  static void build(const std::vector<Section>& secs, std::vector<uint64_t>& toks, std::vector<sb_tag_range>& tags) {
    for (const auto& s : secs) append_section(toks, tags, s);
  }
  uint64_t stream_key(size_t r, size_t i) const {
    return hash_combine(rp::fnv1a(trace[r].id), static_cast<uint64_t>(i));
  }
  void split(size_t r, size_t i, std::vector<Section>& indep, std::vector<Section>& dep) const {
    const int32_t prev = static_cast<int32_t>(i) - 1;
    for (const auto& s : trace[r].iters[i].sections)
      (s.tag == kTool && s.src == prev ? dep : indep).push_back(s);
  }
  void submit_iteration(size_t r, size_t i) {
    ReqRt& req = reqs[r];
    IterRt& it = req.iters[i];
    const Iter& spec = trace[r].iters[i];
    if (req.continuation && req.continuation_for == i) {
      const int64_t h = *req.continuation;
      req.continuation.reset();
      std::vector<Section> indep, dep;
      split(r, i, indep, dep);
      std::vector<uint64_t> toks;
      std::vector<sb_tag_range> tags;
      build(dep, toks, tags);
      it.call = h;
      sim.extend(h, toks, tags, spec.decode_len, [this, r, i](Time at) { on_decoded(r, i, at); });
      note(r, "extend_prefill iteration=" + std::to_string(i));
    } else {
      Call c;
      c.agentic_arrival = trace[r].arrival;
      c.iteration = static_cast<int32_t>(i);
      build(spec.sections, c.prompt, c.tags);
      c.decode_len = spec.decode_len;
      c.stream_key = stream_key(r, i);
      c.on_decoded = [this, r, i](Time at) { on_decoded(r, i, at); };
      it.call = sim.submit(std::move(c));
      note(r, "submit iteration=" + std::to_string(i));
    }
    if (spec.final) return;
    it.transcript = make_transcript(spec, trace[r].id, i);
    it.tools.assign(spec.tools.size(), ToolRt{});
    it.pending = spec.tools.size();
    if (sim.streaming) {
      it.parser = std::make_unique<ToolParser>();
      sim.calls.at(it.call).on_token = [this, r, i](int64_t tok, Time at) { on_token(r, i, tok, at); };
    }
  }
  void on_token(size_t r, size_t i, int64_t tok, Time at) {
    IterRt& it = reqs[r].iters[i];
    if (!it.parser || it.fallback) return;
    const auto idx = static_cast<size_t>(tok);
    if (idx >= it.transcript.spans.size()) return;
    const auto [b, e] = it.transcript.spans[idx];
    const auto& tools = trace[r].iters[i].tools;
    for (const std::string& name : it.parser->feed(it.transcript.text.data() + b, e - b)) {
      if (it.next_dispatch >= tools.size() || name != tools[it.next_dispatch].name) {
        it.fallback = true;
        break;
      }
      dispatch(r, i, it.next_dispatch, at, tok);
      ++it.next_dispatch;
    }
    if (it.parser->malformed()) it.fallback = true;
  }
  void dispatch(size_t r, size_t i, size_t j, Time now, int64_t close) {
    IterRt& it = reqs[r].iters[i];
    const Tool& t = trace[r].iters[i].tools[j];
    Time lat;
    if (t.fixed_ms >= 0) {
      lat = t.fixed_ms;
    } else {
      const Time llm = it.decoded ? sim.actual(it.call) : sim.projected(it.call, close);
      lat = std::max<Time>(static_cast<Time>(std::ceil(t.ratio * static_cast<double>(llm))), 1);
    }
    it.tools[j].dispatched = now;
    note(r, "dispatch_tool iteration=" + std::to_string(i) + " tool=" + std::to_string(j) + " name=" + t.name);
    sim.loop.at(now + lat, [this, r, i, j] { on_tool_done(r, i, j); });
  }
  void on_tool_done(size_t r, size_t i, size_t j) {
    IterRt& it = reqs[r].iters[i];
    it.tools[j].done = true;
    it.pending -= 1;
    note(r, "tool_complete iteration=" + std::to_string(i) + " tool=" + std::to_string(j));
    advance(r, i);
  }
  void submit_partial(size_t r, size_t i) {
    ReqRt& req = reqs[r];
    const size_t next = i + 1;
    std::vector<Section> indep, dep;
    split(r, next, indep, dep);
    if (indep.empty()) return;
    Call c;
    build(indep, c.prompt, c.tags);
    if (c.prompt.empty()) return;
    c.partial = true;
    c.agentic_arrival = trace[r].arrival;
    c.iteration = static_cast<int32_t>(next);
    c.stream_key = stream_key(r, next);
    c.on_pin_failed = [this, r, next](Time) {
      reqs[r].continuation.reset();
      note(r, "partial_pin_failed iteration=" + std::to_string(next));
    };
    const int64_t id = sim.submit(std::move(c));
    req.continuation = id;
    req.continuation_for = next;
    req.iters[next].call = id;
    note(r, "submit_partial iteration=" + std::to_string(next));
  }
  void on_decoded(size_t r, size_t i, Time at) {
    ReqRt& req = reqs[r];
    IterRt& it = req.iters[i];
    const Iter& spec = trace[r].iters[i];
    it.decoded = true;
    note(r, "decode_complete iteration=" + std::to_string(i));
    if (spec.final) {
      req.done = true;
      note(r, "request_done");
      return;
    }
    if (!sim.streaming || it.fallback || it.next_dispatch < spec.tools.size()) {
      for (size_t j = it.next_dispatch; j < spec.tools.size(); ++j) dispatch(r, i, j, at, spec.tools[j].emit);
      it.next_dispatch = spec.tools.size();
    }
    if (sim.splitting && it.pending > 0) submit_partial(r, i);
    advance(r, i);
  }
  void advance(size_t r, size_t i) {
    IterRt& it = reqs[r].iters[i];
    if (it.advanced || !it.decoded || it.pending > 0) return;
    if (trace[r].iters[i].final) return;
    it.advanced = true;
    submit_iteration(r, i + 1);
  }
  void run() {
    reqs.resize(trace.size());
    for (size_t r = 0; r < trace.size(); ++r) {
      reqs[r].iters.resize(trace[r].iters.size());
      sim.loop.at(trace[r].arrival, [this, r] {
        note(r, "arrival");
        submit_iteration(r, 0);
      });
    }
    sim.loop.run();
  }
};

}  // namespace rp
}  // namespace sb

using namespace sb;

extern "C" int sb_replay_generated(const char* workload, const double* gen, int32_t n_requests, uint64_t seed,
                                   int32_t preset, int64_t capacity, int64_t block_size, const double* cost,
                                   int32_t device, int64_t* ftr, int64_t* e2e, int64_t* hit, int64_t* prompt,
                                   uint64_t* evictions) {
  return guard([&] {
    rp::GenConfig g;
    const std::string w = workload ? workload : "default";
    if (w == "tool_heavy" || w == "tool-heavy") {
      g.fanout_p = 0.22;
      g.ratio_scale = 1.2;
      g.tool_out_median = 1500.0;
      g.qps = 0.03;
    } else if (w == "iteration_heavy" || w == "iteration-heavy") {
      g.depth_p = 0.25;
      g.fanout_p = 0.6;
      g.ratio_scale = 0.25;
      g.tool_out_median = 900.0;
      g.qps = 0.03;
    } else if (w != "default") {
      throw Error(SB_ERR_CONFIG, "unknown workload '" + w + "'");
    }
    g.num_requests = n_requests;
    if (gen) {
      if (gen[0] > 0) g.prompt_base_median = gen[0];
      if (gen[1] > 0) g.tool_out_median = gen[1];
      if (gen[2] > 0) g.decode_inter_median = gen[2];
      if (gen[3] > 0) g.decode_final_median = gen[3];
      if (gen[4] > 0) g.qps = gen[4];
      if (gen[5] > 0) g.depth_p = gen[5];
      if (gen[6] > 0) g.fanout_p = gen[6];
      if (gen[7] > 0) g.ratio_scale = gen[7];
    }
    const auto trace = rp::generate(g, seed);
    rp::Sim sim;
    // presets (runner.cpp:120-153): baseline = FCFS/LRU, baseline_sched =
    // request-aware/LRU, sutradhara = request-aware/tiered + PS + DS
    const bool tiered = preset == 2;
    sim.request_aware = preset != 0;
    sim.splitting = sim.streaming = preset == 2;
    sim.bs = block_size;
    if (cost) {
      sim.cost.prefill_ms_per_token = cost[0];
      sim.cost.decode_ms_per_token = cost[1];
      sim.cost.overhead_ms = cost[2];
      sim.cost.chunk = static_cast<int64_t>(cost[3]);
    }
    int st = sb_kv_create(block_size, capacity, tiered ? SB_POLICY_TIERED : SB_POLICY_LRU, device, &sim.pool.c);
    if (st) return st;
    try {
      rp::Orchestrator orch(sim, trace);
      orch.run();
      for (size_t r = 0; r < trace.size(); ++r) {
        if (!orch.reqs[r].done) throw Error(SB_ERR_INVALID, "request " + trace[r].id + " did not complete");
        int64_t h = 0, p = 0;
        for (size_t i = 0; i < trace[r].iters.size(); ++i) {
          const rp::Call& c = sim.calls.at(orch.reqs[r].iters[i].call);
          h += c.cached_prefix;
          p += c.prompt_tokens;
          if (trace[r].iters[i].final) {
            if (ftr) ftr[r] = c.first_token - trace[r].arrival;
            if (e2e) e2e[r] = c.decode_complete - trace[r].arrival;
          }
        }
        if (hit) hit[r] = h;
        if (prompt) prompt[r] = p;
      }
      if (evictions) *evictions = sb_kv_total_evicted(sim.pool.c);
    } catch (...) {
      sb_kv_destroy(sim.pool.c);
      throw;
    }
    sb_kv_destroy(sim.pool.c);
    return int(SB_OK);
  });
}
