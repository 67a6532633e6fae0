// ref_engine.cpp — TEST INFRASTRUCTURE ONLY.
//
// Scripted driver of the UNMODIFIED reference engine
// (/root/reference/proj/src/engine.cpp over src/kv_cache.cpp and src/sim.cpp):
// a caller issues the engine-boundary actions the orchestrator would issue
// (submit_call / submit_partial_prefill / extend_prefill / abandon_partial,
// engine.hpp:104-111) at chosen virtual times, the reference event loop runs
// the engine in between, and every engine-internal KV transition is recorded
// with the pool's audit dump right after it:
//   pin        Engine::pin_partial           engine.cpp:250-286 (on_ready)
//   pin_failed Engine::pin_partial CacheFull engine.cpp:255-259 (on_pin_failed)
//   complete   Engine::complete_prefill      engine.cpp:305-322
//   finish     Engine::finish_decode         engine.cpp:324-347 (on_decode_complete)
// The resulting event list is the golden sequence the B200 engine lifecycle
// (sb_engine_*, csrc/engine.cu) must reproduce: same transitions, same
// virtual times, byte-identical dumps (tests/test_engine_lifecycle_gpu.py).
//
// A `complete` that shares an engine step with `finish`es has no separate
// observation point (the reference runs them inside one finish_inflight,
// engine.cpp:354-379): it is recorded without a dump and the following
// finish's dump covers both.
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "agentsim/engine.hpp"
#include "agentsim/kv_cache.hpp"
#include "agentsim/sim.hpp"
#include "agentsim/trace.hpp"

using namespace agentsim;

namespace {

thread_local std::string g_err;

std::string json_escape(const std::string& s) {
  std::string o;
  o.reserve(s.size() + 8);
  for (char c : s) {
    if (c == '\n') o += "\\n";
    else if (c == '"') o += "\\\"";
    else if (c == '\\') o += "\\\\";
    else o += c;
  }
  return o;
}

std::vector<TagRange> tags_of(const int64_t* t, int64_t n) {
  std::vector<TagRange> v;
  for (int64_t i = 0; i < n; ++i) v.push_back(TagRange{t[3 * i], t[3 * i + 1], static_cast<KvTag>(t[3 * i + 2])});
  return v;
}

int status_of(const std::exception& e) {
  if (dynamic_cast<const CacheFull*>(&e)) return 1;
  if (dynamic_cast<const UnknownBlock*>(&e)) return 2;
  if (dynamic_cast<const ZeroRefRelease*>(&e)) return 3;
  if (dynamic_cast<const CacheError*>(&e)) return 4;
  if (dynamic_cast<const ConfigError*>(&e)) return 5;
  if (dynamic_cast<const StaleHandle*>(&e)) return 9;
  if (dynamic_cast<const InvalidState*>(&e)) return 10;
  if (dynamic_cast<const UnknownCall*>(&e)) return 11;
  if (dynamic_cast<const DuplicateCallId*>(&e)) return 12;
  return 99;
}

struct Harness {
  EventLoop loop;
  KvCache cache;
  Engine engine;
  std::map<CallId, CallState> seen;     // last observed state per call
  std::map<CallId, bool> completed;     // complete event already recorded
  std::vector<std::string> events;

  Harness(const CacheConfig& cc, CostModel cost, SchedulerPolicy sched)
      : cache(cc), engine(loop, cache, cost, sched) {}

  void record(const char* ev, CallId call, SimTime t, const std::string& extra, bool with_dump) {
    std::ostringstream o;
    o << "{\"ev\":\"" << ev << "\",\"call\":" << call << ",\"t\":" << t << extra;
    if (with_dump) o << ",\"dump\":\"" << json_escape(cache.dump()) << "\"";
    o << "}";
    events.push_back(o.str());
  }

  // complete_prefill transitions observed since the last poll (call order;
  // at most one chunk call completes per engine step)
  void poll_completes(bool with_dump) {
    for (auto& [id, st] : seen) {
      if (!engine.has_call(id)) continue;
      const CallRecord& r = engine.call(id);
      const bool decoding_now = r.state == CallState::kDecoding || r.state == CallState::kDone;
      if (decoding_now && !completed[id]) {
        completed[id] = true;
        record("complete", id, r.prefill_complete_time, "", with_dump);
      }
      st = r.state;
    }
  }

  CallCallback on_finish() {
    return [this](CallId id, SimTime at) {
      poll_completes(false);
      const CallRecord& r = engine.call(id);
      record("finish", id, at, ",\"emitted\":" + std::to_string(r.emitted), true);
    };
  }
};

}  // namespace

extern "C" {

const char* refeng_last_error() { return g_err.c_str(); }

// cost: [prefill_ms_per_token, decode_ms_per_token, batch_decode_overhead_ms,
// chunk_size] or NULL for the reference defaults (engine.hpp:19-30).
void* refeng_create(int64_t block_size, int64_t capacity, int32_t policy, int32_t sched, const double* cost) {
  try {
    CacheConfig cc;
    cc.block_size = block_size;
    cc.capacity_blocks = capacity;
    cc.policy = policy ? EvictionPolicy::kTiered : EvictionPolicy::kLru;
    CostModel cm;
    if (cost) {
      cm.prefill_ms_per_token = cost[0];
      cm.decode_ms_per_token = cost[1];
      cm.batch_decode_overhead_ms = cost[2];
      cm.chunk_size = static_cast<int64_t>(cost[3]);
    }
    return new Harness(cc, cm, sched ? SchedulerPolicy::kRequestAware : SchedulerPolicy::kFcfs);
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void refeng_destroy(void* h) { delete static_cast<Harness*>(h); }

int64_t refeng_now(void* h) { return static_cast<Harness*>(h)->loop.now(); }

int refeng_submit_call(void* hp, const uint64_t* tok, int64_t n, const int64_t* tags, int64_t n_tags,
                       int64_t decode_len, uint64_t key, int64_t* id) {
  auto* h = static_cast<Harness*>(hp);
  try {
    CallSubmission s;
    s.prompt.assign(tok, tok + n);
    s.tags = tags_of(tags, n_tags);
    s.decode_length = decode_len;
    s.decode_stream_key = key;
    s.on_decode_complete = h->on_finish();
    const CallId c = h->engine.submit_call(std::move(s));
    *id = static_cast<int64_t>(c);
    h->seen[c] = CallState::kQueued;
    h->record("submit_call", c, h->loop.now(),
              ",\"cached\":" + std::to_string(h->engine.call(c).cached_prefix), true);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

int refeng_submit_partial(void* hp, const uint64_t* tok, int64_t n, const int64_t* tags, int64_t n_tags,
                          uint64_t key, int64_t* id) {
  auto* h = static_cast<Harness*>(hp);
  try {
    PartialSubmission s;
    s.prefix.assign(tok, tok + n);
    s.tags = tags_of(tags, n_tags);
    s.decode_stream_key = key;
    s.on_ready = [h](CallId c, SimTime at) { h->record("pin", c, at, "", true); };
    s.on_pin_failed = [h](CallId c, SimTime at) { h->record("pin_failed", c, at, "", true); };
    const CallId c = h->engine.submit_partial_prefill(std::move(s)).call_id;
    *id = static_cast<int64_t>(c);
    h->seen[c] = CallState::kQueued;
    h->record("submit_partial", c, h->loop.now(),
              ",\"cached\":" + std::to_string(h->engine.call(c).cached_prefix), true);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

int refeng_extend(void* hp, int64_t id, const uint64_t* tok, int64_t n, const int64_t* tags, int64_t n_tags,
                  int64_t decode_len) {
  auto* h = static_cast<Harness*>(hp);
  try {
    h->engine.extend_prefill(ContinuationHandle{static_cast<CallId>(id)}, std::vector<TokenId>(tok, tok + n),
                             tags_of(tags, n_tags), decode_len, h->on_finish());
    h->record("extend", static_cast<CallId>(id), h->loop.now(), "", true);
    h->poll_completes(true);  // an empty suffix completes at once (engine.cpp:212-215)
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

int refeng_abandon(void* hp, int64_t id) {
  auto* h = static_cast<Harness*>(hp);
  try {
    h->engine.abandon_partial(ContinuationHandle{static_cast<CallId>(id)});
    h->record("abandon", static_cast<CallId>(id), h->loop.now(), "", true);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// Runs the loop one virtual millisecond at a time, recording transitions as
// they happen: up to `until` (then the clock is moved to `until` with a no-op
// event, so the caller's next action happens at that virtual time, after
// every event already due then), or with until < 0 until the queue empties.
int refeng_run(void* hp, int64_t until) {
  auto* h = static_cast<Harness*>(hp);
  try {
    SimTime t = h->loop.now();
    while (!h->loop.empty() && (until < 0 || t < until)) {
      ++t;
      h->loop.run(t);
      h->poll_completes(true);
    }
    if (until >= 0) {
      if (until < h->loop.now()) throw TimeTravel("refeng_run: until before now");
      h->loop.schedule(until, EventKind::kRequestArrival, "script", [] {});
      h->loop.run(until);
      h->poll_completes(true);
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return status_of(e);
  }
}

// Events recorded so far as JSON lines; returns the full length.
int64_t refeng_events(void* hp, char* buf, int64_t cap) {
  auto* h = static_cast<Harness*>(hp);
  std::string s;
  for (const auto& e : h->events) s += e + "\n";
  if (buf && cap > 0) {
    const size_t m = std::min<size_t>(s.size(), static_cast<size_t>(cap - 1));
    std::memcpy(buf, s.data(), m);
    buf[m] = 0;
  }
  return static_cast<int64_t>(s.size());
}

}  // extern "C"

#include "agentsim/runner.hpp"
#include "agentsim/scenarios.hpp"

// The paper's overlap-timeline scenario (scenarios.cpp:193-240) through the
// reference orchestrator: split = 1 runs it with prompt splitting + decode
// streaming.  Copies the run's timeline text (engine-boundary actions with
// their virtual times) into buf and returns its length; per-request FTR in
// *ftr.  In libagentsim_kvlog.so every KvCache op of the run is recorded too.
extern "C" int64_t refeng_overlap_scenario(int32_t split, char* buf, int64_t cap, int64_t* ftr) {
  try {
    SimulationResult r = run_trace(overlap_trace(), overlap_config(split != 0));
    if (ftr) *ftr = r.metrics.at(0).ftr_ms;
    const std::string& s = r.timeline_text;
    if (buf && cap > 0) {
      const size_t m = std::min<size_t>(s.size(), static_cast<size_t>(cap - 1));
      std::memcpy(buf, s.data(), m);
      buf[m] = 0;
    }
    return static_cast<int64_t>(s.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// Orchestrator::decode_stream_key (orchestrator.cpp:179-181).
extern "C" uint64_t refeng_stream_key(const char* request_id, uint64_t iteration) {
  return hash_combine(hash_string(request_id), iteration);
}
