// agentsim_run.cpp — C entry point that replays one shard of a synthetic
// agent trace through the reference simulator (trace_gen.cpp:96-193,
// runner.cpp preset resolution, orchestrator.cpp run_trace), compiled into
//   integration/_build/libagentsim_b200.so  — the UNMODIFIED reference
//       engine/orchestrator with its KvCache implemented by the B200 block
//       pool (agentsim_kvcache_b200.cpp): the drop-in, and
//   oracle/_ref/libagentsim_ref.so  — the pure reference (its CPU arm).
// Shard s of n keeps requests i with i % n == s of ONE generated trace (the
// multi-GPU layout of BASELINE configs[3]: each rank replays its shard on its
// own pool, the per-request results are gathered).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "agentsim/runner.hpp"
#include "agentsim/trace_gen.hpp"

using namespace agentsim;

namespace {
thread_local std::string g_err;
}

extern "C" {

const char* agentsim_run_last_error() { return g_err.c_str(); }

// gen: [prompt_base_median, tool_out_median, decode_inter_median,
// decode_final_median, qps, depth_p, fanout_p, ratio_scale] (<= 0 keeps the
// workload's value); kv_tiering: -1 = the preset's, 0 = LRU, 1 = hint-aware; cost: [prefill_ms_per_token, decode_ms_per_token,
// batch_decode_overhead_ms, chunk_size] or NULL.  Per kept request: FTR, e2e,
// prefix-hit and prompt tokens, and the FTR breakdown (metrics.cpp:104-129:
// critical tool, waiting, prefill, decode ms).  Returns the number of kept
// requests, or -1 (agentsim_run_last_error).
int64_t agentsim_run_shard(const char* workload, const double* gen, int32_t n_requests, uint64_t seed,
                           int32_t preset, int32_t kv_tiering, int64_t capacity, int64_t block_size,
                           const double* cost, int32_t shard, int32_t n_shards, int64_t* ftr, int64_t* e2e, int64_t* hit, int64_t* prompt,
                           int64_t* tool_ms, int64_t* wait_ms, int64_t* prefill_ms, int64_t* decode_ms,
                           uint64_t* evictions, double* wall_s) {
  try {
    GeneratorConfig g = workload ? *workload_by_name(workload) : default_workload();
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
    std::vector<AgenticRequestSpec> all = generate_synthetic_trace(g, seed), mine;
    for (size_t i = 0; i < all.size(); ++i)
      if (n_shards <= 1 || static_cast<int32_t>(i % static_cast<size_t>(n_shards)) == shard) mine.push_back(all[i]);
    RunConfig rc;
    rc.preset = preset == 0 ? RunPreset::kBaseline : (preset == 1 ? RunPreset::kBaselineSched : RunPreset::kSutradhara);
    if (kv_tiering >= 0) rc.kv_override = kv_tiering != 0;  // hint-aware vs LRU eviction (runner.cpp)
    rc.capacity_blocks = capacity;
    rc.block_size = block_size;
    rc.seed = seed;
    if (cost) {
      rc.cost.prefill_ms_per_token = cost[0];
      rc.cost.decode_ms_per_token = cost[1];
      rc.cost.batch_decode_overhead_ms = cost[2];
      rc.cost.chunk_size = static_cast<int64_t>(cost[3]);
    }
    const SimConfig sim = resolve_sim_config(rc);
    const auto t0 = std::chrono::steady_clock::now();
    const SimulationResult res = run_trace(mine, sim);
    const auto t1 = std::chrono::steady_clock::now();
    if (wall_s) *wall_s = std::chrono::duration<double>(t1 - t0).count();
    for (size_t i = 0; i < res.metrics.size(); ++i) {
      const RequestMetrics& m = res.metrics[i];
      if (ftr) ftr[i] = m.ftr_ms;
      if (e2e) e2e[i] = m.e2e_ms;
      if (hit) hit[i] = m.hit_tokens();
      if (prompt) prompt[i] = m.prompt_tokens();
      if (tool_ms) tool_ms[i] = m.breakdown.critical_tool_ms;
      if (wait_ms) wait_ms[i] = m.breakdown.waiting_ms;
      if (prefill_ms) prefill_ms[i] = m.breakdown.prefill_ms;
      if (decode_ms) decode_ms[i] = m.breakdown.decode_ms;
    }
    if (evictions) *evictions = res.cache_evictions;
    return static_cast<int64_t>(res.metrics.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

}  // extern "C"

#include "agentsim/scenarios.hpp"

// The paper's KV-thrashing scenario (scenarios.cpp:45-85: three two-iteration
// requests whose first-iteration chains exactly fill the pool) under LRU
// (tiered = 0) or hint-aware tiered eviction (tiered = 1): iteration-2 prefix
// hit tokens per request, and the run's hit rate.
extern "C" int agentsim_thrashing(int32_t tiered, int64_t* it2_hits, double* hit_rate, uint64_t* evictions) {
  try {
    const SimulationResult r = run_trace(thrashing_trace(), thrashing_config(tiered != 0));
    for (size_t i = 0; i < r.metrics.size(); ++i) it2_hits[i] = r.metrics[i].cache.at(1).hit_tokens;
    if (hit_rate) *hit_rate = cache_hit_rate(r.metrics);
    if (evictions) *evictions = r.cache_evictions;
    return static_cast<int>(r.metrics.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}
