// ref_runapi.cpp — TEST INFRASTRUCTURE ONLY.
//
// C entry points that drive the UNMODIFIED reference simulator
// (/root/reference/proj/src/{trace_gen,orchestrator,runner,scenarios}.cpp):
// generate a synthetic agent trace, replay it under a preset, and return the
// per-request metrics.  Used for golden vectors and as the reference arm of
// bench.py (the reference's own CPU code path, timed on the host).
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "agentsim/runner.hpp"
#include "agentsim/scenarios.hpp"
#include "agentsim/trace_gen.hpp"

using namespace agentsim;

namespace {
thread_local std::string g_err;

SimConfig preset_config(int32_t preset, int64_t capacity, int64_t block_size, uint64_t seed) {
  RunConfig rc;
  rc.preset = preset == 0 ? RunPreset::kBaseline
                          : (preset == 1 ? RunPreset::kBaselineSched : RunPreset::kSutradhara);
  rc.capacity_blocks = capacity;
  rc.block_size = block_size;
  rc.seed = seed;
  return resolve_sim_config(rc);
}

int write_results(const SimulationResult& res, int64_t* ftr, int64_t* e2e, int64_t* hit,
                  int64_t* prompt, uint64_t* evictions) {
  for (size_t i = 0; i < res.metrics.size(); ++i) {
    if (ftr) ftr[i] = res.metrics[i].ftr_ms;
    if (e2e) e2e[i] = res.metrics[i].e2e_ms;
    if (hit) hit[i] = res.metrics[i].hit_tokens();
    if (prompt) prompt[i] = res.metrics[i].prompt_tokens();
  }
  if (evictions) *evictions = res.cache_evictions;
  return 0;
}
}  // namespace

extern "C" {

const char* refrun_last_error() { return g_err.c_str(); }

// gen: [prompt_base_median, tool_out_median, decode_inter_median,
//       decode_final_median, qps, depth_p, fanout_p, ratio_scale]
// (values <= 0 keep the default_workload() setting).  workload: NULL or a
// reference workload name used as the base config.
int refrun_generate_and_run(const char* workload, const double* gen, int32_t n_requests,
                            uint64_t seed, int32_t preset, int64_t capacity, int64_t block_size,
                            int64_t* ftr, int64_t* e2e, int64_t* hit, int64_t* prompt,
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
    auto trace = generate_synthetic_trace(g, seed);
    SimConfig sim = preset_config(preset, capacity, block_size, seed);
    auto t0 = std::chrono::steady_clock::now();
    SimulationResult res = run_trace(trace, sim);
    auto t1 = std::chrono::steady_clock::now();
    if (wall_s) *wall_s = std::chrono::duration<double>(t1 - t0).count();
    return write_results(res, ftr, e2e, hit, prompt, evictions);
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

// Runs the embedded paper scenarios; returns 1 when all pass.  The report
// text is copied into buf.
int refrun_scenarios(char* buf, int64_t cap) {
  bool ok = false;
  std::string rep = run_all_scenarios_report(&ok);
  if (buf && cap > 0) {
    size_t m = std::min<size_t>(rep.size(), static_cast<size_t>(cap - 1));
    std::memcpy(buf, rep.data(), m);
    buf[m] = 0;
  }
  return ok ? 1 : 0;
}

// Thrashing scenario replay (scenarios.cpp:45-85) under LRU (tiered=0) or
// tiered (tiered=1): per-request hit tokens of iteration 2.
int refrun_thrashing(int32_t tiered, int64_t* it2_hits) {
  try {
    SimulationResult r = run_trace(thrashing_trace(), thrashing_config(tiered != 0));
    for (size_t i = 0; i < r.metrics.size(); ++i) it2_hits[i] = r.metrics[i].cache[1].hit_tokens;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

}  // extern "C"

extern "C" int64_t refrun_timeline(const double* gen, int32_t n_requests, uint64_t seed, int32_t preset,
                                   int64_t capacity, int64_t block_size, char* buf, int64_t cap) {
  GeneratorConfig g = default_workload();
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
  auto trace = generate_synthetic_trace(g, seed);
  SimConfig sim = preset_config(preset, capacity, block_size, seed);
  SimulationResult res = run_trace(trace, sim);
  const std::string& s = res.timeline_text;
  if (buf && cap > 0) {
    size_t m = std::min<size_t>(s.size(), static_cast<size_t>(cap - 1));
    std::memcpy(buf, s.data(), m);
    buf[m] = 0;
  }
  return static_cast<int64_t>(s.size());
}
