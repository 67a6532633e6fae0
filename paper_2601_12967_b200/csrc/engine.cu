// engine.cu — host-side continuation engine (C++), the B200 counterpart of
// the reference engine's KV lifecycle (/root/reference/proj/src/engine.cpp):
//   submit_call / submit_partial_prefill  engine.cpp:128-182 (admission lookup)
//   complete_prefill -> pin_partial       engine.cpp:250-286, 305-322
//   extend_prefill                        engine.cpp:184-223
//   release_partial_pins                  engine.cpp:288-303
//   abandon_partial                       engine.cpp:234-248
//   finish_decode                         engine.cpp:324-347
// Every KV transition is one op of the block pool's op program
// (pool_program.cuh): the per-call API below runs one op per call, the
// batched step (sb_batch_*) runs one op per continuation of the batch, in
// batch order, with the same code and therefore the same semantics.
//
// Where the reference only charges a prefill cost (CostModel::chunk_ms,
// engine.cpp:35-39) this engine runs the computation: KV append + the
// tcgen05 continuation attention over the paged pool (csrc/attention.cu),
// optionally the full Llama-shaped layers around it (csrc/model.cu).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <numeric>
#include <vector>

#include "common.h"
#include "hash.cuh"
#include "program.h"

namespace sb {

// suffix tokens (packed in batch order) into each slot's prompt buffer
__global__ void k_scatter_suffix(const uint64_t* __restrict__ suffix, const int64_t* __restrict__ suffix_off,
                                 const int64_t* __restrict__ slot_off, int32_t n_seqs, uint64_t* __restrict__ prompts) {
  const int64_t total = suffix_off[n_seqs];
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int lo = 0, hi = n_seqs;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (suffix_off[mid] <= i) lo = mid; else hi = mid;
    }
    prompts[slot_off[lo] + (i - suffix_off[lo])] = suffix[i];
  }
}

// response tokens of a finish: the model's greedy token (when given) else
// decode_token(stream_key, 0) (trace.cpp:80-83), written after each prompt
__global__ void k_response_tokens(const int32_t* __restrict__ model_tok, const uint64_t* __restrict__ keys,
                                  const int64_t* __restrict__ resp_pos, int n, uint64_t* __restrict__ prompts) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n) return;
  prompts[resp_pos[s]] = model_tok ? static_cast<uint64_t>(model_tok[s]) : decode_token(keys[s], 0);
}

// dense page table [n, max_blocks] from per-slot chain arrays
__global__ void k_slot_table(const int32_t* __restrict__ chains, const int64_t* __restrict__ chain_off,
                             const int32_t* __restrict__ n_blocks, int32_t n, int32_t max_blocks, int32_t* __restrict__ table) {
  const int64_t total = static_cast<int64_t>(n) * max_blocks;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int s = static_cast<int>(i / max_blocks), j = static_cast<int>(i % max_blocks);
    table[i] = j < n_blocks[s] ? chains[chain_off[s] + j] : -1;
  }
}

struct ModelWorkspace;
ModelWorkspace* model_workspace_create(sb_model* m, const std::vector<int64_t>& prefix_len,
                                       const std::vector<int64_t>& suffix_len);
void model_workspace_destroy(ModelWorkspace* w);
void model_embed(sb_model* m, ModelWorkspace* w, const uint64_t* d_suffix, cudaStream_t st);
void model_layer_pre(sb_model* m, ModelWorkspace* w, int l, void* k_pool, void* v_pool, const int32_t* q_off,
                     const int32_t* kv_len, const int32_t* table, int32_t n_seqs, int32_t max_blocks,
                     cudaStream_t st);
void model_layer_post(sb_model* m, ModelWorkspace* w, int l, cudaStream_t st);
void model_head(sb_model* m, ModelWorkspace* w, cudaStream_t st);
double model_flops(const sb_model* m, int64_t rows);
struct ModelIO {  // the few workspace buffers the engine touches (model.cu)
  __nv_bfloat16 *q, *a;
  float* logits;
  int32_t* next_tok;
};
ModelIO model_io(ModelWorkspace* w);

template <class T>
static T* dmalloc(size_t n) {
  T* p = nullptr;
  SB_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
  return p;
}

template <class T>
static T* upload(const std::vector<T>& v) {
  T* p = dmalloc<T>(v.size());
  if (!v.empty()) SB_CUDA(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return p;
}

static bool tags_cover_host(const sb_tag_range* t, int64_t nt, int64_t n) {
  int64_t covered = 0;
  for (int64_t i = 0; i < nt; ++i) {
    if (t[i].begin != covered || t[i].end < t[i].begin) return false;
    covered = t[i].end;
  }
  return covered == n;
}

}  // namespace sb

using namespace sb;

// agentsim::CallState order (engine.hpp:35)
enum { CS_QUEUED = 0, CS_PREFILLING = 1, CS_AWAITING = 2, CS_DECODING = 3, CS_DONE = 4, CS_ABORTED = 5 };

struct Call {
  bool partial = false, ext = false;
  int state = CS_QUEUED;
  std::vector<uint64_t> prompt;
  std::vector<sb_tag_range> tags;
  int64_t cached = 0;
  int64_t decode_len = 0;
  int64_t hashed_full = 0;  // full blocks whose chain hashes are current in d_hash
  // device
  uint64_t* d_tok = nullptr;
  uint64_t* d_hash = nullptr;
  sb_tag_range* d_tags = nullptr;
  int32_t *d_ids = nullptr, *d_chain = nullptr, *d_pinned = nullptr;
  int64_t cap_tok = 0, cap_blk = 0, cap_tags = 0;
  int32_t n_chain = 0, n_pinned = 0;
  std::vector<int32_t> chain, pinned;  // host mirrors
  ~Call() {
    for (void* p : {static_cast<void*>(d_tok), static_cast<void*>(d_hash), static_cast<void*>(d_tags),
                    static_cast<void*>(d_ids), static_cast<void*>(d_chain), static_cast<void*>(d_pinned)})
      if (p) cudaFree(p);
  }
};

struct sb_engine {
  int32_t n_layers, hq, hkv, hd, device, policy;
  int64_t cap;
  sb_kv_cache* cache = nullptr;
  std::vector<__nv_bfloat16*> k_pools, v_pools;
  int32_t* d_pin_cnt = nullptr;  // Engine::partial_pin_counts_ (engine.hpp:187), per block id
  int8_t* d_real_tag = nullptr;  // Engine::partial_real_tags_ (engine.hpp:188), -1 = none
  int64_t* d_scratch = nullptr;  // [0] lookup hit, [2..6) hashing segment meta
  std::map<int32_t, Call> calls;
  int32_t next_id = 1;
  ~sb_engine() {
    cudaSetDevice(device);
    calls.clear();
    for (auto* p : k_pools) cudaFree(p);
    for (auto* p : v_pools) cudaFree(p);
    for (void* p : {static_cast<void*>(d_pin_cnt), static_cast<void*>(d_real_tag), static_cast<void*>(d_scratch)})
      if (p) cudaFree(p);
    if (cache) sb_kv_destroy(cache);
  }
};

namespace {

Call& find_call(sb_engine* e, int32_t id, int missing_code) {
  auto it = e->calls.find(id);
  if (it == e->calls.end()) throw Error(missing_code, "call " + std::to_string(id) + " unknown");
  return it->second;
}

// device buffers of a call sized for n tokens (+ the response) and nt tags,
// keeping their contents
void ensure_call_dev(Call& c, int64_t n, int64_t nt) {
  auto grow = [](auto*& p, int64_t& cap, int64_t need, int64_t keep) {
    if (need <= cap) return;
    using T = std::remove_pointer_t<std::remove_reference_t<decltype(p)>>;
    const int64_t nc = std::max<int64_t>(need, 2 * cap);
    T* q = dmalloc<T>(nc);
    if (p && keep > 0) SB_CUDA(cudaMemcpy(q, p, sizeof(T) * keep, cudaMemcpyDeviceToDevice));
    if (p) cudaFree(p);
    p = q;
    cap = nc;
  };
  const int64_t blk = (n + 15) / 16 + 1;
  int64_t ct = c.cap_tok, cb = c.cap_blk;
  grow(c.d_tok, ct, n + 1, c.cap_tok);
  c.cap_tok = ct;
  int64_t cb1 = c.cap_blk, cb2 = c.cap_blk, cb3 = c.cap_blk, cb4 = c.cap_blk;
  grow(c.d_hash, cb1, blk, c.cap_blk);
  grow(c.d_ids, cb2, blk, c.cap_blk);
  grow(c.d_chain, cb3, blk, c.cap_blk);
  grow(c.d_pinned, cb4, blk, c.cap_blk);
  c.cap_blk = std::max(cb, cb1);
  int64_t cg = c.cap_tags;
  grow(c.d_tags, cg, nt + 1, c.cap_tags);
  c.cap_tags = cg;
}

// chain hashes of blocks [from, ceil(n/16)) of the call's prompt buffer
// (the fold continues from block from-1's hash): incremental hashing
void hash_call(sb_engine* e, Call& c, int64_t n, int64_t from, cudaStream_t st) {
  const int64_t nb = (n + 15) / 16;
  if (from >= nb) return;
  int64_t meta[3] = {16 * from, n, from};
  SB_CUDA(cudaMemcpyAsync(e->d_scratch + 2, meta, sizeof(meta), cudaMemcpyHostToDevice, st));
  const int rc = sb_chain_hash_segments(c.d_tok, e->d_scratch + 2, e->d_scratch + 4,
                                        from ? c.d_hash + from - 1 : nullptr, 1, 16, c.d_hash, st);
  if (rc) throw Error(rc, sb_last_error());
}

ProgOp call_op(Call& c, int kind, int64_t n, int64_t n_ins_tags) {
  ProgOp o{};
  o.kind = kind;
  o.n = n;
  o.tokens = c.d_tok;
  o.hashes = c.d_hash;
  o.ins_tags = c.d_tags;
  o.n_ins_tags = static_cast<int32_t>(n_ins_tags);
  o.real_tags = c.d_tags;
  o.n_real_tags = static_cast<int32_t>(c.tags.size());
  o.ids = c.d_ids;
  o.chain = c.d_chain;
  o.pinned = c.d_pinned;
  o.n_chain = c.n_chain;
  o.n_pinned = c.n_pinned;
  return o;
}

ProgRes run_one(sb_engine* e, Call& c, const ProgOp& op, int64_t now) {
  cudaStream_t st = pool_stream(e->cache);
  ProgRes r{};
  pool_run_ops(e->cache, &op, 1, e->d_pin_cnt, e->d_real_tag, now, st, &r);
  c.n_chain = r.n_chain;
  c.n_pinned = r.n_pinned;
  c.chain.resize(static_cast<size_t>(c.n_chain));
  c.pinned.resize(static_cast<size_t>(c.n_pinned));
  if (c.n_chain)
    SB_CUDA(cudaMemcpy(c.chain.data(), c.d_chain, sizeof(int32_t) * c.n_chain, cudaMemcpyDeviceToHost));
  if (c.n_pinned)
    SB_CUDA(cudaMemcpy(c.pinned.data(), c.d_pinned, sizeof(int32_t) * c.n_pinned, cudaMemcpyDeviceToHost));
  if (r.status != SB_OK && r.status != SB_ERR_CACHE_FULL) throw Error(r.status, "engine KV op failed");
  return r;
}

int32_t submit(sb_engine* e, const uint64_t* tokens, int64_t n, const sb_tag_range* tags, int64_t n_tags, int64_t now,
               bool partial, int64_t decode_len) {
  if (n <= 0)
    throw Error(SB_ERR_INVALID_STATE, partial ? "submit_partial_prefill: prefix must be non-empty"
                                              : "submit_call: prompt must be non-empty");
  if (!partial && decode_len < 1) throw Error(SB_ERR_INVALID_STATE, "submit_call: decode_length must be >= 1");
  if (!tags_cover_host(tags, n_tags, n)) throw Error(SB_ERR_INVALID_STATE, "tag ranges must cover the prompt");
  SB_CUDA(cudaSetDevice(e->device));
  cudaStream_t st = pool_stream(e->cache);
  const int32_t id = e->next_id++;
  Call& c = e->calls[id];
  c.partial = partial;
  c.decode_len = decode_len;
  c.prompt.assign(tokens, tokens + n);
  c.tags.assign(tags, tags + n_tags);
  ensure_call_dev(c, n, n_tags);
  SB_CUDA(cudaMemcpyAsync(c.d_tok, tokens, sizeof(uint64_t) * n, cudaMemcpyHostToDevice, st));
  SB_CUDA(cudaMemcpyAsync(c.d_tags, tags, sizeof(sb_tag_range) * n_tags, cudaMemcpyHostToDevice, st));
  hash_call(e, c, n, 0, st);
  c.hashed_full = n / 16;
  // admission lookup (engine.cpp:141, 170)
  ProgOp op = call_op(c, PK_INSERT, n, n_tags);
  pool_lookup(e->cache, &op, 1, now, e->d_scratch, st);
  SB_CUDA(cudaMemcpyAsync(&c.cached, e->d_scratch, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  SB_CUDA(cudaStreamSynchronize(st));
  return id;
}

// Engine::complete_prefill (engine.cpp:305-322); a partial not yet extended
// is pinned instead (pin_partial, engine.cpp:250-286).  Returns the outcome.
int complete(sb_engine* e, Call& c, int64_t now) {
  const int64_t n = static_cast<int64_t>(c.prompt.size());
  if (c.partial && !c.ext) {
    const ProgRes r = run_one(e, c, call_op(c, PK_PIN, n, 1), now);
    c.state = r.outcome == PO_PINNED ? CS_AWAITING : CS_ABORTED;
    return r.outcome;
  }
  run_one(e, c, call_op(c, PK_COMPLETE, n, static_cast<int64_t>(c.tags.size())), now);
  c.state = CS_DECODING;
  return PO_COMPLETED;
}

}  // namespace

extern "C" {

int sb_engine_create(int32_t n_layers, int32_t n_q_heads, int32_t n_kv_heads, int32_t head_dim,
                     int64_t capacity_blocks, int32_t policy, int32_t device, uint64_t seed, sb_engine** out) {
  return guard([&] {
    if (head_dim != 128) throw Error(SB_ERR_UNSUPPORTED, "head_dim must be 128");
    if (n_layers < 1 || n_kv_heads < 1 || n_q_heads % n_kv_heads) throw Error(SB_ERR_INVALID, "bad model shape");
    SB_CUDA(cudaSetDevice(device));
    auto* e = new sb_engine();
    try {
      e->n_layers = n_layers;
      e->hq = n_q_heads;
      e->hkv = n_kv_heads;
      e->hd = head_dim;
      e->device = device;
      e->policy = policy;
      e->cap = capacity_blocks;
      int st = sb_kv_create(16, capacity_blocks, policy, device, &e->cache);
      if (st) throw Error(st, sb_last_error());
      e->d_pin_cnt = dmalloc<int32_t>(capacity_blocks);
      e->d_real_tag = dmalloc<int8_t>(capacity_blocks);
      e->d_scratch = dmalloc<int64_t>(16);
      SB_CUDA(cudaMemset(e->d_pin_cnt, 0, sizeof(int32_t) * capacity_blocks));
      SB_CUDA(cudaMemset(e->d_real_tag, 0xff, capacity_blocks));
      const int64_t elems = capacity_blocks * n_kv_heads * 16 * head_dim;
      for (int l = 0; l < n_layers; ++l) {
        e->k_pools.push_back(dmalloc<__nv_bfloat16>(elems));
        e->v_pools.push_back(dmalloc<__nv_bfloat16>(elems));
        // seeded KV for pages never prefilled here (the partial prefill of a
        // model-backed batch overwrites the pages it computes)
        st = sb_fill_random_bf16(e->k_pools.back(), elems, seed * 131 + 2 * l, 1.f, nullptr);
        if (!st) st = sb_fill_random_bf16(e->v_pools.back(), elems, seed * 131 + 2 * l + 1, 1.f, nullptr);
        if (st) throw Error(st, sb_last_error());
      }
      SB_CUDA(cudaDeviceSynchronize());
    } catch (...) {
      delete e;
      throw;
    }
    *out = e;
    return int(SB_OK);
  });
}

void sb_engine_destroy(sb_engine* e) { delete e; }
sb_kv_cache* sb_engine_cache(sb_engine* e) { return e->cache; }
void* sb_engine_k_pool(sb_engine* e, int32_t layer) { return e->k_pools.at(layer); }
void* sb_engine_v_pool(sb_engine* e, int32_t layer) { return e->v_pools.at(layer); }

int sb_engine_submit_call(sb_engine* e, const uint64_t* tokens, int64_t n, const sb_tag_range* tags, int64_t n_tags,
                          int64_t decode_length, int64_t now, int32_t* call) {
  return guard([&] {
    *call = submit(e, tokens, n, tags, n_tags, now, false, decode_length);
    return int(SB_OK);
  });
}

int sb_engine_submit_partial(sb_engine* e, const uint64_t* tokens, int64_t n, const sb_tag_range* tags,
                             int64_t n_tags, int64_t now, int32_t* handle) {
  return guard([&] {
    *handle = submit(e, tokens, n, tags, n_tags, now, true, 0);
    return int(SB_OK);
  });
}

int sb_engine_prefill_done(sb_engine* e, int32_t call, int64_t now, int32_t* outcome) {
  return guard([&] {
    Call& c = find_call(e, call, SB_ERR_UNKNOWN_CALL);
    if (c.state != CS_QUEUED && c.state != CS_PREFILLING)
      throw Error(SB_ERR_INVALID_STATE, "prefill_done: call is not prefilling");
    SB_CUDA(cudaSetDevice(e->device));
    const int oc = complete(e, c, now);
    if (outcome) *outcome = oc;
    return int(SB_OK);
  });
}

int sb_engine_extend(sb_engine* e, int32_t handle, const uint64_t* suffix, int64_t n, const sb_tag_range* tags,
                     int64_t n_tags, int64_t decode_length, int64_t now, int32_t* completed) {
  return guard([&] {
    auto it = e->calls.find(handle);
    if (it == e->calls.end()) throw Error(SB_ERR_STALE_HANDLE, "unknown continuation handle");
    Call& c = it->second;
    if (!c.partial || c.ext) throw Error(SB_ERR_STALE_HANDLE, "continuation handle already consumed");
    if (c.state == CS_DONE || c.state == CS_ABORTED || c.state == CS_DECODING)
      throw Error(SB_ERR_STALE_HANDLE, "continuation no longer extendable");
    if (decode_length < 1) throw Error(SB_ERR_INVALID_STATE, "extend_prefill: decode_length must be >= 1");
    if (!tags_cover_host(tags, n_tags, n)) throw Error(SB_ERR_INVALID_STATE, "tag ranges must cover the suffix");
    SB_CUDA(cudaSetDevice(e->device));
    cudaStream_t st = pool_stream(e->cache);
    const int64_t p = static_cast<int64_t>(c.prompt.size());
    c.ext = true;
    c.decode_len = decode_length;
    c.prompt.insert(c.prompt.end(), suffix, suffix + n);
    for (int64_t i = 0; i < n_tags; ++i) c.tags.push_back(sb_tag_range{tags[i].begin + p, tags[i].end + p, tags[i].tag, 0});
    ensure_call_dev(c, p + n, static_cast<int64_t>(c.tags.size()));
    if (n) SB_CUDA(cudaMemcpyAsync(c.d_tok + p, suffix, sizeof(uint64_t) * n, cudaMemcpyHostToDevice, st));
    SB_CUDA(cudaMemcpyAsync(c.d_tags, c.tags.data(), sizeof(sb_tag_range) * c.tags.size(), cudaMemcpyHostToDevice, st));
    hash_call(e, c, p + n, p / 16, st);  // the prefix's full blocks keep their hashes
    c.hashed_full = (p + n) / 16;
    int done = 0;
    if (c.state == CS_AWAITING) {
      if (n == 0) {  // nothing left to prefill (engine.cpp:212-215)
        complete(e, c, now);
        done = 1;
      } else {
        c.state = CS_PREFILLING;
      }
    }
    SB_CUDA(cudaStreamSynchronize(st));
    if (completed) *completed = done;
    return int(SB_OK);
  });
}

int sb_engine_abandon_partial(sb_engine* e, int32_t handle) {
  return guard([&] {
    auto it = e->calls.find(handle);
    if (it == e->calls.end()) throw Error(SB_ERR_STALE_HANDLE, "unknown continuation handle");
    Call& c = it->second;
    if (!c.partial || c.ext || c.state == CS_DONE || c.state == CS_ABORTED)
      throw Error(SB_ERR_STALE_HANDLE, "continuation handle no longer abandonable");
    SB_CUDA(cudaSetDevice(e->device));
    run_one(e, c, call_op(c, PK_ABANDON, 0, 0), 0);
    c.state = CS_ABORTED;
    return int(SB_OK);
  });
}

int sb_engine_finish(sb_engine* e, int32_t call, const uint64_t* response, int64_t n_response, int64_t now) {
  return guard([&] {
    Call& c = find_call(e, call, SB_ERR_UNKNOWN_CALL);
    if (c.state != CS_DECODING) throw Error(SB_ERR_INVALID_STATE, "finish: call is not decoding");
    SB_CUDA(cudaSetDevice(e->device));
    cudaStream_t st = pool_stream(e->cache);
    const int64_t p = static_cast<int64_t>(c.prompt.size());
    const int64_t nt = static_cast<int64_t>(c.tags.size());
    ensure_call_dev(c, p + n_response, nt + 1);
    if (n_response)
      SB_CUDA(cudaMemcpyAsync(c.d_tok + p, response, sizeof(uint64_t) * n_response, cudaMemcpyHostToDevice, st));
    const sb_tag_range resp{p, p + n_response, SB_TAG_RESPONSE, 0};
    SB_CUDA(cudaMemcpyAsync(c.d_tags + nt, &resp, sizeof(resp), cudaMemcpyHostToDevice, st));
    hash_call(e, c, p + n_response, p / 16, st);
    run_one(e, c, call_op(c, PK_FINISH, p + n_response, nt + 1), now);
    c.state = CS_DONE;
    return int(SB_OK);
  });
}

int sb_engine_call_info(sb_engine* e, int32_t call, int32_t* state, int64_t* cached_prefix, int64_t* prompt_tokens,
                        int32_t* n_chain, int32_t* n_pinned) {
  return guard([&] {
    Call& c = find_call(e, call, SB_ERR_UNKNOWN_CALL);
    if (state) *state = c.state;
    if (cached_prefix) *cached_prefix = c.cached;
    if (prompt_tokens) *prompt_tokens = static_cast<int64_t>(c.prompt.size());
    if (n_chain) *n_chain = c.n_chain;
    if (n_pinned) *n_pinned = c.n_pinned;
    return int(SB_OK);
  });
}

int sb_engine_call_blocks(sb_engine* e, int32_t call, int32_t which, int32_t* out, int64_t cap, int64_t* n_out) {
  return guard([&] {
    Call& c = find_call(e, call, SB_ERR_UNKNOWN_CALL);
    const std::vector<int32_t>& v = which ? c.pinned : c.chain;
    *n_out = static_cast<int64_t>(v.size());
    for (int64_t i = 0; i < std::min<int64_t>(cap, *n_out); ++i) out[i] = v[static_cast<size_t>(i)];
    return int(SB_OK);
  });
}

int sb_engine_partial_blocks(sb_engine* e, int32_t handle, int32_t* out, int64_t cap, int64_t* n_out) {
  return sb_engine_call_blocks(e, handle, 0, out, cap, n_out);
}

int sb_engine_partial_cached(sb_engine* e, int32_t handle, int64_t* cached_tokens) {
  return sb_engine_call_info(e, handle, nullptr, cached_tokens, nullptr, nullptr, nullptr);
}

// The partial prefill compute of pinned partials: tokens [cached, P) of each
// prefix run through the model, attending to [0, P) through the call's pinned
// chain (the pages allocated when the prefix was admitted).
int sb_engine_prefill_partials(sb_engine* e, sb_model* m, const int32_t* handles, int32_t n, void* stream) {
  return guard([&] {
    SB_CUDA(cudaSetDevice(e->device));
    int32_t nl = 0, hq = 0, hkv = 0;
    sb_model_shape(m, &nl, &hq, &hkv);
    if (nl != e->n_layers || hq != e->hq || hkv != e->hkv)
      throw Error(SB_ERR_INVALID, "model shape differs from the engine's KV shape");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::vector<int64_t> pre, suf;
    std::vector<int32_t> qo{0}, kl, table;
    std::vector<uint64_t> toks;
    int32_t max_blocks = 1, max_q = 0;
    for (int i = 0; i < n; ++i) {
      Call& c = find_call(e, handles[i], SB_ERR_STALE_HANDLE);
      if (c.state != CS_AWAITING) throw Error(SB_ERR_INVALID_STATE, "prefill_partials: partial not pinned");
      max_blocks = std::max<int32_t>(max_blocks, c.n_chain);
    }
    for (int i = 0; i < n; ++i) {
      const Call& c = e->calls.find(handles[i])->second;
      const int64_t P = static_cast<int64_t>(c.prompt.size()), H = std::min(c.cached, P);
      pre.push_back(H);
      suf.push_back(P - H);
      toks.insert(toks.end(), c.prompt.begin() + H, c.prompt.end());
      qo.push_back(qo.back() + static_cast<int32_t>(P - H));
      kl.push_back(static_cast<int32_t>(P));
      max_q = std::max<int32_t>(max_q, static_cast<int32_t>(P - H));
      for (int32_t j = 0; j < max_blocks; ++j) table.push_back(j < c.n_chain ? c.chain[static_cast<size_t>(j)] : -1);
    }
    const int64_t T = qo.back();
    if (T == 0) return int(SB_OK);
    ModelWorkspace* mw = model_workspace_create(m, pre, suf);
    uint64_t* d_tok = upload(toks);
    int32_t *d_qo = upload(qo), *d_kl = upload(kl), *d_tb = upload(table), *d_work = nullptr;
    int32_t n_work = 0;
    auto cleanup = [&] {
      model_workspace_destroy(mw);
      for (void* p : {static_cast<void*>(d_tok), static_cast<void*>(d_qo), static_cast<void*>(d_kl),
                      static_cast<void*>(d_tb), static_cast<void*>(d_work)})
        if (p) cudaFree(p);
    };
    try {
      const int tpt = 128 / (e->hq / e->hkv);
      int64_t cap_items = 0;
      for (int i = 0; i < n; ++i) cap_items += (suf[static_cast<size_t>(i)] + 2 * tpt - 1) / (2 * tpt) * e->hkv;
      std::vector<int32_t> work(static_cast<size_t>(2 * cap_items + 2));
      int stt = sb_attention_work_list(qo.data(), kl.data(), n, e->hq, e->hkv, work.data(),
                                       static_cast<int32_t>(cap_items + 1), &n_work);
      if (stt) throw Error(stt, sb_last_error());
      work.resize(static_cast<size_t>(2 * n_work));
      d_work = upload(work);
      const ModelIO io = model_io(mw);
      const float scale = 1.f / std::sqrt(static_cast<float>(e->hd));
      model_embed(m, mw, d_tok, st);
      for (int l = 0; l < e->n_layers; ++l) {
        model_layer_pre(m, mw, l, e->k_pools[l], e->v_pools[l], d_qo, d_kl, d_tb, n, max_blocks, st);
        stt = sb_continuation_attention(io.q, e->k_pools[l], e->v_pools[l], io.a, d_qo, d_kl, d_tb, n, max_blocks,
                                        max_q, static_cast<int32_t>(T), e->hq, e->hkv, e->hd, 16, e->cap, scale,
                                        d_work, n_work, stream);
        if (stt) throw Error(stt, sb_last_error());
        model_layer_post(m, mw, l, st);
      }
      SB_CUDA(cudaStreamSynchronize(st));
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
    return int(SB_OK);
  });
}

}  // extern "C"

// ===================================================================== step
// A batch of continuations run through the whole engine-side lifecycle per
// step: admission lookups of the tool-independent prefixes, pin_partial,
// extend with the tool outputs, complete_prefill, KV append + attention over
// the pages (or the full dense layers), finish_decode with one response
// token.  Slot s keeps its device buffers across steps; each step is a new
// set of calls over them.
struct sb_batch {
  sb_engine* eng = nullptr;
  int32_t n = 0;
  std::vector<int64_t> prefix_len, suffix_len, full_len, tok_off_h, blk_off_h, n_prefix_tags;
  int64_t total_q = 0, total_blocks = 0, total_tokens = 0, total_blk_cap = 0;
  int32_t max_blocks = 0, max_q = 0;
  // slot buffers: tokens (prefix + suffix + response), hashes, ids / chain / pinned, tags
  uint64_t *tokens = nullptr, *hashes = nullptr, *suffix = nullptr, *keys = nullptr;
  int32_t *ids = nullptr, *chain = nullptr, *pinned = nullptr;
  sb_tag_range* tags = nullptr;
  std::vector<int64_t> tag_off_h;
  int64_t *suffix_off = nullptr, *slot_off = nullptr, *resp_pos = nullptr, *chain_off = nullptr, *hits = nullptr;
  int64_t *seg_pre = nullptr, *seg_sfx = nullptr, *seg_resp = nullptr;  // hashing segments
  int64_t *blk_pre = nullptr, *blk_sfx = nullptr, *blk_resp = nullptr;
  uint64_t *par_sfx = nullptr, *par_resp = nullptr;
  int32_t *n_blocks = nullptr, *table = nullptr, *q_off = nullptr, *kv_len = nullptr, *work = nullptr;
  int32_t n_work = 0;
  std::vector<ProgOp> pin_ops, complete_ops, finish_ops, lookup_ops;
  std::vector<ProgRes> res;
  std::vector<int32_t> pin_outcome, complete_status;
  __nv_bfloat16 *q = nullptr, *k_new = nullptr, *v_new = nullptr, *out = nullptr;
  std::vector<cudaEvent_t> ev0, ev1;
  cudaEvent_t evp[6] = {};  // pool phases of a timed run: [0,1) submit+pin, [2,3) extend+complete, [4,5) finish
  // Prefix hashing of the NEXT step's calls runs on a side stream while this
  // step's attention runs (the tool-independent prefix is known before the
  // tool returns, paper section 4.2): two hash buffers, the next step's
  // prefix blocks hashed into the one this step does not use.
  uint64_t* hbuf[2] = {nullptr, nullptr};
  int hsel = 0;
  bool hready[2] = {false, false};
  cudaStream_t side = nullptr;
  cudaEvent_t ev_side_in = nullptr, ev_side_out[2] = {nullptr, nullptr};
  double attn_flops = 0;
  sb_model* model = nullptr;
  ModelWorkspace* mw = nullptr;
  ~sb_batch() {
    cudaSetDevice(eng->device);
    for (auto e : evp)
      if (e) cudaEventDestroy(e);
    for (auto e : {ev_side_in, ev_side_out[0], ev_side_out[1]})
      if (e) cudaEventDestroy(e);
    if (side) cudaStreamDestroy(side);
    for (auto* h : hbuf)  // (hashes aliases one of them)
      if (h) cudaFree(h);
    hashes = nullptr;
    model_workspace_destroy(mw);
    void* ptrs[] = {tokens, hashes, suffix, keys, ids, chain, pinned, tags, suffix_off, slot_off, resp_pos, chain_off, hits,
                    seg_pre, seg_sfx, seg_resp, blk_pre, blk_sfx, blk_resp, par_sfx, par_resp, n_blocks, table, q_off,
                    kv_len, work, q, k_new, v_new, out};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    for (auto e : ev0) cudaEventDestroy(e);
    for (auto e : ev1) cudaEventDestroy(e);
  }
};

namespace {
// parent hash of a hashing segment that starts at (absolute) block from[s]
// of slot s, whose blocks start at base[s]
__global__ void k_seg_parents(const uint64_t* hashes, const int64_t* base, const int64_t* from, int n,
                              uint64_t* parent) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < n) parent[s] = from[s] > base[s] ? hashes[from[s] - 1] : kRootHash;
}
}  // namespace

extern "C" {

int sb_batch_create(sb_engine* e, int32_t n, const uint64_t* prefix_tokens, const int64_t* prefix_off,
                    const sb_tag_range* prefix_tags, const int64_t* tag_off, const int64_t* suffix_lens,
                    const uint64_t* stream_keys, sb_batch** out) {
  return guard([&] {
    if (n <= 0) throw Error(SB_ERR_INVALID, "empty batch");
    SB_CUDA(cudaSetDevice(e->device));
    auto* b = new sb_batch();
    try {
      b->eng = e;
      b->n = n;
      std::vector<uint64_t> toks;
      std::vector<sb_tag_range> tags;
      std::vector<int64_t> suffix_off{0}, slot_off, resp_pos, chain_off, seg_pre, seg_sfx, seg_resp, blk_pre, blk_sfx,
          blk_resp;
      b->tok_off_h = {0};
      b->blk_off_h = {0};
      b->tag_off_h = {0};
      for (int i = 0; i < n; ++i) {
        const int64_t pl = prefix_off[i + 1] - prefix_off[i], sl = suffix_lens[i];
        if (pl <= 0) throw Error(SB_ERR_INVALID_STATE, "submit_partial_prefill: prefix must be non-empty");
        if (sl <= 0) throw Error(SB_ERR_INVALID, "suffix must be non-empty");
        const int64_t nt = tag_off[i + 1] - tag_off[i];
        if (!tags_cover_host(prefix_tags + tag_off[i], nt, pl))
          throw Error(SB_ERR_INVALID_STATE, "tag ranges must cover the prefix");
        const int64_t cap = pl + sl + 1;  // + one response token
        const int64_t base = b->tok_off_h.back(), bb = b->blk_off_h.back();
        b->prefix_len.push_back(pl);
        b->suffix_len.push_back(sl);
        b->full_len.push_back(pl + sl);
        b->n_prefix_tags.push_back(nt);
        toks.insert(toks.end(), prefix_tokens + prefix_off[i], prefix_tokens + prefix_off[i + 1]);
        toks.resize(static_cast<size_t>(base + cap), 0);
        slot_off.push_back(base + pl);
        resp_pos.push_back(base + pl + sl);
        chain_off.push_back(bb);
        for (int64_t k = 0; k < nt; ++k) tags.push_back(prefix_tags[tag_off[i] + k]);
        tags.push_back(sb_tag_range{pl, pl + sl, SB_TAG_TOOL_OUTPUT, 0});
        tags.push_back(sb_tag_range{pl + sl, pl + sl + 1, SB_TAG_RESPONSE, 0});
        b->tag_off_h.push_back(static_cast<int64_t>(tags.size()));
        // hashing segments: the prefix from the root; the suffix from the
        // prefix's last full block; the response from the prompt's last full block
        seg_pre.push_back(base);
        seg_pre.push_back(base + pl);
        blk_pre.push_back(bb);
        seg_sfx.push_back(base + 16 * (pl / 16));
        seg_sfx.push_back(base + pl + sl);
        blk_sfx.push_back(bb + pl / 16);
        seg_resp.push_back(base + 16 * ((pl + sl) / 16));
        seg_resp.push_back(base + pl + sl + 1);
        blk_resp.push_back(bb + (pl + sl) / 16);
        suffix_off.push_back(suffix_off.back() + sl);
        b->tok_off_h.push_back(base + cap);
        b->blk_off_h.push_back(bb + (cap + 15) / 16);
        b->max_blocks = std::max<int32_t>(b->max_blocks, static_cast<int32_t>((pl + sl + 15) / 16));
        b->max_q = std::max<int32_t>(b->max_q, static_cast<int32_t>(sl));
        const double keys = static_cast<double>(sl) * pl + static_cast<double>(sl) * (sl + 1) / 2;
        b->attn_flops += 4.0 * e->hd * e->hq * keys;
      }
      b->total_tokens = 0;
      for (int i = 0; i < n; ++i) b->total_tokens += b->full_len[i];
      b->total_blk_cap = b->blk_off_h.back();
      b->total_q = suffix_off.back();
      b->tokens = upload(toks);
      b->tags = upload(tags);
      b->hashes = dmalloc<uint64_t>(b->total_blk_cap);
      b->hbuf[0] = b->hashes;
      b->hbuf[1] = dmalloc<uint64_t>(b->total_blk_cap);
      SB_CUDA(cudaStreamCreateWithFlags(&b->side, cudaStreamNonBlocking));
      SB_CUDA(cudaEventCreateWithFlags(&b->ev_side_in, cudaEventDisableTiming));
      for (auto& ev : b->ev_side_out) SB_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      b->ids = dmalloc<int32_t>(b->total_blk_cap);
      b->chain = dmalloc<int32_t>(b->total_blk_cap);
      b->pinned = dmalloc<int32_t>(b->total_blk_cap);
      b->suffix = dmalloc<uint64_t>(b->total_q);
      b->suffix_off = upload(suffix_off);
      b->slot_off = upload(slot_off);
      b->resp_pos = upload(resp_pos);
      b->chain_off = upload(chain_off);
      b->seg_pre = upload(seg_pre);
      b->seg_sfx = upload(seg_sfx);
      b->seg_resp = upload(seg_resp);
      b->blk_pre = upload(blk_pre);
      b->blk_sfx = upload(blk_sfx);
      b->blk_resp = upload(blk_resp);
      b->par_sfx = dmalloc<uint64_t>(n);
      b->par_resp = dmalloc<uint64_t>(n);
      b->hits = dmalloc<int64_t>(n);
      std::vector<uint64_t> keys(stream_keys ? stream_keys : nullptr, stream_keys ? stream_keys + n : nullptr);
      if (!stream_keys)
        for (int i = 0; i < n; ++i) keys.push_back(hash_combine(0x5eedull, static_cast<uint64_t>(i)));
      b->keys = upload(keys);
      std::vector<int32_t> nb, qo{0}, kl;
      for (int i = 0; i < n; ++i) {
        nb.push_back(static_cast<int32_t>((b->full_len[i] + 15) / 16));
        qo.push_back(qo.back() + static_cast<int32_t>(b->suffix_len[i]));
        kl.push_back(static_cast<int32_t>(b->full_len[i]));
      }
      b->total_blocks = std::accumulate(nb.begin(), nb.end(), int64_t(0));
      b->n_blocks = upload(nb);
      b->table = dmalloc<int32_t>(static_cast<size_t>(n) * b->max_blocks);
      b->q_off = upload(qo);
      b->kv_len = upload(kl);
      b->q = dmalloc<__nv_bfloat16>(static_cast<size_t>(b->total_q) * e->hq * e->hd);
      b->out = dmalloc<__nv_bfloat16>(static_cast<size_t>(b->total_q) * e->hq * e->hd);
      b->k_new = dmalloc<__nv_bfloat16>(static_cast<size_t>(b->total_q) * e->hkv * e->hd);
      b->v_new = dmalloc<__nv_bfloat16>(static_cast<size_t>(b->total_q) * e->hkv * e->hd);
      {  // seeded stand-ins for the projection outputs (attention-path mode, no model attached)
        const int64_t nq = b->total_q * e->hq * e->hd, nkv = b->total_q * e->hkv * e->hd;
        int st = sb_fill_random_bf16(b->q, nq, 0x51ull, 1.f, nullptr);
        if (!st) st = sb_fill_random_bf16(b->k_new, nkv, 0x52ull, 1.f, nullptr);
        if (!st) st = sb_fill_random_bf16(b->v_new, nkv, 0x53ull, 1.f, nullptr);
        if (st) throw Error(st, sb_last_error());
      }
      const int tpt = 128 / (e->hq / e->hkv);
      int64_t cap_items = 0;
      for (int i = 0; i < n; ++i) cap_items += (b->suffix_len[i] + 2 * tpt - 1) / (2 * tpt) * e->hkv;
      std::vector<int32_t> work(static_cast<size_t>(2 * cap_items + 2));
      int st = sb_attention_work_list(qo.data(), kl.data(), n, e->hq, e->hkv, work.data(),
                                      static_cast<int32_t>(cap_items + 1), &b->n_work);
      if (st) throw Error(st, sb_last_error());
      work.resize(static_cast<size_t>(2 * b->n_work));
      b->work = upload(work);
      // op descriptors (device pointers fixed per slot)
      for (int i = 0; i < n; ++i) {
        const int64_t bo = b->blk_off_h[static_cast<size_t>(i)], to = b->tok_off_h[static_cast<size_t>(i)];
        const int64_t tg = b->tag_off_h[static_cast<size_t>(i)];
        ProgOp o{};
        o.tokens = b->tokens + to;
        o.hashes = b->hashes + bo;
        o.ids = b->ids + bo;
        o.chain = b->chain + bo;
        o.pinned = b->pinned + bo;
        o.ins_tags = b->tags + tg;
        o.real_tags = b->tags + tg;
        o.n_real_tags = static_cast<int32_t>(b->n_prefix_tags[i]);
        ProgOp l = o, p = o, c = o, f = o;
        l.n = b->prefix_len[i];
        p.kind = PK_PIN;
        p.n = b->prefix_len[i];
        p.n_ins_tags = 1;
        c.kind = PK_COMPLETE;
        c.n = b->full_len[i];
        c.n_ins_tags = static_cast<int32_t>(b->n_prefix_tags[i] + 1);
        f.kind = PK_FINISH;
        f.n = b->full_len[i] + 1;
        f.n_ins_tags = static_cast<int32_t>(b->n_prefix_tags[i] + 2);
        b->lookup_ops.push_back(l);
        b->pin_ops.push_back(p);
        b->complete_ops.push_back(c);
        b->finish_ops.push_back(f);
      }
      b->res.resize(static_cast<size_t>(n));
      b->ev0.resize(e->n_layers);
      b->ev1.resize(e->n_layers);
      for (int l = 0; l < e->n_layers; ++l) {
        SB_CUDA(cudaEventCreate(&b->ev0[l]));
        SB_CUDA(cudaEventCreate(&b->ev1[l]));
      }
      for (auto& ev : b->evp) SB_CUDA(cudaEventCreate(&ev));
    } catch (...) {
      delete b;
      throw;
    }
    *out = b;
    return int(SB_OK);
  });
}

void sb_batch_destroy(sb_batch* b) { delete b; }

int sb_batch_stage_suffix(sb_batch* b, const uint64_t* tokens, int32_t on_device, void* stream) {
  return guard([&] {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    SB_CUDA(cudaMemcpyAsync(b->suffix, tokens, sizeof(uint64_t) * b->total_q,
                            on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    const int grid = static_cast<int>(std::min<int64_t>((b->total_q + 255) / 256, 148 * 8));
    k_scatter_suffix<<<std::max(grid, 1), 256, 0, st>>>(b->suffix, b->suffix_off, b->slot_off, b->n, b->tokens);
    SB_CHECK_LAUNCH();
    return int(SB_OK);
  });
}

// One step of the batch's lifecycle at virtual time `now` (all transitions of
// the step happen at `now`, in batch order per transition kind).
int sb_batch_run(sb_batch* b, int64_t now, uint64_t seed, int32_t time_attention, void* stream, int32_t* launches) {
  return guard([&] {
    (void)seed;
    sb_engine* e = b->eng;
    SB_CUDA(cudaSetDevice(e->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int n = b->n;
    int n_launch = 0;
    auto chk = [](int s) {
      if (s) throw Error(s, sb_last_error());
    };
    if (time_attention) SB_CUDA(cudaEventRecord(b->evp[0], st));
    // this step's hash buffer (the ops read their chain hashes from it)
    b->hashes = b->hbuf[b->hsel];
    for (auto* v : {&b->lookup_ops, &b->pin_ops, &b->complete_ops, &b->finish_ops})
      for (int i = 0; i < n; ++i) (*v)[i].hashes = b->hashes + b->blk_off_h[static_cast<size_t>(i)];
    // 1. submit_partial_prefill x n: prefix chain hashes (hashed ahead on the
    // side stream during the previous step when possible) + admission lookups (engine.cpp:170)
    if (b->hready[b->hsel]) {
      SB_CUDA(cudaStreamWaitEvent(st, b->ev_side_out[b->hsel], 0));
      b->hready[b->hsel] = false;
    } else {
      chk(sb_chain_hash_segments(b->tokens, b->seg_pre, b->blk_pre, nullptr, n, 16, b->hashes, st));
      n_launch += 1;
    }
    SB_CUDA(cudaEventRecord(b->ev_side_in, st));  // the other buffer's last readers (previous step) are done
    const uint64_t pool_l0 = pool_launches(e->cache);
    pool_lookup(e->cache, b->lookup_ops.data(), n, now, b->hits, st);
    // 2. the prefix prefill completes: pin_partial x n (program)
    for (auto& o : b->pin_ops) o.n_chain = o.n_pinned = 0;
    pool_run_ops(e->cache, b->pin_ops.data(), n, e->d_pin_cnt, e->d_real_tag, now, st, b->res.data());
    if (time_attention) SB_CUDA(cudaEventRecord(b->evp[1], st));
    b->pin_outcome.assign(static_cast<size_t>(n), 0);
    for (int i = 0; i < n; ++i) {
      b->pin_outcome[i] = b->res[i].outcome;
      b->complete_ops[i].n_chain = b->res[i].n_chain;
      b->complete_ops[i].n_pinned = b->res[i].n_pinned;
    }
    // 3. extend_prefill x n (suffix tokens staged by sb_batch_stage_suffix):
    //    incremental hashing of the suffix from the prefix's last full block
    if (time_attention) SB_CUDA(cudaEventRecord(b->evp[2], st));
    k_seg_parents<<<(n + 127) / 128, 128, 0, st>>>(b->hashes, b->chain_off, b->blk_sfx, n, b->par_sfx);
    chk(sb_chain_hash_segments(b->tokens, b->seg_sfx, b->blk_sfx, b->par_sfx, n, 16, b->hashes, st));
    n_launch += 2;
    // 4. complete_prefill x n (program)
    pool_run_ops(e->cache, b->complete_ops.data(), n, e->d_pin_cnt, e->d_real_tag, now, st, b->res.data());
    if (time_attention) SB_CUDA(cudaEventRecord(b->evp[3], st));
    b->complete_status.assign(static_cast<size_t>(n), 0);
    for (int i = 0; i < n; ++i) {
      b->complete_status[i] = b->res[i].status;
      b->finish_ops[i].n_chain = b->res[i].n_chain;
      if (b->res[i].n_chain != (b->full_len[i] + 15) / 16)  // the pool state is the reference's; the compute has no pages
        throw Error(SB_ERR_CACHE_FULL, "complete_prefill proceeded uncached (CacheFull): the pool is too small for "
                                       "this step's continuations");
    }
    // 5. pages = the chains; per layer KV append + attention (or the model)
    k_slot_table<<<std::max(1, static_cast<int>(std::min<int64_t>((int64_t(n) * b->max_blocks + 255) / 256, 1184))),
                   256, 0, st>>>(b->chain, b->chain_off, b->n_blocks, n, b->max_blocks, b->table);
    n_launch += 1;
    const float scale = 1.f / std::sqrt(static_cast<float>(e->hd));
    const int32_t* model_tok = nullptr;
    if (b->model) {
      const ModelIO io = model_io(b->mw);
      model_embed(b->model, b->mw, b->suffix, st);
      n_launch += 1;
      for (int l = 0; l < e->n_layers; ++l) {
        model_layer_pre(b->model, b->mw, l, e->k_pools[l], e->v_pools[l], b->q_off, b->kv_len, b->table, n,
                        b->max_blocks, st);
        if (time_attention) SB_CUDA(cudaEventRecord(b->ev0[l], st));
        chk(sb_continuation_attention(io.q, e->k_pools[l], e->v_pools[l], io.a, b->q_off, b->kv_len, b->table, n,
                                      b->max_blocks, b->max_q, static_cast<int32_t>(b->total_q), e->hq, e->hkv, e->hd,
                                      16, e->cap, scale, b->work, b->n_work, stream));
        if (time_attention) SB_CUDA(cudaEventRecord(b->ev1[l], st));
        model_layer_post(b->model, b->mw, l, st);
        n_launch += 5;  // rmsnorm, rope+scatter, attention, rmsnorm, swiglu (+ cuBLAS GEMMs)
      }
      model_head(b->model, b->mw, st);
      n_launch += 2;
      model_tok = io.next_tok;
    } else {
      for (int l = 0; l < e->n_layers; ++l) {
        chk(sb_kv_append(b->k_new, b->v_new, e->k_pools[l], e->v_pools[l], b->q_off, b->kv_len, b->table, n,
                         b->max_blocks, e->hkv, e->hd, 16, stream));
        if (time_attention) SB_CUDA(cudaEventRecord(b->ev0[l], st));
        chk(sb_continuation_attention(b->q, e->k_pools[l], e->v_pools[l], b->out, b->q_off, b->kv_len, b->table, n,
                                      b->max_blocks, b->max_q, static_cast<int32_t>(b->total_q), e->hq, e->hkv, e->hd,
                                      16, e->cap, scale, b->work, b->n_work, stream));
        if (time_attention) SB_CUDA(cudaEventRecord(b->ev1[l], st));
        n_launch += 2;
      }
    }
    // the next step's prefix hashes, overlapping this step's attention
    {
      const int nx = b->hsel ^ 1;
      SB_CUDA(cudaStreamWaitEvent(b->side, b->ev_side_in, 0));
      chk(sb_chain_hash_segments(b->tokens, b->seg_pre, b->blk_pre, nullptr, n, 16, b->hbuf[nx], b->side));
      SB_CUDA(cudaEventRecord(b->ev_side_out[nx], b->side));
      b->hready[nx] = true;
      n_launch += 1;
    }
    // 6. finish_decode x n with the first response token (program)
    if (time_attention) SB_CUDA(cudaEventRecord(b->evp[4], st));
    k_response_tokens<<<(n + 127) / 128, 128, 0, st>>>(model_tok, b->keys, b->resp_pos, n, b->tokens);
    k_seg_parents<<<(n + 127) / 128, 128, 0, st>>>(b->hashes, b->chain_off, b->blk_resp, n, b->par_resp);
    chk(sb_chain_hash_segments(b->tokens, b->seg_resp, b->blk_resp, b->par_resp, n, 16, b->hashes, st));
    n_launch += 3;
    pool_run_ops(e->cache, b->finish_ops.data(), n, e->d_pin_cnt, e->d_real_tag, now, st, b->res.data());
    if (time_attention) SB_CUDA(cudaEventRecord(b->evp[5], st));
    n_launch += static_cast<int>(pool_launches(e->cache) - pool_l0);  // lookups + op programs, counted by the pool
    b->hsel ^= 1;
    if (launches) *launches = n_launch;
    return int(SB_OK);
  });
}

// Pool-side phases of the last timed run (ms): submit + pin_partial,
// extend + complete_prefill, finish_decode (each including its host sync).
int sb_batch_pool_ms(sb_batch* b, float* out) {
  return guard([&] {
    for (int k = 0; k < 3; ++k) {
      SB_CUDA(cudaEventSynchronize(b->evp[2 * k + 1]));
      SB_CUDA(cudaEventElapsedTime(&out[k], b->evp[2 * k], b->evp[2 * k + 1]));
    }
    return int(SB_OK);
  });
}

int sb_batch_attention_ms(sb_batch* b, float* out) {
  return guard([&] {
    for (int l = 0; l < b->eng->n_layers; ++l) {
      SB_CUDA(cudaEventSynchronize(b->ev1[l]));
      SB_CUDA(cudaEventElapsedTime(&out[l], b->ev0[l], b->ev1[l]));
    }
    return int(SB_OK);
  });
}

// Admission-lookup hits of the last step (tokens per call), pin outcomes
// (ProgOutcome), complete_prefill statuses and the chains the continuation
// ran over (packed, ceil(full_len / 16) ids per call).
int sb_batch_results(sb_batch* b, int64_t* hits, int32_t* status, int32_t* block_ids, void* stream) {
  return guard([&] {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (hits) SB_CUDA(cudaMemcpyAsync(hits, b->hits, sizeof(int64_t) * b->n, cudaMemcpyDeviceToHost, st));
    if (block_ids) {
      int64_t o = 0;
      std::vector<int32_t> tab(static_cast<size_t>(b->n) * b->max_blocks);
      SB_CUDA(cudaMemcpyAsync(tab.data(), b->table, sizeof(int32_t) * tab.size(), cudaMemcpyDeviceToHost, st));
      SB_CUDA(cudaStreamSynchronize(st));
      for (int i = 0; i < b->n; ++i) {
        const int64_t nb = (b->full_len[i] + 15) / 16;
        for (int64_t j = 0; j < nb; ++j) block_ids[o++] = tab[static_cast<size_t>(i) * b->max_blocks + j];
      }
    }
    SB_CUDA(cudaStreamSynchronize(st));
    if (status)
      for (int i = 0; i < b->n; ++i) status[i] = i < static_cast<int>(b->complete_status.size()) ? b->complete_status[i] : 0;
    return int(SB_OK);
  });
}

int sb_batch_pin_outcomes(sb_batch* b, int32_t* outcomes) {
  return guard([&] {
    for (int i = 0; i < b->n; ++i) outcomes[i] = i < static_cast<int>(b->pin_outcome.size()) ? b->pin_outcome[i] : 0;
    return int(SB_OK);
  });
}

int sb_batch_copy_output(sb_batch* b, int64_t first_row, int64_t n_rows, void* host_dst, void* stream) {
  return guard([&] {
    if (first_row < 0 || first_row + n_rows > b->total_q) throw Error(SB_ERR_INVALID, "row range");
    const size_t row = static_cast<size_t>(b->eng->hq) * b->eng->hd;
    const __nv_bfloat16* src = b->model ? model_io(b->mw).a : b->out;
    SB_CUDA(cudaMemcpyAsync(host_dst, src + first_row * row, n_rows * row * sizeof(__nv_bfloat16),
                            cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream)));
    return int(SB_OK);
  });
}

int sb_batch_set_model(sb_batch* b, sb_model* m) {
  return guard([&] {
    SB_CUDA(cudaSetDevice(b->eng->device));
    model_workspace_destroy(b->mw);
    b->mw = nullptr;
    b->model = nullptr;
    if (!m) return int(SB_OK);
    int32_t nl = 0, hq = 0, hkv = 0;
    sb_model_shape(m, &nl, &hq, &hkv);
    if (nl != b->eng->n_layers || hq != b->eng->hq || hkv != b->eng->hkv)
      throw Error(SB_ERR_INVALID, "model shape differs from the engine's KV shape");
    b->mw = model_workspace_create(m, b->prefix_len, b->suffix_len);
    b->model = m;
    return int(SB_OK);
  });
}

int sb_batch_model_result(sb_batch* b, int32_t* next_tokens, float* logits, void* stream) {
  return guard([&] {
    if (!b->model) throw Error(SB_ERR_INVALID, "no model attached");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const ModelIO io = model_io(b->mw);
    if (next_tokens)
      SB_CUDA(cudaMemcpyAsync(next_tokens, io.next_tok, sizeof(int32_t) * b->n, cudaMemcpyDeviceToHost, st));
    if (logits) {
      int64_t vocab = 0;
      sb_model_vocab(b->model, &vocab);
      SB_CUDA(cudaMemcpyAsync(logits, io.logits, sizeof(float) * b->n * vocab, cudaMemcpyDeviceToHost, st));
    }
    SB_CUDA(cudaStreamSynchronize(st));
    return int(SB_OK);
  });
}

int sb_batch_dense_flops(const sb_batch* b, double* flops) {
  *flops = b->model ? model_flops(b->model, b->total_q) : 0.0;
  return SB_OK;
}

int sb_batch_info(const sb_batch* b, int64_t* total_q, int64_t* total_blocks, int64_t* prompt_tokens,
                  double* attention_flops, void** out_ptr) {
  if (total_q) *total_q = b->total_q;
  if (total_blocks) *total_blocks = b->total_blocks;
  if (prompt_tokens) *prompt_tokens = b->total_tokens;
  if (attention_flops) *attention_flops = b->attn_flops;
  if (out_ptr) *out_ptr = b->out;
  return SB_OK;
}

}  // extern "C"
