// engine.cu — host-side continuation engine (C++), the B200 counterpart of
// the reference engine's prompt-splitting path:
//   Engine::submit_partial_prefill + pin_partial  engine.cpp:153-182, 250-286
//   Engine::extend_prefill + complete_prefill     engine.cpp:184-223, 305-322
//   Engine::abandon_partial                       engine.cpp:234-248
// where the reference only charges a prefill cost (engine.cpp:35-39), this
// engine runs the computation: the partial prefill of a prefix's uncached
// tokens (sb_engine_prefill_partials, while the tool runs) and the
// continuation step: chain hashes -> admission lookup -> insert (hint-aware
// eviction) -> page table -> per layer {KV append, tcgen05 attention} (or the
// full dense layers with an attached model, csrc/model.cu) -> release, all
// stream-ordered on one stream.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <numeric>
#include <vector>

#include "common.h"
#include "hash.cuh"

namespace sb {

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

}  // namespace sb

using namespace sb;

struct PartialCall {
  std::vector<uint64_t> tokens;
  std::vector<sb_tag_range> tags;
  std::vector<int32_t> ids;
  int64_t cached = 0;  // prefix tokens already in the pool at submit (engine.cpp:170)
  bool live = true;
};

struct sb_engine {
  int32_t n_layers, hq, hkv, hd, device, policy;
  int64_t cap;
  sb_kv_cache* cache = nullptr;
  std::vector<__nv_bfloat16*> k_pools, v_pools;
  std::map<int32_t, PartialCall> partials;
  int32_t next_handle = 1;
  ~sb_engine() {
    cudaSetDevice(device);
    for (auto* p : k_pools) cudaFree(p);
    for (auto* p : v_pools) cudaFree(p);
    if (cache) sb_kv_destroy(cache);
  }
};

struct sb_batch {
  sb_engine* eng = nullptr;
  int32_t n = 0;
  std::vector<int64_t> prefix_len, suffix_len, full_len, seq_off_h, blk_off_h;
  int64_t total_blocks = 0, total_q = 0, total_tokens = 0;
  int32_t max_blocks = 0, max_q = 0;
  uint64_t* tokens = nullptr;  // packed prompts
  int64_t *seq_off = nullptr, *blk_off = nullptr, *tag_off = nullptr;
  sb_tag_range* tags = nullptr;
  uint64_t* hashes = nullptr;
  int32_t *ids = nullptr, *status = nullptr, *table = nullptr, *q_off = nullptr, *kv_len = nullptr, *work = nullptr;
  int32_t n_work = 0;
  int64_t* hits = nullptr;
  int64_t *suffix_off = nullptr, *slot_off = nullptr;
  // incremental hashing: prefix chain hashes gathered from the pinned blocks,
  // only the suffix segments folded (parent = last prefix block's hash)
  int32_t *pre_ids = nullptr, *last_pre = nullptr;
  int64_t *pre_pos = nullptr, *sfx_seq_off = nullptr, *sfx_blk_off = nullptr;
  int64_t n_pre = 0;
  uint64_t* parent0 = nullptr;
  uint64_t* suffix = nullptr;
  __nv_bfloat16 *q = nullptr, *k_new = nullptr, *v_new = nullptr, *out = nullptr;
  std::vector<cudaEvent_t> ev0, ev1;
  double attn_flops = 0;
  sb_model* model = nullptr;  // dense layers around the attention (optional)
  ModelWorkspace* mw = nullptr;
  ~sb_batch() {
    cudaSetDevice(eng->device);
    model_workspace_destroy(mw);
    void* ptrs[] = {tokens, seq_off, blk_off, tag_off, tags, hashes, ids, status, table, q_off, kv_len, work,
                    hits, suffix_off, slot_off, suffix, q, k_new, v_new, out, pre_ids, last_pre, pre_pos,
                    sfx_seq_off, sfx_blk_off, parent0};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    for (auto e : ev0) cudaEventDestroy(e);
    for (auto e : ev1) cudaEventDestroy(e);
  }
};

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
      const int64_t elems = capacity_blocks * n_kv_heads * 16 * head_dim;
      for (int l = 0; l < n_layers; ++l) {
        e->k_pools.push_back(dmalloc<__nv_bfloat16>(elems));
        e->v_pools.push_back(dmalloc<__nv_bfloat16>(elems));
        // seeded KV for pages never prefilled here (sb_engine_prefill_partials overwrites
        // the pages of the prefixes it computes)
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

int sb_engine_submit_partial(sb_engine* e, const uint64_t* tokens, int64_t n, const sb_tag_range* tags,
                             int64_t n_tags, int64_t now, int32_t* handle) {
  return guard([&] {
    if (n <= 0) throw Error(SB_ERR_INVALID, "submit_partial_prefill: prefix must be non-empty");
    PartialCall pc;
    pc.tokens.assign(tokens, tokens + n);
    pc.tags.assign(tags, tags + n_tags);
    pc.ids.resize(static_cast<size_t>((n + 15) / 16));
    // admission lookup (engine.cpp:170): the prefix tokens whose KV is already
    // cached; the partial prefill computes the rest (the insert below touches
    // the same blocks at the same time, so the pool state is unchanged by it)
    int st = sb_kv_lookup_prefix(e->cache, tokens, n, now, &pc.cached);
    if (st) return st;
    int64_t n_out = 0;
    st = sb_kv_insert(e->cache, tokens, n, tags, n_tags, now, pc.ids.data(), &n_out);
    if (st) return st;
    // pinned at the PARTIAL_PREFILL tier until extended or abandoned (engine.cpp:280-281)
    st = sb_kv_set_reuse_priority(e->cache, pc.ids.data(), n_out, 1, SB_TAG_PARTIAL_PREFILL);
    if (st) return st;
    *handle = e->next_handle++;
    e->partials.emplace(*handle, std::move(pc));
    return int(SB_OK);
  });
}

int sb_engine_abandon_partial(sb_engine* e, int32_t handle) {
  return guard([&] {
    auto it = e->partials.find(handle);
    if (it == e->partials.end() || !it->second.live) throw Error(SB_ERR_INVALID, "stale continuation handle");
    auto& ids = it->second.ids;
    int st = sb_kv_set_reuse_priority(e->cache, ids.data(), static_cast<int64_t>(ids.size()), 0, -1);
    if (!st) st = sb_kv_release(e->cache, ids.data(), static_cast<int64_t>(ids.size()));
    it->second.live = false;
    return st;
  });
}

int sb_engine_partial_blocks(sb_engine* e, int32_t handle, int32_t* out, int64_t cap, int64_t* n_out) {
  return guard([&] {
    auto it = e->partials.find(handle);
    if (it == e->partials.end()) throw Error(SB_ERR_INVALID, "unknown handle");
    const auto& ids = it->second.ids;
    *n_out = static_cast<int64_t>(ids.size());
    for (int64_t i = 0; i < std::min<int64_t>(cap, *n_out); ++i) out[i] = ids[i];
    return int(SB_OK);
  });
}

int sb_engine_prefill_partials(sb_engine* e, sb_model* m, const int32_t* handles, int32_t n, void* stream) {
  return guard([&] {
    SB_CUDA(cudaSetDevice(e->device));
    int32_t nl = 0, hq = 0, hkv = 0;
    sb_model_shape(m, &nl, &hq, &hkv);
    if (nl != e->n_layers || hq != e->hq || hkv != e->hkv)
      throw Error(SB_ERR_INVALID, "model shape differs from the engine's KV shape");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // per partial: tokens [cached, P) are computed, attending to [0, P)
    std::vector<int64_t> pre, suf;
    std::vector<int32_t> qo{0}, kl, table;
    std::vector<uint64_t> toks;
    int32_t max_blocks = 1, max_q = 0;
    for (int i = 0; i < n; ++i) {
      auto it = e->partials.find(handles[i]);
      if (it == e->partials.end() || !it->second.live) throw Error(SB_ERR_INVALID, "stale continuation handle");
      max_blocks = std::max<int32_t>(max_blocks, static_cast<int32_t>(it->second.ids.size()));
    }
    for (int i = 0; i < n; ++i) {
      const PartialCall& pc = e->partials.find(handles[i])->second;
      const int64_t P = static_cast<int64_t>(pc.tokens.size()), H = std::min(pc.cached, P);
      pre.push_back(H);
      suf.push_back(P - H);
      toks.insert(toks.end(), pc.tokens.begin() + H, pc.tokens.end());
      qo.push_back(qo.back() + static_cast<int32_t>(P - H));
      kl.push_back(static_cast<int32_t>(P));
      max_q = std::max<int32_t>(max_q, static_cast<int32_t>(P - H));
      for (int32_t j = 0; j < max_blocks; ++j)
        table.push_back(j < static_cast<int32_t>(pc.ids.size()) ? pc.ids[static_cast<size_t>(j)] : -1);
    }
    const int64_t T = qo.back();
    if (T == 0) return int(SB_OK);
    ModelWorkspace* mw = model_workspace_create(m, pre, suf);
    uint64_t* d_tok = upload(toks);
    int32_t *d_qo = upload(qo), *d_kl = upload(kl), *d_tb = upload(table), *d_work = nullptr;
    int32_t n_work = 0;
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
      model_workspace_destroy(mw);
      for (void* p : {static_cast<void*>(d_tok), static_cast<void*>(d_qo), static_cast<void*>(d_kl),
                      static_cast<void*>(d_tb), static_cast<void*>(d_work)})
        if (p) cudaFree(p);
      throw;
    }
    model_workspace_destroy(mw);
    for (void* p : {static_cast<void*>(d_tok), static_cast<void*>(d_qo), static_cast<void*>(d_kl),
                    static_cast<void*>(d_tb), static_cast<void*>(d_work)})
      if (p) cudaFree(p);
    return int(SB_OK);
  });
}

int sb_engine_partial_cached(sb_engine* e, int32_t handle, int64_t* cached_tokens) {
  return guard([&] {
    auto it = e->partials.find(handle);
    if (it == e->partials.end()) throw Error(SB_ERR_INVALID, "unknown handle");
    *cached_tokens = it->second.cached;
    return int(SB_OK);
  });
}

int sb_batch_create(sb_engine* e, const int32_t* handles, const int64_t* suffix_lens, int32_t n, sb_batch** out) {
  return guard([&] {
    if (n <= 0) throw Error(SB_ERR_INVALID, "empty batch");
    SB_CUDA(cudaSetDevice(e->device));
    auto* b = new sb_batch();
    try {
      b->eng = e;
      b->n = n;
      std::vector<uint64_t> toks;
      std::vector<sb_tag_range> tags;
      std::vector<int64_t> tag_off{0}, slot_off, suffix_off{0}, pre_pos, sfx_blk;
      std::vector<int32_t> pre_ids, last_pre;
      b->seq_off_h = {0};
      b->blk_off_h = {0};
      for (int i = 0; i < n; ++i) {
        auto it = e->partials.find(handles[i]);
        if (it == e->partials.end() || !it->second.live) throw Error(SB_ERR_INVALID, "stale continuation handle");
        const PartialCall& pc = it->second;
        const int64_t pl = static_cast<int64_t>(pc.tokens.size()), sl = suffix_lens[i];
        if (pl % 16) throw Error(SB_ERR_UNSUPPORTED, "tool-independent prefix must end on a 16-token block boundary");
        if (sl <= 0) throw Error(SB_ERR_INVALID, "suffix must be non-empty");
        for (int64_t k = 0; k < pl / 16; ++k) {
          pre_ids.push_back(pc.ids[static_cast<size_t>(k)]);
          pre_pos.push_back(b->blk_off_h.back() + k);
        }
        last_pre.push_back(pc.ids[static_cast<size_t>(pl / 16 - 1)]);
        sfx_blk.push_back(b->blk_off_h.back() + pl / 16);
        b->prefix_len.push_back(pl);
        b->suffix_len.push_back(sl);
        b->full_len.push_back(pl + sl);
        slot_off.push_back(static_cast<int64_t>(toks.size()) + pl);
        toks.insert(toks.end(), pc.tokens.begin(), pc.tokens.end());
        toks.resize(toks.size() + static_cast<size_t>(sl), 0);
        for (auto t : pc.tags) tags.push_back(t);
        tags.push_back(sb_tag_range{pl, pl + sl, SB_TAG_TOOL_OUTPUT, 0});
        tag_off.push_back(static_cast<int64_t>(tags.size()));
        b->seq_off_h.push_back(static_cast<int64_t>(toks.size()));
        b->blk_off_h.push_back(b->blk_off_h.back() + (pl + sl + 15) / 16);
        suffix_off.push_back(suffix_off.back() + sl);
        b->max_blocks = std::max<int32_t>(b->max_blocks, static_cast<int32_t>((pl + sl + 15) / 16));
        b->max_q = std::max<int32_t>(b->max_q, static_cast<int32_t>(sl));
        const double keys = static_cast<double>(sl) * pl + static_cast<double>(sl) * (sl + 1) / 2;
        b->attn_flops += 4.0 * e->hd * e->hq * keys;
      }
      b->total_tokens = static_cast<int64_t>(toks.size());
      b->total_blocks = b->blk_off_h.back();
      b->total_q = suffix_off.back();
      b->tokens = upload(toks);
      b->seq_off = upload(b->seq_off_h);
      b->blk_off = upload(b->blk_off_h);
      b->tag_off = upload(tag_off);
      b->tags = upload(tags);
      b->hashes = dmalloc<uint64_t>(b->total_blocks);
      b->ids = dmalloc<int32_t>(b->total_blocks);
      b->status = dmalloc<int32_t>(n);
      b->hits = dmalloc<int64_t>(n);
      b->table = dmalloc<int32_t>(static_cast<size_t>(n) * b->max_blocks);
      std::vector<int32_t> qo{0}, kl;
      for (int i = 0; i < n; ++i) {
        qo.push_back(qo.back() + static_cast<int32_t>(b->suffix_len[i]));
        kl.push_back(static_cast<int32_t>(b->full_len[i]));
      }
      b->q_off = upload(qo);
      b->kv_len = upload(kl);
      b->suffix_off = upload(suffix_off);
      b->slot_off = upload(slot_off);
      // suffix-only hashing: segment s = tokens[slot_off[s], seq_off[s+1]), its blocks from
      // blk_off[s] + prefix_blocks (sb_chain_hash_segments)
      std::vector<int64_t> so;
      for (int i = 0; i < n; ++i) {
        so.push_back(slot_off[static_cast<size_t>(i)]);
        so.push_back(b->seq_off_h[static_cast<size_t>(i) + 1]);
      }
      const std::vector<int64_t>& bo = sfx_blk;
      b->sfx_seq_off = upload(so);
      b->sfx_blk_off = upload(bo);
      b->pre_ids = upload(pre_ids);
      b->pre_pos = upload(pre_pos);
      b->last_pre = upload(last_pre);
      b->n_pre = static_cast<int64_t>(pre_ids.size());
      b->parent0 = dmalloc<uint64_t>(n);
      b->suffix = dmalloc<uint64_t>(b->total_q);
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
      // LPT-ordered attention work list
      const int tpt = 128 / (e->hq / e->hkv);
      int64_t cap_items = 0;
      for (int i = 0; i < n; ++i) cap_items += (b->suffix_len[i] + 2 * tpt - 1) / (2 * tpt) * e->hkv;
      std::vector<int32_t> work(static_cast<size_t>(2 * cap_items + 2));
      int st = sb_attention_work_list(qo.data(), kl.data(), n, e->hq, e->hkv, work.data(),
                                      static_cast<int32_t>(cap_items + 1), &b->n_work);
      if (st) throw Error(st, sb_last_error());
      work.resize(static_cast<size_t>(2 * b->n_work));
      b->work = upload(work);
      b->ev0.resize(e->n_layers);
      b->ev1.resize(e->n_layers);
      for (int l = 0; l < e->n_layers; ++l) {
        SB_CUDA(cudaEventCreate(&b->ev0[l]));
        SB_CUDA(cudaEventCreate(&b->ev1[l]));
      }
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

int sb_batch_run(sb_batch* b, int64_t now, uint64_t seed, int32_t time_attention, void* stream,
                 int32_t* launches) {
  return guard([&] {
    sb_engine* e = b->eng;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int n_launch = 0;
    auto chk = [](int s) {
      if (s) throw Error(s, sb_last_error());
    };
    // incremental hashing: the pinned prefix's chain hashes come from the pool,
    // only the suffix (tool output) tokens are folded, from the prefix's last hash
    chk(sb_kv_gather_chain_hashes(e->cache, b->pre_ids, b->pre_pos, b->n_pre, b->hashes, stream));
    chk(sb_kv_gather_chain_hashes(e->cache, b->last_pre, nullptr, b->n, b->parent0, stream));
    chk(sb_chain_hash_segments(b->tokens, b->sfx_seq_off, b->sfx_blk_off, b->parent0, b->n, 16, b->hashes, stream));
    n_launch += 3;
    chk(sb_kv_lookup_prefix_batch(e->cache, b->tokens, b->seq_off, b->blk_off, b->blk_off_h.data(), b->hashes, b->n,
                                  now, b->hits, stream));
    n_launch += 3;
    chk(sb_kv_insert_batch(e->cache, b->tokens, b->seq_off, b->tags, b->tag_off, b->blk_off, b->blk_off_h.data(),
                           b->hashes, b->n, now, b->ids, b->status, stream));
    n_launch += 5 * b->n;
    chk(sb_build_block_table(b->ids, b->blk_off, b->n, b->max_blocks, b->table, stream));
    n_launch += 1;
    const float scale = 1.f / std::sqrt(static_cast<float>(e->hd));
    const int64_t nq = b->total_q * e->hq * e->hd, nkv = b->total_q * e->hkv * e->hd;
    if (b->model) {  // the real Llama-shaped layers (model.cu) around the attention
      const ModelIO io = model_io(b->mw);
      model_embed(b->model, b->mw, b->suffix, st);
      n_launch += 1;
      for (int l = 0; l < e->n_layers; ++l) {
        model_layer_pre(b->model, b->mw, l, e->k_pools[l], e->v_pools[l], b->q_off, b->kv_len, b->table, b->n,
                        b->max_blocks, st);
        if (time_attention) SB_CUDA(cudaEventRecord(b->ev0[l], st));
        chk(sb_continuation_attention(io.q, e->k_pools[l], e->v_pools[l], io.a, b->q_off, b->kv_len, b->table, b->n,
                                      b->max_blocks, b->max_q, static_cast<int32_t>(b->total_q), e->hq, e->hkv, e->hd,
                                      16, e->cap, scale, b->work, b->n_work, stream));
        if (time_attention) SB_CUDA(cudaEventRecord(b->ev1[l], st));
        model_layer_post(b->model, b->mw, l, st);
        n_launch += 5;  // rmsnorm, rope+scatter, attention, rmsnorm, swiglu (+ cuBLAS GEMMs)
      }
      model_head(b->model, b->mw, st);
      n_launch += 2;
      chk(sb_kv_release_batch(e->cache, b->ids, b->total_blocks, nullptr, stream));
      n_launch += 3;
      if (launches) *launches = n_launch;
      return int(SB_OK);
    }
    (void)seed;
    (void)nq;
    (void)nkv;
    for (int l = 0; l < e->n_layers; ++l) {
      // q / k / v: the seeded stand-ins of the batch (the dense layers are sb_batch_set_model)
      chk(sb_kv_append(b->k_new, b->v_new, e->k_pools[l], e->v_pools[l], b->q_off, b->kv_len, b->table, b->n,
                       b->max_blocks, e->hkv, e->hd, 16, stream));
      if (time_attention) SB_CUDA(cudaEventRecord(b->ev0[l], st));
      chk(sb_continuation_attention(b->q, e->k_pools[l], e->v_pools[l], b->out, b->q_off, b->kv_len, b->table, b->n,
                                    b->max_blocks, b->max_q, static_cast<int32_t>(b->total_q), e->hq, e->hkv, e->hd, 16,
                                    e->cap, scale, b->work, b->n_work, stream));
      if (time_attention) SB_CUDA(cudaEventRecord(b->ev1[l], st));
      n_launch += 2;
    }
    chk(sb_kv_release_batch(e->cache, b->ids, b->total_blocks, nullptr, stream));
    n_launch += 3;
    if (launches) *launches = n_launch;
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

int sb_batch_results(sb_batch* b, int64_t* hits, int32_t* status, int32_t* block_ids, void* stream) {
  return guard([&] {
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (hits) SB_CUDA(cudaMemcpyAsync(hits, b->hits, sizeof(int64_t) * b->n, cudaMemcpyDeviceToHost, st));
    if (status) SB_CUDA(cudaMemcpyAsync(status, b->status, sizeof(int32_t) * b->n, cudaMemcpyDeviceToHost, st));
    if (block_ids)
      SB_CUDA(cudaMemcpyAsync(block_ids, b->ids, sizeof(int32_t) * b->total_blocks, cudaMemcpyDeviceToHost, st));
    SB_CUDA(cudaStreamSynchronize(st));
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
