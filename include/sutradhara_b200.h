/*
 * sutradhara_b200.h — C-ABI of the B200-native engine-side hot path of
 * Sutradhara (arXiv 2601.12967): paged-KV block pool + block table, prefix
 * block hashing and prefix match, hint-aware (tiered) eviction scoring, and
 * the continuation-prefill attention over the paged KV pool.
 *
 * Plain C types only (no torch types).  Device pointers are raw CUDA device
 * addresses; `stream` is a cudaStream_t passed as void* (0 = legacy stream).
 *
 * Each entry point names the reference interface it replaces
 * (paths relative to the reference tree proj/).  Status codes mirror the
 * reference's exception hierarchy (include/agentsim/common.hpp:72-115) so a
 * binding can re-raise the same exception type.
 */
#ifndef SUTRADHARA_B200_H_
#define SUTRADHARA_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mirror common.hpp exception classes) ---------------- */
enum {
  SB_OK = 0,
  SB_ERR_CACHE_FULL = 1,       /* CacheFull        common.hpp:77  */
  SB_ERR_UNKNOWN_BLOCK = 2,    /* UnknownBlock     common.hpp:82  */
  SB_ERR_ZERO_REF_RELEASE = 3, /* ZeroRefRelease   common.hpp:87  */
  SB_ERR_CACHE = 4,            /* CacheError       common.hpp:72  */
  SB_ERR_CONFIG = 5,           /* ConfigError      common.hpp:25  */
  SB_ERR_CUDA = 6,             /* CUDA runtime / launch failure   */
  SB_ERR_INVALID = 7,          /* bad argument to this C-ABI      */
  SB_ERR_UNSUPPORTED = 8,      /* shape/config outside the kernels' range */
  SB_ERR_STALE_HANDLE = 9,     /* StaleHandle      common.hpp:102 */
  SB_ERR_INVALID_STATE = 10,   /* InvalidState     common.hpp:107 */
  SB_ERR_UNKNOWN_CALL = 11     /* UnknownCall      common.hpp:112 */
};

/* ---- semantic tags (order == agentsim::KvTag, kv_cache.hpp:21-28) ---- */
enum {
  SB_TAG_RESPONSE = 0,
  SB_TAG_TOOL_OUTPUT = 1,
  SB_TAG_USER_QUERY = 2,
  SB_TAG_SYSTEM_PROMPT = 3,
  SB_TAG_PARTIAL_PREFILL = 4,
  SB_TAG_HISTORY = 5
};

/* ---- eviction policy (agentsim::EvictionPolicy, kv_cache.hpp:36) ------ */
enum { SB_POLICY_LRU = 0, SB_POLICY_TIERED = 1 };

/* Half-open token range with a tag (agentsim::TagRange, kv_cache.hpp:45). */
typedef struct sb_tag_range {
  int64_t begin;
  int64_t end;
  int32_t tag;
  int32_t _pad;
} sb_tag_range;

/* Read-back of one block's metadata (agentsim::KvBlock, kv_cache.hpp:51). */
typedef struct sb_block_info {
  int32_t block_id;
  int32_t tag;
  int32_t tier;
  int32_t ref_count;
  int64_t last_used;
  uint64_t chain_hash;
  uint64_t parent_hash;
  int32_t pinned;
  int32_t n_tokens;
} sb_block_info;

typedef struct sb_kv_cache sb_kv_cache; /* opaque, device-resident pool */

/* Last error message of the calling thread (never NULL). */
const char* sb_last_error(void);
/* Library version string. */
const char* sb_version(void);

/* ---- hashing (common.hpp:136-145, kv_cache.cpp:35-41, trace.cpp:60-83) */
uint64_t sb_kv_root_hash(void);
/* Host-side single chain hash, for bindings that need one value. */
uint64_t sb_kv_chain_hash_host(uint64_t parent, const uint64_t* tokens, int64_t n);

/* Batched chain hashing on the device.  Sequence s spans
 * d_tokens[d_seq_offsets[s] .. d_seq_offsets[s+1]); its blocks of
 * `block_size` tokens (last one partial) get their chain hashes written to
 * d_block_hashes[d_block_offsets[s] + j].  The chain for sequence s starts
 * from d_parent[s] (NULL = kv_root_hash()).  Replaces the per-block
 * kv_chain_hash loop inside KvCache::lookup_prefix / insert
 * (kv_cache.cpp:90-98, 138-141). */
int sb_chain_hash_batch(const uint64_t* d_tokens, const int64_t* d_seq_offsets,
                        const int64_t* d_block_offsets, const uint64_t* d_parent,
                        int32_t n_seqs, int64_t block_size, uint64_t* d_block_hashes,
                        void* stream);

/* Same fold over token segments: segment s is d_tokens[d_seg_bounds[2s] ..
 * d_seg_bounds[2s+1]), its blocks' chain hashes go to d_block_hashes
 * [d_seg_blocks[s] + j], the chain starting from d_parent[s] (NULL = root).
 * With d_parent = the hash of a cached prefix's last block this is the
 * incremental (suffix-only) hashing of an extended prompt. */
int sb_chain_hash_segments(const uint64_t* d_tokens, const int64_t* d_seg_bounds,
                           const int64_t* d_seg_blocks, const uint64_t* d_parent, int32_t n_segs,
                           int64_t block_size, uint64_t* d_block_hashes, void* stream);

/* Device-side synthetic token materialisation (trace.cpp:70-78 and
 * decode_token trace.cpp:80-83).  section_tag uses agentsim::SectionTag order
 * (trace.hpp:18): 0 system, 1 user, 2 tool_output, 3 history. */
int sb_materialize_tokens(int32_t section_tag, int64_t length, uint64_t content_key,
                          int32_t src_iteration, uint64_t* d_out, void* stream);
int sb_decode_tokens(uint64_t stream_key, int64_t first_index, int64_t count, uint64_t* d_out,
                     void* stream);

/* ---- KV block pool / block table: agentsim::KvCache (kv_cache.hpp:70) -- */
/* KvCache::KvCache(const CacheConfig&)          kv_cache.cpp:43 */
int sb_kv_create(int64_t block_size, int64_t capacity_blocks, int32_t policy, int32_t device,
                 sb_kv_cache** out);
void sb_kv_destroy(sb_kv_cache* cache);

/* KvCache::lookup_prefix(tokens, now)            kv_cache.cpp:85  (host tokens) */
int sb_kv_lookup_prefix(sb_kv_cache* cache, const uint64_t* tokens, int64_t n_tokens,
                        int64_t now, int64_t* hit_tokens);
/* KvCache::insert(tokens, tags, now)             kv_cache.cpp:103
 * out_ids must hold ceil(n_tokens / block_size) entries.  On CacheFull the
 * reference's rollback is reproduced (kv_cache.cpp:130-136, 148-154). */
int sb_kv_insert(sb_kv_cache* cache, const uint64_t* tokens, int64_t n_tokens,
                 const sb_tag_range* tags, int64_t n_tags, int64_t now, int32_t* out_ids,
                 int64_t* n_out);
/* KvCache::evict(needed)                         kv_cache.cpp:177
 * out_ids must hold `needed` entries; *n_out < needed signals shortfall. */
int sb_kv_evict(sb_kv_cache* cache, int64_t needed, int32_t* out_ids, int64_t* n_out);
/* KvCache::set_reuse_priority(ids, update)       kv_cache.cpp:209
 * pinned: -1 = leave, 0 = unpin, 1 = pin; tier_override: -1 = none, else tag. */
int sb_kv_set_reuse_priority(sb_kv_cache* cache, const int32_t* ids, int64_t n, int32_t pinned,
                             int32_t tier_override);
/* KvCache::set_tag(id, tag)                      kv_cache.cpp:222 */
int sb_kv_set_tag(sb_kv_cache* cache, int32_t id, int32_t tag);
/* KvCache::release(ids)                          kv_cache.cpp:228 */
int sb_kv_release(sb_kv_cache* cache, const int32_t* ids, int64_t n);
/* KvCache::touch(ids, now)                       kv_cache.cpp:238 */
int sb_kv_touch(sb_kv_cache* cache, const int32_t* ids, int64_t n, int64_t now);

int64_t sb_kv_block_size(const sb_kv_cache* cache);
int64_t sb_kv_resident_blocks(const sb_kv_cache* cache); /* kv_cache.hpp:101 */
int64_t sb_kv_capacity_blocks(const sb_kv_cache* cache); /* kv_cache.hpp:102 */
int64_t sb_kv_free_blocks(const sb_kv_cache* cache);     /* kv_cache.hpp:103 */
uint64_t sb_kv_total_evicted(const sb_kv_cache* cache);  /* kv_cache.hpp:104 */
int32_t sb_kv_policy(const sb_kv_cache* cache);
/* KvCache::contains(id) — 1 resident, 0 not      kv_cache.hpp:106 */
int sb_kv_contains(const sb_kv_cache* cache, int32_t id);
/* Ids evicted by the most recent sb_kv_insert / sb_kv_evict on this pool
 * (kv_cache.cpp:147-149, 177-197), in eviction order: with the ids an insert
 * returns, the residency change of one call — what a binding mirroring
 * KvCache::blocks_ needs, in O(change) instead of O(capacity).  *n_out gets
 * the full count; at most cap ids are copied. */
int sb_kv_last_evicted(const sb_kv_cache* cache, int32_t* out, int64_t cap, int64_t* n_out);
/* Resident block ids in ascending order (the key set of KvCache::blocks_,
 * kv_cache.hpp:124); out holds capacity entries. */
int sb_kv_resident_ids(const sb_kv_cache* cache, int32_t* out, int64_t* n_out);
/* KvCache::block(id); tokens_out may be NULL, else holds block_size u64. */
int sb_kv_block(const sb_kv_cache* cache, int32_t id, sb_block_info* info, uint64_t* tokens_out);
/* Batched KvCache::contains / KvCache::block (kv_cache.hpp:106-107): one
 * record per id in a single device round trip; a record with n_tokens == 0
 * means the id is not resident (block() would throw for it). */
int sb_kv_blocks(sb_kv_cache* cache, const int32_t* ids, int64_t n, sb_block_info* infos);
/* KvCache::audit()                                kv_cache.cpp:242 */
int sb_kv_audit(const sb_kv_cache* cache);
/* KvCache::dump() — byte-identical text; *len receives the full length
 * (call with buf=NULL to size).                   kv_cache.cpp:268 */
int sb_kv_dump(const sb_kv_cache* cache, char* buf, int64_t cap, int64_t* len);

/* ---- batched, stream-ordered engine path (no host round trip) --------- */
/* `stream` is used literally (NULL = the legacy default stream); the per-op
 * calls above run on the pool's own stream and synchronise before
 * returning. */
/* Batched lookup_prefix: sequence s is d_tokens[d_seq_offsets[s]..[s+1]);
 * d_hit_tokens[s] receives its hit length.  Touch semantics are identical to
 * calling lookup_prefix for each sequence at the same `now`.  Optional
 * precomputed chain hashes (d_block_hashes, laid out by d_block_offsets with
 * ceil(len/block_size) entries per sequence, as for insert) skip hashing;
 * pass NULL for both to hash here.  h_block_offsets (optional host copy of
 * d_block_offsets) avoids a device->host read, keeping the call fully
 * stream-ordered. */
int sb_kv_lookup_prefix_batch(sb_kv_cache* cache, const uint64_t* d_tokens,
                              const int64_t* d_seq_offsets, const int64_t* d_block_offsets,
                              const int64_t* h_block_offsets, const uint64_t* d_block_hashes,
                              int32_t n_seqs, int64_t now, int64_t* d_hit_tokens, void* stream);
/* Batched insert with the reference's sequential semantics (sequence 0 is
 * applied first).  Tag ranges for sequence s are
 * d_tags[d_tag_offsets[s]..[s+1]) with sequence-local token positions.
 * d_out_ids[d_block_offsets[s] + j] receive block ids; d_status[s] a status
 * code.  Optional d_block_hashes (NULL = computed here) are precomputed chain
 * hashes laid out like d_out_ids; optional h_block_offsets is a host copy of
 * d_block_offsets (NULL = read back, one synchronisation). */
int sb_kv_insert_batch(sb_kv_cache* cache, const uint64_t* d_tokens,
                       const int64_t* d_seq_offsets, const sb_tag_range* d_tags,
                       const int64_t* d_tag_offsets, const int64_t* d_block_offsets,
                       const int64_t* h_block_offsets, const uint64_t* d_block_hashes,
                       int32_t n_seqs, int64_t now, int32_t* d_out_ids, int32_t* d_status,
                       void* stream);
/* Batched release of d_ids[0..n) (all-or-nothing like release(); negative
 * ids — the outputs of failed inserts — are skipped).  d_status (optional,
 * device int32) receives SB_OK or, when nothing was released, the status of
 * the first failing id in order (UnknownBlock / ZeroRefRelease). */
int sb_kv_release_batch(sb_kv_cache* cache, const int32_t* d_ids, int64_t n, int32_t* d_status,
                        void* stream);
/* Counters for the cross-GPU statistics reduction: [lookups, hit_tokens,
 * looked_up_tokens, inserted_blocks, evicted_blocks, cache_full_events]. */
int sb_kv_stats(const sb_kv_cache* cache, uint64_t out[6]);
/* Diagnostics of the batched op programs (no reference counterpart):
 * [programs run, programs applied by the parallel path]. */
int sb_kv_program_stats(const sb_kv_cache* cache, uint64_t out[2]);

/* ---- continuation-prefill attention over the paged pool --------------- */
/* Replaces the prefill cost model of the reference engine
 * (CostModel::chunk_ms, engine.cpp:35-39; charged in Engine::start_step,
 * engine.cpp:424-427) with the real computation for extend_prefill
 * (engine.cpp:184-223): each sequence's new (suffix) tokens attend to its
 * cached prefix plus causally to themselves.
 *
 *  q        [total_q, n_q_heads, head_dim] bf16 (suffix queries, packed)
 *  k_pool,v_pool [n_pool_blocks, n_kv_heads, page_size, head_dim] bf16
 *  out      [total_q, n_q_heads, head_dim] bf16
 *  d_q_offsets[s]..[s+1]   suffix tokens of sequence s within q (total_q = d_q_offsets[n_seqs])
 *  d_kv_lens[s]            total keys of s (prefix + suffix); the suffix
 *                          occupies the last (q_len) positions
 *  d_block_table[s*max_blocks + j]  pool block of key positions
 *                          [j*page_size, (j+1)*page_size)
 * head_dim must be 128, page_size 16, n_q_heads % n_kv_heads == 0. */
int sb_continuation_attention(const void* q, const void* k_pool, const void* v_pool, void* out,
                              const int32_t* d_q_offsets, const int32_t* d_kv_lens,
                              const int32_t* d_block_table, int32_t n_seqs,
                              int32_t max_blocks_per_seq, int32_t max_q_len, int32_t total_q,
                              int32_t n_q_heads,
                              int32_t n_kv_heads, int32_t head_dim, int32_t page_size,
                              int64_t n_pool_blocks, float softmax_scale, const int32_t* d_work,
                              int32_t n_work, void* stream);

/* The same op in fp32 on CUDA cores (fp32 q / pages / out; outputs within
 * 1e-5 of an fp32 reference): the precision contract of fp32 pipelines such
 * as the toy model of BASELINE configs[0].  Same layouts and arguments. */
int sb_continuation_attention_f32(const float* q, const float* k_pool, const float* v_pool, float* out,
                                  const int32_t* d_q_offsets, const int32_t* d_kv_lens,
                                  const int32_t* d_block_table, int32_t n_seqs,
                                  int32_t max_blocks_per_seq, int32_t total_q, int32_t n_q_heads,
                                  int32_t n_kv_heads, int32_t head_dim, int32_t page_size,
                                  float softmax_scale, void* stream);

/* Work list for sb_continuation_attention (host): one item per (sequence, kv
 * head, pair of 128-row query tiles) that has queries, longest first (LPT),
 * as int32 pairs {seq, kv_head << 16 | pair}.  out holds 2*cap ints; returns
 * the item count in *n_out.  With d_work = NULL the kernel walks a dense
 * (n_seqs x n_kv_heads x pairs(max_q_len)) grid instead. */
int sb_attention_work_list(const int32_t* h_q_offsets, const int32_t* h_kv_lens, int32_t n_seqs,
                           int32_t n_q_heads, int32_t n_kv_heads, int32_t* out, int32_t cap,
                           int32_t* n_out);

/* Scatter the suffix K/V rows into their pool pages (the KV write of
 * extend_prefill).  k_new/v_new [total_q, n_kv_heads, head_dim]. */
int sb_kv_append(const void* k_new, const void* v_new, void* k_pool, void* v_pool,
                 const int32_t* d_q_offsets, const int32_t* d_kv_lens,
                 const int32_t* d_block_table, int32_t n_seqs, int32_t max_blocks_per_seq,
                 int32_t n_kv_heads, int32_t head_dim, int32_t page_size, void* stream);

/* Device gather of the chain hashes of resident blocks (KvBlock::chain_hash,
 * kv_cache.hpp:53): d_out[d_pos ? d_pos[i] : i] = chain hash of d_ids[i].
 * Lets an engine reuse the hashes of a pinned prefix instead of re-folding
 * its tokens (incremental, suffix-only hashing). */
int sb_kv_gather_chain_hashes(sb_kv_cache* cache, const int32_t* d_ids, const int64_t* d_pos, int64_t n,
                              uint64_t* d_out, void* stream);

/* ---- engine-path helpers ---------------------------------------------- */
/* Dense block table from the per-sequence chain ids returned by
 * sb_kv_insert_batch: table[s*max_blocks + j] = ids[block_offsets[s] + j]
 * for j < block_offsets[s+1]-block_offsets[s], -1 elsewhere. */
int sb_build_block_table(const int32_t* d_ids, const int64_t* d_block_offsets, int32_t n_seqs,
                         int32_t max_blocks, int32_t* d_table, void* stream);
/* Deterministic pseudo-random bf16 fill in [-amp, amp) keyed by `seed`: the
 * stand-in for projection outputs / prefilled pages with random-init
 * weights. */
int sb_fill_random_bf16(void* d_out, int64_t n_elems, uint64_t seed, float amp, void* stream);

/* ---- continuation engine (host C++): Engine prompt-splitting path ------ */
typedef struct sb_engine sb_engine; /* pool + per-layer K/V page pools */
typedef struct sb_batch sb_batch;   /* static layout of a batch of continuations */

/* Model shape of the paged KV (head_dim 128), pool of capacity_blocks 16-token
 * pages per layer; pages are filled with seeded random-init KV. */
int sb_engine_create(int32_t n_layers, int32_t n_q_heads, int32_t n_kv_heads, int32_t head_dim,
                     int64_t capacity_blocks, int32_t policy, int32_t device, uint64_t seed,
                     sb_engine** out);
void sb_engine_destroy(sb_engine* engine);
sb_kv_cache* sb_engine_cache(sb_engine* engine);
void* sb_engine_k_pool(sb_engine* engine, int32_t layer);
void* sb_engine_v_pool(sb_engine* engine, int32_t layer);
/* Engine lifecycle, one call at a time (engine.hpp:104-111, engine.cpp).
 * Calls are engine-owned records; each KV transition is one op of the pool's
 * op program, with the reference's exact block-pool effects.  All run on the
 * pool's stream and return when done.  Errors mirror the reference's
 * exceptions: SB_ERR_STALE_HANDLE, SB_ERR_INVALID_STATE, SB_ERR_UNKNOWN_CALL.
 *
 * Engine::submit_call (engine.cpp:128-151): admission lookup_prefix at now. */
int sb_engine_submit_call(sb_engine* engine, const uint64_t* tokens, int64_t n,
                          const sb_tag_range* tags, int64_t n_tags, int64_t decode_length,
                          int64_t now, int32_t* call);
/* Engine::submit_partial_prefill (engine.cpp:153-182): admission lookup of the
 * tool-independent prefix; returns the continuation handle (= call id). */
int sb_engine_submit_partial(sb_engine* engine, const uint64_t* tokens, int64_t n,
                             const sb_tag_range* tags, int64_t n_tags, int64_t now,
                             int32_t* handle);
/* The call's prefill finished (Engine::complete_prefill, engine.cpp:305-322):
 * a partial not yet extended is pinned (pin_partial, engine.cpp:250-286:
 * insert at PARTIAL_PREFILL, pin counts, remembered real tags) -> outcome 1,
 * or fails to pin (CacheFull, the call is aborted) -> outcome 2; otherwise the
 * prompt is inserted with its tags (CacheFull: proceed uncached), the partial
 * pins released (engine.cpp:288-303) and the old refs dropped -> outcome 3. */
int sb_engine_prefill_done(sb_engine* engine, int32_t call, int64_t now, int32_t* outcome);
/* Engine::extend_prefill (engine.cpp:184-223).  *completed = 1 when an empty
 * suffix completed the prefill at once. */
int sb_engine_extend(sb_engine* engine, int32_t handle, const uint64_t* suffix, int64_t n,
                     const sb_tag_range* tags, int64_t n_tags, int64_t decode_length, int64_t now,
                     int32_t* completed);
/* Engine::abandon_partial (engine.cpp:234-248): release pins (restoring real
 * tags), drop the chain refs. */
int sb_engine_abandon_partial(sb_engine* engine, int32_t handle);
/* Engine::finish_decode (engine.cpp:324-347): insert prompt + response
 * (RESPONSE tag), release it, release the chain refs. */
int sb_engine_finish(sb_engine* engine, int32_t call, const uint64_t* response, int64_t n_response,
                     int64_t now);
/* CallRecord view: state (agentsim::CallState order), cached prefix at
 * admission, prompt tokens, chain refs held, partial pins held. */
int sb_engine_call_info(sb_engine* engine, int32_t call, int32_t* state, int64_t* cached_prefix,
                        int64_t* prompt_tokens, int32_t* n_chain, int32_t* n_pinned);
/* which = 0: the chain refs; 1: the partial-prefill pins. */
int sb_engine_call_blocks(sb_engine* engine, int32_t call, int32_t which, int32_t* out, int64_t cap,
                          int64_t* n_out);
int sb_engine_partial_blocks(sb_engine* engine, int32_t handle, int32_t* out, int64_t cap,
                             int64_t* n_out);

/* ---- the batched engine step ------------------------------------------
 * n continuations per step, slot i with a fixed tool-independent prefix
 * (tokens prefix_tokens[prefix_off[i] .. prefix_off[i+1]), tags
 * prefix_tags[tag_off[i] .. tag_off[i+1]) in prefix-local positions) and a
 * fixed tool-output length.  One sb_batch_run is the engine-side lifecycle of
 * n new calls at `now`, each transition for all n calls as one op program
 * (same semantics as the per-call API applied in slot order):
 *   submit_partial_prefill (prefix hashes + admission lookups) -> pin_partial
 *   -> extend_prefill (the staged tool-output tokens, suffix-only hashing)
 *   -> complete_prefill (insert with hint-aware eviction, release pins and
 *   partial refs) -> per layer {KV append, continuation attention} (or the
 *   dense model) -> finish_decode with one response token (the model's greedy
 *   token, else decode_token(stream_keys[i], 0)).
 * Without an attached model the per-layer q / k / v are seeded stand-ins
 * generated once at batch creation (the dense layers are sb_batch_set_model). */
int sb_batch_create(sb_engine* engine, int32_t n, const uint64_t* prefix_tokens,
                    const int64_t* prefix_off, const sb_tag_range* prefix_tags,
                    const int64_t* tag_off, const int64_t* suffix_lens,
                    const uint64_t* stream_keys, sb_batch** out);
void sb_batch_destroy(sb_batch* batch);
/* This step's tool-output tokens, packed in slot order (host or device array). */
int sb_batch_stage_suffix(sb_batch* batch, const uint64_t* tokens, int32_t on_device,
                          void* stream);
int sb_batch_run(sb_batch* batch, int64_t now, uint64_t seed, int32_t time_attention,
                 void* stream, int32_t* launches);
/* Per-layer attention times of the last timed run (ms, n_layers floats). */
int sb_batch_attention_ms(sb_batch* batch, float* out);
/* Pool-side phases of the last timed run (ms, 3 floats): submit + pin_partial,
 * extend + complete_prefill, finish_decode. */
int sb_batch_pool_ms(sb_batch* batch, float* out);
/* Last step: admission-lookup hits (tokens per call), complete_prefill
 * statuses, and the chains the continuation attended over (ceil(full/16)
 * ids per call, packed). */
int sb_batch_results(sb_batch* batch, int64_t* hits, int32_t* status, int32_t* block_ids,
                     void* stream);
/* Last step's pin_partial outcomes (1 pinned, 2 pin failed). */
int sb_batch_pin_outcomes(sb_batch* batch, int32_t* outcomes);
/* Async D2H of query rows [first_row, first_row+n_rows) of the last layer's
 * attention output (bf16) into host_dst. */
int sb_batch_copy_output(sb_batch* batch, int64_t first_row, int64_t n_rows, void* host_dst,
                         void* stream);
int sb_batch_info(const sb_batch* batch, int64_t* total_q, int64_t* total_blocks,
                  int64_t* prompt_tokens, double* attention_flops, void** out);

/* ---- dense layers around the attention (csrc/model.cu) ----------------
 * A Llama-3-shaped decoder with seeded random-init bf16 weights (BASELINE
 * configs[2]); the reference charges this compute as a cost
 * (CostModel::chunk_ms, engine.cpp:35-39).  d_model = 128 * n_q_heads. */
typedef struct sb_model sb_model;

/* The projections' GEMM (csrc/gemm.cu, tcgen05 + TMA, persistent):
 * Y[rows, n] (op)= X[rows, k] W[n, k]^T, row-major bf16, fp32 accumulate.
 * mode 0: Y = acc (bf16); 1: Y += acc (bf16 residual); 2: Y = acc (fp32);
 * 3: SwiGLU — W is [2n, k] (gate rows, then up rows), Y[rows, n] =
 * silu(gate) * up.  n and k multiples of 8. */
int sb_gemm_bf16(const void* x, const void* w, void* y, int64_t rows, int64_t n, int64_t k,
                 int32_t mode, void* stream);

int sb_model_create(int32_t n_layers, int32_t d_model, int32_t n_q_heads, int32_t n_kv_heads,
                    int32_t d_ff, int64_t vocab, float rope_theta, uint64_t seed, int32_t device,
                    sb_model** out);
void sb_model_destroy(sb_model* model);
void sb_model_shape(const sb_model* model, int32_t* n_layers, int32_t* n_q_heads,
                    int32_t* n_kv_heads);
void sb_model_vocab(const sb_model* model, int64_t* vocab);
/* Device pointer + element count of a weight (bf16, nn.Linear [out, in]
 * layout).  layer >= 0: which = 0 Wqkv [(Hq+2Hkv)*128, d] (q, k, v rows),
 * 1 Wo [d, d], 2 Wgate_up [2*d_ff, d] (gate rows then up rows),
 * 3 Wdown [d, d_ff], 4 attention RMSNorm [d], 5 MLP RMSNorm [d];
 * layer < 0: 0 embedding [vocab, d], 1 LM head [vocab, d], 2 final norm [d]. */
int sb_model_weight(sb_model* model, int32_t layer, int32_t which, void** ptr, int64_t* n_elems);
/* Attach a model to a batch: sb_batch_run then embeds the suffix tokens
 * (token id mod vocab), runs every layer (RMSNorm, QKV, RoPE at the token's
 * absolute position, KV append into the pages, continuation attention, O
 * projection, SwiGLU MLP) and the LM head on each sequence's last token.
 * NULL detaches (attention-path mode with stand-in projections). */
int sb_batch_set_model(sb_batch* batch, sb_model* model);
/* The partial prefill itself (paper §4.2: the tool-independent prompt is
 * prefilled while the tool runs; Engine::start_step charges it,
 * engine.cpp:424-427): for each pinned partial call (sb_engine_prefill_done
 * allocated its pages), the prefix tokens not cached at submit (the
 * admission lookup, engine.cpp:170) run through the model, their K/V written
 * into the call's pinned pages.  A later continuation batch then attends over a prefix whose
 * KV is the model's own. */
int sb_engine_prefill_partials(sb_engine* engine, sb_model* model, const int32_t* handles, int32_t n,
                               void* stream);
/* Prefix tokens of a partial call that were already cached at submit. */
int sb_engine_partial_cached(sb_engine* engine, int32_t handle, int64_t* cached_tokens);
/* Greedy next token per sequence (int32 [n]) and/or fp32 logits [n, vocab]. */
int sb_batch_model_result(sb_batch* batch, int32_t* next_tokens, float* logits, void* stream);
/* Dense-layer FLOPs of one run (2 * tokens * weights of all layers). */
int sb_batch_dense_flops(const sb_batch* batch, double* flops);

#ifdef __cplusplus
}
#endif

#endif /* SUTRADHARA_B200_H_ */
