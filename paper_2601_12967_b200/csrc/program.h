// program.h — host/device descriptors of the block pool's op program
// (pool_program.cuh) and the internal entry points the engine (engine.cu)
// uses.  Not part of the C-ABI.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/sutradhara_b200.h"

struct sb_kv_cache;

namespace sb {

enum ProgKind { PK_INSERT = 0, PK_PIN = 1, PK_COMPLETE = 2, PK_FINISH = 3, PK_ABANDON = 4 };
enum ProgOutcome { PO_NONE = 0, PO_PINNED = 1, PO_PIN_FAILED = 2, PO_COMPLETED = 3, PO_FINISHED = 4, PO_ABANDONED = 5 };
enum ProgStop { PS_NONE = 0, PS_BEFORE = 1, PS_AFTER = 2, PS_ERROR = 3 };

struct ProgOp {
  int32_t kind;
  int32_t n_ins_tags;    // tags of the insert
  int32_t n_real_tags;   // PK_PIN: the call's own tags (real tag of fresh blocks, engine.cpp:267-276)
  int32_t n_chain;       // the call's chain refs (engine.hpp:153)
  int32_t n_pinned;      // the call's partial-prefill pins (engine.hpp:154)
  int32_t _pad;
  int64_t n;             // insert tokens
  int64_t pos_off;       // first slot of this op's block positions in the pre-program probe array (host-filled)
  const uint64_t* tokens;
  const uint64_t* hashes;  // chain hash of every insert block
  const sb_tag_range* ins_tags;
  const sb_tag_range* real_tags;
  int32_t* ids;     // insert output (ceil(n / bs))
  int32_t* chain;   // in: chain refs; PK_PIN / PK_COMPLETE: out (the new chain)
  int32_t* pinned;  // in: pinned ids; PK_PIN: out
};

struct ProgRes {
  int32_t status;   // SB_OK / SB_ERR_CACHE_FULL / release errors / SB_ERR_CACHE (tags)
  int32_t outcome;  // ProgOutcome
  int32_t n_chain;
  int32_t n_pinned;
};


// Applies ops [0, n) (host descriptors holding device pointers) to the pool
// on stream st with the reference's sequential semantics; per-op results in
// h_res.  Synchronises st.  Returns the number of ops applied.
int64_t pool_run_ops(sb_kv_cache* c, const ProgOp* h_ops, int64_t n, int32_t* d_pin_cnt, int8_t* d_real_tag,
                     int64_t now, cudaStream_t st, ProgRes* h_res);

// KvCache::lookup_prefix (kv_cache.cpp:85-101) of n sequences described by
// (tokens, n, hashes) of h_ops; hit lengths (tokens) into d_hits[n].
// Stream-ordered (no synchronisation).
void pool_lookup(sb_kv_cache* c, const ProgOp* h_ops, int64_t n, int64_t now, int64_t* d_hits, cudaStream_t st);

// The pool's own stream (per-op C-ABI calls run there).
cudaStream_t pool_stream(sb_kv_cache* c);
// Kernels the pool's op programs and batched lookups have launched so far.
uint64_t pool_launches(const sb_kv_cache* c);
int pool_device(sb_kv_cache* c);

}  // namespace sb
