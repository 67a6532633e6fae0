// pool_batch.cuh — the op program's parallel path.  Included into
// kv_pool.cu after pool_program.cuh (same namespace and translation unit).
//
// A program of engine ops (PK_INSERT / PK_PIN / PK_COMPLETE / PK_FINISH /
// PK_ABANDON, each the reference's KvCache call sequence for one engine call,
// see pool_program.cuh) is applied op after op by ONE CTA in k_program: the
// reference's semantics are sequential (kv_cache.cpp:138-175 decides every
// insert position in order; evict(1) per miss, kv_cache.cpp:147-149, sorts
// the candidates by (tier, last_used, id), kv_cache.cpp:184-188).  Most
// programs the engine runs are nevertheless order-independent except for
// WHICH victim each miss takes, and that order is cheap to compute.  This
// path proves it for the given program on the device and then applies every
// op at once across the GPU; when the proof fails nothing has been written
// and k_program runs as before.
//
// What must hold (checked in the pre-program state, which the pre-program
// probe k_prog_bound and the select describe exactly):
//   * every op's tag ranges cover its tokens (else CacheError in order);
//   * no position hits a block with ref -1 ("late" candidates);
//   * no two missing positions share a chain hash (a later op could hit the
//     block an earlier op creates);
//   * a pool block that gets released or unpinned in the program either never
//     returns to ref 0 & unpinned, or does so at its LAST event (op z) and is
//     hit by no op after z: then it is a new candidate from op z on, with
//     key (tier after its tag restore, now if it was hit else its last_used,
//     id) — "monotone" blocks, i.e. no unmatched ref increment anywhere in
//     the program (an increment paired with the release of the same block by
//     the same op, COMPLETE's prompt vs its old chain, is matched);
//   * every release is valid (ref_count >= the number of releases of refs
//     held before the program) and every unpin acts (pin count >= unpins);
//   * the free ids the misses take are all listed, and the victims come from
//     the sorted candidate list (select) and the new candidates only; a
//     listed candidate that an op hits is never taken before that op (it is
//     skipped after it, being referenced), the list is never exhausted while
//     unlisted candidates exist, and nothing runs out (CacheFull).
// Under these conditions the sequential program's decisions are: the r-th
// miss in (op, position) order takes the r-th lowest free id while any is
// left, else the smaller of the next list entry and the smallest new
// candidate of the ops before it.  k_fast_plan replays exactly that (one warp,
// O(misses + ops)); when no op creates a candidate the mapping is direct
// (miss r -> free id r, else list entry r - free) and fully parallel.
// A block created by one op and evicted by a later op of the same program
// (FINISH's response block, tier 0, taken by the next call's miss) is
// "superseded": its id is reported to its op but its contents never written.
#pragma once
// (included inside namespace sb)

enum FastFlag { FF_POS = 1, FF_TOUCH = 2, FF_CLAIM = 4 };
enum FastCtl { FC_FAIL = 0, FC_DONE, FC_M, FC_FREE_USED, FC_NV, FC_NPEND, FC_DIRECT, FC_N = 8 };
enum MissFlag { MF_EXISTING = 1, MF_SUPERSEDED = 2 };
constexpr int kFastThreads = 1024;
constexpr int kFastMaxOps = 1024;  // ops of a program whose new candidates are tracked per op (kFastPlan smem)
constexpr int32_t kNoOp = 0x7fffffff;
constexpr int kPlanWin = 4096;     // victim-list entries k_fast_plan stages in shared memory
constexpr int kPlanNew = 4096;     // new blocks of FINISH ops tracked as candidates (shared memory)
constexpr size_t kPlanSmem = (2 * kFastMaxOps + kPlanWin + kPlanNew) * sizeof(uint64_t) +
                             (7 * kFastMaxOps + 2 + kPlanWin + 2 * kPlanNew) * sizeof(int32_t);

struct FastBuf {
  // per pool block (cap), neutral values restored by k_fast_reset
  int32_t* hit_op;   // kNoOp: smallest op hitting the block while it is a candidate
  int32_t* hit_max;  // -1: largest op hitting the block
  int32_t* dref;     // 0: net unmatched ref_count change
  int32_t* ev_max;   // -1: last op releasing / unpinning the block (or FINISH re-releasing a candidate it hit)
  int32_t* nrel;     // 0: releases of refs held before the program
  int32_t* nunp;     // 0: unpins
  int32_t* flags;    // 0: FastFlag bits
  // per op (n_ops + 1)
  int32_t* miss_cnt;
  int32_t* miss_base;
  // per position of all ops (pos_off layout)
  int32_t* mrank;  // rank of a missing position among its op's misses, -1 hit
  int32_t* mpos;   // [pos_off + k] = position of the op's k-th miss
  // per miss, global (op, position) order
  int32_t* miss_id;
  uint8_t* mflag;
  // new candidates: (key, op z) from k_fast_blocks; per-op segments in k_fast_plan
  uint64_t* pend_raw_key;
  int32_t* pend_raw_op;
  uint64_t* pend_key;  // the pool blocks' new candidates by op (k_fast_plan)
  unsigned long long* dup;  // chain hashes of missing positions (open addressing, 0 = empty)
  int64_t dup_mask;
  int64_t* ctl;
};

__device__ __forceinline__ void fast_fail(const FastBuf& F) { F.ctl[FC_FAIL] = 1; }

// returns true if h was already present
__device__ __forceinline__ bool dup_insert(const FastBuf& F, uint64_t h) {
  const unsigned long long v0 = h ? h : 1ull;  // 0 marks empty; hash 0 shares the slot of 1 (a false dup only)
  uint64_t s = (v0 ^ (v0 >> 29)) & static_cast<uint64_t>(F.dup_mask);
  for (;;) {
    const unsigned long long v = atomicCAS(&F.dup[s], 0ull, v0);
    if (v == 0) return false;
    if (v == v0) return true;
    s = (s + 1) & static_cast<uint64_t>(F.dup_mask);
  }
}

// Block-wide exclusive scan of one flag per thread (blockDim.x <= 1024).
__device__ __forceinline__ int block_scan_flag(bool f, uint32_t* warp_sums, int* total) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5, nw = blockDim.x >> 5;
  const unsigned bal = __ballot_sync(0xffffffffu, f);
  if (lane == 0) warp_sums[w] = __popc(bal);
  __syncthreads();
  if (w == 0) {
    const uint32_t c = lane < nw ? warp_sums[lane] : 0;
    uint32_t x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane < nw) warp_sums[lane] = x - c;
    if (lane == 31) warp_sums[32] = x;
  }
  __syncthreads();
  const int r = static_cast<int>(warp_sums[w]) + __popc(bal & ((1u << lane) - 1u));
  *total = static_cast<int>(warp_sums[32]);
  __syncthreads();
  return r;
}

__device__ __forceinline__ int64_t op_positions(const Pool& P, const ProgOp& op) {
  return op.kind == PK_ABANDON ? 0 : (op.n + P.bs - 1) / P.bs;
}
__device__ __forceinline__ bool op_releases_chain(int kind) {
  return kind == PK_COMPLETE || kind == PK_FINISH || kind == PK_ABANDON;
}
__device__ __forceinline__ bool op_unpins(int kind) { return kind == PK_COMPLETE || kind == PK_ABANDON; }
// COMPLETE's prompt position p referencing the same block as its old chain
// entry p: the increment and the release cancel (engine.cpp:305-322)
__device__ __forceinline__ bool complete_matched(const ProgOp& op, int64_t p, int32_t b) {
  return op.kind == PK_COMPLETE && p < op.n_chain && op.chain[p] == b;
}

// ---- 1. events of every op: misses ranked per op, per-block ref / pin events
__global__ void __launch_bounds__(kFastThreads) k_fast_events(Pool P, const ProgOp* __restrict__ ops,
                                                               const int32_t* __restrict__ pre_all,
                                                               const int32_t* __restrict__ pin_cnt, FastBuf F) {
  __shared__ uint32_t warp_sums[33];
  const int o = blockIdx.x, t = threadIdx.x;
  const ProgOp op = ops[o];
  const int64_t Pn = op_positions(P, op);
  if (t == 0 && op.kind != PK_ABANDON && op.kind != PK_PIN && !tags_cover(op.ins_tags, op.n_ins_tags, op.n))
    fast_fail(F);
  if (t == 0 && op.kind > PK_ABANDON) fast_fail(F);
  int base = 0;
  for (int64_t p0 = 0; p0 < Pn; p0 += blockDim.x) {
    const int64_t p = p0 + t;
    const int32_t b = p < Pn ? pre_all[op.pos_off + p] : 0;
    const bool miss = p < Pn && b < 0;
    int tot;
    const int r = block_scan_flag(miss, warp_sums, &tot);
    if (p < Pn) {
      if (miss) {
        F.mrank[op.pos_off + p] = base + r;
        F.mpos[op.pos_off + base + r] = static_cast<int32_t>(p);
        if (dup_insert(F, op.hashes[p])) fast_fail(F);
      } else {
        F.mrank[op.pos_off + p] = -1;
        const int rf = P.ref[b], pn = P.pinned[b];
        if (pn == 0 && rf < 0) fast_fail(F);
        const bool cand = pn == 0 && rf == 0;
        atomicMax(&F.hit_max[b], o);
        if (cand) atomicMin(&F.hit_op[b], o);
        if (op.kind == PK_FINISH) {  // +1 then its own release: ref unchanged, last_used = now
          atomicOr(&F.flags[b], FF_TOUCH);
          if (cand) atomicMax(&F.ev_max[b], o);
        } else if (complete_matched(op, p, b)) {
          atomicOr(&F.flags[b], FF_TOUCH);
        } else {
          atomicAdd(&F.dref[b], 1);
          atomicOr(&F.flags[b], FF_POS | FF_TOUCH);
        }
      }
    }
    base += tot;
  }
  if (t == 0) F.miss_cnt[o] = base;
  if (op_releases_chain(op.kind))
    for (int64_t k = t; k < op.n_chain; k += blockDim.x) {
      const int32_t b = op.chain[k];
      if (k < Pn && complete_matched(op, k, b) && pre_all[op.pos_off + k] == b) continue;
      if (b < 0 || b >= P.cap || P.ntok[b] <= 0) {  // UnknownBlock: the sequential program reports it
        fast_fail(F);
        continue;
      }
      atomicAdd(&F.nrel[b], 1);
      atomicAdd(&F.dref[b], -1);
      atomicMax(&F.ev_max[b], o);
    }
  if (op_unpins(op.kind))
    for (int64_t k = t; k < op.n_pinned; k += blockDim.x) {
      const int32_t b = op.pinned[k];
      if (b < 0 || b >= P.cap) continue;  // not in the pin map (prog_unpin skips it)
      if (!pin_cnt) {
        fast_fail(F);
        continue;
      }
      if (pin_cnt[b] <= 0) continue;
      atomicAdd(&F.nunp[b], 1);
      atomicMax(&F.ev_max[b], o);
    }
}

// ---- 2. per block with events: does it become a candidate, when, with which key
__global__ void __launch_bounds__(256) k_fast_blocks(Pool P, const ProgOp* __restrict__ ops,
                                                     const int32_t* __restrict__ pre_all,
                                                     const int32_t* __restrict__ pin_cnt,
                                                     const int8_t* __restrict__ real_tag, int64_t now, FastBuf F) {
  if (F.ctl[FC_FAIL]) return;
  const int o = blockIdx.x;
  const ProgOp op = ops[o];
  const int64_t Pn = op_positions(P, op);
  const int64_t nc = op_releases_chain(op.kind) ? op.n_chain : 0;
  const int64_t np = op_unpins(op.kind) ? op.n_pinned : 0;
  for (int64_t e = threadIdx.x; e < Pn + nc + np; e += blockDim.x) {
    const int32_t b = e < Pn ? pre_all[op.pos_off + e] : e < Pn + nc ? op.chain[e - Pn] : op.pinned[e - Pn - nc];
    if (b < 0 || b >= P.cap) continue;
    const int z = F.ev_max[b];
    if (z < 0) continue;  // never released / unpinned: it cannot become a candidate here
    if (atomicOr(&F.flags[b], FF_CLAIM) & FF_CLAIM) continue;  // one thread per block
    const int fl = F.flags[b];
    if ((fl & FF_POS) || F.hit_max[b] > z) {  // order-dependent: a reference after a release
      fast_fail(F);
      continue;
    }
    const int rf0 = P.ref[b];
    if (rf0 < F.nrel[b]) {  // a release fails in order (ZeroRefRelease)
      fast_fail(F);
      continue;
    }
    const int nu = F.nunp[b];
    const int pc = pin_cnt ? pin_cnt[b] : 0;
    if (nu > pc) {
      fast_fail(F);
      continue;
    }
    const bool unpinned_here = nu > 0 && pc == nu;
    const bool pinned_end = P.pinned[b] != 0 && !unpinned_here;
    if (rf0 + F.dref[b] != 0 || pinned_end || P.ntok[b] <= 0) continue;
    int tg = P.tag[b];
    if (unpinned_here && real_tag && real_tag[b] >= 0) tg = real_tag[b];
    const int64_t last = (fl & FF_TOUCH) ? now : P.last[b];
    uint64_t key = (static_cast<uint64_t>(last + P.lbias) << P.idb) | static_cast<uint64_t>(b);
    if (P.policy == SB_POLICY_TIERED) key |= static_cast<uint64_t>(tier_of(tg)) << 61;
    const unsigned long long at = atomicAdd(reinterpret_cast<unsigned long long*>(&F.ctl[FC_NPEND]), 1ull);
    F.pend_raw_key[at] = key;
    F.pend_raw_op[at] = z;
  }
}

// ---- 3. one CTA: rank the misses, decide every miss's id in the reference's order
__global__ void __launch_bounds__(kFastThreads) k_fast_plan(Pool P, Scratch S, const ProgOp* __restrict__ ops,
                                                            int n_ops, int64_t now, FastBuf F,
                                                            unsigned long long* prof) {
  const unsigned long long c0 = clock64();
  __shared__ uint32_t warp_sums[33];
  __shared__ int any_finish_miss, fail_sh;
  const int t = threadIdx.x, lane = t & 31;
  if (F.ctl[FC_FAIL]) return;
  if (t == 0) {
    any_finish_miss = 0;
    fail_sh = 0;
  }
  // exclusive scan of the per-op miss counts
  int run = 0;
  for (int o0 = 0; o0 < n_ops; o0 += blockDim.x) {
    const int o = o0 + t;
    const int c = o < n_ops ? F.miss_cnt[o] : 0;
    if (o < n_ops && c > 0 && ops[o].kind == PK_FINISH) any_finish_miss = 1;
    // block scan of c (values, not flags): warp then block
    int x = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= d) x += y;
    }
    if (lane == 31) warp_sums[t >> 5] = x;
    __syncthreads();
    if (t < 32) {
      const int nw = blockDim.x >> 5;
      const int ws = lane < nw ? static_cast<int>(warp_sums[lane]) : 0;
      int z = ws;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, z, d);
        if (lane >= d) z += y;
      }
      if (lane < nw) warp_sums[lane] = z - ws;
      if (lane == 31) warp_sums[32] = z;
    }
    __syncthreads();
    if (o < n_ops) F.miss_base[o] = run + static_cast<int>(warp_sums[t >> 5]) + x - c;
    run += static_cast<int>(warp_sums[32]);
    __syncthreads();
  }
  const int64_t M = run;
  if (t == 0) F.miss_base[n_ops] = static_cast<int32_t>(M);
  const int64_t free0 = P.cap - static_cast<int64_t>(P.ctr[C_NRES]);
  const int64_t Fp = S.scal[S_FREE], K = S.scal[S_K], ncand = S.scal[S_NCAND];
  const int64_t free_used = min64(M, free0);
  const int64_t npend = F.ctl[FC_NPEND];
  __syncthreads();
  if (free_used > Fp) return fast_fail(F);  // unlisted free ids (uniform)
  const bool direct = npend == 0 && !any_finish_miss;
  if (direct) {
    // miss r -> free id r, else list entry r - free_used; a listed block some
    // op hits must not be taken (it would have to be skipped or turn a hit into a miss)
    const int64_t nv = M - free_used;
    if (nv > K) return fast_fail(F);
    for (int64_t r = t; r < M; r += blockDim.x) {
      if (r < free_used) {
        F.miss_id[r] = S.freel[r];
        F.mflag[r] = 0;
      } else {
        const int32_t v = static_cast<int32_t>(S.victims[r - free_used] & P.idmask);
        if (F.hit_op[v] != kNoOp) fail_sh = 1;
        F.miss_id[r] = v;
        F.mflag[r] = MF_EXISTING;
      }
    }
    __syncthreads();
    if (t == 0) {
      if (fail_sh) {
        fast_fail(F);
      } else {
        F.ctl[FC_M] = M;
        F.ctl[FC_FREE_USED] = free_used;
        F.ctl[FC_NV] = nv;
        F.ctl[FC_DIRECT] = 1;
        F.ctl[FC_DONE] = 1;
      }
    }
    return;
  }
  if (n_ops > kFastMaxOps) return fast_fail(F);
  // ---- new candidates by the op z from which they are candidates:
  //   E part: pool blocks reaching ref 0 & unpinned at their last event
  //           (k_fast_blocks), segment [segE[z], segE[z + 1]) of F.pend_key;
  //   N part: FINISH's own new blocks (candidates once it releases its
  //           insert's refs), [noff[z], noff[z + 1]) of nkey in shared memory.
  extern __shared__ __align__(16) uint8_t plan_dyn[];
  uint64_t* minE = reinterpret_cast<uint64_t*>(plan_dyn);
  uint64_t* minN = minE + kFastMaxOps;
  uint64_t* lkey = minN + kFastMaxOps;    // list window: keys
  uint64_t* nkey = lkey + kPlanWin;       // N entries: key (id or-ed in when assigned)
  int32_t* segE = reinterpret_cast<int32_t*>(nkey + kPlanNew);
  int32_t* noff = segE + kFastMaxOps + 1;
  int32_t* fillE = noff + kFastMaxOps + 1;
  int32_t* argE = fillE + kFastMaxOps;
  int32_t* argN = argE + kFastMaxOps;
  int32_t* mc = argN + kFastMaxOps;
  int32_t* mb = mc + kFastMaxOps;
  int32_t* lho = mb + kFastMaxOps;        // list window: hit_op of each entry
  int32_t* nwho = lho + kPlanWin;         // N entries: creating miss rank
  int32_t* nsup = nwho + kPlanNew;        // N entries: evicted later in the program (superseded)
  for (int o = t; o < n_ops; o += blockDim.x) {
    fillE[o] = 0;
    mc[o] = F.miss_cnt[o];
    mb[o] = F.miss_base[o];
    minE[o] = kNoKey;
    minN[o] = kNoKey;
    argE[o] = -1;
    argN[o] = -1;
  }
  const int64_t W = min64(K, kPlanWin);
  for (int64_t i = t; i < W; i += blockDim.x) {
    const uint64_t k = S.victims[i];
    lkey[i] = k;
    lho[i] = F.hit_op[static_cast<int32_t>(k & P.idmask)];
  }
  __syncthreads();
  for (int64_t i = t; i < npend; i += blockDim.x) atomicAdd(&fillE[F.pend_raw_op[i]], 1);
  __syncthreads();
  if (t == 0) {
    int acc = 0, accn = 0;
    for (int o = 0; o < n_ops; ++o) {
      segE[o] = acc;
      noff[o] = accn;
      acc += fillE[o];
      accn += ops[o].kind == PK_FINISH ? mc[o] : 0;
      fillE[o] = 0;
    }
    segE[n_ops] = acc;
    noff[n_ops] = accn;
    if (accn > kPlanNew) fail_sh = 1;
  }
  __syncthreads();
  if (fail_sh) return fast_fail(F);  // uniform
  for (int64_t i = t; i < npend; i += blockDim.x) {
    const int z = F.pend_raw_op[i];
    const int at = segE[z] + atomicAdd(&fillE[z], 1);
    F.pend_key[at] = F.pend_raw_key[i];
  }
  // N entries: key without the id (tier of the position's tag, last_used now)
  const uint64_t now_bits = static_cast<uint64_t>(now + P.lbias) << P.idb;
  for (int i = t; i < noff[n_ops]; i += blockDim.x) {
    int lo = 0, hi = n_ops;  // op z with noff[z] <= i < noff[z + 1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (noff[mid] <= i) lo = mid; else hi = mid;
    }
    while (noff[lo + 1] <= i) ++lo;  // (ops without N entries share an offset)
    const ProgOp& op = ops[lo];
    const int32_t pos = F.mpos[op.pos_off + (i - noff[lo])];
    uint64_t key = now_bits;
    if (P.policy == SB_POLICY_TIERED)
      key |= static_cast<uint64_t>(tier_of(tag_at(op.ins_tags, op.n_ins_tags, static_cast<int64_t>(pos) * P.bs))) << 61;
    nkey[i] = key;
    nwho[i] = mb[lo] + (i - noff[lo]);
    nsup[i] = 0;
  }
  __syncthreads();
  __syncthreads();
  for (int o = t >> 5; o < n_ops; o += blockDim.x >> 5) {  // min / argmin of every E segment: a warp each
    uint64_t mk = kNoKey;
    int ma = -1;
    for (int i = segE[o] + lane; i < segE[o + 1]; i += 32) {
      const uint64_t k = F.pend_key[i];
      if (k < mk) {
        mk = k;
        ma = i;
      }
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) {
      const uint64_t ok = __shfl_xor_sync(0xffffffffu, mk, d);
      const int oa = __shfl_xor_sync(0xffffffffu, ma, d);
      if (ok < mk) {
        mk = ok;
        ma = oa;
      }
    }
    if (lane == 0) {
      minE[o] = mk;
      argE[o] = ma;
    }
  }
  __syncthreads();
  if (t >= 32) return;
  const unsigned long long c1 = clock64();
  // ---- warp 0: the sequential decisions
  uint64_t best = kNoKey;  // smallest available new candidate (segments of ops before the current one)
  int best_op = -1;
  int64_t ptr = 0;  // next list entry
  bool failed = false;
  auto rescan = [&](int o, bool part_n) {  // min / argmin of one part of op o's candidates (warp)
    const int lo = part_n ? noff[o] : segE[o], hi = part_n ? noff[o + 1] : segE[o + 1];
    uint64_t mk = kNoKey;
    int ma = -1;
    for (int i = lo + lane; i < hi; i += 32) {
      const uint64_t k = part_n ? nkey[i] : F.pend_key[i];
      if (k < mk) {
        mk = k;
        ma = i;
      }
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) {
      const uint64_t ok = __shfl_xor_sync(0xffffffffu, mk, d);
      const int oa = __shfl_xor_sync(0xffffffffu, ma, d);
      if (ok < mk) {
        mk = ok;
        ma = oa;
      }
    }
    if (lane == 0) {
      if (part_n) {
        minN[o] = mk;
        argN[o] = ma;
      } else {
        minE[o] = mk;
        argE[o] = ma;
      }
    }
    __syncwarp();
  };
  auto find_best = [&](int upto) {  // over ops [0, upto)
    uint64_t mk = kNoKey;
    int ms = -1;
    for (int o = lane; o < upto; o += 32) {
      const uint64_t k = min(minE[o], minN[o]);
      if (k < mk) {
        mk = k;
        ms = o;
      }
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) {
      const uint64_t ok = __shfl_xor_sync(0xffffffffu, mk, d);
      const int os = __shfl_xor_sync(0xffffffffu, ms, d);
      if (ok < mk) {
        mk = ok;
        ms = os;
      }
    }
    best = mk;
    best_op = ms;
  };
  // the id taken by miss k of op o (N entries of a FINISH op record it)
  auto assign = [&](int o, int64_t base, int k, int32_t id, uint8_t fl) {
    F.miss_id[base + k] = id;
    F.mflag[base + k] = fl;
    if (noff[o + 1] > noff[o]) nkey[noff[o] + k] |= static_cast<uint64_t>(id);
  };
  for (int o = 0; o < n_ops && !failed; ++o) {
    const int m = mc[o];
    const int64_t base = mb[o];
    int k = 0;
    // free ids first (alloc_block_id, kv_cache.cpp:62-67)
    if (base < free_used) {
      const int nf = static_cast<int>(min64(m, free_used - base));
      for (int i = lane; i < nf; i += 32) assign(o, base, i, S.freel[base + i], 0);
      k = nf;
    }
    while (k < m) {
      const int need = m - k;
      // the next 32 list entries: skip (hit by an earlier op: referenced),
      // take (key below every new candidate), else stop: the list end, a key
      // above the best new candidate, or a block this or a later op hits
      const int64_t e = ptr + lane;
      uint64_t key = kNoKey;
      int ho = kNoOp;
      if (e < W) {
        key = lkey[e];
        ho = lho[e];
      } else if (e < K) {
        key = S.victims[e];
        ho = F.hit_op[static_cast<int32_t>(key & P.idmask)];
      }
      const bool in = e < K;
      const bool skip = in && ho < o;
      const bool take = in && !skip && ho == kNoOp && key < best;
      const unsigned stopm = __ballot_sync(0xffffffffu, !skip && !take);
      const int f = stopm ? __ffs(stopm) - 1 : 32;
      const unsigned tm = __ballot_sync(0xffffffffu, take) & (f == 32 ? 0xffffffffu : ((1u << f) - 1u));
      const int c = __popc(tm);
      const int ntake = min(c, need);
      if ((tm >> lane) & 1u) {
        const int j = __popc(tm & ((1u << lane) - 1u));
        if (j < ntake) assign(o, base, k + j, static_cast<int32_t>(key & P.idmask), MF_EXISTING);
      }
      k += ntake;
      __syncwarp();
      if (ntake < c) {  // satisfied before the stop: resume right after the last entry taken
        unsigned rest = tm;
        for (int j = 1; j < ntake; ++j) rest &= rest - 1u;
        ptr += __ffs(rest);
        continue;
      }
      ptr += f;  // skipped and taken entries before the stop are consumed for good
      if (k == m || f == 32) continue;
      const int64_t ef = __shfl_sync(0xffffffffu, e, f);
      const uint64_t kf = __shfl_sync(0xffffffffu, key, f);
      const bool list_end = ef >= K;
      if (!list_end && kf < best) {  // a listed block that this or a later op hits
        failed = true;
        break;
      }
      if (list_end && K < ncand && (K == 0 || best > S.victims[K - 1])) {  // an unlisted candidate may be next
        failed = true;
        break;
      }
      if (best == kNoKey) {  // nothing left: CacheFull, left to the program
        failed = true;
        break;
      }
      // take the best new candidate
      const bool from_n = minN[best_op] <= minE[best_op];
      const int at = from_n ? argN[best_op] : argE[best_op];
      if (lane == 0) {
        assign(o, base, k, static_cast<int32_t>(best & P.idmask), from_n ? 0 : MF_EXISTING);
        if (from_n) {
          nsup[at] = 1;
          nkey[at] = kNoKey;
        }
        else F.pend_key[at] = kNoKey;
      }
      __syncwarp();
      ++k;
      rescan(best_op, from_n);
      find_best(o);
    }
    if (failed) break;
    // op o's candidates become available (its N keys are complete now)
    if (noff[o + 1] > noff[o]) rescan(o, true);
    const uint64_t so = min(minE[o], minN[o]);
    if (so < best) {
      best = so;
      best_op = o;
    }
  }
  __syncwarp();
  if (!failed)
    for (int i = lane; i < noff[n_ops]; i += 32)
      if (nsup[i]) F.mflag[nwho[i]] |= MF_SUPERSEDED;
  if (lane == 0) {
    if (failed) {
      fast_fail(F);
    } else {
      F.ctl[FC_M] = M;
      F.ctl[FC_FREE_USED] = free_used;
      F.ctl[FC_NV] = M - free_used;  // every miss past the free ids is one eviction
      F.ctl[FC_DIRECT] = 0;
      F.ctl[FC_DONE] = 1;
    }
    if (prof) {
      const unsigned long long c2 = clock64();
      prof[60] += c1 - c0;
      prof[61] += c2 - c1;
      prof[62] += 1;
    }
  }
}

// ---- 4. effects on pool blocks: hits (ref + 1 unless matched or released
// by the same FINISH, last_used = now), releases of held refs, unpins with
// the real tag restored (release_partial_pins, engine.cpp:288-303).  Before
// the evictions: a block released to ref 0 here may be evicted by a later op.
__global__ void __launch_bounds__(256) k_fast_touch(Pool P, const ProgOp* __restrict__ ops,
                                                    const int32_t* __restrict__ pre_all, int32_t* pin_cnt,
                                                    int8_t* real_tag, int64_t now, FastBuf F) {
  if (!F.ctl[FC_DONE]) return;
  const int o = blockIdx.x;
  const ProgOp op = ops[o];
  const int64_t Pn = op_positions(P, op);
  for (int64_t p = blockIdx.y * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < Pn;
       p += static_cast<int64_t>(gridDim.y) * blockDim.x) {
    const int32_t b = pre_all[op.pos_off + p];
    if (b < 0) continue;
    if (op.kind != PK_FINISH && !complete_matched(op, p, b)) atomicAdd(&P.ref[b], 1);
    P.last[b] = now;
    op.ids[p] = b;
  }
  if (blockIdx.y != 0) return;
  if (op_releases_chain(op.kind))
    for (int64_t k = threadIdx.x; k < op.n_chain; k += blockDim.x) {
      const int32_t b = op.chain[k];
      if (k < Pn && complete_matched(op, k, b) && pre_all[op.pos_off + k] == b) continue;
      atomicSub(&P.ref[b], 1);
    }
  if (op_unpins(op.kind))
    for (int64_t k = threadIdx.x; k < op.n_pinned; k += blockDim.x) {
      const int32_t b = op.pinned[k];
      // a block's unpins all act or none (k_fast_blocks): the count stays > 0 until the last
      if (b < 0 || b >= P.cap || pin_cnt[b] <= 0) continue;
      if (atomicSub(&pin_cnt[b], 1) == 1) {
        if (P.ntok[b] > 0) {
          P.pinned[b] = 0;
          const int rt = real_tag[b];
          if (rt >= 0) P.tag[b] = rt;
        }
        real_tag[b] = -1;
      }
    }
}

// ---- 5. evictions: the index slots of evicted pool blocks become tombstones
// Also the evicted ids in eviction order into S.evicted, as the sequential
// program leaves them (sb_kv_insert reports them: sb_kv_last_evicted, which
// the drop-in binding's residency mirror consumes).
__global__ void k_fast_evict(Pool P, Scratch S, FastBuf F) {
  if (!F.ctl[FC_DONE]) return;
  const int64_t M = F.ctl[FC_M], fu = F.ctl[FC_FREE_USED];
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < M;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (r >= fu) S.evicted[r - fu] = F.miss_id[r];
    if (!(F.mflag[r] & MF_EXISTING)) continue;
    const int32_t v = F.miss_id[r];
    P.idx[P.slot[v]].id = -2;
    P.ntok[v] = 0;
  }
}

// ---- 6. new blocks (a superseded one only reports its id)
__global__ void __launch_bounds__(256) k_fast_create(Pool P, const ProgOp* __restrict__ ops,
                                                     const int32_t* __restrict__ pre_all, int64_t now, FastBuf F) {
  if (!F.ctl[FC_DONE]) return;
  const int o = blockIdx.x;
  const ProgOp op = ops[o];
  const int64_t Pn = op_positions(P, op);
  const int64_t mb = F.miss_base[o];
  const sb_tag_range pin_range{0, op.n, SB_TAG_PARTIAL_PREFILL, 0};
  const sb_tag_range* tags = op.kind == PK_PIN ? &pin_range : op.ins_tags;
  const int64_t ntags = op.kind == PK_PIN ? 1 : op.n_ins_tags;
  for (int64_t p = blockIdx.y * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < Pn;
       p += static_cast<int64_t>(gridDim.y) * blockDim.x) {
    if (pre_all[op.pos_off + p] >= 0) continue;
    const int64_t r = mb + F.mrank[op.pos_off + p];
    const int32_t id = F.miss_id[r];
    op.ids[p] = id;
    if (F.mflag[r] & MF_SUPERSEDED) continue;
    const int64_t off = p * P.bs;
    const int len = static_cast<int>(min(P.bs, op.n - off));
    uint64_t* dst = P.tok + static_cast<int64_t>(id) * P.bs;
    if (len == 16) {
      uint64_t v[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) v[i] = op.tokens[off + i];
#pragma unroll
      for (int i = 0; i < 16; ++i) dst[i] = v[i];
    } else {
      for (int i = 0; i < len; ++i) dst[i] = op.tokens[off + i];
    }
    const uint64_t h = op.hashes[p];
    const uint64_t par = p ? op.hashes[p - 1] : kRootHash;
    P.ntok[id] = len;
    P.chain[id] = h;
    P.parent[id] = par;
    P.tag[id] = tag_at(tags, ntags, off);
    P.ref[id] = op.kind == PK_FINISH ? 0 : 1;  // FINISH releases its own insert's refs (engine.cpp:333-337)
    P.last[id] = now;
    P.pinned[id] = 0;
    index_insert(P, h, id, par, len);
  }
}

// ---- 7. pin_partial's pins (engine.cpp:273-285): first op per block records the real tag
__global__ void __launch_bounds__(256) k_fast_pin_a(Pool P, const ProgOp* __restrict__ ops, int32_t* first_op,
                                                    FastBuf F) {
  if (!F.ctl[FC_DONE]) return;
  const int o = blockIdx.x;
  const ProgOp op = ops[o];
  if (op.kind != PK_PIN) return;
  const int64_t Pn = op_positions(P, op);
  for (int64_t p = blockIdx.y * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < Pn;
       p += static_cast<int64_t>(gridDim.y) * blockDim.x)
    atomicMin(&first_op[op.ids[p]], o);
}
__global__ void __launch_bounds__(256) k_fast_pin_b(Pool P, const ProgOp* __restrict__ ops,
                                                    const int32_t* __restrict__ pin_cnt, const int32_t* first_op,
                                                    int8_t* real_tag, FastBuf F) {
  if (!F.ctl[FC_DONE]) return;
  const int o = blockIdx.x;
  const ProgOp op = ops[o];
  if (op.kind != PK_PIN) return;
  const int64_t Pn = op_positions(P, op);
  for (int64_t p = blockIdx.y * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < Pn;
       p += static_cast<int64_t>(gridDim.y) * blockDim.x) {
    const int32_t b = op.ids[p];
    if (first_op[b] == o && pin_cnt[b] == 0) {
      const int cur = P.tag[b];
      real_tag[b] = static_cast<int8_t>(cur != SB_TAG_PARTIAL_PREFILL ? cur
                                                                      : engine_tag_at(op.real_tags, op.n_real_tags,
                                                                                      p * P.bs));
    }
  }
}
__global__ void __launch_bounds__(256) k_fast_pin_c(Pool P, const ProgOp* __restrict__ ops, int32_t* pin_cnt,
                                                    int32_t* first_op, FastBuf F) {
  if (!F.ctl[FC_DONE]) return;
  const int o = blockIdx.x;
  const ProgOp op = ops[o];
  if (op.kind != PK_PIN) return;
  const int64_t Pn = op_positions(P, op);
  for (int64_t p = blockIdx.y * static_cast<int64_t>(blockDim.x) + threadIdx.x; p < Pn;
       p += static_cast<int64_t>(gridDim.y) * blockDim.x) {
    const int32_t b = op.ids[p];
    atomicAdd(&pin_cnt[b], 1);
    P.pinned[b] = 1;
    P.tag[b] = SB_TAG_PARTIAL_PREFILL;
    op.chain[p] = b;
    op.pinned[p] = b;
    first_op[b] = kNoOp;
  }
}

// ---- 8. one CTA per op: the per-block scratch neutral again (always, also
// when the program falls back: before any chain is rewritten), then the
// op's results and chain
__global__ void __launch_bounds__(256) k_fast_finish(Pool P, Scratch S, const ProgOp* __restrict__ ops,
                                                     const int32_t* __restrict__ pre_all, ProgRes* res, int n_ops,
                                                     int64_t* out, FastBuf F) {
  const int o = blockIdx.x;
  const ProgOp op = ops[o];
  const int64_t Pn = op_positions(P, op);
  {
    const int64_t nc = op_releases_chain(op.kind) ? op.n_chain : 0;
    const int64_t np = op_unpins(op.kind) ? op.n_pinned : 0;
    for (int64_t e = threadIdx.x; e < Pn + nc + np; e += blockDim.x) {
      const int32_t b = e < Pn ? pre_all[op.pos_off + e] : e < Pn + nc ? op.chain[e - Pn] : op.pinned[e - Pn - nc];
      if (b < 0 || b >= P.cap) continue;
      F.hit_op[b] = kNoOp;
      F.hit_max[b] = -1;
      F.dref[b] = 0;
      F.ev_max[b] = -1;
      F.nrel[b] = 0;
      F.nunp[b] = 0;
      F.flags[b] = 0;
    }
  }
  if (!F.ctl[FC_DONE]) return;  // uniform
  __syncthreads();  // this op's chain entries were read above
  if (op.kind == PK_COMPLETE)
    for (int64_t p = threadIdx.x; p < Pn; p += blockDim.x) op.chain[p] = op.ids[p];
  if (threadIdx.x == 0) {
    ProgRes r{SB_OK, PO_NONE, op.n_chain, op.n_pinned};
    switch (op.kind) {
      case PK_PIN:
        r = ProgRes{SB_OK, PO_PINNED, static_cast<int32_t>(Pn), static_cast<int32_t>(Pn)};
        break;
      case PK_COMPLETE:
        r = ProgRes{SB_OK, PO_COMPLETED, static_cast<int32_t>(Pn), 0};
        break;
      case PK_FINISH:
        r.n_chain = 0;
        r.outcome = PO_FINISHED;
        break;
      case PK_ABANDON:
        r = ProgRes{SB_OK, PO_ABANDONED, 0, 0};
        break;
      default:
        break;
    }
    res[o] = r;
  }
  if (o != 0) return;
  const int64_t M = F.ctl[FC_M], nv = F.ctl[FC_NV];
  // select's rank marks (S.rank_of, read only by the per-insert path)
  for (int64_t i = threadIdx.x; i < S.scal[S_K]; i += blockDim.x) S.rank_of[S.victims[i] & P.idmask] = -1;
  if (threadIdx.x == 0) {
    if (nv > 0) {
      P.ctr[C_EVICTED] += static_cast<unsigned long long>(nv);
      P.ctr[C_EV_BLOCKS] += static_cast<unsigned long long>(nv);
    }
    P.ctr[C_NRES] += static_cast<unsigned long long>(M - nv);
    P.ctr[C_INS_BLOCKS] += static_cast<unsigned long long>(M);
    out[0] = n_ops;
    out[1] = PS_NONE;
    out[2] = nv;
    out[3] = M;
  }
}
