// pool_program.cuh — the block pool's op program: ONE cooperative-free CTA
// applies a list of engine operations to the device pool with the
// reference's sequential semantics, op after op, with no host round trip.
// Included into kv_pool.cu (same translation unit: Pool, Scratch, the index
// and probe helpers are shared).
//
// Ops (each = the reference's KvCache call sequence for one engine call):
//   PK_INSERT    KvCache::insert                              kv_cache.cpp:103-175
//   PK_PIN       Engine::pin_partial                          engine.cpp:250-286
//                insert(prefix, PARTIAL) -> per-block pin count, real tag,
//                set_reuse_priority(pinned, PARTIAL); CacheFull -> pin failed
//   PK_COMPLETE  Engine::complete_prefill                     engine.cpp:305-322
//                insert(prompt, tags) (CacheFull: proceed uncached) ->
//                release_partial_pins (engine.cpp:288-303) -> release(old refs)
//   PK_FINISH    Engine::finish_decode                        engine.cpp:324-347
//                insert(prompt + response, tags + RESPONSE) -> release(ids)
//                -> release(chain refs)
//   PK_ABANDON   Engine::abandon_partial                      engine.cpp:234-248
//
// Victims.  Before the program, one hint-aware scoring pass + select (the
// all-SM k_score / k_select_coop or the one-CTA k_select, mode 2) lists the
// K smallest (tier, last_used, id) keys of the pool's candidates and the
// lowest F free ids, K and F bounded by the misses the program can make
// (k_prog_bound: pre-state probe of every insert position).  Inside the
// program the list is consumed lazily: an entry is a victim only if the
// block is STILL a candidate with the SAME key (ref 0, unpinned, resident,
// unchanged tier/last_used) and was not touched by the current insert.
// Blocks that become candidates inside the program (a release to ref 0, an
// unpin, a tag restore, a ref -1 block raised to 0 by a hit) are appended as
// sorted "runs"; the next victim is the smallest valid key over the list
// head, the run heads and the current insert's late candidates — exactly
// the reference's sort by (tier, last_used, block_id) (kv_cache.cpp:184-188)
// taken one evict(1) at a time (kv_cache.cpp:147-149).
//
// Resources the program cannot see past (the list or the free-id list used
// up while unselected candidates / unlisted free ids exist, the run table
// full) stop it BEFORE the op that needs them: the walk has no global side
// effects until the op commits, so the op is simply left for the next
// program (the host re-scores and continues).  An op that fails (CacheFull
// with its rollback, or a release error) ends the program AFTER it.
#pragma once
// (included inside namespace sb)

struct ProgState {
  const ProgOp* ops;
  ProgRes* res;
  int32_t n_ops;
  int32_t first;          // first op of this launch
  int32_t* pin_cnt;       // engine pin counts per block (engine.hpp:187), may be null for PK_INSERT only
  int8_t* real_tag;       // engine real tags per block (engine.hpp:188), -1 = none
  uint64_t* runk;         // storage of the candidate runs
  int64_t runk_cap;
  int64_t* out;           // [0] next op to run, [1] stop kind, [2] evictions, [3] inserted blocks
  int64_t now;
  const int32_t* pre_all; // pre-program probe result of every insert position (k_prog_bound)
  unsigned long long* created;  // chain hashes of blocks created by this program (open addressing, 0 = empty)
  int64_t created_mask;
  unsigned long long* prof;     // SB_PROG_PROFILE: cycles per program phase (thread 0), else null
  const int64_t* skip;          // non-null and set: the parallel path (pool_batch.cuh) applied the program
};
// phase clock (thread 0, at barrier points): cycles since the previous mark
#define PROG_T(k)                                                    \
  do {                                                               \
    if (G.prof && threadIdx.x == 0) {                                \
      const unsigned long long c_ = clock64();                       \
      G.prof[sh.pkind * 11 + (k)] += c_ - sh.tlast;                  \
      sh.tlast = c_;                                                 \
    }                                                                \
  } while (0)

constexpr int kProgThreads = 1024;
constexpr int kSetSlots = 16384;   // per-insert "touched" id set (evicted or referenced), shared memory
constexpr int kRunMax = 512;       // candidate runs
constexpr int kRunBuf = 2048;      // keys per run (one sort in shared memory)
constexpr int kProgMaxPos = kSetSlots / 2;  // block positions of one insert
// dynamic shared memory: touched-id set | run sort buffer | per-position id,
// probe list, kind
constexpr int kWin = 2048;  // list entries pre-validated per insert (victim window)
constexpr int kTagSmem = 256;  // insert tag ranges staged in shared memory
constexpr size_t kProgSmem = kSetSlots * sizeof(int32_t) + kRunBuf * sizeof(uint64_t) +
                             kWin * (sizeof(uint64_t) + sizeof(int32_t)) +
                             kProgMaxPos * (2 * sizeof(int32_t) + sizeof(int8_t));

struct ProgShared {
  uint64_t run_head[kRunMax];  // key at the head of each run (kNoKey: exhausted)
  int64_t run_pos[kRunMax], run_end[kRunMax];
  uint64_t lkey[kLateMax];
  uint64_t wtmp[32];
  int32_t lpos[kLateMax];
  int64_t K, F, ncand0, free0, list_ptr, free_ptr, runk_used;
  int64_t nev, nnew, failpos;
  unsigned long long err;
  int n_runs, n_late, status, stop, n_sort, sort_overflow, n_probe;
  // victim window of the current insert: valid list entries [win_beg, win_end)
  // compacted in list order into wkey / widx, consumed from wptr
  int64_t win_end;
  unsigned long long tlast;
  int pkind;
  int nwin, wptr, nm;
  uint32_t warp_sums[33];
  sb_tag_range tags_s[kTagSmem];
};

__device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
__device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }

__device__ __forceinline__ uint32_t set_hash(int32_t id) {
  return (static_cast<uint32_t>(id) * 0x9E3779B1u) >> (32 - 14);  // kSetSlots = 2^14
}
__device__ __forceinline__ bool set_has(const int32_t* set, int32_t id) {
  uint32_t s = set_hash(id);
  for (;;) {
    const int32_t v = set[s];
    if (v == id) return true;
    if (v == -1) return false;
    s = (s + 1) & (kSetSlots - 1);
  }
}
__device__ __forceinline__ void set_add(int32_t* set, int32_t id) {
  uint32_t s = set_hash(id);
  for (;;) {
    const int32_t v = atomicCAS(&set[s], -1, id);
    if (v == -1 || v == id) return;
    s = (s + 1) & (kSetSlots - 1);
  }
}

// Chain hashes of blocks this program created: a pre-program probe result
// may be stale only for those (a miss may now hit one; a hit's id may hold a
// re-created block), every other position's pre-program result stands.
__device__ __forceinline__ bool created_has(const ProgState& G, uint64_t h) {
  if (h == 0) return true;  // 0 marks an empty slot: never trust the hint
  uint64_t s = (h ^ (h >> 31)) & static_cast<uint64_t>(G.created_mask);
  for (;;) {
    const unsigned long long v = G.created[s];
    if (v == h) return true;
    if (v == 0) return false;
    s = (s + 1) & static_cast<uint64_t>(G.created_mask);
  }
}
__device__ __forceinline__ void created_add(const ProgState& G, uint64_t h) {
  if (h == 0) return;
  uint64_t s = (h ^ (h >> 31)) & static_cast<uint64_t>(G.created_mask);
  for (;;) {
    const unsigned long long v = atomicCAS(&G.created[s], 0ull, static_cast<unsigned long long>(h));
    if (v == 0 || v == h) return;
    s = (s + 1) & static_cast<uint64_t>(G.created_mask);
  }
}

// Still a candidate with exactly this key (the pool state; constant during
// one insert's walk).
__device__ __forceinline__ bool victim_valid_g(const Pool& P, uint64_t k) {
  const int32_t id = static_cast<int32_t>(k & P.idmask);
  if (P.ntok[id] <= 0 || P.ref[id] != 0 || P.pinned[id] != 0) return false;
  return victim_key(P, id) == k;
}
// ... and not touched by the current insert.
__device__ __forceinline__ bool victim_valid(const Pool& P, const int32_t* set, uint64_t k) {
  return victim_valid_g(P, k) && !set_has(set, static_cast<int32_t>(k & P.idmask));
}

// Engine::pin_partial's tag_at: first range containing pos, else USER_QUERY
// (engine.cpp:267-272).
__device__ __forceinline__ int engine_tag_at(const sb_tag_range* tags, int64_t ntags, int64_t pos) {
  for (int64_t r = 0; r < ntags; ++r)
    if (pos >= tags[r].begin && pos < tags[r].end) return tags[r].tag;
  return SB_TAG_USER_QUERY;
}

// ---- candidate runs ---------------------------------------------------
// Phase protocol: threads call prog_push(key) for blocks that just became
// candidates; after a __syncthreads the CTA calls prog_flush(), which sorts
// the pushed keys and registers them as one run.
__device__ __forceinline__ void prog_push(ProgShared& sh, uint64_t* buf, uint64_t key) {
  const int at = atomicAdd(&sh.n_sort, 1);
  if (at < kRunBuf) buf[at] = key;
  else sh.sort_overflow = 1;  // callers chunk their pushes to kRunBuf; never expected
}
__device__ void prog_flush(ProgShared& sh, uint64_t* buf, const ProgState& G) {
  const int n = min(sh.n_sort, kRunBuf);
  if (n == 0) return;  // uniform (read after a barrier)
  int n2 = 1;
  while (n2 < n) n2 <<= 1;
  for (int i = n + threadIdx.x; i < n2; i += blockDim.x) buf[i] = kNoKey;
  __syncthreads();
  bitonic_smem(buf, n2);
  __syncthreads();
  const int64_t base = sh.runk_used;
  for (int i = threadIdx.x; i < n; i += blockDim.x) G.runk[base + i] = buf[i];
  if (threadIdx.x == 0) {
    const int r = sh.n_runs++;
    sh.run_pos[r] = base;
    sh.run_end[r] = base + n;
    sh.run_head[r] = buf[0];
    sh.runk_used = base + n;
    sh.n_sort = 0;
  }
  __syncthreads();
}

// ---- the walk's next victim (warp 0, all lanes, uniform) ---------------
// Returns a block id, or -1 (no candidate left: CacheFull), or -2 (the
// smallest candidate cannot be decided from what the program holds: stop).
// *late_i receives the late-list index when the victim came from there.
__device__ int32_t prog_pop(const Pool& P, const Scratch& S, const int32_t* set, const uint64_t* wkey,
                            const int32_t* widx, ProgShared& sh, const ProgState& G, int* late_i) {
  const int lane = threadIdx.x & 31;
  *late_i = -1;
  for (;;) {
    // list head: the insert's pre-validated window first, then the list
    // beyond it validated here
    uint64_t lk = kNoKey;
    int from_win = 0;
    if (lane == 0) {
      while (sh.wptr < sh.nwin) {
        const uint64_t k = wkey[sh.wptr];
        if (!set_has(set, static_cast<int32_t>(k & P.idmask))) {
          lk = k;
          from_win = 1;
          break;
        }
        ++sh.wptr;
      }
      if (!from_win) {
        int64_t p = max64(sh.list_ptr, sh.win_end);
        while (p < sh.K) {
          const uint64_t k = S.victims[p];
          if (victim_valid(P, set, k)) {
            lk = k;
            break;
          }
          ++p;
        }
        sh.list_ptr = p;
      }
    }
    lk = __shfl_sync(0xffffffffu, lk, 0);
    from_win = __shfl_sync(0xffffffffu, from_win, 0);
    // run heads (keys cached in shared memory, validated when chosen)
    uint64_t rk = kNoKey;
    int rr = -1;
    for (int r = lane; r < sh.n_runs; r += 32)
      if (sh.run_head[r] < rk) {
        rk = sh.run_head[r];
        rr = r;
      }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const uint64_t ok = __shfl_xor_sync(0xffffffffu, rk, o);
      const int orr = __shfl_xor_sync(0xffffffffu, rr, o);
      if (ok < rk || (ok == rk && orr < rr && orr >= 0)) {
        rk = ok;
        rr = orr;
      }
    }
    // late candidates of the current insert
    uint64_t tk = kNoKey;
    int ti = -1;
    if (lane == 0)
      for (int i = 0; i < sh.n_late; ++i)
        if (sh.lkey[i] < tk) {
          tk = sh.lkey[i];
          ti = i;
        }
    tk = __shfl_sync(0xffffffffu, tk, 0);
    ti = __shfl_sync(0xffffffffu, ti, 0);
    const uint64_t best = min(lk, min(rk, tk));
    const bool list_short = lk == kNoKey && sh.K < sh.ncand0;  // list used up, unselected candidates exist
    if (best == kNoKey) return list_short ? -2 : -1;
    // every unselected candidate's key is above the last selected one
    if (list_short && (sh.K == 0 || best > S.victims[sh.K - 1])) return -2;
    if (best == lk) {
      if (lane == 0) {
        if (from_win) {
          sh.list_ptr = widx[sh.wptr] + 1;
          sh.wptr += 1;
        } else {
          sh.list_ptr += 1;
        }
      }
      __syncwarp();
      return static_cast<int32_t>(lk & P.idmask);
    }
    if (best == tk) {
      *late_i = ti;
      if (lane == 0) {
        sh.lkey[ti] = kNoKey;  // consumed
      }
      __syncwarp();
      return static_cast<int32_t>(tk & P.idmask);
    }
    // a run head: validate it, advance the run either way
    bool ok = false;
    if (lane == 0) {
      ok = victim_valid(P, set, rk);
      const int64_t np = ++sh.run_pos[rr];
      sh.run_head[rr] = np < sh.run_end[rr] ? G.runk[np] : kNoKey;
    }
    ok = __shfl_sync(0xffffffffu, ok, 0);
    __syncwarp();
    if (ok) return static_cast<int32_t>(rk & P.idmask);
  }
}

// ---- one insert (KvCache::insert, kv_cache.cpp:103-175), whole CTA -------
// Returns the status; sh.stop = PS_BEFORE when the op must be left for the
// next program (no global state was modified).
__device__ int prog_insert(const Pool& P, const Scratch& S, const ProgState& G, ProgShared& sh, int32_t* set,
                           uint64_t* buf, uint64_t* wkey, int32_t* widx, int32_t* pb, int8_t* pk, int32_t* pprobe,
                           const ProgOp& op, const sb_tag_range* tags, int64_t ntags) {
  const int t = threadIdx.x, lane = t & 31;
  const int64_t n = op.n;
  const int64_t Pn = (n + P.bs - 1) / P.bs;
  const int64_t now = G.now;
  // the insert's tag ranges, staged in shared memory when they fit
  if (ntags <= kTagSmem) {
    for (int64_t i = t; i < ntags; i += blockDim.x) sh.tags_s[i] = tags[i];
    __syncthreads();
    tags = sh.tags_s;
  }
  // tag coverage (kv_cache.cpp:105-115): a CacheError with no effect
  if (!tags_cover(tags, ntags, n)) return SB_ERR_CACHE;
  if (Pn == 0) return SB_OK;
  for (int i = t; i < kSetSlots; i += blockDim.x) set[i] = -1;
  if (t == 0) {
    sh.n_late = 0;
    sh.nev = 0;
    sh.nnew = 0;
    sh.failpos = -1;
    sh.status = SB_OK;
  }
  // block of every position: the pre-program probe result (k_prog_bound),
  // re-probed against the live index only where this program may have
  // changed the answer (positions of one insert never match blocks created
  // by the same insert)
  if (t == 0) sh.n_probe = 0;
  __syncthreads();
  PROG_T(0);
  for (int64_t p = t; p < Pn; p += blockDim.x) {
    const int64_t off = p * P.bs;
    const int len = static_cast<int>(min(P.bs, n - off));
    const uint64_t h = op.hashes[p];
    const uint64_t par = p ? op.hashes[p - 1] : kRootHash;
    int32_t b = G.pre_all[op.pos_off + p];
    bool probe = created_has(G, h);
    if (b >= 0 && !(P.ntok[b] == len && P.chain[b] == h && P.parent[b] == par)) probe = true;  // evicted / reused
    if (probe) {
      pprobe[atomicAdd(&sh.n_probe, 1)] = static_cast<int32_t>(p);
      b = -1;
    }
    pb[p] = b;
  }
  __syncthreads();
  PROG_T(1);
  {
    const int pair = t >> 1, part = t & 1;
    const int pairs = blockDim.x >> 1;
    const int np = sh.n_probe;
    for (int base = 0; base < np; base += pairs) {
      const int i = base + pair;
      const bool active = i < np;
      const int64_t pc = active ? pprobe[i] : pprobe[np - 1];
      const int64_t off = pc * P.bs;
      const int len = static_cast<int>(min(P.bs, n - off));
      const uint64_t h = op.hashes[pc];
      const uint64_t parent = pc ? op.hashes[pc - 1] : kRootHash;
      const int32_t b = P.bs == 16 ? probe_find_g<true>(P, active, h, parent, op.tokens + off, len, part)
                                   : probe_find_g<false>(P, active, h, parent, op.tokens + off, len, part);
      if (active && part == 0) pb[pc] = b;
    }
  }
  __syncthreads();
  PROG_T(2);
  if (t == 0) sh.nm = 0;
  __syncthreads();
  for (int64_t p0 = 0; p0 < Pn; p0 += blockDim.x) {  // warp-uniform trip count
    const int64_t p = p0 + t;
    int8_t fl = 0;  // 1: candidate, 2: late (ref -1, reachable through duplicate releases)
    int w = 0;      // victims this position may consume
    if (p < Pn) {
      const int32_t b = pb[p];
      if (b >= 0 && P.pinned[b] == 0) {
        const int32_t rf = P.ref[b];
        fl = rf == 0 ? 1 : (rf == -1 ? 2 : 0);
      }
      pk[p] = fl;
      w = b < 0 ? 1 : (fl == 1 ? 2 : 0);
    }
    w = __reduce_add_sync(0xffffffffu, w);
    if ((t & 31) == 0 && w) atomicAdd(&sh.nm, w);
  }
  __syncthreads();
  PROG_T(3);
  // victim window: the list entries this insert's walk may take, validated
  // against the pool state (which the walk does not change) by every thread
  // and compacted in list order
  {
    const int64_t ptr0 = sh.list_ptr;
    const int W = static_cast<int>(min64(min64(sh.K - ptr0, kWin), sh.nm > 0 ? sh.nm + 32 : 0));
    uint32_t* flag = reinterpret_cast<uint32_t*>(buf);  // run buffer unused until the commit
    uint64_t k0 = kNoKey, k1 = kNoKey;
    uint32_t f0 = 0, f1 = 0;
    if (W > 0) {
      if (2 * t < W) {
        k0 = S.victims[ptr0 + 2 * t];
        f0 = victim_valid_g(P, k0);
      }
      if (2 * t + 1 < W) {
        k1 = S.victims[ptr0 + 2 * t + 1];
        f1 = victim_valid_g(P, k1);
      }
      flag[2 * t] = f0;
      flag[2 * t + 1] = f1;
      __syncthreads();
      const uint32_t total = block_scan_2048(flag, sh.warp_sums);
      if (f0) {
        wkey[flag[2 * t]] = k0;
        widx[flag[2 * t]] = static_cast<int32_t>(ptr0 + 2 * t);
      }
      if (f1) {
        wkey[flag[2 * t + 1]] = k1;
        widx[flag[2 * t + 1]] = static_cast<int32_t>(ptr0 + 2 * t + 1);
      }
      if (t == 0) sh.nwin = static_cast<int>(total);
    } else if (t == 0) {
      sh.nwin = 0;
    }
    if (t == 0) {
      sh.wptr = 0;
      sh.win_end = ptr0 + max(W, 0);
    }
  }
  __syncthreads();
  PROG_T(4);
  // ---- the walk: warp 0 replays the sequential decisions
  if (t < 32) {
    const uint64_t now_bits = static_cast<uint64_t>(now + P.lbias) << P.idb;
    int64_t fi = sh.free_ptr;
    int status = SB_OK, stop = PS_NONE;
    int64_t nev = 0, nnew = 0, failpos = -1;
    for (int64_t p0 = 0; p0 < Pn && status == SB_OK && stop == PS_NONE; p0 += 32) {
      const int64_t p = p0 + lane;
      const int cnt = static_cast<int>(min64(32, Pn - p0));
      int32_t b = -1;
      int8_t fl = 0;
      if (p < Pn) {
        b = pb[p];
        fl = pk[p];
      }
      // a candidate hit may have been evicted earlier in this insert
      const bool touched = b >= 0 && fl == 1 && set_has(set, b);
      // leading positions that need no decision: hits on non-candidates and
      // hits on candidates not evicted earlier in this insert (no eviction
      // happens among them, so their order does not matter; referenced
      // candidates are marked so no later miss of this insert evicts them)
      const bool easy_hit = lane < cnt && b >= 0 && (fl == 0 || (fl == 1 && !touched));
      const unsigned hard = __ballot_sync(0xffffffffu, lane < cnt && !easy_hit);
      const int m = hard ? __ffs(hard) - 1 : cnt;
      if (lane < m) {
        pk[p] = 0;
        pb[p] = b;
        if (fl == 1) set_add(set, b);
      }
      __syncwarp();
      if (m == cnt) continue;
      const bool runs_live = __shfl_sync(0xffffffffu, sh.n_runs, 0) > 0;
      const bool miss = lane < m || lane >= cnt || b < 0;
      if (__all_sync(0xffffffffu, miss) && sh.n_late == 0 && !runs_live) {
        // positions m.. all miss: the i-th takes the next free id, else the
        // next valid list victim — all lanes at once
        const int nm = cnt - m, mi = lane - m;  // misses, this lane's miss index
        const int64_t a = min64(nm, max64(0, sh.F - fi));
        int32_t id = -1;
        if (mi >= 0 && mi < a) id = S.freel[fi + mi];
        int64_t need = nm - a, got = 0;
        const bool free_short = need > 0 && sh.F < sh.free0;  // unlisted free ids: cannot decide
        if (free_short) {
          stop = PS_BEFORE;
          break;
        }
        while (got < need) {
          // the next 32 candidates in list order: window entries (validated
          // before the walk; only this insert's touched set is checked), then
          // list entries beyond the window, validated here
          const bool win = sh.wptr < sh.nwin;
          const int64_t base = win ? sh.wptr : max64(sh.list_ptr, sh.win_end);
          const int64_t lim = win ? sh.nwin : sh.K;
          if (base >= lim) break;
          const int64_t e = base + lane;
          uint64_t k = kNoKey;
          bool v = false;
          if (e < lim) {
            k = win ? wkey[e] : S.victims[e];
            v = win ? !set_has(set, static_cast<int32_t>(k & P.idmask)) : victim_valid(P, set, k);
          }
          const unsigned bal = __ballot_sync(0xffffffffu, v);
          const int rk = __popc(bal & ((1u << lane) - 1));
          const int take = static_cast<int>(min64(__popc(bal), need - got));
          if (v && rk < take) sh.wtmp[rk] = k;
          __syncwarp();
          const int r = mi - static_cast<int>(a + got);
          if (mi >= 0 && r >= 0 && r < take) id = static_cast<int32_t>(sh.wtmp[r] & P.idmask);
          const unsigned last = __ballot_sync(0xffffffffu, v && rk == take - 1);
          const int64_t next = (take > 0 && take < __popc(bal)) ? base + (__ffs(last) - 1) + 1 : min64(base + 32, lim);
          if (lane == 0) {
            if (win) {
              if (take > 0) sh.list_ptr = widx[base + (__ffs(last) - 1)] + 1;
              sh.wptr = static_cast<int>(next);
            } else {
              sh.list_ptr = next;
            }
          }
          got += take;
          __syncwarp();
        }
        int64_t nok = nm;
        if (got < need) {
          if (sh.K < sh.ncand0) {  // unselected candidates: cannot decide
            stop = PS_BEFORE;
            break;
          }
          nok = a + got;  // CacheFull at the first unassigned miss
          status = SB_ERR_CACHE_FULL;
          failpos = p0 + m + nok;
        }
        if (mi >= 0 && mi < nok) {
          pk[p] = 1;
          pb[p] = id;
          if (mi >= a) {
            set_add(set, id);
            S.evicted[nev + (mi - a)] = id;
          }
        }
        nev += max64(0, nok - a);
        nnew += nok;
        fi += min64(nok, a);
        __syncwarp();
        continue;
      }
      // general path: position by position (warp-uniform loop)
      for (int i = m; i < cnt; ++i) {
        const int32_t bb = __shfl_sync(0xffffffffu, b, i);
        const int8_t ff = static_cast<int8_t>(__shfl_sync(0xffffffffu, static_cast<int>(fl), i));
        const bool tt = __shfl_sync(0xffffffffu, touched, i);
        const int64_t q = p0 + i;
        bool ms = bb < 0;
        if (!ms && ff == 1 && (tt || set_has(set, bb))) ms = true;  // evicted earlier in this insert
        if (!ms) {
          if (lane == 0) {
            if (ff == 1) set_add(set, bb);  // referenced: no longer a candidate
            if (ff == 2 && sh.n_late < kLateMax) {
              uint64_t k = now_bits | static_cast<uint64_t>(bb);
              if (P.policy == SB_POLICY_TIERED) k |= static_cast<uint64_t>(tier_of(P.tag[bb])) << 61;
              sh.lkey[sh.n_late] = k;
              sh.lpos[sh.n_late] = static_cast<int32_t>(q);
              sh.n_late += 1;
            }
            pk[q] = 0;
            pb[q] = bb;
          }
          __syncwarp();
          continue;
        }
        int32_t id = -1;
        if (fi < sh.F) {
          if (lane == 0) id = S.freel[fi];
          id = __shfl_sync(0xffffffffu, id, 0);
          ++fi;
        } else {
          if (sh.F < sh.free0) {
            stop = PS_BEFORE;
            break;
          }
          int li = -1;
          id = prog_pop(P, S, set, wkey, widx, sh, G, &li);
          if (id == -2) {
            stop = PS_BEFORE;
            break;
          }
          if (id == -1) {
            status = SB_ERR_CACHE_FULL;
            failpos = q;
            break;
          }
          if (lane == 0) {
            if (li >= 0) pk[sh.lpos[li]] = 2;  // hit, then evicted later in this insert
            set_add(set, id);
            S.evicted[nev] = id;
          }
          ++nev;
        }
        if (lane == 0) {
          pk[q] = 1;
          pb[q] = id;
        }
        ++nnew;
        __syncwarp();
      }
    }
    if (lane == 0) {
      sh.nev = nev;
      sh.nnew = nnew;
      sh.failpos = failpos;
      sh.status = status;
      sh.stop = stop;
      if (stop == PS_NONE && status == SB_OK) sh.free_ptr = fi;
    }
  }
  __syncthreads();
  PROG_T(5);
  if (sh.stop != PS_NONE) return SB_OK;
  const int status = sh.status;
  const int64_t nev = sh.nev;
  // ---- commit: evictions first (their index slots become tombstones)
  for (int64_t i = t; i < nev; i += blockDim.x) {
    const int32_t v = S.evicted[i];
    P.idx[P.slot[v]].id = -2;
    P.ntok[v] = 0;
  }
  __syncthreads();
  PROG_T(6);
  const int64_t limit = status == SB_OK ? Pn : sh.failpos;
  for (int64_t p = t; p < Pn; p += blockDim.x) {
    if (p < limit) {
      const int kd = pk[p];
      const int32_t id = pb[p];
      if (kd == 0) {
        if (status == SB_OK) P.ref[id] += 1;  // distinct blocks per position
        P.last[id] = now;
      } else if (kd == 1 && status == SB_OK) {
        const int64_t off = p * P.bs;
        const int len = static_cast<int>(min(P.bs, n - off));
        uint64_t* dst = P.tok + static_cast<int64_t>(id) * P.bs;
        if (len == 16) {  // all loads in flight before the stores
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
        P.ref[id] = 1;
        P.last[id] = now;
        P.pinned[id] = 0;
        index_insert(P, h, id, par, len);
        created_add(G, h);
      }
    }
    op.ids[p] = status == SB_OK ? pb[p] : -1;
  }
  if (t == 0) {
    if (nev > 0) {
      P.ctr[C_NRES] -= static_cast<unsigned long long>(nev);
      P.ctr[C_EVICTED] += static_cast<unsigned long long>(nev);
      P.ctr[C_EV_BLOCKS] += static_cast<unsigned long long>(nev);
    }
    if (status == SB_OK) {
      P.ctr[C_NRES] += static_cast<unsigned long long>(sh.nnew);
      P.ctr[C_INS_BLOCKS] += static_cast<unsigned long long>(sh.nnew);
    } else {
      P.ctr[C_FULL] += 1ull;
    }
    G.out[2] += nev;
    G.out[3] += status == SB_OK ? sh.nnew : 0;
  }
  __syncthreads();
  PROG_T(7);
  // late candidates raised to ref 0 and not evicted are candidates from now on
  if (status == SB_OK) {
    if (t < sh.n_late && sh.lkey[t] != kNoKey) {
      const int32_t id = static_cast<int32_t>(sh.lkey[t] & P.idmask);
      if (P.ntok[id] > 0 && P.ref[id] == 0 && P.pinned[id] == 0) prog_push(sh, buf, victim_key(P, id));
    }
    __syncthreads();
    prog_flush(sh, buf, G);
  }
  PROG_T(8);
  (void)lane;
  return status;
}

// KvCache::release (kv_cache.cpp:228-236): all ids validated first (first
// failing id in order decides UnknownBlock / ZeroRefRelease), then each
// decremented; blocks reaching ref 0 unpinned become candidates.
__device__ int prog_release(const Pool& P, const ProgState& G, ProgShared& sh, uint64_t* buf, const int32_t* ids,
                            int64_t m) {
  const int t = threadIdx.x;
  if (t == 0) sh.err = ~0ull;
  __syncthreads();
  for (int64_t i = t; i < m; i += blockDim.x) {
    const int32_t id = ids[i];
    const bool known = id >= 0 && id < P.cap && P.ntok[id] > 0;
    if (!known) atomicMin(&sh.err, static_cast<unsigned long long>(2 * i));
    else if (P.ref[id] < 1) atomicMin(&sh.err, static_cast<unsigned long long>(2 * i + 1));
  }
  __syncthreads();
  const unsigned long long err = sh.err;
  if (err != ~0ull) return (err & 1) ? SB_ERR_ZERO_REF_RELEASE : SB_ERR_UNKNOWN_BLOCK;
  for (int64_t c0 = 0; c0 < m; c0 += kRunBuf) {
    for (int64_t i = c0 + t; i < min64(m, c0 + kRunBuf); i += blockDim.x) {
      const int32_t id = ids[i];
      const int old = atomicSub(&P.ref[id], 1);
      if (old == 1 && P.pinned[id] == 0) prog_push(sh, buf, victim_key(P, id));
    }
    __syncthreads();
    prog_flush(sh, buf, G);
  }
  return SB_OK;
}

// Engine::release_partial_pins (engine.cpp:288-303).
__device__ void prog_unpin(const Pool& P, const ProgState& G, ProgShared& sh, uint64_t* buf, const int32_t* ids,
                           int64_t m) {
  const int t = threadIdx.x;
  for (int64_t c0 = 0; c0 < m; c0 += kRunBuf) {
    for (int64_t i = c0 + t; i < min64(m, c0 + kRunBuf); i += blockDim.x) {
      const int32_t id = ids[i];
      if (id < 0 || id >= P.cap) continue;
      const int c = G.pin_cnt[id];
      if (c <= 0) continue;  // not in the pin map
      G.pin_cnt[id] = c - 1;  // pinned ids of one call are distinct
      if (c - 1 > 0) continue;
      if (P.ntok[id] > 0) {
        P.pinned[id] = 0;
        const int rt = G.real_tag[id];
        if (rt >= 0) P.tag[id] = rt;
        if (P.ref[id] == 0) prog_push(sh, buf, victim_key(P, id));
      }
      G.real_tag[id] = -1;
    }
    __syncthreads();
    prog_flush(sh, buf, G);
  }
}

__global__ void __launch_bounds__(kProgThreads, 1) k_program(Pool P, Scratch S, ProgState G) {
  extern __shared__ __align__(16) uint8_t prog_dyn[];
  int32_t* set = reinterpret_cast<int32_t*>(prog_dyn);
  uint64_t* buf = reinterpret_cast<uint64_t*>(prog_dyn + kSetSlots * sizeof(int32_t));
  uint64_t* wkey = buf + kRunBuf;                            // victim window keys
  int32_t* widx = reinterpret_cast<int32_t*>(wkey + kWin);   // ... and their list positions
  int32_t* pb = widx + kWin;                                 // per position: block (after the walk: the chain id)
  int32_t* pprobe = pb + kProgMaxPos;                       // positions to re-probe
  int8_t* pk = reinterpret_cast<int8_t*>(pprobe + kProgMaxPos);  // per position: candidacy, then kind
  __shared__ ProgShared sh;
  __shared__ sb_tag_range pin_range;
  const int t = threadIdx.x;
  if (G.skip && *G.skip) return;
  if (t == 0) {
    sh.K = S.scal[S_K];
    sh.F = S.scal[S_FREE];
    sh.ncand0 = S.scal[S_NCAND];
    sh.free0 = P.cap - static_cast<int64_t>(P.ctr[C_NRES]);
    sh.list_ptr = 0;
    sh.free_ptr = 0;
    sh.runk_used = 0;
    sh.n_runs = 0;
    sh.n_sort = 0;
    sh.sort_overflow = 0;
    sh.stop = PS_NONE;
    sh.n_late = 0;
    sh.tlast = clock64();
  }
  __syncthreads();
  int c = G.first;
  for (; c < G.n_ops; ++c) {
    const ProgOp op = G.ops[c];
    const int64_t Pn = (op.n + P.bs - 1) / P.bs;
    if (t == 0) sh.pkind = op.kind;
    // resources this op may need: runs and run storage (worst case)
    const int64_t pushes = (op.kind == PK_INSERT ? 0 : op.n_chain + op.n_pinned + Pn) + kLateMax;
    const int64_t runs_needed = 3 + (pushes + kRunBuf - 1) / kRunBuf * 2;
    if (t == 0 && sh.n_runs + runs_needed > kRunMax) {  // drop exhausted runs
      int w = 0;
      for (int r = 0; r < sh.n_runs; ++r)
        if (sh.run_head[r] != kNoKey) {
          sh.run_head[w] = sh.run_head[r];
          sh.run_pos[w] = sh.run_pos[r];
          sh.run_end[w] = sh.run_end[r];
          ++w;
        }
      sh.n_runs = w;
    }
    __syncthreads();
    if (sh.n_runs + runs_needed > kRunMax || sh.runk_used + pushes + kRunBuf > G.runk_cap || Pn > kProgMaxPos ||
        Pn > S.pmax) {
      break;  // left for the next program
    }
    PROG_T(9);
    ProgRes r{SB_OK, PO_NONE, op.n_chain, op.n_pinned};
    int stop_after = 0;
    const bool inserts = op.kind != PK_ABANDON;
    int ist = SB_OK;
    if (inserts) {
      const sb_tag_range* tg = op.ins_tags;
      int64_t ntg = op.n_ins_tags;
      if (op.kind == PK_PIN) {  // one PARTIAL_PREFILL range over the prefix (engine.cpp:251-252)
        if (t == 0) pin_range = sb_tag_range{0, op.n, SB_TAG_PARTIAL_PREFILL, 0};
        __syncthreads();
        tg = &pin_range;
        ntg = 1;
      }
      ist = prog_insert(P, S, G, sh, set, buf, wkey, widx, pb, pk, pprobe, op, tg, ntg);
      if (sh.stop == PS_BEFORE) break;
      if (ist == SB_ERR_CACHE_FULL) stop_after = 1;
    }
    switch (op.kind) {
      case PK_INSERT:
        r.status = ist;
        break;
      case PK_PIN:
        if (ist == SB_OK) {
          for (int64_t i = t; i < Pn; i += blockDim.x) {
            const int32_t id = op.ids[i];
            const int old = G.pin_cnt[id];
            G.pin_cnt[id] = old + 1;
            if (old == 0) {
              const int cur = P.tag[id];
              G.real_tag[id] = static_cast<int8_t>(
                  cur != SB_TAG_PARTIAL_PREFILL ? cur : engine_tag_at(op.real_tags, op.n_real_tags, i * P.bs));
            }
            P.pinned[id] = 1;
            P.tag[id] = SB_TAG_PARTIAL_PREFILL;
            op.chain[i] = id;
            op.pinned[i] = id;
          }
          r.n_chain = static_cast<int32_t>(Pn);
          r.n_pinned = static_cast<int32_t>(Pn);
          r.outcome = PO_PINNED;
        } else {
          r.status = ist;
          r.outcome = PO_PIN_FAILED;
        }
        break;
      case PK_COMPLETE: {
        if (op.n_pinned > 0) prog_unpin(P, G, sh, buf, op.pinned, op.n_pinned);
        r.n_pinned = 0;
        if (op.n_chain > 0) {
          const int rs = prog_release(P, G, sh, buf, op.chain, op.n_chain);
          if (rs != SB_OK) {
            r.status = rs;
            stop_after = 2;
          }
        }
        __syncthreads();
        if (ist == SB_OK) {
          for (int64_t i = t; i < Pn; i += blockDim.x) op.chain[i] = op.ids[i];
          r.n_chain = static_cast<int32_t>(Pn);
        } else {
          r.n_chain = 0;
          if (r.status == SB_OK) r.status = ist;
        }
        r.outcome = PO_COMPLETED;
        break;
      }
      case PK_FINISH: {
        if (ist == SB_OK) {
          const int rs = prog_release(P, G, sh, buf, op.ids, Pn);
          if (rs != SB_OK) {
            r.status = rs;
            stop_after = 2;
          }
        } else {
          r.status = ist;
        }
        if (stop_after != 2) {
          if (op.n_chain > 0) {
            const int rs = prog_release(P, G, sh, buf, op.chain, op.n_chain);
            if (rs != SB_OK) {
              r.status = rs;
              stop_after = 2;
            }
          }
        }
        r.n_chain = 0;
        r.outcome = PO_FINISHED;
        break;
      }
      case PK_ABANDON: {
        if (op.n_pinned > 0) prog_unpin(P, G, sh, buf, op.pinned, op.n_pinned);
        r.n_pinned = 0;
        if (op.n_chain > 0) {
          const int rs = prog_release(P, G, sh, buf, op.chain, op.n_chain);
          if (rs != SB_OK) {
            r.status = rs;
            stop_after = 2;
          }
        }
        r.n_chain = 0;
        r.outcome = PO_ABANDONED;
        break;
      }
      default:
        r.status = SB_ERR_INVALID;
        stop_after = 2;
    }
    __syncthreads();
    PROG_T(10);
    if (t == 0) G.res[c] = r;
    if (stop_after) {
      if (t == 0) sh.stop = stop_after == 2 ? PS_ERROR : PS_AFTER;
      ++c;
      break;
    }
  }
  __syncthreads();
  // select's rank marks (S.rank_of, read only by the per-insert path)
  for (int64_t i = t; i < sh.K; i += blockDim.x) S.rank_of[S.victims[i] & P.idmask] = -1;
  if (t == 0) {
    G.out[0] = c;
    G.out[1] = sh.stop;
  }
}

// Pre-program probe of every insert position (kept for the program as a
// hint) and the bound of the victims / free ids the program can consume:
// every position that misses in the pre-program state, plus twice every
// position that hits a current candidate (it may be evicted first, and its
// list entry is then skipped), plus slack — and none at all when no position
// misses (a hit can only turn into a miss after an eviction, which needs a
// miss first).  One lane pair per position.
__global__ void __launch_bounds__(256) k_prog_bound(Pool P, const ProgOp* __restrict__ ops, int first, int n_ops,
                                                    int64_t* scal, int32_t* pre_all) {
  const int o = first + blockIdx.x;
  const ProgOp op = ops[o];
  if (op.kind == PK_ABANDON) return;
  const int64_t Pn = (op.n + P.bs - 1) / P.bs;
  const int64_t p = static_cast<int64_t>(blockIdx.y) * (blockDim.x / 2) + (threadIdx.x >> 1);
  if (static_cast<int64_t>(blockIdx.y) * (blockDim.x / 2) + ((threadIdx.x & ~31) >> 1) >= Pn) return;  // warp-uniform
  const int part = threadIdx.x & 1;
  const bool active = p < Pn;
  const int64_t pc = active ? p : Pn - 1;
  const int64_t off = pc * P.bs;
  const int len = static_cast<int>(min(P.bs, op.n - off));
  const uint64_t h = op.hashes[pc];
  const uint64_t parent = pc ? op.hashes[pc - 1] : kRootHash;
  const int32_t b = P.bs == 16 ? probe_find_g<true>(P, active, h, parent, op.tokens + off, len, part)
                               : probe_find_g<false>(P, active, h, parent, op.tokens + off, len, part);
  if (!active || part) return;
  pre_all[op.pos_off + p] = b;
  if (b < 0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&scal[S_NMISS]), 1ull);
    atomicAdd(reinterpret_cast<unsigned long long*>(&scal[S_BOUND]), 1ull);
  } else if (P.pinned[b] == 0 && P.ref[b] <= 0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(&scal[S_BOUND]), 2ull);
    if (P.ref[b] < 0) atomicAdd(reinterpret_cast<unsigned long long*>(&scal[S_NLATEHIT]), 1ull);
  }
}

// ---- descriptor lookups: KvCache::lookup_prefix (kv_cache.cpp:85-101) of
// op o = (tokens, n, hashes): full blocks only, stop at the first miss,
// touch the hit prefix.  op.ids is per-op scratch for the probe results.
__global__ void __launch_bounds__(256) k_lookup_ops_probe(Pool P, const ProgOp* __restrict__ ops,
                                                          int64_t* __restrict__ first_miss) {
  const int o = blockIdx.x;
  const ProgOp op = ops[o];
  const int64_t nf = op.n / P.bs;  // a lookup never matches a partial block (kv_cache.cpp:90)
  const int64_t p = static_cast<int64_t>(blockIdx.y) * (blockDim.x / 2) + (threadIdx.x >> 1);
  if (static_cast<int64_t>(blockIdx.y) * (blockDim.x / 2) + ((threadIdx.x & ~31) >> 1) >= nf) return;
  const int part = threadIdx.x & 1;
  const bool active = p < nf;
  const int64_t pc = active ? p : nf - 1;
  const uint64_t h = op.hashes[pc];
  const uint64_t parent = pc ? op.hashes[pc - 1] : kRootHash;
  const int32_t b = P.bs == 16 ? probe_find_g<true>(P, active, h, parent, op.tokens + pc * P.bs, static_cast<int>(P.bs), part)
                               : probe_find_g<false>(P, active, h, parent, op.tokens + pc * P.bs, static_cast<int>(P.bs), part);
  if (!active || part) return;
  op.ids[p] = b;
  if (b < 0) atomicMin(reinterpret_cast<unsigned long long*>(first_miss + o), static_cast<unsigned long long>(p));
}
__global__ void k_lookup_ops_init(Pool P, const ProgOp* __restrict__ ops, int n, int64_t* first_miss) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o < n) first_miss[o] = ops[o].n / P.bs;
}
__global__ void __launch_bounds__(256) k_lookup_ops_finish(Pool P, const ProgOp* __restrict__ ops,
                                                           const int64_t* __restrict__ first_miss, int64_t now,
                                                           int64_t* __restrict__ hits) {
  const int o = blockIdx.x;
  const int64_t f = first_miss[o];
  const ProgOp op = ops[o];
  if (blockIdx.y == 0 && threadIdx.x == 0) {
    hits[o] = f * P.bs;
    atomicAdd(&P.ctr[C_LOOKUPS], 1ull);
    atomicAdd(&P.ctr[C_HIT_TOK], static_cast<unsigned long long>(f * P.bs));
    atomicAdd(&P.ctr[C_LOOK_TOK], static_cast<unsigned long long>(op.n));
  }
  for (int64_t p = static_cast<int64_t>(blockIdx.y) * blockDim.x + threadIdx.x; p < f;
       p += static_cast<int64_t>(gridDim.y) * blockDim.x)
    P.last[op.ids[p]] = now;
}

// ---- miss-free pin batches: pin_partial x n in parallel --------------------
// When no insert position of a program of PK_PIN ops misses in the
// pre-program state (k_prog_bound: S_NMISS == 0) and none hits a ref -1
// block, no insert can evict anything (a hit turns into a miss only after an
// eviction, which needs a miss first), so every op's effects commute: each
// position references its pre-probe block (ref + 1, last_used = now), every
// block gets pinned at PARTIAL_PREFILL with its pin count raised once per op,
// and a block's real tag is recorded by the FIRST op (in op order) that pins
// it from count 0 (engine.cpp:273-279) — found with an atomicMin over op
// indices.  Three grid-wide passes instead of a sequential program.
__global__ void __launch_bounds__(256) k_pin_nomiss_a(Pool P, const ProgOp* __restrict__ ops, int first,
                                                      const int32_t* __restrict__ pre_all, int32_t* first_op,
                                                      int64_t now) {
  const int o = first + blockIdx.x;
  const ProgOp op = ops[o];
  const int64_t Pn = (op.n + P.bs - 1) / P.bs;
  for (int64_t p = static_cast<int64_t>(blockIdx.y) * blockDim.x + threadIdx.x; p < Pn;
       p += static_cast<int64_t>(gridDim.y) * blockDim.x) {
    const int32_t b = pre_all[op.pos_off + p];
    atomicAdd(&P.ref[b], 1);
    P.last[b] = now;
    op.ids[p] = b;
    atomicMin(&first_op[b], o);
  }
}
__global__ void __launch_bounds__(256) k_pin_nomiss_b(Pool P, const ProgOp* __restrict__ ops, int first,
                                                      const int32_t* __restrict__ pin_cnt, const int32_t* first_op,
                                                      int8_t* real_tag) {
  const int o = first + blockIdx.x;
  const ProgOp op = ops[o];
  const int64_t Pn = (op.n + P.bs - 1) / P.bs;
  for (int64_t p = static_cast<int64_t>(blockIdx.y) * blockDim.x + threadIdx.x; p < Pn;
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
__global__ void __launch_bounds__(256) k_pin_nomiss_c(Pool P, const ProgOp* __restrict__ ops, int first,
                                                      int32_t* pin_cnt, int32_t* first_op, ProgRes* res) {
  const int o = first + blockIdx.x;
  const ProgOp op = ops[o];
  const int64_t Pn = (op.n + P.bs - 1) / P.bs;
  for (int64_t p = static_cast<int64_t>(blockIdx.y) * blockDim.x + threadIdx.x; p < Pn;
       p += static_cast<int64_t>(gridDim.y) * blockDim.x) {
    const int32_t b = op.ids[p];
    atomicAdd(&pin_cnt[b], 1);
    P.pinned[b] = 1;
    P.tag[b] = SB_TAG_PARTIAL_PREFILL;
    op.chain[p] = b;
    op.pinned[p] = b;
    first_op[b] = 0x7fffffff;
  }
  if (blockIdx.y == 0 && threadIdx.x == 0)
    res[o] = ProgRes{SB_OK, PO_PINNED, static_cast<int32_t>(Pn), static_cast<int32_t>(Pn)};
}
