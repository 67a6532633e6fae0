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
};

constexpr int kProgThreads = 1024;
constexpr int kSetSlots = 16384;   // per-insert "touched" id set (evicted or referenced), shared memory
constexpr int kRunMax = 512;       // candidate runs
constexpr int kRunBuf = 2048;      // keys per run (one sort in shared memory)
constexpr int kProgMaxPos = kSetSlots / 2;  // block positions of one insert
constexpr size_t kProgSmem = kSetSlots * sizeof(int32_t) + kRunBuf * sizeof(uint64_t);

struct ProgShared {
  uint64_t run_head[kRunMax];  // key at the head of each run (kNoKey: exhausted)
  int64_t run_pos[kRunMax], run_end[kRunMax];
  uint64_t lkey[kLateMax];
  uint64_t wtmp[32];
  int32_t lpos[kLateMax];
  int64_t K, F, ncand0, free0, list_ptr, free_ptr, runk_used;
  int64_t nev, nnew, failpos;
  unsigned long long err;
  int n_runs, n_late, status, stop, n_sort, sort_overflow;
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

// Still a candidate with exactly this key, and not touched by this insert.
__device__ __forceinline__ bool victim_valid(const Pool& P, const int32_t* set, uint64_t k) {
  const int32_t id = static_cast<int32_t>(k & P.idmask);
  if (P.ntok[id] <= 0 || P.ref[id] != 0 || P.pinned[id] != 0) return false;
  if (victim_key(P, id) != k) return false;
  return !set_has(set, id);
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
__device__ int32_t prog_pop(const Pool& P, const Scratch& S, const int32_t* set, ProgShared& sh, const ProgState& G,
                            int* late_i) {
  const int lane = threadIdx.x & 31;
  *late_i = -1;
  for (;;) {
    // list head (validated)
    uint64_t lk = kNoKey;
    if (lane == 0) {
      int64_t p = sh.list_ptr;
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
    lk = __shfl_sync(0xffffffffu, lk, 0);
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
    const bool list_short = sh.list_ptr >= sh.K && sh.K < sh.ncand0;  // unselected candidates exist
    if (best == kNoKey) return list_short ? -2 : -1;
    // every unselected candidate's key is above the last selected one
    if (list_short && (sh.K == 0 || best > S.victims[sh.K - 1])) return -2;
    if (best == lk) {
      if (lane == 0) sh.list_ptr += 1;
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
                           uint64_t* buf, const ProgOp& op, const sb_tag_range* tags, int64_t ntags) {
  const int t = threadIdx.x, lane = t & 31;
  const int64_t n = op.n;
  const int64_t Pn = (n + P.bs - 1) / P.bs;
  const int64_t now = G.now;
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
  // live probe of every position against the current index (positions of
  // one insert never match blocks created by the same insert)
  {
    const int pair = t >> 1, part = t & 1;
    const int pairs = blockDim.x >> 1;
    for (int64_t base = 0; base < Pn; base += pairs) {
      const int64_t p = base + pair;
      const bool active = p < Pn;
      const int64_t pc = active ? p : Pn - 1;
      const int64_t off = pc * P.bs;
      const int len = static_cast<int>(min(P.bs, n - off));
      const uint64_t h = op.hashes[pc];
      const uint64_t parent = pc ? op.hashes[pc - 1] : kRootHash;
      const int32_t b = P.bs == 16 ? probe_find_g<true>(P, active, h, parent, op.tokens + off, len, part)
                                   : probe_find_g<false>(P, active, h, parent, op.tokens + off, len, part);
      if (active && part == 0) {
        int8_t fl = 0;  // 1: candidate, 2: late (ref -1, reachable through duplicate releases)
        if (b >= 0 && P.pinned[b] == 0) {
          const int32_t rf = P.ref[b];
          fl = rf == 0 ? 1 : (rf == -1 ? 2 : 0);
        }
        S.prehit[p] = b;
        S.kind[p] = fl;
      }
    }
  }
  __syncthreads();
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
        b = S.prehit[p];
        fl = S.kind[p];
      }
      // a candidate hit may have been evicted earlier in this insert
      const bool touched = b >= 0 && fl == 1 && set_has(set, b);
      const bool plain = lane >= cnt || (b >= 0 && fl == 0);
      const bool miss = lane >= cnt || b < 0;
      if (__all_sync(0xffffffffu, plain)) {  // hits on non-candidates: nothing to decide
        if (lane < cnt) {
          S.kind[p] = 0;
          S.chain_out[p] = b;
        }
        continue;
      }
      const bool runs_live = __shfl_sync(0xffffffffu, sh.n_runs, 0) > 0;
      if (__all_sync(0xffffffffu, miss) && sh.n_late == 0 && !runs_live) {
        // every position misses: the i-th takes the next free id, else the
        // next valid list victim — all lanes at once
        const int64_t a = min64(cnt, max64(0, sh.F - fi));
        int32_t id = -1;
        if (lane < a) id = S.freel[fi + lane];
        int64_t need = cnt - a, got = 0;
        const bool free_short = need > 0 && sh.F < sh.free0;  // unlisted free ids: cannot decide
        if (free_short) {
          stop = PS_BEFORE;
          break;
        }
        int64_t ptr = sh.list_ptr;
        while (got < need && ptr < sh.K) {
          // lanes validate the next 32 list entries; the r-th valid one goes
          // to the (a + got + r)-th miss of the chunk
          const int64_t e = ptr + lane;
          const uint64_t k = e < sh.K ? S.victims[e] : kNoKey;
          const bool v = e < sh.K && victim_valid(P, set, k);
          const unsigned bal = __ballot_sync(0xffffffffu, v);
          const int rk = __popc(bal & ((1u << lane) - 1));
          const int take = static_cast<int>(min64(__popc(bal), need - got));
          if (v && rk < take) sh.wtmp[rk] = k;
          __syncwarp();
          const int r = lane - static_cast<int>(a + got);
          if (r >= 0 && r < take) id = static_cast<int32_t>(sh.wtmp[r] & P.idmask);
          const unsigned last = __ballot_sync(0xffffffffu, v && rk == take - 1);
          ptr = (take > 0 && take < __popc(bal)) ? ptr + (__ffs(last) - 1) + 1 : min64(ptr + 32, sh.K);
          got += take;
          __syncwarp();
        }
        int64_t nok = cnt;
        if (got < need) {
          if (sh.K < sh.ncand0) {  // unselected candidates: cannot decide
            stop = PS_BEFORE;
            break;
          }
          nok = a + got;  // CacheFull at the first unassigned miss
          status = SB_ERR_CACHE_FULL;
          failpos = p0 + nok;
        }
        if (lane < nok) {
          S.kind[p] = 1;
          S.chain_out[p] = id;
          if (lane >= a) {
            set_add(set, id);
            S.evicted[nev + (lane - a)] = id;
          }
        }
        if (lane == 0) sh.list_ptr = ptr;
        nev += max64(0, nok - a);
        nnew += nok;
        fi += min64(nok, a);
        __syncwarp();
        continue;
      }
      // general path: position by position (warp-uniform loop)
      for (int i = 0; i < cnt; ++i) {
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
            S.kind[q] = 0;
            S.chain_out[q] = bb;
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
          id = prog_pop(P, S, set, sh, G, &li);
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
            if (li >= 0) S.kind[sh.lpos[li]] = 2;  // hit, then evicted later in this insert
            set_add(set, id);
            S.evicted[nev] = id;
          }
          ++nev;
        }
        if (lane == 0) {
          S.kind[q] = 1;
          S.chain_out[q] = id;
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
  const int64_t limit = status == SB_OK ? Pn : sh.failpos;
  for (int64_t p = t; p < Pn; p += blockDim.x) {
    if (p < limit) {
      const int kd = S.kind[p];
      const int32_t id = S.chain_out[p];
      if (kd == 0) {
        if (status == SB_OK) P.ref[id] += 1;  // distinct blocks per position
        P.last[id] = now;
      } else if (kd == 1 && status == SB_OK) {
        const int64_t off = p * P.bs;
        const int len = static_cast<int>(min(P.bs, n - off));
        uint64_t* dst = P.tok + static_cast<int64_t>(id) * P.bs;
        for (int i = 0; i < len; ++i) dst[i] = op.tokens[off + i];
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
      }
    }
    op.ids[p] = status == SB_OK ? S.chain_out[p] : -1;
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
  // late candidates raised to ref 0 and not evicted are candidates from now on
  if (status == SB_OK) {
    if (t < sh.n_late && sh.lkey[t] != kNoKey) {
      const int32_t id = static_cast<int32_t>(sh.lkey[t] & P.idmask);
      if (P.ntok[id] > 0 && P.ref[id] == 0 && P.pinned[id] == 0) prog_push(sh, buf, victim_key(P, id));
    }
    __syncthreads();
    prog_flush(sh, buf, G);
  }
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
  __shared__ ProgShared sh;
  __shared__ sb_tag_range pin_range;
  const int t = threadIdx.x;
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
  }
  __syncthreads();
  int c = G.first;
  for (; c < G.n_ops; ++c) {
    const ProgOp op = G.ops[c];
    const int64_t Pn = (op.n + P.bs - 1) / P.bs;
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
      ist = prog_insert(P, S, G, sh, set, buf, op, tg, ntg);
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

// Upper bound of the victims / free ids a program can consume: every insert
// position that misses in the pre-program state, plus twice every position
// that hits a current candidate (it may be evicted first, and its list
// entry is then skipped), plus slack.  One lane pair per position.
__global__ void __launch_bounds__(256) k_prog_bound(Pool P, const ProgOp* __restrict__ ops, int first, int n_ops,
                                                    int64_t* scal) {
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
  int64_t add = 0;
  if (b < 0) add = 1;
  else if (P.pinned[b] == 0 && P.ref[b] <= 0) add = 2;
  if (add) atomicAdd(reinterpret_cast<unsigned long long*>(&scal[S_BOUND]), static_cast<unsigned long long>(add));
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
