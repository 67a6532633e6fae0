// kv_pool.cu — device-resident paged-KV block pool + prefix-indexed block
// table with hint-aware (tiered) eviction, bit-exact with the reference
// KvCache (/root/reference/proj/src/kv_cache.cpp).
//
// Layout in HBM (structure of arrays, one slot per pool block id):
//   tok[cap*bs] u64   block token contents (full-token compare on hash match)
//   ntok[cap]   i32   tokens in block, 0 = free slot
//   chain/parent[cap] u64  chain hash of the block / of its predecessor
//   tag, ref, pinned [cap] i32, last[cap] i64
//   index: open-addressed multimap chain_hash -> block id (tcap = 4*cap
//          slots, -1 empty, -2 tombstone), slot[cap] = index slot of a block
//
// One insert (kv_cache.cpp:103-175) is five stream-ordered kernels, no host
// round trip:
//   k_probe   (all positions in parallel) find the resident block of each
//             position in the PRE-insert state (chain hash + parent + tokens)
//   k_select  (1 CTA) hint-aware eviction scoring: key = (tier, last_used,
//             id) per candidate, radix-select of the K smallest, sorted
//   k_walk    (1 thread) replays the reference's sequential decisions from
//             the first pre-miss: hit / allocate lowest free id / evict the
//             next victim (skipping blocks hit earlier in this insert) /
//             CacheFull with rollback
//   k_commit_evict, k_commit_apply  apply evictions, then hits + new blocks
// Chain hashes are computed by k_chain_hash (one thread per sequence; the
// hash is a sequential fold over tokens) or supplied precomputed.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include <cooperative_groups.h>

#include "common.h"
#include "hash.cuh"
#include "sm100.cuh"
#include "program.h"

namespace sb {

// Victim keys pack (tier:3 | last_used + bias | block id) into 64 bits, so
// one unsigned compare orders candidates exactly as the reference's sort
// (kv_cache.cpp:184-188).  The id field is idb = max(21, ceil(log2(cap)))
// bits wide (pools up to 2^kMaxIdBits blocks); last_used gets the remaining
// 61 - idb bits, i.e. |now| < 2^(60 - idb) (2^39 for pools up to 2M blocks).
constexpr int kMinIdBits = 21;
constexpr int kMaxIdBits = 24;
constexpr uint64_t kNoKey = ~uint64_t(0);
constexpr int kSelectThreads = 1024;
constexpr int kSortSmemKeys = 8192;
constexpr int kCandSmem = 16384;  // candidate keys staged in shared memory (128 KB)
constexpr int64_t kCoopMinCap = 16384;  // pools at least this large use the all-SM scorer
constexpr int64_t kProgCoopMinCap = 65536;  // ... for op programs (see use_coop)

enum Ctr { C_NRES = 0, C_EVICTED, C_LOOKUPS, C_HIT_TOK, C_LOOK_TOK, C_INS_BLOCKS, C_EV_BLOCKS, C_FULL, C_N };
enum Scal { S_F = 0, S_K, S_FREE, S_NEV, S_STATUS, S_FAILPOS, S_NNEW, S_NCAND, S_ERRIDX, S_NLATE, S_BOUND, S_NMISS, S_NLATEHIT, S_N };
// Blocks whose ref_count is -1 (reachable only through duplicate releases)
// become eviction candidates the moment an insert hits them; at most this
// many are tracked per insert.
constexpr int kLateMax = 64;

// One 32 B index slot (= one DRAM sector): a probe learns from a single
// sector whether the slot is empty/tombstone, its chain hash, and the parent
// hash and token count the reference's find_chain_block compares
// (kv_cache.cpp:77) — only the block's tokens remain a second access.
// parent/ntok of a resident block never change, so the copies stay valid.
struct alignas(32) IdxEntry {
  uint64_t key;     // chain hash
  uint64_t parent;  // parent chain hash of the block
  int32_t id;       // block id, -1 empty, -2 tombstone
  int32_t ntok;     // tokens in the block
  int64_t pad;
};

struct Pool {
  int64_t bs, cap, tcap;
  int32_t policy;
  int32_t idb;      // id bits of a victim key
  uint64_t idmask;  // (1 << idb) - 1
  int64_t lbias;    // 2^(60 - idb): last_used + lbias is non-negative
  uint64_t* tok;
  int32_t* ntok;
  uint64_t* chain;
  uint64_t* parent;
  int32_t* tag;
  int32_t* ref;
  int32_t* pinned;
  int64_t* last;
  IdxEntry* idx;
  int32_t* slot;
  unsigned long long* ctr;
};

struct Scratch {
  int64_t pmax = 0, kmax = 0;
  uint64_t* hashes = nullptr;   // pmax
  int32_t* prehit = nullptr;    // pmax
  int32_t* chain_out = nullptr; // pmax
  int8_t* kind = nullptr;       // pmax (0 hit, 1 new)
  int32_t* freel = nullptr;     // pmax
  int32_t* evicted = nullptr;   // max(pmax, cap)
  uint64_t* victims = nullptr;  // kmax
  uint8_t* taken = nullptr;     // kmax
  int32_t* rank_of = nullptr;   // cap
  uint64_t* keys = nullptr;     // cap
  uint64_t* sortbuf = nullptr;  // kmax (global sort fallback)
  int64_t* scal = nullptr;      // S_N
  int32_t* late = nullptr;      // 2 * kLateMax: (position, id) of hits on ref==-1 blocks before the first miss
};

__device__ __forceinline__ uint64_t index_slot(uint64_t h, int64_t tcap) {
  return (h ^ (h >> 29) ^ (h >> 47)) & static_cast<uint64_t>(tcap - 1);
}

__device__ __forceinline__ bool is_candidate(const Pool& P, int32_t id) {
  return P.ntok[id] > 0 && P.ref[id] == 0 && P.pinned[id] == 0;
}

__device__ __forceinline__ uint64_t victim_key(const Pool& P, int32_t id) {
  uint64_t k = (static_cast<uint64_t>(P.last[id] + P.lbias) << P.idb) | static_cast<uint64_t>(id);
  if (P.policy == SB_POLICY_TIERED) k |= static_cast<uint64_t>(tier_of(P.tag[id])) << 61;
  return k;
}

// find_chain_block (kv_cache.cpp:70-83) is probe_find_g below.

// Entries are written by commit/rebuild kernels and read by probes of later
// launches only, so no reader ever sees a half-written slot.
__device__ void index_insert(const Pool& P, uint64_t h, int32_t id, uint64_t parent, int32_t ntok) {
  uint64_t s = index_slot(h, P.tcap);
  for (;;) {
    int32_t v = P.idx[s].id;
    if (v < 0 && atomicCAS(&P.idx[s].id, v, id) == v) {
      P.idx[s].key = h;
      P.idx[s].parent = parent;
      P.idx[s].ntok = ntok;
      P.slot[id] = static_cast<int32_t>(s);
      return;
    }
    s = (s + 1) & static_cast<uint64_t>(P.tcap - 1);
  }
}

// ------------------------------------------------------------------ hashing
// One thread per sequence; the chain is a sequential fold (kv_chain_hash),
// tokens are prefetched one block ahead so only the dependent hash path is
// exposed.  Writes the chain hash after every block (last block may be
// partial unless full_only).
__global__ void k_chain_hash(const uint64_t* __restrict__ tokens, const int64_t* __restrict__ seq_off,
                             const int64_t* __restrict__ blk_off, const uint64_t* __restrict__ parent0, int n_seqs,
                             int64_t bs, int full_only, uint64_t* __restrict__ out, int segs) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_seqs) return;
  const int64_t b = seq_off[segs ? 2 * s : s], e = seq_off[segs ? 2 * s + 1 : s + 1];
  uint64_t h = parent0 ? parent0[s] : kRootHash;
  const int64_t ob = blk_off[s];
  const int64_t nblk = full_only ? (e - b) / bs : (e - b + bs - 1) / bs;
  constexpr int U = 8;
  int64_t pos = b;
  for (int64_t j = 0; j < nblk; ++j) {
    const int64_t end = min(pos + bs, e);
    int64_t i = pos;
    for (; i + U <= end; i += U) {
      uint64_t v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = __ldg(reinterpret_cast<const unsigned long long*>(tokens + i + u)) + kGolden;
#pragma unroll
      for (int u = 0; u < U; ++u) h = chain_step(h, v[u]);
    }
    for (; i < end; ++i) h = chain_step(h, tokens[i] + kGolden);
    out[ob + j] = h;
    pos = end;
  }
}

// Few sequences (the engine's tool-output and prefix hashes: tens of
// sequences of thousands of tokens): the kernel time is the dependent chain
// of the longest sequence, so each lane runs its own sequence with nothing
// but the fold on its critical path — the next block's 16 tokens are loaded
// into registers (16 B vector loads) while the current block is folded, no
// shared-memory staging or warp synchronisation per block.
__global__ void __launch_bounds__(32) k_chain_hash_lat(const uint64_t* __restrict__ tokens,
                                                        const int64_t* __restrict__ seq_off,
                                                        const int64_t* __restrict__ blk_off,
                                                        const uint64_t* __restrict__ parent0, int n_seqs,
                                                        int full_only, uint64_t* __restrict__ out, int segs) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_seqs) return;
  const int64_t b = seq_off[segs ? 2 * s : s], e = seq_off[segs ? 2 * s + 1 : s + 1];
  uint64_t h = parent0 ? parent0[s] : kRootHash;
  const int64_t ob = blk_off[s];
  const int64_t nblk = full_only ? (e - b) / 16 : (e - b + 15) / 16;
  const int64_t nfull = (e - b) / 16;
  const bool vec = (reinterpret_cast<uintptr_t>(tokens + b) & 15) == 0;
  uint64_t cur[16], nxt[16];
  auto load = [&](int64_t j, uint64_t (&v)[16]) {
    const uint64_t* p = tokens + b + 16 * j;
    if (j < nfull && vec) {
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const ulonglong2 w = __ldg(reinterpret_cast<const ulonglong2*>(p) + r);
        v[2 * r] = w.x;
        v[2 * r + 1] = w.y;
      }
    } else {
#pragma unroll
      for (int r = 0; r < 16; ++r)
        v[r] = b + 16 * j + r < e ? __ldg(reinterpret_cast<const unsigned long long*>(p + r)) : 0ull;
    }
  };
  if (nblk > 0) load(0, cur);
  for (int64_t j = 0; j < nblk; ++j) {
    if (j + 1 < nblk) load(j + 1, nxt);
    const int len = static_cast<int>(min(static_cast<int64_t>(16), e - (b + 16 * j)));
    if (len == 16) {
#pragma unroll
      for (int r = 0; r < 16; ++r) h = chain_step(h, cur[r] + kGolden);
    } else {  // the partial last block (registers, no dynamic indexing)
#pragma unroll
      for (int r = 0; r < 16; ++r)
        if (r < len) h = chain_step(h, cur[r] + kGolden);
    }
    out[ob + j] = h;
#pragma unroll
    for (int r = 0; r < 16; ++r) cur[r] = nxt[r];
  }
}

// 16-token blocks: a warp hashes 32 sequences (one per lane) but loads their
// tokens cooperatively — each warp load instruction covers the current block
// of two sequences (16 lanes x 8 B, contiguous), staged through shared memory
// and prefetched one block ahead in registers — instead of 32 scattered 8 B
// loads per instruction (which made the per-lane fold L1-wavefront bound).
// The fold itself is ALU-pipe bound (ncu: alu 77 %, math-pipe throttle), so
// the load path is kept off the ALU pipe: while every sequence of the warp
// still has a full block j (warp-uniform), a load is one LDS of the
// sequence's base pointer + one IMAD.WIDE + the LDG, no bounds checks.
// Persistent grid (whole waves): warps stride over 32-sequence groups.
constexpr int kHashWarps = 4;
// kTok tokens of each of the warp's 32 sequences are staged per step (a
// 16-token block in 16 / kTok steps): each warp load instruction covers
// 32 / kTok sequences x kTok contiguous tokens.  kTok = 16 is used: kTok = 8
// (half the prefetch registers, 40 instead of 32 resident warps) measured
// 7 % slower — the fold is ALU-pipe bound, not latency bound.
template <int kTok>
__global__ void __launch_bounds__(32 * kHashWarps, kTok == 8 ? 10 : 8)
    k_chain_hash16(const uint64_t* __restrict__ tokens, const int64_t* __restrict__ seq_off,
                   const int64_t* __restrict__ blk_off, const uint64_t* __restrict__ parent0, int n_seqs,
                   int full_only, uint64_t* __restrict__ out, int segs) {
  constexpr int kPer = 32 / kTok;  // sequences per warp load instruction
  __shared__ uint64_t stage[kHashWarps][32][kTok + 1];  // padded rows: conflict-free reads
  __shared__ const uint64_t* seq_p[kHashWarps][32];
  __shared__ int64_t seq_b[kHashWarps][32], seq_e[kHashWarps][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qi = lane / kTok, k = lane % kTok;
  const int n_groups = (n_seqs + 31) >> 5;
  for (int grp = blockIdx.x * kHashWarps + w; grp < n_groups; grp += gridDim.x * kHashWarps) {
    const int s = grp * 32 + lane;
    int64_t b = 0, e = 0, ob = 0, nblk = 0;
    uint64_t h = kRootHash;
    if (s < n_seqs) {
      b = seq_off[segs ? 2 * s : s];  // segs: sequence s = tokens [seq_off[2s], seq_off[2s+1])
      e = seq_off[segs ? 2 * s + 1 : s + 1];
      ob = blk_off[s];
      if (parent0) h = parent0[s];
      nblk = full_only ? (e - b) / 16 : (e - b + 15) / 16;
    }
    __syncwarp();
    seq_b[w][lane] = b;
    seq_e[w][lane] = e;
    seq_p[w][lane] = tokens + b;
    const int nb_max = static_cast<int>(__reduce_max_sync(0xffffffffu, static_cast<unsigned>(nblk)));
    // steps every sequence of the group holds in full (empty lanes hold none)
    const int ns_full = static_cast<int>(
        __reduce_min_sync(0xffffffffu, s < n_seqs ? static_cast<unsigned>((e - b) / kTok) : 0u));
    const int n_steps = nb_max * (16 / kTok);
    __syncwarp();
    uint64_t v[kTok];
    auto load = [&](int j) {  // step j: tokens [kTok j, kTok j + kTok) of every sequence
      if (j < ns_full) {
#pragma unroll
        for (int r = 0; r < kTok; ++r)
          v[r] = __ldg(reinterpret_cast<const unsigned long long*>(seq_p[w][kPer * r + qi] + kTok * j + k));
      } else {
#pragma unroll
        for (int r = 0; r < kTok; ++r) {
          const int q = kPer * r + qi;
          const int64_t pos = seq_b[w][q] + kTok * static_cast<int64_t>(j) + k;
          v[r] = pos < seq_e[w][q] ? __ldg(reinterpret_cast<const unsigned long long*>(tokens + pos)) : 0ull;
        }
      }
    };
    if (n_steps > 0) load(0);
    for (int j = 0; j < n_steps; ++j) {
      __syncwarp();
#pragma unroll
      for (int r = 0; r < kTok; ++r) stage[w][kPer * r + qi][k] = v[r];
      __syncwarp();
      if (j + 1 < n_steps) load(j + 1);
      const int blk = j / (16 / kTok);
      if (blk < nblk) {
        const int64_t len = e - (b + kTok * static_cast<int64_t>(j));
        if (len >= kTok) {
#pragma unroll
          for (int i = 0; i < kTok; ++i) h = chain_step(h, stage[w][lane][i] + kGolden);
        } else if (len > 0) {
          for (int i = 0; i < len; ++i) h = chain_step(h, stage[w][lane][i] + kGolden);
        }
        // the block's hash once its last step is folded (or the sequence ends inside it)
        if ((j + 1) % (16 / kTok) == 0 || len <= kTok) {
          if (len > 0 || (j + 1) % (16 / kTok) == 0) out[ob + blk] = h;
        }
      }
    }
  }
}

static void launch_chain_hash(const uint64_t* tokens, const int64_t* seq_off, const int64_t* blk_off,
                              const uint64_t* parent0, int n_seqs, int64_t bs, int full_only, uint64_t* out,
                              cudaStream_t st, int segs = 0) {
  if (n_seqs <= 0) return;
  if (bs == 16) {
    static int grid_cap = 0;  // whole waves of resident CTAs
    auto kern = k_chain_hash16<16>;
    if (!grid_cap) {
      int dev = 0, sms = 0, per_sm = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * kHashWarps, 0);
      grid_cap = std::max(1, sms * std::max(per_sm, 1));
    }
    // the per-lane kernel up to this many sequences (SB_HASH_LAT_MAX); measured
    // (profiles/run_r02aw.sh): 4096 x 1024 tokens 60 vs 72 us, 65536 x 512
    // 73 vs 82 us; the staged kernel wins from ~8K warps (262144 sequences)
    static int lat_max = -1;
    if (lat_max < 0) {
      const char* e = getenv("SB_HASH_LAT_MAX");
      lat_max = e ? atoi(e) : 65536;
    }
    if (n_seqs <= lat_max) {
      k_chain_hash_lat<<<(n_seqs + 31) / 32, 32, 0, st>>>(tokens, seq_off, blk_off, parent0, n_seqs, full_only, out,
                                                         segs);
      return;
    }
    const int groups = (n_seqs + 31) / 32;
    const int grid = std::min(grid_cap, (groups + kHashWarps - 1) / kHashWarps);
    kern<<<grid, 32 * kHashWarps, 0, st>>>(tokens, seq_off, blk_off, parent0, n_seqs, full_only, out, segs);
  } else {
    k_chain_hash<<<(n_seqs + 63) / 64, 64, 0, st>>>(tokens, seq_off, blk_off, parent0, n_seqs, bs, full_only, out,
                                                    segs);
  }
}

// --------------------------------------------------------------- lookups

// Group probe: the kGroup = 2 lanes of an aligned lane pair look up ONE block
// position together.  Both walk the index identically (same 32 B slot, one
// sector, broadcast), and on a slot whose (chain hash, parent, ntok) match,
// each lane compares one half of the block's tokens with the query's (16 B
// vector loads of the pool's 128 B token row) and the pair votes.  The
// dependent chain per position is chain hash -> index slot -> block tokens;
// the query tokens are loaded before the walk.
// The walk is WARP-converged: every lane runs the loop until all 16 pairs of
// the warp are done and the vote is one full-warp ballot.  (A per-pair
// __all_sync inside a data-dependent loop left the warp diverged, so the
// pairs' probes — and their loads — ran one after another: ncu counted 16
// vote executions per warp.)  `active` is false for lanes with no position.
constexpr int kGroup = 2;
__device__ __forceinline__ void ld_slot(const IdxEntry* e, uint64_t& key, uint64_t& parent, int32_t& id,
                                        int32_t& ntok) {
  asm volatile(
      "ld.global.v2.u64 {%0, %1}, [%4];\n\t"
      "ld.global.v2.s32 {%2, %3}, [%4+16];"
      : "=l"(key), "=l"(parent), "=r"(id), "=r"(ntok)
      : "l"(e));
}
__device__ __forceinline__ void ld_v2(const uint64_t* p, uint64_t& a, uint64_t& b) {
  asm volatile("ld.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
}
template <bool kVec>
__device__ int32_t probe_find_g(const Pool& P, bool active, uint64_t h, uint64_t parent,
                                const uint64_t* __restrict__ t, int len, int part) {
  constexpr int R = 16 / kGroup;  // tokens per lane of a 16-token block: [R*part, R*part + R)
  const int lane = threadIdx.x & 31;
  uint64_t s = index_slot(h, P.tcap);
  bool done = !active;
  int32_t found = -1;
  // query tokens are only needed once a slot matches: loaded in the same
  // round trip as the block's tokens (no registers held across the walk)
  const bool q_vec = kVec && len == 16 && (reinterpret_cast<uintptr_t>(t + R * part) & 15) == 0;  // (a partial block must not read past its tokens)
  while (__any_sync(0xffffffffu, !done)) {
    bool eq = false, empty = false;
    int32_t id = -1;
    if (!done) {
      uint64_t key, par;
      int32_t nt;
      ld_slot(P.idx + s, key, par, id, nt);
      empty = id == -1;
      if (id >= 0 && key == h && par == parent && nt == len) {
        const uint64_t* bt = P.tok + static_cast<int64_t>(id) * P.bs;
        eq = true;
        if (kVec) {  // bs == 16: 128 B aligned rows
          uint64_t x[R], q[R];
#pragma unroll
          for (int r = 0; r < R / 2; ++r) ld_v2(bt + R * part + 2 * r, x[2 * r], x[2 * r + 1]);
          if (q_vec) {
#pragma unroll
            for (int r = 0; r < R / 2; ++r) {
              const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(t + R * part) + r);
              q[2 * r] = v.x;
              q[2 * r + 1] = v.y;
            }
          } else {
#pragma unroll
            for (int r = 0; r < R; ++r) q[r] = R * part + r < len ? __ldg(reinterpret_cast<const unsigned long long*>(t + R * part + r)) : 0ull;
          }
#pragma unroll
          for (int r = 0; r < R; ++r)
            if (R * part + r < len) eq &= x[r] == q[r];
        } else {
          for (int i = part; i < len; i += kGroup) eq &= bt[i] == t[i];
        }
      }
    }
    const unsigned vote = __ballot_sync(0xffffffffu, eq);
    const unsigned pair = (vote >> (lane & ~(kGroup - 1))) & ((1u << kGroup) - 1);
    if (!done) {
      if (pair == (1u << kGroup) - 1) {
        found = id;
        done = true;
      } else if (empty) {
        done = true;
      } else {
        s = (s + 1) & static_cast<uint64_t>(P.tcap - 1);
      }
    }
  }
  return found;
}

// Warp-wide 32-ary search: s with blk_off[s] <= x < blk_off[s + 1]
// (requires blk_off[0] <= x < blk_off[n]).  All 32 lanes call it with the
// same x; two rounds cover 1000+ sequences.
__device__ __forceinline__ int warp_search(const int64_t* __restrict__ blk_off, int n, int64_t x) {
  const int lane = threadIdx.x & 31;
  int lo = 0, hi = n;
  while (hi - lo > 1) {
    const int64_t span = hi - lo;
    const int piv = lo + static_cast<int>((span * (lane + 1)) / 33);  // in [lo, hi), nondecreasing in lane
    const unsigned m = __ballot_sync(0xffffffffu, blk_off[piv] <= x);
    const int k = __popc(m);
    const int a = __shfl_sync(0xffffffffu, piv, k > 0 ? k - 1 : 0);
    const int b = __shfl_sync(0xffffffffu, piv, k < 32 ? k : 31);
    const int nlo = k > 0 ? a : lo, nhi = k < 32 ? b : hi;
    lo = nlo;
    hi = nhi;
  }
  return lo;
}

// Sequence of position g for every lane of a warp whose positions ascend
// with the lane: bracket the warp's range with two warp searches, then a
// per-lane binary search inside the bracket (usually empty).
__device__ __forceinline__ int find_seq_warp(const int64_t* __restrict__ blk_off, int n_seqs, int64_t g,
                                             int64_t total) {
  const int64_t gc = min(g, total - 1);
  const int64_t g0 = __shfl_sync(0xffffffffu, gc, 0), g1 = __shfl_sync(0xffffffffu, gc, 31);
  int lo = warp_search(blk_off, n_seqs, g0);
  int hi = warp_search(blk_off, n_seqs, g1) + 1;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (blk_off[mid] <= gc) lo = mid; else hi = mid;
  }
  return lo;
}

// Pre-state probe of the block positions of a batch of sequences, one CTA
// per (sequence, run of kProbeRun consecutive positions): grid = (n_seqs,
// max runs).  The sequence's offsets are three broadcast loads (no search).
// Each lane pair works through kProbePer positions (j0 + pair + 128 k) as a
// small state machine — every trip round the loop is ONE memory round trip
// for every pair: either its current position's index slot (SLOT) or the
// matched block's tokens + the query's tokens (TOK).  A pair that resolves a
// position starts the next one in the same trip (its chain hashes were
// prefetched a position ahead), so extra probes of one pair no longer stall
// the other 15 pairs of the warp, and a warp keeps 16 positions in flight.
constexpr int kProbePairs = 128;                   // lane pairs per CTA
template <int kProbePer>                           // positions per pair
__global__ void __launch_bounds__(kProbePairs * kGroup, 4) k_probe_rows(Pool P, const uint64_t* __restrict__ tokens,
                                                                       const int64_t* __restrict__ seq_off,
                                                                       const int64_t* __restrict__ blk_off,
                                                                       const uint64_t* __restrict__ hashes,
                                                                       int32_t* __restrict__ prehit,
                                                                       int64_t* __restrict__ first_miss,
                                                                       int full_only_check) {
  static_assert(kGroup == 2, "pair protocol");
  constexpr int kProbeRun = kProbePairs * kProbePer;  // positions per CTA
  const int sq = blockIdx.x;
  const int64_t b0 = blk_off[sq], np = blk_off[sq + 1] - b0;
  const int64_t j0 = static_cast<int64_t>(blockIdx.y) * kProbeRun;
  if (j0 >= np) return;  // CTA-uniform
  const int64_t t0 = seq_off[sq], t1 = seq_off[sq + 1];
  const int lane = threadIdx.x & 31, part = lane & 1;
  const int pair = threadIdx.x >> 1;
  constexpr int R = 16 / kGroup;
  const bool vec = P.bs == 16;
  // position k of this pair
  auto pos = [&](int k) { return j0 + pair + static_cast<int64_t>(kProbePairs) * k; };
  int k = 0;
  int64_t j = pos(0);
  bool live = j < np;  // pair has a position to resolve
  uint64_t h = 0, parent = kRootHash, h_nx = 0, parent_nx = kRootHash;
  if (live) {
    h = hashes[b0 + j];
    if (j) parent = hashes[b0 + j - 1];
  }
  if (pos(1) < np) {
    h_nx = hashes[b0 + pos(1)];
    parent_nx = hashes[b0 + pos(1) - 1];
  }
  int len = 0;
  int64_t base = 0;
  auto setup = [&]() {  // per-position constants of j
    base = t0 + j * P.bs;
    len = static_cast<int>(min(P.bs, t1 - base));
  };
  if (live) setup();
  uint64_t s = index_slot(h, P.tcap);
  bool tok_phase = false;
  int32_t cand = -1;
  // a lookup never matches a partial block (kv_cache.cpp:90)
  bool skip = live && full_only_check && len < P.bs;
  while (__any_sync(0xffffffffu, live)) {
    bool eq = false, resolved = false;
    const bool was_tok = live && tok_phase && !skip;
    int32_t result = -1;
    if (live && skip) {
      resolved = true;
    } else if (live && !tok_phase) {
      uint64_t key, par;
      int32_t id, nt;
      ld_slot(P.idx + s, key, par, id, nt);
      if (id == -1) {
        resolved = true;
      } else if (id >= 0 && key == h && par == parent && nt == len) {
        tok_phase = true;
        cand = id;
      } else {
        s = (s + 1) & static_cast<uint64_t>(P.tcap - 1);
      }
    } else if (live) {
      const uint64_t* bt = P.tok + static_cast<int64_t>(cand) * P.bs;
      const uint64_t* q = tokens + base;
      eq = true;
      if (vec) {
        uint64_t x[R], y[R];
#pragma unroll
        for (int r = 0; r < R / 2; ++r) ld_v2(bt + R * part + 2 * r, x[2 * r], x[2 * r + 1]);
#pragma unroll
        for (int r = 0; r < R; ++r)
          y[r] = R * part + r < len ? __ldg(reinterpret_cast<const unsigned long long*>(q + R * part + r)) : 0ull;
#pragma unroll
        for (int r = 0; r < R; ++r)
          if (R * part + r < len) eq &= x[r] == y[r];
      } else {
        for (int i = part; i < len; i += kGroup) eq &= bt[i] == q[i];
      }
    }
    // pair vote (both lanes of a pair are always in the same state)
    const unsigned vote = __ballot_sync(0xffffffffu, eq);
    if (was_tok) {
      if (((vote >> (lane & ~1)) & 3u) == 3u) {
        resolved = true;
        result = cand;
      } else {  // hash collision: keep walking
        tok_phase = false;
        s = (s + 1) & static_cast<uint64_t>(P.tcap - 1);
      }
    }
    if (resolved) {
      if (part == 0) {
        prehit[b0 + j] = result;
        if (result < 0 && first_miss)
          atomicMin(reinterpret_cast<unsigned long long*>(first_miss + sq), static_cast<unsigned long long>(j));
      }
      ++k;
      j = pos(k);
      live = k < kProbePer && j < np;
      if (live) {
        h = h_nx;
        parent = parent_nx;
        setup();
        s = index_slot(h, P.tcap);
        tok_phase = false;
        skip = full_only_check && len < P.bs;
        const int64_t jn = pos(k + 1);
        if (k + 1 < kProbePer && jn < np) {  // prefetch the next position's chain hashes
          h_nx = hashes[b0 + jn];
          parent_nx = hashes[b0 + jn - 1];
        }
      }
    }
  }
}

// Pre-state probe of the block positions of insert sequence s (kGroup lanes
// per position).
__global__ void k_probe_seq(Pool P, const uint64_t* __restrict__ tokens, const int64_t* __restrict__ seq_off,
                            const int64_t* __restrict__ blk_off, const uint64_t* __restrict__ hashes, int s,
                            int32_t* __restrict__ prehit) {
  const int64_t b0 = blk_off[s];
  const int64_t np = blk_off[s + 1] - b0;
  const int64_t p = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / kGroup;
  const int part = threadIdx.x % kGroup;
  if (blockIdx.x * static_cast<int64_t>(blockDim.x) / kGroup + (threadIdx.x & ~31) / kGroup >= np) return;
  const bool active = p < np;
  const int64_t pc = min(p, np - 1);
  const int64_t base = seq_off[s] + pc * P.bs;
  const int len = static_cast<int>(min(P.bs, seq_off[s + 1] - base));
  const uint64_t parent = pc ? hashes[b0 + pc - 1] : kRootHash;
  const uint64_t h = hashes[b0 + pc];
  const int32_t id = P.bs == 16 ? probe_find_g<true>(P, active, h, parent, tokens + base, len, part)
                                 : probe_find_g<false>(P, active, h, parent, tokens + base, len, part);
  if (part == 0 && active) prehit[b0 + p] = id;
}

__global__ void k_lookup_init(const int64_t* __restrict__ blk_off, int n_seqs, int64_t* first_miss) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < n_seqs) first_miss[s] = blk_off[s + 1] - blk_off[s];
}

// Touch the hit prefix (kv_cache.cpp:99) and emit hit lengths.
__global__ void k_lookup_finish(Pool P, const int64_t* __restrict__ seq_off, const int64_t* __restrict__ blk_off,
                                int n_seqs, int64_t total_blocks, const int32_t* __restrict__ prehit,
                                const int64_t* __restrict__ first_miss, int64_t now, int64_t* __restrict__ hit_tokens) {
  const int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (g < n_seqs) {
    hit_tokens[g] = first_miss[g] * P.bs;
    atomicAdd(&P.ctr[C_LOOKUPS], 1ull);
    atomicAdd(&P.ctr[C_HIT_TOK], static_cast<unsigned long long>(first_miss[g] * P.bs));
    atomicAdd(&P.ctr[C_LOOK_TOK], static_cast<unsigned long long>(seq_off[g + 1] - seq_off[g]));
  }
  if (total_blocks == 0 || blockIdx.x * static_cast<int64_t>(blockDim.x) + (threadIdx.x & ~31) >= total_blocks) return;
  const int s = find_seq_warp(blk_off, n_seqs, g, total_blocks);  // whole warp
  if (g >= total_blocks) return;
  if (g - blk_off[s] < first_miss[s]) P.last[prehit[g]] = now;
}

// ---------------------------------------------------------------- scoring
// Block-wide exclusive scan of 2 values per thread over kSelectThreads
// threads (2048 bins); returns the inclusive total.
__device__ uint32_t block_scan_2048(uint32_t* hist, uint32_t* warp_sums) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  uint32_t a = hist[2 * t], b = hist[2 * t + 1];
  uint32_t v = a + b, x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[w] = x;
  __syncthreads();
  if (w == 0) {
    uint32_t ws = warp_sums[lane], z = ws;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, z, o);
      if (lane >= o) z += y;
    }
    warp_sums[lane] = z - ws;  // exclusive warp offsets
    if (lane == 31) warp_sums[32] = z;
  }
  __syncthreads();
  const uint32_t excl = warp_sums[w] + x - v;
  hist[2 * t] = excl;
  hist[2 * t + 1] = excl + a;
  const uint32_t total = warp_sums[32];
  __syncthreads();
  return total;
}

// Bitonic sort of n (power of two) keys in shared memory, block-wide.
// Stages with a compare distance j >= 64 run over shared memory, indexed by
// compare-exchange pair (q -> i = 2j*(q/j) + q%j, partner i + j) so every
// thread works; the stages with j <= 32 of each merge run in registers: a
// warp loads a 64-key segment (two keys per lane), does them with shuffles
// (j = 32 inside the lane) and writes the segment back — one block barrier
// per shared-memory stage and per register phase instead of one per stage.
__device__ __forceinline__ uint64_t cx_keep(uint64_t v, uint64_t p, bool keep_min) {
  return keep_min ? (v < p ? v : p) : (v > p ? v : p);
}
__device__ void bitonic_warp_stages(uint64_t* a, int n, int k_lo, int k_hi, bool all_ascending = false) {
  // merges k_lo..k_hi (powers of two, k_hi <= 64 or k_lo == k_hi), stages j <= min(k/2, 32);
  // all_ascending: the k = 64 merge sorts every 64-key segment ascending
  const int lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int seg = (threadIdx.x >> 5) * 64; seg < n; seg += nw * 64) {
    const int i0 = seg + lane, i1 = i0 + 32;
    uint64_t v0 = a[i0], v1 = a[i1];
    for (int k = k_lo; k <= k_hi; k <<= 1) {
      for (int j = min(k >> 1, 32); j > 0; j >>= 1) {
        const bool asc = all_ascending && k == 64;
        const bool up0 = asc || (i0 & k) == 0, up1 = asc || (i1 & k) == 0;
        if (j == 32) {  // both keys of the pair sit in this lane
          const uint64_t lo = v0 < v1 ? v0 : v1, hi = v0 < v1 ? v1 : v0;
          v0 = up0 ? lo : hi;
          v1 = up0 ? hi : lo;
        } else {
          const bool lower = (lane & j) == 0;
          const uint64_t p0 = __shfl_xor_sync(0xffffffffu, v0, j);
          const uint64_t p1 = __shfl_xor_sync(0xffffffffu, v1, j);
          v0 = cx_keep(v0, p0, lower == up0);
          v1 = cx_keep(v1, p1, lower == up1);
        }
      }
    }
    a[i0] = v0;
    a[i1] = v1;
  }
}
__device__ void bitonic_smem(uint64_t* a, int n) {
  if (n < 64) {  // tiny: plain network
    for (int k = 2; k <= n; k <<= 1)
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int q = threadIdx.x; q < (n >> 1); q += blockDim.x) {
          const int i = ((q & ~(j - 1)) << 1) | (q & (j - 1));
          const int ixj = i | j;
          const uint64_t x = a[i], y = a[ixj];
          if ((x > y) == ((i & k) == 0)) {
            a[i] = y;
            a[ixj] = x;
          }
        }
        __syncthreads();
      }
    return;
  }
  const int half = n >> 1;
  bitonic_warp_stages(a, n, 2, 64);
  __syncthreads();
  for (int k = 128; k <= n; k <<= 1) {
    for (int j = k >> 1; j >= 64; j >>= 1) {
      for (int q = threadIdx.x; q < half; q += blockDim.x) {
        const int i = ((q & ~(j - 1)) << 1) | (q & (j - 1));
        const int ixj = i | j;
        const uint64_t x = a[i], y = a[ixj];
        if ((x > y) == ((i & k) == 0)) {
          a[i] = y;
          a[ixj] = x;
        }
      }
      __syncthreads();
    }
    bitonic_warp_stages(a, n, k, k);
    __syncthreads();
  }
}

// Merge sort of n keys (power of two, 128 <= n, 2n keys of shared memory):
// 64-key segments sorted ascending per warp in registers, then merge passes
// in which each thread emits n / blockDim.x consecutive outputs of a merged
// run, located by a merge-path binary search (A before B on ties).  Every
// pass moves the keys through shared memory once — the bitonic network moves
// them once per stage.  Returns the buffer holding the sorted keys.
__device__ uint64_t* merge_sort_smem(uint64_t* a, uint64_t* tmp, int n) {
  bitonic_warp_stages(a, n, 2, 64, true);
  __syncthreads();
  const int per = max(1, n / static_cast<int>(blockDim.x));
  uint64_t *src = a, *dst = tmp;
  for (int w = 64; w < n; w <<= 1) {
    for (int o = threadIdx.x * per; o < n; o += blockDim.x * per) {
      const int base = o & ~(2 * w - 1), d = o - base;
      const uint64_t* A = src + base;
      const uint64_t* B = A + w;
      int lo = max(0, d - w), hi = min(d, w);
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (A[mid] <= B[d - 1 - mid]) lo = mid + 1;
        else hi = mid;
      }
      int ia = lo, ib = d - lo;
      for (int e = 0; e < per; ++e) {
        const bool take_a = ib >= w || (ia < w && A[ia] <= B[ib]);
        dst[base + d + e] = take_a ? A[ia++] : B[ib++];
      }
    }
    __syncthreads();
    uint64_t* t = src;
    src = dst;
    dst = t;
  }
  return src;
}

// Same network in global memory (fallback for very large victim lists).
__device__ void bitonic_global(uint64_t* a, int64_t n) {
  for (int64_t k = 2; k <= n; k <<= 1) {
    for (int64_t j = k >> 1; j > 0; j >>= 1) {
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        const int64_t ixj = i ^ j;
        if (ixj > i) {
          const uint64_t x = a[i], y = a[ixj];
          const bool up = (i & k) == 0;
          if ((x > y) == up) {
            a[i] = y;
            a[ixj] = x;
          }
        }
      }
      __syncthreads();
    }
  }
}

// Hint-aware eviction scoring of pool blocks [lo, hi) (lo % 4 == 0): every
// field the decision needs is read with 16 B vector loads, unconditionally
// (no dependent short-circuit loads), and the keys (tier, last_used, id) of
// the candidates — resident, ref 0, unpinned, not excluded (rank_of -2) —
// are appended with one shared/global atomic per warp and element slot.
template <int U, bool kRank, class Emit>
__device__ __forceinline__ void score_slice(const Pool& P, const int32_t* rank_of, int64_t lo, int64_t hi, Emit emit) {
  const int64_t hi4 = lo + ((hi - lo) & ~int64_t(3));
  const bool tiered = P.policy == SB_POLICY_TIERED;
  auto one = [&](int32_t id, int nt, int rf, int pn, int rk, int tg, int64_t last) {
    const bool c = nt > 0 && rf == 0 && pn == 0 && rk != -2;
    uint64_t k = (static_cast<uint64_t>(last + P.lbias) << P.idb) | static_cast<uint64_t>(id);
    if (tiered) k |= static_cast<uint64_t>(tier_of(tg)) << 61;
    emit(c, k, nt == 0);
  };
  // U 4-block groups per thread in flight before any decision
  const int64_t step = 4 * static_cast<int64_t>(blockDim.x);
  for (int64_t i0 = lo + 4 * static_cast<int64_t>(threadIdx.x); i0 < hi4; i0 += U * step) {
    int4 nt[U], rf[U], pn[U], rk[U], tg[U];
    longlong2 l0[U], l1[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * step;
      if (i < hi4) {
        nt[u] = *reinterpret_cast<const int4*>(P.ntok + i);
        rf[u] = *reinterpret_cast<const int4*>(P.ref + i);
        pn[u] = *reinterpret_cast<const int4*>(P.pinned + i);
        if (kRank) rk[u] = *reinterpret_cast<const int4*>(rank_of + i);
        else rk[u] = make_int4(0, 0, 0, 0);
        tg[u] = *reinterpret_cast<const int4*>(P.tag + i);
        l0[u] = *reinterpret_cast<const longlong2*>(P.last + i);
        l1[u] = *reinterpret_cast<const longlong2*>(P.last + i + 2);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * step;
      if (i < hi4) {
        const int32_t id = static_cast<int32_t>(i);
        one(id, nt[u].x, rf[u].x, pn[u].x, rk[u].x, tg[u].x, l0[u].x);
        one(id + 1, nt[u].y, rf[u].y, pn[u].y, rk[u].y, tg[u].y, l0[u].y);
        one(id + 2, nt[u].z, rf[u].z, pn[u].z, rk[u].z, tg[u].z, l1[u].x);
        one(id + 3, nt[u].w, rf[u].w, pn[u].w, rk[u].w, tg[u].w, l1[u].y);
      }
    }
  }
  for (int64_t i = hi4 + threadIdx.x; i < hi; i += blockDim.x)
    one(static_cast<int32_t>(i), P.ntok[i], P.ref[i], P.pinned[i], kRank ? rank_of[i] : 0, P.tag[i], P.last[i]);
}

// Warp-aggregated append: one atomic per warp for the set lanes.
template <class Counter>
__device__ __forceinline__ uint64_t warp_append_slot(bool c, Counter* cnt, bool& mine) {
  const unsigned act = __activemask();
  const unsigned m = __ballot_sync(act, c);
  mine = c;
  if (!m) return 0;
  const int lane = threadIdx.x & 31;
  const int leader = __ffs(m) - 1;
  uint64_t base = 0;
  if (lane == leader) base = static_cast<uint64_t>(atomicAdd(cnt, static_cast<Counter>(__popc(m))));
  base = __shfl_sync(act, base, leader);
  return base + __popc(m & ((1u << lane) - 1));
}

// Tag coverage check (kv_cache.cpp:105-115): ranges must tile [0, n).
__device__ bool tags_cover(const sb_tag_range* tags, int64_t ntags, int64_t n) {
  int64_t covered = 0;
  for (int64_t r = 0; r < ntags; ++r) {
    if (tags[r].begin != covered || tags[r].end < tags[r].begin) return false;
    covered = tags[r].end;
  }
  return covered == n;
}

struct InsertArgs {
  const uint64_t* tokens;
  const int64_t* seq_off;
  const sb_tag_range* tags;
  const int64_t* tag_off;
  const int64_t* blk_off;
  const uint64_t* hashes;  // all sequences, laid out by blk_off
  int32_t* out_ids;        // laid out by blk_off
  int32_t* status;         // per sequence
  int64_t now;
};

// mode 0: plan one insert (sequence s).  mode 1: evict(needed) — K = needed.
// Hint-aware eviction scoring: the key (tier, last_used, id) of every
// candidate block (resident, unpinned, ref 0, not referenced before the first
// miss of this insert) is compacted into shared memory, the K smallest are
// radix-selected there (11-bit digits from the top, early exit once the
// boundary bin is exactly consumed), sorted, and published with their ranks.
// The lowest free ids are listed as well.  Pools whose candidate set exceeds
// the shared-memory budget run the same passes over global memory.
__global__ void __launch_bounds__(kSelectThreads, 1)
    k_select(Pool P, Scratch S, InsertArgs A, int s, int mode, int64_t needed) {
  __shared__ uint32_t hist[2048];
  __shared__ uint32_t bmin[2048], bmax[2048];  // per bin: min / max of the 32 key bits below the digit
  __shared__ uint32_t warp_sums[33];
  __shared__ int64_t sh[8];
  __shared__ uint32_t cnt_b;
  __shared__ unsigned long long n_cand, n_hc;
  __shared__ unsigned long long key_range[2];
  extern __shared__ uint64_t dyn[];  // [kCandSmem] candidates | [kSortSmemKeys] selection
  uint64_t* cand_s = dyn;
  uint64_t* sel_s = dyn + kCandSmem;
  const int t = threadIdx.x;
  int64_t P_ = 0, f = 0, b0 = 0;
  if (mode == 0) {
    b0 = A.blk_off[s];
    P_ = A.blk_off[s + 1] - b0;
    const int64_t n = A.seq_off[s + 1] - A.seq_off[s];
    const bool ok = tags_cover(A.tags + A.tag_off[s], A.tag_off[s + 1] - A.tag_off[s], n);
    if (t == 0) sh[0] = P_;
    __syncthreads();
    for (int64_t p = t; p < P_; p += blockDim.x)
      if (S.prehit[b0 + p] < 0) atomicMin(reinterpret_cast<unsigned long long*>(&sh[0]), (unsigned long long)p);
    __syncthreads();
    f = sh[0];
    if (!ok) {
      if (t == 0) {
        S.scal[S_STATUS] = SB_ERR_CACHE;
        S.scal[S_F] = 0;
        S.scal[S_K] = 0;
        S.scal[S_FREE] = 0;
      }
      return;
    }
    if (t == 0) S.scal[S_NLATE] = 0;
    // blocks referenced before the first miss cannot be evicted by this insert
    for (int64_t p = t; p < f; p += blockDim.x) {
      const int32_t id = S.prehit[b0 + p];
      S.kind[p] = 0;
      S.rank_of[id] = -2;  // temporary exclusion mark (rank_of is -1 elsewhere)
    }
  }
  if (t == 0) {
    n_cand = 0;
    n_hc = 0;
    key_range[0] = ~0ull;
    key_range[1] = 0;
  }
  __syncthreads();
  if (mode == 0) {
    for (int64_t p = t; p < P_; p += blockDim.x) {
      const int32_t id = S.prehit[b0 + p];
      if (id < 0) continue;
      if (p < f && P.ref[id] == -1 && P.pinned[id] == 0) {
        const int64_t at = atomicAdd(reinterpret_cast<unsigned long long*>(&S.scal[S_NLATE]), 1ull);
        if (at < kLateMax) {
          S.late[2 * at] = static_cast<int32_t>(p);
          S.late[2 * at + 1] = id;
        }
      } else if (p >= f && is_candidate(P, id)) {
        atomicAdd(&n_hc, 1ull);
      }
    }
  }
  // ---- score every block, compact the candidates
  // (first into shared memory; overflow keeps going into global S.keys)
  uint64_t kmn = ~0ull, kmx = 0;  // key range of the candidates: radix passes skip the shared high bits
  score_slice<1, true>(P, S.rank_of, 0, P.cap, [&](bool c, uint64_t k, bool) {
    bool mine;
    const uint64_t at = warp_append_slot(c, &n_cand, mine);
    if (mine) {
      if (at < kCandSmem) cand_s[at] = k; else S.keys[at - kCandSmem] = k;
      kmn = min(kmn, k);
      kmx = max(kmx, k);
    }
  });
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    kmn = min(kmn, __shfl_xor_sync(0xffffffffu, kmn, o));
    kmx = max(kmx, __shfl_xor_sync(0xffffffffu, kmx, o));
  }
  if ((t & 31) == 0) {
    atomicMin(&key_range[0], kmn);
    atomicMax(&key_range[1], kmx);
  }
  __syncthreads();
  if (mode == 0)
    for (int64_t p = t; p < f; p += blockDim.x) S.rank_of[S.prehit[b0 + p]] = -1;
  const int64_t ncand = static_cast<int64_t>(n_cand);
  const int64_t nres = static_cast<int64_t>(P.ctr[C_NRES]);
  const int64_t free_cnt = P.cap - nres;
  int64_t K, Fp = 0;
  if (mode == 0) {
    const int64_t rest = P_ - f;
    Fp = min(free_cnt, rest);
    K = min(ncand, (rest > free_cnt ? rest - free_cnt : int64_t(0)) + static_cast<int64_t>(n_hc));
  } else if (mode == 2) {  // op program: K and F bounded by k_prog_bound
    const int64_t bnd = S.scal[S_NMISS] > 0 ? S.scal[S_BOUND] : 0;
    K = min(ncand, bnd);
    Fp = min(free_cnt, bnd);
  } else {
    K = min(ncand, needed);
  }
  auto key_at = [&](int64_t i) -> uint64_t { return i < kCandSmem ? cand_s[i] : S.keys[i - kCandSmem]; };
  // ---- radix select of the K smallest keys (keys are unique)
  if (K > 0) {
    uint64_t prefix = 0, mask = 0;
    if (K < ncand) {
      int64_t need = K;
      // start at the highest bit in which the candidates differ (the bits above are shared)
      int hi_bit = 64 - __clzll(static_cast<long long>(key_range[0] ^ key_range[1]));
      mask = hi_bit >= 64 ? 0ull : ~((uint64_t(1) << hi_bit) - 1);
      prefix = key_range[0] & mask;
      while (hi_bit > 0) {
        const int wd = min(11, hi_bit), sh_ = hi_bit - wd;
        hi_bit = sh_;
        const uint64_t bmask = (uint64_t(1) << wd) - 1;
        const int s2 = sh_ > 32 ? sh_ - 32 : 0;  // the 32 key bits below the digit: [s2, s2 + 32)
        hist[2 * t] = 0;
        hist[2 * t + 1] = 0;
        bmin[2 * t] = bmin[2 * t + 1] = ~0u;
        bmax[2 * t] = bmax[2 * t + 1] = 0u;
        __syncthreads();
        // warp-aggregated: the keys of one pass crowd into a few bins (same
        // tier / last_used high bits), so lanes with equal digits combine
        // first and one lane per distinct digit updates shared memory
        for (int64_t i0 = 0; i0 < ncand; i0 += blockDim.x) {
          const int64_t i = i0 + t;
          const uint64_t k = i < ncand ? key_at(i) : 0;
          const bool part = i < ncand && (k & mask) == prefix;
          const uint32_t d = part ? static_cast<uint32_t>((k >> sh_) & bmask) : 0xFFFFFFFFu;
          const uint32_t low = static_cast<uint32_t>(k >> s2);
          const unsigned peers = __match_any_sync(0xffffffffu, d);
          const uint32_t mn = __reduce_min_sync(peers, low), mxv = __reduce_max_sync(peers, low);
          if (part && (t & 31) == __ffs(peers) - 1) {
            atomicAdd(&hist[d], static_cast<uint32_t>(__popc(peers)));
            atomicMin(&bmin[d], mn);
            atomicMax(&bmax[d], mxv);
          }
        }
        __syncthreads();
        const uint32_t a0 = hist[2 * t], a1 = hist[2 * t + 1];
        block_scan_2048(hist, warp_sums);
        const uint32_t e0 = hist[2 * t], e1 = hist[2 * t + 1];
        if (e0 < need && need <= e0 + a0) {
          sh[4] = 2 * t;
          sh[5] = e0;
          cnt_b = a0;
        }
        if (e1 < need && need <= e1 + a1) {
          sh[4] = 2 * t + 1;
          sh[5] = e1;
          cnt_b = a1;
        }
        __syncthreads();
        need -= sh[5];
        prefix |= static_cast<uint64_t>(sh[4]) << sh_;
        mask |= bmask << sh_;
        const bool done = (static_cast<int64_t>(cnt_b) == need);
        if (!done && sh_ > 0) {
          // skip the bits below the digit that every key of the chosen bin
          // shares (tiered keys: same tier and last_used high bits)
          const uint32_t lo = bmin[sh[4]], hi = bmax[sh[4]];
          const int top = sh_ - s2;                           // valid bits of lo/hi: [0, top)
          const uint32_t vmask = top >= 32 ? ~0u : ((1u << top) - 1);
          const uint32_t diff = (lo ^ hi) & vmask;
          const int nb = diff ? 32 - __clz(diff) : 0;         // differing bits are [0, nb)
          const int new_hi = s2 + nb;                         // next digit starts below new_hi
          if (new_hi < sh_) {
            const uint64_t shared_bits = (((uint64_t(1) << (sh_ - new_hi)) - 1)) << new_hi;
            prefix |= (static_cast<uint64_t>(lo) << s2) & shared_bits;
            mask |= shared_bits;
            hi_bit = new_hi;
          }
        }
        __syncthreads();
        if (done) break;
      }
    }
    // gather the selected keys: exactly K of them
    if (t == 0) sh[6] = 0;
    __syncthreads();
    const bool in_smem = K <= kSortSmemKeys;
    uint64_t* dst = in_smem ? sel_s : S.sortbuf;
    for (int64_t i = t; i < ncand; i += blockDim.x) {
      const uint64_t k = key_at(i);
      if (K == ncand || (k & mask) <= prefix) {
        const int64_t at = atomicAdd(reinterpret_cast<unsigned long long*>(&sh[6]), 1ull);
        dst[at] = k;
      }
    }
    __syncthreads();
    int64_t n2 = 1;
    while (n2 < K) n2 <<= 1;
    for (int64_t i = K + t; i < n2; i += blockDim.x) dst[i] = kNoKey;
    __syncthreads();
    if (in_smem) bitonic_smem(dst, static_cast<int>(n2));
    else bitonic_global(dst, n2);
    for (int64_t r = t; r < K; r += blockDim.x) {
      const uint64_t k = dst[r];
      S.victims[r] = k;
      S.taken[r] = 0;
      S.rank_of[k & P.idmask] = static_cast<int32_t>(r);
    }
  }
  // ---- lowest Fp free ids, ascending (std::set<int32_t> order)
  if (Fp > 0) {
    __shared__ uint32_t wcnt[33];
    __shared__ int64_t found;
    if (t == 0) found = 0;
    __syncthreads();
    const int lane = t & 31, w = t >> 5;
    for (int64_t base = 0; base < P.cap; base += blockDim.x) {
      if (found >= Fp) break;  // uniform: read after a barrier
      const int64_t i = base + t;
      const bool fr = i < P.cap && P.ntok[i] == 0;
      const unsigned ball = __ballot_sync(0xffffffffu, fr);
      if (lane == 0) wcnt[w] = __popc(ball);
      __syncthreads();
      if (t == 0) {
        uint32_t acc = 0;
        for (int k = 0; k < 32; ++k) {
          const uint32_t cnt = wcnt[k];
          wcnt[k] = acc;
          acc += cnt;
        }
        wcnt[32] = acc;
      }
      __syncthreads();
      const int64_t rank = found + wcnt[w] + __popc(ball & ((1u << lane) - 1));
      if (fr && rank < Fp) S.freel[rank] = static_cast<int32_t>(i);
      __syncthreads();
      if (t == 0) found += wcnt[32];
      __syncthreads();
    }
  }
  if (t == 0) {
    S.scal[S_F] = f;
    S.scal[S_K] = K;
    S.scal[S_FREE] = Fp;
    S.scal[S_STATUS] = 0;
    S.scal[S_NCAND] = ncand;
  }
}

// Sequential decisions of one insert (kv_cache.cpp:138-173), from the first
// pre-miss position on.  Single thread: each step is a handful of
// L1/L2-resident accesses.
// ---------------------------------------------------------------------------
// Large pools (>= kCoopMinCap blocks): the same decisions as k_select, split
// into three kernels so the HBM pass runs on every SM at streaming rate:
//   k_plan         1 CTA: first miss, tag check, exclusion marks, late
//                  candidates (phase A of k_select)
//   k_score        all SMs: hint-aware key (tier, last_used, id) of every
//                  block (24 B read per block, 16 B vectors), candidates
//                  compacted per CTA in shared memory then appended to a
//                  global key list; free blocks counted per slice; key range
//   k_select_coop  cooperative: radix select of the K smallest keys from the
//                  highest differing bit of the key range (histograms
//                  exchanged between grid barriers), CTA 0 sorts them; the
//                  lowest free ids are listed in parallel from the per-slice
//                  free counts.
struct CoopBuf {
  uint32_t* hist;            // [6][2048]
  unsigned long long* ctr;   // [0] candidates [1] selected [2] pre-hit candidates [3] min key [4] max key
                             // [5] keys compacted from the chosen radix bin
  uint64_t* keys;            // candidate keys, slice sl at [sl * slice, + ncnt[sl])
  uint32_t* fcnt;            // free blocks per score slice, [n_slices]
  uint32_t* ncnt;            // candidates per score slice, [n_slices]
  uint64_t* kmin;            // smallest / largest candidate key per slice, [n_slices]
  uint64_t* kmax;
  int n_slices;
  int64_t slice;             // blocks per score slice (multiple of 4)
  int64_t sort_keys;         // keys k_select_coop's dynamic shared memory holds (its final sort)
  unsigned long long* tprof; // SB_SELECT_PROF=1: phase timestamps (%globaltimer) of the last evict, else null
  int64_t rank_early_max = 6144;  // radix passes stop once <= this many keys remain (SB_RANK_EARLY)
};
// SB_SELECT_PROF slots: 0/1 k_plan start/end, 2/3 k_score first/last CTA entry, 4 k_score last exit,
// 5/6 k_select_coop first/last entry, 7 CTA 0 after the prologue, 8+2p / 9+2p last arrival at / CTA 0
// leaving grid barrier p (p < 6), 20 CTA 0 sort start, 21 CTA 0 end, 29 / 30 CTA 0 rank step: keys loaded /
// ranks written, 31 the rank step's key count M
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void tp_set(const CoopBuf& G, int slot) {
  if (G.tprof && threadIdx.x == 0) G.tprof[slot] = gtimer();
}
__device__ __forceinline__ void tp_max(const CoopBuf& G, int slot) {
  if (G.tprof && threadIdx.x == 0) atomicMax(G.tprof + slot, gtimer());
}
__device__ __forceinline__ void tp_min(const CoopBuf& G, int slot) {
  if (G.tprof && threadIdx.x == 0) atomicMin(G.tprof + slot, gtimer());
}
constexpr int kScoreThreads = 512;
constexpr int kSlicesPerSm = 2;  // score slices per SM; k_score CTA c scans slices c and c + n_sm
constexpr int kMaxSlicesPerCta = 4;
constexpr int kMaxLiveSlices = 1024;
constexpr int64_t kRankEarlyMax = 6144;  // k_select_coop stops its radix passes at this many candidate winners  // k_select_coop's list of slices a filtered pass visits (>= n_slices)  // k_select_coop's staging table (kSlicesPerSm, grids of >= n_sm / 2 CTAs)
// k_score streams the metadata through shared memory with 1-D bulk copies
// (TMA engine): per stage, kScoreChunk blocks of ntok/ref/pinned/tag (4 B)
// and last (8 B) = 48 KB; kScoreStages stages in flight per SM.
constexpr int kScoreChunk = 2048;
constexpr int kScoreStages = 4;
constexpr size_t kScoreStageBytes = kScoreChunk * 24;
constexpr size_t kScoreSmem = kScoreStages * kScoreStageBytes;
static_assert(kScoreChunk == 4 * kScoreThreads, "k_score: 4 blocks per thread per chunk");

__global__ void __launch_bounds__(kSelectThreads, 1)
    k_plan(Pool P, Scratch S, InsertArgs A, int s, int mode, CoopBuf G) {
  __shared__ int64_t first;
  const int t = threadIdx.x;
  if (G.tprof && t < 32) G.tprof[t] = (t == 2 || t == 5) ? ~0ull : 0ull;
  tp_set(G, 0);
  for (int i = t; i < 6 * 2048; i += blockDim.x) G.hist[i] = 0;
  if (t < 3) G.ctr[t] = 0;
  if (t == 3) G.ctr[3] = ~0ull;
  if (t == 4 || t == 5) G.ctr[t] = 0;
  if (mode != 0) {
    if (t == 0) {
      S.scal[S_F] = 0;
      S.scal[S_STATUS] = 0;
    }
    tp_set(G, 1);
    return;
  }
  const int64_t b0 = A.blk_off[s];
  const int64_t P_ = A.blk_off[s + 1] - b0;
  const int64_t n = A.seq_off[s + 1] - A.seq_off[s];
  const bool ok = tags_cover(A.tags + A.tag_off[s], A.tag_off[s + 1] - A.tag_off[s], n);
  if (t == 0) first = P_;
  __syncthreads();
  for (int64_t p = t; p < P_; p += blockDim.x)
    if (S.prehit[b0 + p] < 0) atomicMin(reinterpret_cast<unsigned long long*>(&first), (unsigned long long)p);
  __syncthreads();
  const int64_t f = first;
  if (t == 0) {
    S.scal[S_F] = f;
    S.scal[S_STATUS] = ok ? 0 : SB_ERR_CACHE;
    S.scal[S_NLATE] = 0;
    if (!ok) {
      S.scal[S_K] = 0;
      S.scal[S_FREE] = 0;
    }
  }
  if (!ok) return;
  for (int64_t p = t; p < P_; p += blockDim.x) {
    const int32_t id = S.prehit[b0 + p];
    if (p < f) {
      S.kind[p] = 0;
      const int32_t pn = P.pinned[id];
      if (P.ref[id] == -1 && pn == 0) {
        const int64_t at = atomicAdd(reinterpret_cast<unsigned long long*>(&S.scal[S_NLATE]), 1ull);
        if (at < kLateMax) {
          S.late[2 * at] = static_cast<int32_t>(p);
          S.late[2 * at + 1] = id;
        }
      }
      // temporary exclusion mark read by k_score (pinned blocks are never
      // candidates), cleared by k_select_coop; blocks at distinct positions
      // are distinct
      P.pinned[id] = pn | 2;
    } else if (id >= 0 && is_candidate(P, id)) {
      atomicAdd(&G.ctr[2], 1ull);
    }
  }
}

// One persistent CTA per SM.  Thread 0 keeps kScoreStages chunks in flight
// (5 bulk copies each, completion on the stage's mbarrier); all threads
// score a landed chunk from shared memory and append the candidates' keys
// to the slice's own region of the key list (one shared atomic per warp and
// element slot).  The metadata of a pool block is read from HBM exactly once.
// The scoring pass over kScoreThreads threads (the fused kernel's other
// threads skip it).
__device__ __forceinline__ void score_body(const Pool& P, const CoopBuf& G, uint8_t* stage_mem) {
  __shared__ uint64_t full[kScoreStages];
  // named barrier over the kScoreThreads scoring threads: the fused kernel's
  // other warps go straight to its grid barrier instead of polling the ring
  auto score_sync = []() { asm volatile("bar.sync 1, %0;" ::"n"(kScoreThreads) : "memory"); };
  if (threadIdx.x >= kScoreThreads) return;
  __shared__ unsigned int n_c, n_free;
  __shared__ unsigned long long kmin, kmax;
  const int t = threadIdx.x;
  const int n_my = (G.n_slices - static_cast<int>(blockIdx.x) + gridDim.x - 1) / gridDim.x;  // slices of this CTA
  const int64_t chunks_per_slice = (G.slice + kScoreChunk - 1) / kScoreChunk;
  auto slice_of = [&](int k) { return static_cast<int>(blockIdx.x) + k * static_cast<int>(gridDim.x); };
  auto range = [&](int64_t c, int64_t& lo, int64_t& n) {  // chunk c of this CTA -> pool block range
    const int sl = slice_of(static_cast<int>(c / chunks_per_slice));
    const int64_t s_lo = sl * G.slice, s_hi = min(P.cap, s_lo + G.slice);
    lo = s_lo + (c % chunks_per_slice) * kScoreChunk;
    n = s_hi - lo < 0 ? 0 : (s_hi - lo < kScoreChunk ? s_hi - lo : int64_t(kScoreChunk));
  };
  const int64_t n_chunks = n_my * chunks_per_slice;
  tp_min(G, 2);
  tp_max(G, 3);
  auto issue = [&](int64_t c) {
    int64_t lo, n;
    range(c, lo, n);
    uint64_t* bar = &full[c % kScoreStages];
    if (n == 0) {  // empty tail chunk: complete the phase without traffic
      mbar_arrive(bar);
      return;
    }
    uint8_t* st = stage_mem + (c % kScoreStages) * kScoreStageBytes;
    const uint32_t b4 = static_cast<uint32_t>((n + 3) & ~int64_t(3)) * 4;  // arrays padded to a multiple of 4
    const uint32_t b8 = static_cast<uint32_t>((n + 1) & ~int64_t(1)) * 8;
    mbar_arrive_expect_tx(bar, 4 * b4 + b8);
    bulk_g2s(st, P.ntok + lo, b4, bar);
    bulk_g2s(st + 4 * kScoreChunk, P.ref + lo, b4, bar);
    bulk_g2s(st + 8 * kScoreChunk, P.pinned + lo, b4, bar);
    bulk_g2s(st + 12 * kScoreChunk, P.tag + lo, b4, bar);
    bulk_g2s(st + 16 * kScoreChunk, P.last + lo, b8, bar);
  };
  if (t == 0) {
    for (int i = 0; i < kScoreStages; ++i) mbar_init(&full[i], 1);
    fence_barrier_init();
    n_c = 0;
    n_free = 0;
    kmin = ~0ull;
    kmax = 0;
  }
  score_sync();
  if (t == 0)
    for (int64_t c = 0; c < n_chunks && c < kScoreStages; ++c) issue(c);
  const bool tiered = P.policy == SB_POLICY_TIERED;
  const int lane = t & 31;
  uint64_t mn = ~0ull, mx = 0;
  unsigned nf = 0;
  for (int64_t c = 0; c < n_chunks; ++c) {
    int64_t lo, n;
    range(c, lo, n);
    const int sl = slice_of(static_cast<int>(c / chunks_per_slice));
    mbar_wait_suspend(&full[c % kScoreStages], static_cast<uint32_t>((c / kScoreStages) & 1));
    const uint8_t* st = stage_mem + (c % kScoreStages) * kScoreStageBytes;
    // thread t scores blocks 4t .. 4t+3 of the chunk: 16 B shared loads
    const int i0 = 4 * t;
    const int4 nt4 = reinterpret_cast<const int4*>(st)[t];
    const int4 rf4 = reinterpret_cast<const int4*>(st + 4 * kScoreChunk)[t];
    const int4 pn4 = reinterpret_cast<const int4*>(st + 8 * kScoreChunk)[t];
    const int4 tg4 = reinterpret_cast<const int4*>(st + 12 * kScoreChunk)[t];
    const longlong2 la0 = reinterpret_cast<const longlong2*>(st + 16 * kScoreChunk)[2 * t];
    const longlong2 la1 = reinterpret_cast<const longlong2*>(st + 16 * kScoreChunk)[2 * t + 1];
    const int nt[4] = {nt4.x, nt4.y, nt4.z, nt4.w}, rf[4] = {rf4.x, rf4.y, rf4.z, rf4.w};
    const int pn[4] = {pn4.x, pn4.y, pn4.z, pn4.w}, tg[4] = {tg4.x, tg4.y, tg4.z, tg4.w};
    const int64_t la[4] = {la0.x, la0.y, la1.x, la1.y};
    uint64_t key[4];
    unsigned cm = 0;  // candidate mask of the thread's 4 blocks
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool in = i0 + u < n;
      const bool cnd = in && nt[u] > 0 && rf[u] == 0 && pn[u] == 0;
      nf += in && nt[u] == 0;
      // tier_of as a nibble table: tags 0..5 -> 0,1,2,3,4,2 (kv_cache.cpp:23-33)
      const uint64_t tier = tiered && static_cast<unsigned>(tg[u]) < 6u ? (0x243210u >> (4 * tg[u])) & 0xFu : 0u;
      key[u] = (tier << 61) | (static_cast<uint64_t>(la[u] + P.lbias) << P.idb) | static_cast<uint64_t>(lo + i0 + u);
      cm |= static_cast<unsigned>(cnd) << u;
      if (cnd) {
        mn = min(mn, key[u]);
        mx = max(mx, key[u]);
      }
    }
    // warp-aggregated append: exclusive scan of the per-thread counts
    const unsigned cnt = __popc(cm);
    unsigned incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    unsigned base = 0;
    if (lane == 31 && incl) base = atomicAdd(&n_c, incl);
    base = __shfl_sync(0xffffffffu, base, 31) + incl - cnt;
    uint64_t* out = G.keys + sl * G.slice;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (cm >> u & 1) out[base++] = key[u];
    score_sync();  // stage consumed by every thread
    if (t == 0 && c + kScoreStages < n_chunks) {
      fence_proxy_async();
      issue(c + kScoreStages);
    }
    if ((c + 1) % chunks_per_slice == 0) {  // slice done: publish its counts and key range
      nf = __reduce_add_sync(0xffffffffu, nf);
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      }
      if ((t & 31) == 0) {
        atomicAdd(&n_free, nf);
        atomicMin(&kmin, mn);
        atomicMax(&kmax, mx);
      }
      score_sync();
      if (t == 0) {
        G.fcnt[sl] = n_free;
        G.ncnt[sl] = n_c;
        G.kmin[sl] = kmin;
        G.kmax[sl] = kmax;
        n_c = 0;
        n_free = 0;
        kmin = ~0ull;
        kmax = 0;
      }
      score_sync();
      mn = ~0ull;
      mx = 0;
      nf = 0;
    }
  }
  tp_max(G, 4);
}

__global__ void __launch_bounds__(kScoreThreads, 1) k_score(Pool P, Scratch S, CoopBuf G) {
  extern __shared__ __align__(128) uint8_t stage_mem[];
  score_body(P, G, stage_mem);
}

__device__ __forceinline__ void select_body(const Pool& P, const Scratch& S, const InsertArgs& A, int s, int mode,
                                            int64_t needed, const CoopBuf& G, uint64_t* local_keys) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  __shared__ uint32_t hist[2048];
  __shared__ uint32_t warp_sums[33];
  __shared__ int64_t sh[8];
  __shared__ uint32_t cnt_b;
  tp_min(G, 5);
  tp_max(G, 6);
  int n_sync = 0;
  auto gsync = [&]() {
    if (n_sync < 6) tp_max(G, 8 + 2 * n_sync);
    grid.sync();
    if (blockIdx.x == 0 && n_sync < 6) tp_set(G, 9 + 2 * n_sync);
    ++n_sync;
  };
  if (S.scal[S_STATUS] != 0) return;  // uniform across the grid
  __shared__ unsigned long long red[3];
  const int t = threadIdx.x;
  const int cta = blockIdx.x, n_cta = gridDim.x;
  // per-slice results of k_score: total candidates and key range
  if (t == 0) {
    red[0] = 0;
    red[1] = ~0ull;
    red[2] = 0;
  }
  __syncthreads();
  {
    unsigned long long c = 0, mn = ~0ull, mx = 0;
    for (int i = t; i < G.n_slices; i += blockDim.x)
      if (G.ncnt[i]) {
        c += G.ncnt[i];
        mn = min(mn, static_cast<unsigned long long>(G.kmin[i]));
        mx = max(mx, static_cast<unsigned long long>(G.kmax[i]));
      }
    // warp reduction first: 64-bit shared atomics are CAS loops on sm_100a
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      c += __shfl_xor_sync(0xffffffffu, c, o);
      mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
      mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if ((t & 31) == 0 && c) {
      atomicAdd(&red[0], c);
      atomicMin(&red[1], mn);
      atomicMax(&red[2], mx);
    }
  }
  __syncthreads();
  const int64_t ncand = static_cast<int64_t>(red[0]);
  const uint64_t key_lo = red[1], key_hi = red[2];
  if (cta == 0) tp_set(G, 7);
  if (cta == 0 && mode == 0) {  // drop the exclusion marks (k_score has read them)
    const int64_t f = S.scal[S_F], b0 = A.blk_off[s];
    for (int64_t p = t; p < f; p += blockDim.x) P.pinned[S.prehit[b0 + p]] &= ~2;
  }
  const int64_t free_cnt = P.cap - static_cast<int64_t>(P.ctr[C_NRES]);
  int64_t K, Fp = 0;
  if (mode == 0) {
    const int64_t P_ = A.blk_off[s + 1] - A.blk_off[s];
    const int64_t rest = P_ - S.scal[S_F];
    Fp = min(free_cnt, rest);
    K = min(ncand, (rest > free_cnt ? rest - free_cnt : int64_t(0)) + static_cast<int64_t>(G.ctr[2]));
  } else if (mode == 2) {  // op program: K and F bounded by k_prog_bound
    const int64_t bnd = S.scal[S_NMISS] > 0 ? S.scal[S_BOUND] : 0;
    K = min(ncand, bnd);
    Fp = min(free_cnt, bnd);
  } else {
    K = min(ncand, needed);
  }
  // ---- lowest Fp free ids, ascending: each CTA lists the free ids of its
  // score slices, offset by the free counts of all lower slices
  if (Fp > 0) {
    const int lane = t & 31, w = t >> 5;
    __shared__ uint32_t wcnt[33];
    __shared__ unsigned long long below;
    for (int sl = cta; sl < G.n_slices; sl += n_cta) {
      if (t == 0) below = 0;
      __syncthreads();
      unsigned long long part = 0;
      for (int i = t; i < sl; i += blockDim.x) part += G.fcnt[i];
      part = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(part));
      if (lane == 0 && part) atomicAdd(&below, part);
      __syncthreads();
      int64_t found = static_cast<int64_t>(below);
      __syncthreads();
      if (found >= Fp || G.fcnt[sl] == 0) continue;  // uniform
      const int64_t lo = sl * G.slice, hi = min(P.cap, lo + G.slice);
      for (int64_t b = lo; b < hi && found < Fp; b += blockDim.x) {
        const int64_t i = b + t;
        const bool fr = i < hi && P.ntok[i] == 0;
        const unsigned ball = __ballot_sync(0xffffffffu, fr);
        if (lane == 0) wcnt[w] = __popc(ball);
        __syncthreads();
        if (w == 0) {
          const uint32_t c = lane < 32 ? wcnt[lane] : 0;
          uint32_t x = c;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
          }
          wcnt[lane] = x - c;
          if (lane == 31) wcnt[32] = x;
        }
        __syncthreads();
        const int64_t rank = found + wcnt[w] + __popc(ball & ((1u << lane) - 1));
        if (fr && rank < Fp) S.freel[rank] = static_cast<int32_t>(i);
        found += wcnt[32];
        __syncthreads();
      }
    }
  }
  // ---- radix select of the K smallest candidate keys (keys are unique).
  // The CTA's keys: its score slices' regions of G.keys, staged in shared
  // memory when they fit, else read in place each pass (L2-resident).
  // Staged when EVERY CTA's keys fit (a grid-uniform decision: the
  // compaction below is a grid-wide step): one bulk copy per slice into
  // shared memory, each slice's run padded to an even count (16 B aligned).
  __shared__ unsigned max_cta_keys;
  __shared__ uint64_t stage_bar;
  __shared__ int64_t seg_off[kMaxSlicesPerCta], seg_n[kMaxSlicesPerCta];
  if (t == 0) max_cta_keys = 0;
  __syncthreads();
  for (int c2 = t; c2 < n_cta; c2 += blockDim.x) {
    unsigned n2 = 0;
    for (int sl = c2; sl < G.n_slices; sl += n_cta) n2 += (G.ncnt[sl] + 1u) & ~1u;
    atomicMax(&max_cta_keys, n2);
  }
  __syncthreads();
  const bool staged = static_cast<int64_t>(max_cta_keys) <= G.sort_keys &&
                      (G.n_slices + n_cta - 1) / n_cta <= kMaxSlicesPerCta;
  int nseg = 0;
  if (staged) {
    int64_t off = 0;
    for (int sl = cta; sl < G.n_slices; sl += n_cta, ++nseg) {
      if (t == 0) {  // the segment table (read by all after the barrier below)
        seg_off[nseg] = off;
        seg_n[nseg] = G.ncnt[sl];
      }
      off += (G.ncnt[sl] + 1) & ~int64_t(1);
    }
    if (t == 0) {
      mbar_init(&stage_bar, 1);
      fence_barrier_init();
      fence_proxy_async();  // earlier generic accesses of this shared memory before the async writes
      fence_proxy_async_global();  // the keys were stored through the generic proxy
      mbar_arrive_expect_tx(&stage_bar, static_cast<uint32_t>(off * 8));
      for (int j = 0, sl = cta; j < nseg; ++j, sl += n_cta)
        if (seg_n[j] > 0)
          bulk_g2s(local_keys + seg_off[j], G.keys + sl * G.slice,
                   static_cast<uint32_t>(((seg_n[j] + 1) & ~int64_t(1)) * 8), &stage_bar);
    }
    __syncthreads();
    mbar_wait_suspend(&stage_bar, 0);
  }
  // Large pools (keys read in place): after the first radix pass the keys of
  // the chosen bin are compacted into S.keys (unused by this path) and the
  // lower bins' keys go straight to the victim list, so the later passes and
  // the final gather touch only the bin instead of every candidate.
  bool compacted = false;
  int64_t n_bin = 0;
  // Radix state, and a per-slice filter from the slice's key range: a pass
  // counting keys equal to the prefix (1) or taking keys up to it (2) skips
  // slices that cannot hold such a key (often most of them: ids are handed
  // out in order, so last_used and ids correlate).
  uint64_t prefix = 0, mask = 0;
  int slice_filter = 0;
  __shared__ int live[kMaxLiveSlices];
  __shared__ int n_live;
  auto slice_skip = [&](int sl) {
    if (!slice_filter || G.ncnt[sl] == 0) return slice_filter != 0;
    const uint64_t lo = G.kmin[sl] & mask, hi = G.kmax[sl] & mask;
    return lo > prefix || (slice_filter == 1 && hi < prefix);
  };
  // the slices passing the filter, listed in shared memory (the same list on
  // every CTA: it depends on global data only); returns their count
  auto live_slices = [&]() {
    if (t == 0) n_live = 0;
    __syncthreads();
    for (int sl = t; sl < G.n_slices; sl += blockDim.x)
      if (!slice_skip(sl)) live[atomicAdd(&n_live, 1)] = sl;
    __syncthreads();
    return n_live;
  };
  auto for_keys = [&](auto&& f) {
    if (compacted) {
      for (int64_t i = static_cast<int64_t>(cta) * blockDim.x + t; i < n_bin;
           i += static_cast<int64_t>(n_cta) * blockDim.x)
        f(S.keys[i]);
    } else if (staged) {
      for (int j = 0; j < nseg; ++j) {
        if (slice_skip(cta + j * n_cta)) continue;
        const uint64_t* src = local_keys + seg_off[j];
        for (int64_t i = t; i < seg_n[j]; i += blockDim.x) f(src[i]);
      }
    } else if (slice_filter && live_slices() * 4 <= G.n_slices) {
      // in place, few slices can hold a wanted key (the smallest keys often
      // sit in one slice, not spread over the CTAs' own slices): the whole
      // grid strides over each listed slice
      const int nl2 = n_live;
      for (int q = 0; q < nl2; ++q) {
        const int sl = live[q];
        const int64_t c = G.ncnt[sl];
        const uint64_t* src = G.keys + sl * G.slice;
        for (int64_t i = static_cast<int64_t>(cta) * blockDim.x + t; i < c;
             i += static_cast<int64_t>(n_cta) * blockDim.x)
          f(__ldcg(src + i));
      }
      __syncthreads();  // the list is rebuilt by the next pass
    } else {
      // in place (L2/HBM): key pairs as 16 B loads, four in flight per
      // thread before the keys are consumed, so a pass streams instead of
      // waiting one load latency per key (a slice's keys start 32 B aligned)
      constexpr int kU = 4;
      for (int sl = cta; sl < G.n_slices; sl += n_cta) {
        if (slice_skip(sl)) continue;
        const int64_t c = G.ncnt[sl];
        const uint64_t* src = G.keys + sl * G.slice;
        const ulonglong2* src2 = reinterpret_cast<const ulonglong2*>(src);
        for (int64_t p0 = t; 2 * p0 < c; p0 += kU * static_cast<int64_t>(blockDim.x)) {
          ulonglong2 v[kU];
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int64_t p = p0 + static_cast<int64_t>(u) * blockDim.x;
            v[u] = 2 * p + 1 < c ? __ldcg(src2 + p) : make_ulonglong2(2 * p < c ? __ldcg(src + 2 * p) : 0ull, 0ull);
          }
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int64_t p = p0 + static_cast<int64_t>(u) * blockDim.x;
            if (2 * p < c) f(v[u].x);
            if (2 * p + 1 < c) f(v[u].y);
          }
        }
      }
    }
  };
  __syncthreads();
  if (K > 0 && K < ncand) {
    const uint64_t kmin = key_lo, diff = key_lo ^ key_hi;
    int hi_bit = 64 - __clzll(static_cast<long long>(diff));  // bits above are shared by every candidate
    mask = hi_bit >= 64 ? 0ull : ~((uint64_t(1) << hi_bit) - 1);
    prefix = kmin & mask;
    int64_t need = K;
    for (int pass = 0; hi_bit > 0; ++pass) {
      const int wd = min(11, hi_bit), sh_ = hi_bit - wd;
      hi_bit = sh_;
      const uint64_t bmask = (uint64_t(1) << wd) - 1;
      hist[2 * t] = 0;
      hist[2 * t + 1] = 0;
      __syncthreads();
      if (pass == 0 && G.tprof && cta == 5 && t == 0) G.tprof[32 + 320 + 32] = gtimer();
      // (a warp-aggregated add for warps whose keys share a bin measured
      // slower than these plain shared atomics; the pass is bound by the key
      // loads, profiles/README.md)
      slice_filter = pass > 0 ? 1 : 0;  // pass 1's prefix is the bits every key shares
      for_keys([&](uint64_t k) {
        if ((k & mask) == prefix) atomicAdd(&hist[(k >> sh_) & bmask], 1u);
      });
      slice_filter = 0;
      if (pass == 0 && G.tprof && cta == 5 && (t & 31) == 0) G.tprof[32 + 320 + (t >> 5)] = gtimer();
      __syncthreads();
      if (pass < 2) tp_max(G, 22 + pass);
      if (pass < 2 && cta == 0) tp_set(G, 26 + pass);
      if (pass == 0 && G.tprof && t == 0) G.tprof[32 + cta] = gtimer();  // per-CTA pass-0 finish
      uint32_t* gh = G.hist + pass * 2048;
      if (hist[2 * t]) atomicAdd(&gh[2 * t], hist[2 * t]);
      if (hist[2 * t + 1]) atomicAdd(&gh[2 * t + 1], hist[2 * t + 1]);
      gsync();
      hist[2 * t] = gh[2 * t];
      hist[2 * t + 1] = gh[2 * t + 1];
      __syncthreads();
      const uint32_t a0 = hist[2 * t], a1 = hist[2 * t + 1];
      block_scan_2048(hist, warp_sums);
      const uint32_t e0 = hist[2 * t], e1 = hist[2 * t + 1];
      if (e0 < need && need <= e0 + a0) {
        sh[4] = 2 * t;
        sh[5] = e0;
        cnt_b = a0;
      }
      if (e1 < need && need <= e1 + a1) {
        sh[4] = 2 * t + 1;
        sh[5] = e1;
        cnt_b = a1;
      }
      __syncthreads();
      need -= sh[5];
      prefix |= static_cast<uint64_t>(sh[4]) << sh_;
      mask |= bmask << sh_;
      const bool done = static_cast<int64_t>(cnt_b) == need;
      __syncthreads();
      if (done) break;
      // the chosen bin plus the lower bins are few enough for the rank step
      // (O(M^2) compares spread over the grid: ~2 us at 4K keys, ~7 us at
      // 8K, where another radix pass costs ~3-4 us): gather them all and let
      // the rank step pick the K smallest
      if ((K - need) + static_cast<int64_t>(cnt_b) <= min(G.sort_keys, G.rank_early_max)) break;
      if (!staged && !compacted && hi_bit > 0) {
        const int lane = t & 31;
        auto append = [&](bool take, uint64_t k, unsigned long long* ctr, uint64_t* dst) {
          const unsigned am = __activemask();
          const unsigned b = __ballot_sync(am, take);
          if (!b) return;
          const int leader = __ffs(am) - 1;
          unsigned long long base = 0;
          if (lane == leader) base = atomicAdd(ctr, static_cast<unsigned long long>(__popc(b)));
          base = __shfl_sync(am, base, leader);
          if (take) dst[base + __popc(b & ((1u << lane) - 1u))] = k;
        };
        slice_filter = 2;
        for_keys([&](uint64_t k) {
          const uint64_t km = k & mask;
          append(km < prefix, k, &G.ctr[1], S.sortbuf);  // lower bins: selected
          append(km == prefix, k, &G.ctr[5], S.keys);    // the chosen bin
        });
        slice_filter = 0;
        tp_max(G, 24);
        if (cta == 0) tp_set(G, 28);
        if (G.tprof && t == 0) G.tprof[32 + 160 + cta] = gtimer();  // per-CTA compaction finish
        gsync();
        n_bin = static_cast<int64_t>(*reinterpret_cast<volatile unsigned long long*>(&G.ctr[5]));
        compacted = true;
      }
    }
  }
  if (K > 0) {
    // gather the selected keys (after a compaction only the chosen bin's:
    // the lower bins are listed already): one global atomic per warp
    const int lane = t & 31;
    slice_filter = 2;
    for_keys([&](uint64_t k) {
      const bool sel = K == ncand || (k & mask) <= prefix;
      const unsigned am = __activemask();
      const unsigned b = __ballot_sync(am, sel);
      if (!b) return;
      const int leader = __ffs(am) - 1;
      unsigned long long base = 0;
      if (lane == leader) base = atomicAdd(&G.ctr[1], static_cast<unsigned long long>(__popc(b)));
      base = __shfl_sync(am, base, leader);
      if (sel) S.sortbuf[base + __popc(b & ((1u << lane) - 1u))] = k;
    });
  }
  tp_max(G, 25);
  if (G.tprof && t == 0 && !compacted) G.tprof[32 + 160 + cta] = gtimer();  // per-CTA gather finish
  gsync();
  // gathered keys: K, or the K plus the rest of the chosen bin after an early exit
  const int64_t M = K > 0 ? static_cast<int64_t>(*reinterpret_cast<volatile unsigned long long*>(&G.ctr[1])) : 0;
  if (K > 0 && M <= G.sort_keys) {
    // every CTA: the M gathered keys into shared memory; CTA c ranks its
    // share of them (rank = gathered keys below it; keys are unique), one
    // warp per key, lanes splitting the comparisons; ranks < K are the victims
    tp_set(G, 20);
    constexpr int kLU = 8;  // eight loads in flight per thread, not one round trip per key
    for (int64_t i0 = t; i0 < M; i0 += kLU * static_cast<int64_t>(blockDim.x)) {
      uint64_t v[kLU];
#pragma unroll
      for (int u = 0; u < kLU; ++u) {
        const int64_t i = i0 + static_cast<int64_t>(u) * blockDim.x;
        v[u] = i < M ? __ldcg(S.sortbuf + i) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < kLU; ++u) {
        const int64_t i = i0 + static_cast<int64_t>(u) * blockDim.x;
        if (i < M) local_keys[i] = v[u];
      }
    }
    __syncthreads();
    if (cta == 0) tp_set(G, 29);  // keys loaded
    if (cta == 0 && t == 0 && G.tprof) G.tprof[31] = static_cast<unsigned long long>(M);
    const int64_t per = (M + n_cta - 1) / n_cta, r_lo = cta * per, r_hi = min(M, r_lo + per);
    const int lane = t & 31, nw = blockDim.x >> 5;
    for (int64_t i = r_lo + (t >> 5); i < r_hi; i += nw) {
      const uint64_t k = local_keys[i];
      unsigned c = 0;
      for (int64_t j = lane; j < M; j += 32) c += local_keys[j] < k;
      c = __reduce_add_sync(0xffffffffu, c);
      if (lane == 0 && c < K) {
        S.victims[c] = k;
        S.taken[c] = 0;
        S.rank_of[k & P.idmask] = static_cast<int32_t>(c);
      }
    }
    if (cta == 0 && G.tprof) {  // CTA 0's ranks written (each warp's last one)
      __syncthreads();
      tp_set(G, 30);
    }
    if (cta == 0 && t == 0) {
      S.scal[S_K] = K;
      S.scal[S_FREE] = Fp;
      S.scal[S_STATUS] = 0;
      S.scal[S_NCAND] = ncand;
    }
    tp_set(G, 21);
    return;
  }
  if (cta != 0) return;
  tp_set(G, 20);
  // ---- CTA 0: sort the K selected keys, publish them with their ranks
  if (K > 0) {
    int64_t n2 = 1;
    while (n2 < K) n2 <<= 1;
    uint64_t* dst = S.sortbuf;
    const bool in_smem = n2 <= G.sort_keys;  // dynamic smem holds G.sort_keys keys
    if (in_smem) {
      for (int64_t i = t; i < n2; i += blockDim.x) local_keys[i] = i < K ? S.sortbuf[i] : kNoKey;
      __syncthreads();
      if (n2 >= 1024 && 2 * n2 <= G.sort_keys) {  // merge sort (faster from 1K keys), scratch after the keys
        dst = merge_sort_smem(local_keys, local_keys + n2, static_cast<int>(n2));
      } else {
        bitonic_smem(local_keys, static_cast<int>(n2));
        dst = local_keys;
      }
    } else {
      for (int64_t i = K + t; i < n2; i += blockDim.x) S.sortbuf[i] = kNoKey;
      __syncthreads();
      bitonic_global(S.sortbuf, n2);
    }
    for (int64_t r = t; r < K; r += blockDim.x) {
      const uint64_t k = dst[r];
      S.victims[r] = k;
      S.taken[r] = 0;
      S.rank_of[k & P.idmask] = static_cast<int32_t>(r);
    }
  }
  if (t == 0) {
    S.scal[S_K] = K;
    S.scal[S_FREE] = Fp;
    S.scal[S_STATUS] = 0;
    S.scal[S_NCAND] = ncand;
  }
  tp_set(G, 21);
}

__global__ void __launch_bounds__(kSelectThreads, 1)
    k_select_coop(Pool P, Scratch S, InsertArgs A, int s, int mode, int64_t needed, CoopBuf G) {
  extern __shared__ __align__(128) uint64_t local_keys[];
  select_body(P, S, A, s, mode, needed, G, local_keys);
}

// k_score + k_select_coop as ONE cooperative kernel (one CTA per SM): the
// select reuses the scoring ring's shared memory, and the score -> select
// hand-off is a grid barrier instead of a kernel boundary (a launch gap of
// ~4 us and the select's ramp).  Modes 1 / 2 also take over k_plan's reset
// of the histograms and counters, so evict() is one launch.
__global__ void __launch_bounds__(kSelectThreads, 1)
    k_evict_fused(Pool P, Scratch S, InsertArgs A, int s, int mode, int64_t needed, CoopBuf G) {
  extern __shared__ __align__(128) uint8_t dyn_smem[];
  if (mode != 0 && blockIdx.x == 0) {  // k_plan's work for modes 1 / 2 (read only after the grid barrier)
    const int t = threadIdx.x;
    if (G.tprof && t < 32) G.tprof[t] = (t == 2 || t == 5) ? ~0ull : 0ull;
    __syncthreads();
    tp_set(G, 0);
    for (int i = t; i < 6 * 2048; i += blockDim.x) G.hist[i] = 0;
    if (t < 3) G.ctr[t] = 0;
    if (t == 3) G.ctr[3] = ~0ull;
    if (t == 4 || t == 5) G.ctr[t] = 0;
    if (t == 0) {
      S.scal[S_F] = 0;
      S.scal[S_STATUS] = 0;
    }
  }
  score_body(P, G, dyn_smem);
  cooperative_groups::this_grid().sync();
  select_body(P, S, A, s, mode, needed, G, reinterpret_cast<uint64_t*>(dyn_smem));
}

constexpr int kWalkSmemVictims = 4096;

__global__ void __launch_bounds__(32, 1) k_walk(Pool P, Scratch S, InsertArgs A, int s) {
  __shared__ uint64_t vic_s[kWalkSmemVictims];
  __shared__ uint8_t taken_s[kWalkSmemVictims];
  __shared__ int32_t pb[32], pr[32];
  __shared__ uint8_t pl[32];
  const int lane = threadIdx.x;
  if (S.scal[S_STATUS] != 0) {
    if (lane == 0) {
      S.scal[S_NEV] = 0;
      S.scal[S_NNEW] = 0;
      S.scal[S_FAILPOS] = -1;
    }
    return;
  }
  const int64_t b0 = A.blk_off[s];
  const int64_t P_ = A.blk_off[s + 1] - b0;
  const int64_t f = S.scal[S_F], K = S.scal[S_K], Fp = S.scal[S_FREE];
  const bool vs = K <= kWalkSmemVictims;
  if (vs)
    for (int64_t r = lane; r < K; r += 32) {
      vic_s[r] = S.victims[r];
      taken_s[r] = 0;
    }
  uint8_t* taken = vs ? taken_s : S.taken;
  const uint64_t now_bits = static_cast<uint64_t>(A.now + P.lbias) << P.idb;
  // late candidates: blocks that a hit in this insert raised from ref -1 to 0
  uint64_t lkey[kLateMax];
  int32_t lpos[kLateMax];
  int nl = 0;
  auto late_key = [&](int32_t id) {
    uint64_t k = now_bits | static_cast<uint64_t>(id);
    if (P.policy == SB_POLICY_TIERED) k |= static_cast<uint64_t>(tier_of(P.tag[id])) << 61;
    return k;
  };
  if (lane == 0) {
    const int64_t n_pre_late = S.scal[S_NLATE] < kLateMax ? S.scal[S_NLATE] : int64_t(kLateMax);
    for (int64_t i = 0; i < n_pre_late; ++i) {
      lpos[nl] = S.late[2 * i];
      lkey[nl++] = late_key(S.late[2 * i + 1]);
    }
  }
  __syncwarp();
  int64_t ptr = 0, fi = 0, nev = 0, nnew = 0, failpos = -1;
  int status = 0;
  bool taken_seen = false;  // lane 0: some victim was referenced by a hit of this insert
  for (int64_t p0 = f; p0 < P_ && status == 0; p0 += 32) {
    // the warp prefetches 32 positions' pre-state probe results
    const int64_t p = p0 + lane;
    int32_t b = -1, r = -1;
    uint8_t late = 0;
    if (p < P_) {
      b = S.prehit[b0 + p];
      if (b >= 0) {
        r = S.rank_of[b];
        late = P.ref[b] == -1 && P.pinned[b] == 0;
      }
    }
    // Fast path (the common case of a continuation: fresh tool-output blocks):
    // every position of the chunk misses, no late candidate is pending and no
    // victim was referenced, so the i-th miss takes the next free id, else the
    // next victim in (tier, last_used, id) order — all 32 lanes in parallel.
    const bool all_miss = __all_sync(0xffffffffu, b < 0);
    const bool simple = __shfl_sync(0xffffffffu, static_cast<int>(nl == 0 && !taken_seen), 0) != 0;
    if (all_miss && simple) {
      const int64_t n = (P_ - p0) < 32 ? (P_ - p0) : int64_t(32);
      const int64_t fi0 = __shfl_sync(0xffffffffu, fi, 0), ptr0 = __shfl_sync(0xffffffffu, ptr, 0);
      const int64_t nev0 = __shfl_sync(0xffffffffu, nev, 0);
      const int64_t a = Fp - fi0 > 0 ? Fp - fi0 : 0;  // free ids left
      const int64_t i = lane;
      bool ok = i < n;
      bool fail = false;
      int32_t id = -1;
      if (ok) {
        if (i < a) {
          id = S.freel[fi0 + i];
        } else if (ptr0 + (i - a) < K) {
          const uint64_t vk = vs ? vic_s[ptr0 + (i - a)] : S.victims[ptr0 + (i - a)];
          id = static_cast<int32_t>(vk & P.idmask);
          S.evicted[nev0 + (i - a)] = id;
        } else {
          fail = true;
        }
      }
      const unsigned fm = __ballot_sync(0xffffffffu, fail);
      const int64_t nok = fm ? static_cast<int64_t>(__ffs(fm) - 1) : n;  // positions assigned
      if (ok && i < nok) {
        S.chain_out[p0 + i] = id;
        S.kind[p0 + i] = 1;
      }
      if (lane == 0) {
        const int64_t from_free = nok < a ? nok : a;
        fi = fi0 + from_free;
        ptr = ptr0 + (nok - from_free);
        nev = nev0 + (nok - from_free);
        nnew += nok;
        if (fm) {
          status = SB_ERR_CACHE_FULL;
          failpos = p0 + nok;
        }
      }
      status = __shfl_sync(0xffffffffu, status, 0);
      __syncwarp();
      continue;
    }
    pb[lane] = b;
    pr[lane] = r;
    pl[lane] = late;
    __syncwarp();
    if (lane == 0) {
      const int64_t n = (P_ - p0) < 32 ? (P_ - p0) : int64_t(32);
      for (int64_t i = 0; i < n; ++i) {
        const int64_t q = p0 + i;
        const int32_t bb = pb[i], rr = pr[i];
        bool miss = bb < 0;
        if (!miss && rr >= 0) {
          if (rr < ptr && !taken[rr]) {
            miss = true;  // evicted earlier in this insert
          } else {
            taken[rr] = 1;  // referenced: no longer a candidate
            taken_seen = true;
          }
        }
        if (!miss) {
          S.chain_out[q] = bb;
          S.kind[q] = 0;
          if (pl[i] && nl < kLateMax) {
            lpos[nl] = static_cast<int32_t>(q);
            lkey[nl++] = late_key(bb);
          }
          continue;
        }
        int32_t id;
        if (fi < Fp) {
          id = S.freel[fi++];
        } else {
          while (ptr < K && taken[ptr]) ++ptr;
          int li = -1;
          for (int k = 0; k < nl; ++k)
            if (li < 0 || lkey[k] < lkey[li]) li = k;
          const uint64_t vk = ptr < K ? (vs ? vic_s[ptr] : S.victims[ptr]) : kNoKey;
          const bool use_list = ptr < K && (li < 0 || vk < lkey[li]);
          if (!use_list && li < 0) {
            status = SB_ERR_CACHE_FULL;
            failpos = q;
            break;
          }
          if (use_list) {
            id = static_cast<int32_t>(vk & P.idmask);
            ++ptr;
          } else {
            id = static_cast<int32_t>(lkey[li] & P.idmask);
            S.kind[lpos[li]] = 2;  // hit, then evicted later in this insert
            lkey[li] = lkey[nl - 1];
            lpos[li] = lpos[nl - 1];
            --nl;
          }
          S.evicted[nev++] = id;
        }
        S.chain_out[q] = id;
        S.kind[q] = 1;
        ++nnew;
      }
    }
    status = __shfl_sync(0xffffffffu, status, 0);
    __syncwarp();
  }
  if (lane == 0) {
    S.scal[S_NEV] = nev;
    S.scal[S_NNEW] = nnew;
    S.scal[S_FAILPOS] = failpos;
    S.scal[S_STATUS] = status;
  }
}

__global__ void k_commit_evict(Pool P, Scratch S) {
  const int64_t nev = S.scal[S_NEV];
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nev;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t id = S.evicted[i];
    P.idx[P.slot[id]].id = -2;
    P.ntok[id] = 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && nev > 0) {
    P.ctr[C_NRES] -= static_cast<unsigned long long>(nev);
    P.ctr[C_EVICTED] += static_cast<unsigned long long>(nev);
    P.ctr[C_EV_BLOCKS] += static_cast<unsigned long long>(nev);
  }
}

__device__ __forceinline__ int tag_at(const sb_tag_range* tags, int64_t ntags, int64_t pos) {
  for (int64_t r = 0; r < ntags; ++r)
    if (pos >= tags[r].begin && pos < tags[r].end) return tags[r].tag;
  return ntags ? tags[ntags - 1].tag : SB_TAG_RESPONSE;
}

__global__ void k_commit_apply(Pool P, Scratch S, InsertArgs A, int s) {
  const int64_t b0 = A.blk_off[s];
  const int64_t P_ = A.blk_off[s + 1] - b0;
  const int64_t status = S.scal[S_STATUS];
  const int64_t f = S.scal[S_F];
  const int64_t K = S.scal[S_K];
  const int64_t gid = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t r = gid; r < K; r += stride) S.rank_of[S.victims[r] & P.idmask] = -1;
  if (gid == 0) {
    A.status[s] = static_cast<int32_t>(status);
    if (status == 0) {
      P.ctr[C_NRES] += static_cast<unsigned long long>(S.scal[S_NNEW]);
      P.ctr[C_INS_BLOCKS] += static_cast<unsigned long long>(S.scal[S_NNEW]);
    } else if (status == SB_ERR_CACHE_FULL) {
      P.ctr[C_FULL] += 1ull;
    }
  }
  if (status != 0)
    for (int64_t p = gid; p < P_; p += stride) A.out_ids[b0 + p] = -1;
  if (status == SB_ERR_CACHE) return;
  const int64_t limit = status == 0 ? P_ : S.scal[S_FAILPOS];
  const int64_t n = A.seq_off[s + 1] - A.seq_off[s];
  const uint64_t* tok = A.tokens + A.seq_off[s];
  const sb_tag_range* tags = A.tags + A.tag_off[s];
  const int64_t ntags = A.tag_off[s + 1] - A.tag_off[s];
  for (int64_t p = gid; p < limit; p += stride) {
    const int kd = S.kind[p];
    const bool hit = kd == 0;
    const int32_t id = p < f ? S.prehit[b0 + p] : S.chain_out[p];
    if (kd == 2) {
      // block was hit, then evicted (and possibly re-allocated) later in this insert
    } else if (hit) {
      if (status == 0) atomicAdd(&P.ref[id], 1);
      P.last[id] = A.now;
    } else if (status == 0) {
      const int64_t pos = p * P.bs;
      const int len = static_cast<int>(min(P.bs, n - pos));
      uint64_t* dst = P.tok + static_cast<int64_t>(id) * P.bs;
      for (int i = 0; i < len; ++i) dst[i] = tok[pos + i];
      P.ntok[id] = len;
      const uint64_t h = A.hashes[b0 + p];
      P.chain[id] = h;
      P.parent[id] = p ? A.hashes[b0 + p - 1] : kRootHash;
      P.tag[id] = tag_at(tags, ntags, pos);
      P.ref[id] = 1;
      P.last[id] = A.now;
      P.pinned[id] = 0;
      index_insert(P, h, id, P.parent[id], len);
    }
    if (status == 0) A.out_ids[b0 + p] = id;
  }
}

// --------------------------------------------------------- small ops
// First failing index of a release (kv_cache.cpp:228-236): UnknownBlock /
// ZeroRefRelease, checked in id order; apply only if none.
__global__ void k_validate_ids(Pool P, const int32_t* ids, int64_t n, int check_ref, int64_t* scal,
                               int skip_negative = 0) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t id = ids[i];
    if (skip_negative && id < 0) continue;
    const bool known = id >= 0 && id < P.cap && P.ntok[id] > 0;
    if (!known || (check_ref && P.ref[id] < 1))
      atomicMin(reinterpret_cast<unsigned long long*>(&scal[S_ERRIDX]), (unsigned long long)i);
  }
}
__global__ void k_release_apply(Pool P, const int32_t* ids, int64_t n, const int64_t* scal) {
  if (scal[S_ERRIDX] < n) return;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (ids[i] >= 0) atomicSub(&P.ref[ids[i]], 1);
}
// Batched KvCache::block(id) read-back: one record per id, n_tokens == 0 for
// an id that is out of range or not resident.
__global__ void k_block_info(Pool P, const int32_t* ids, int64_t n, sb_block_info* out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t id = ids[i];
    sb_block_info b{};
    b.block_id = id;
    if (id >= 0 && id < P.cap && P.ntok[id] > 0) {
      b.tag = P.tag[id];
      b.tier = tier_of(b.tag);
      b.ref_count = P.ref[id];
      b.last_used = P.last[id];
      b.chain_hash = P.chain[id];
      b.parent_hash = P.parent[id];
      b.pinned = P.pinned[id];
      b.n_tokens = P.ntok[id];
    }
    out[i] = b;
  }
}
__global__ void k_touch_apply(Pool P, const int32_t* ids, int64_t n, int64_t now, const int64_t* scal) {
  const int64_t lim = min(n, scal[S_ERRIDX]);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < lim;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    P.last[ids[i]] = now;
}
__global__ void k_priority_apply(Pool P, const int32_t* ids, int64_t n, int pinned, int tier, const int64_t* scal) {
  if (scal[S_ERRIDX] < n) return;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (pinned >= 0) P.pinned[ids[i]] = pinned;
    if (tier >= 0) P.tag[ids[i]] = tier;
  }
}
__global__ void k_set_scal(int64_t* scal, int idx, int64_t v) { scal[idx] = v; }
// the op program's bound accumulators (k_prog_bound adds to them)
__global__ void k_init_bound(int64_t* scal) {
  if (threadIdx.x == 0) {
    scal[S_BOUND] = 64;
    scal[S_NMISS] = 0;
    scal[S_NLATEHIT] = 0;
  }
}
__global__ void k_release_status(Pool P, const int32_t* ids, int64_t n, const int64_t* scal, int32_t* status) {
  if (threadIdx.x) return;
  const int64_t e = scal[S_ERRIDX];
  if (e >= n) {
    *status = SB_OK;
    return;
  }
  const int32_t id = ids[e];
  *status = (id < 0 || id >= P.cap || P.ntok[id] == 0) ? SB_ERR_UNKNOWN_BLOCK : SB_ERR_ZERO_REF_RELEASE;
}

__global__ void k_evict_out(Pool P, Scratch S, int32_t* out, int64_t* n_out) {
  const int64_t K = S.scal[S_K];
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < K;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t id = static_cast<int32_t>(S.victims[r] & P.idmask);
    out[r] = id;
    S.evicted[r] = id;
    S.rank_of[id] = -1;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    S.scal[S_NEV] = K;
    *n_out = K;
  }
}

// Rebuild the index without tombstones.
__global__ void k_index_clear(Pool P) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < P.tcap;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    P.idx[i].id = -1;
}
__global__ void k_index_fill(Pool P) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < P.cap;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (P.ntok[i] > 0) index_insert(P, P.chain[i], static_cast<int32_t>(i), P.parent[i], P.ntok[i]);
}

// out[pos ? pos[i] : i] = chain hash of resident block ids[i]
__global__ void k_gather_chain(Pool P, const int32_t* __restrict__ ids, const int64_t* __restrict__ pos, int64_t n,
                               uint64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[pos ? pos[i] : i] = P.chain[ids[i]];
}

__global__ void k_fill_i32(int32_t* p, int64_t n, int32_t v) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] = v;
}

#include "pool_program.cuh"
#include "pool_batch.cuh"

// PK_INSERT descriptors of a device-described batch (sb_kv_insert_batch).
__global__ void k_build_insert_ops(ProgOp* ops, const uint64_t* tokens, const int64_t* seq_off, const sb_tag_range* tags,
                                   const int64_t* tag_off, const int64_t* blk_off, const uint64_t* hashes,
                                   int32_t* out_ids, int n_seqs) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= n_seqs) return;
  ProgOp o{};
  o.kind = PK_INSERT;
  o.n = seq_off[s + 1] - seq_off[s];
  o.tokens = tokens + seq_off[s];
  o.hashes = hashes + blk_off[s];
  o.ins_tags = tags + tag_off[s];
  o.n_ins_tags = static_cast<int32_t>(tag_off[s + 1] - tag_off[s]);
  o.ids = out_ids + blk_off[s];
  o.pos_off = blk_off[s];
  ops[s] = o;
}
__global__ void k_prog_status(const ProgRes* res, int n, int32_t* status) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < n) status[s] = res[s].status;
}

// ==================================================================== host
template <class T>
static T* dalloc(size_t n) {
  T* p = nullptr;
  if (n == 0) n = 1;
  SB_CUDA(cudaMalloc(&p, n * sizeof(T)));
  return p;
}

static void check_now(const Pool& P, int64_t now) {
  if (now < -P.lbias || now >= P.lbias)
    throw Error(SB_ERR_UNSUPPORTED, "now outside +-2^" + std::to_string(60 - P.idb) + " for this pool size");
}

// Batched prefix probe for 16-token blocks, two phases per CTA of
// kProbe2 consecutive positions of one sequence, so every memory access of a
// phase is independent and all of them are in flight at once:
//   A  one thread per position: the position's chain hash (and its parent's,
//      the previous element), the 32 B index slot it hashes to (one random
//      sector); a slot whose (chain hash, parent, ntok) match names the
//      candidate block, an empty slot is a miss, anything else (tombstone,
//      other entry: a longer probe sequence) is left to phase C;
//   B  eight lanes per candidate position: the block's 128 B token row and
//      the position's 128 B of query tokens, 16 B per lane, four positions
//      per warp per round and four rounds in flight; the eight lanes vote;
//   C  positions A or B could not decide (probe chains, a hash collision)
//      run the full lane-pair walk (probe_find_g).
// The old one-kernel state machine (k_probe_rows) issued the slot and the
// token row of a position as two dependent round trips per lane pair; ncu
// showed it latency bound (long_scoreboard 15.3 stalls per issue).
constexpr int kProbe2 = 256;
__global__ void __launch_bounds__(kProbe2, 4) k_probe_rows2(Pool P, const uint64_t* __restrict__ tokens,
                                                            const int64_t* __restrict__ seq_off,
                                                            const int64_t* __restrict__ blk_off,
                                                            const uint64_t* __restrict__ hashes,
                                                            int32_t* __restrict__ prehit,
                                                            int64_t* __restrict__ first_miss, int full_only_check) {
  __shared__ int32_t cand[kProbe2];
  __shared__ int32_t slow[kProbe2];
  __shared__ int n_slow;
  __shared__ int64_t fm;
  const int sq = blockIdx.x, t = threadIdx.x;
  const int64_t b0 = blk_off[sq], np = blk_off[sq + 1] - b0;
  const int64_t j0 = static_cast<int64_t>(blockIdx.y) * kProbe2;
  if (j0 >= np) return;  // CTA-uniform
  const int64_t t0 = seq_off[sq], t1 = seq_off[sq + 1];
  const int nloc = static_cast<int>(min(static_cast<int64_t>(kProbe2), np - j0));
  if (t == 0) {
    n_slow = 0;
    fm = INT64_MAX;
  }
  // ---- A
  int32_t c = -1;
  if (t < nloc) {
    const int64_t j = j0 + t;
    const int64_t base = t0 + j * 16;
    const int len = static_cast<int>(min(static_cast<int64_t>(16), t1 - base));
    if (!(full_only_check && len < 16)) {
      const uint64_t h = hashes[b0 + j];
      const uint64_t parent = j ? hashes[b0 + j - 1] : kRootHash;
      uint64_t key, par;
      int32_t id, nt;
      ld_slot(P.idx + index_slot(h, P.tcap), key, par, id, nt);
      c = id == -1 ? -1 : (id >= 0 && key == h && par == parent && nt == len) ? id : -2;
    }
  }
  cand[t] = c;
  __syncthreads();
  // ---- B: position q = 32 r + (t >> 3), lane part p = t & 7 holds tokens [2p, 2p + 2)
  const int part = t & 7, lane = t & 31;
  for (int r0 = 0; r0 < kProbe2 / 32; r0 += 4) {
    uint64_t x[4][2], y[4][2];
    int lens[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = 32 * (r0 + u) + (t >> 3);
      const int32_t id = q < nloc ? cand[q] : -1;
      const int64_t base = t0 + (j0 + q) * 16;
      const int len = q < nloc ? static_cast<int>(min(static_cast<int64_t>(16), t1 - base)) : 0;
      lens[u] = id >= 0 ? len : 0;
      x[u][0] = x[u][1] = y[u][0] = y[u][1] = 0;
      if (id >= 0) {
        ld_v2(P.tok + static_cast<int64_t>(id) * 16 + 2 * part, x[u][0], x[u][1]);
        if (2 * part + 1 < len && ((base + 2 * part) & 1) == 0) {
          const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(tokens + base + 2 * part));
          y[u][0] = v.x;
          y[u][1] = v.y;
        } else {
          if (2 * part < len) y[u][0] = __ldg(reinterpret_cast<const unsigned long long*>(tokens + base + 2 * part));
          if (2 * part + 1 < len) y[u][1] = __ldg(reinterpret_cast<const unsigned long long*>(tokens + base + 2 * part + 1));
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = 32 * (r0 + u) + (t >> 3);
      const bool eq = (2 * part >= lens[u] || x[u][0] == y[u][0]) && (2 * part + 1 >= lens[u] || x[u][1] == y[u][1]);
      const unsigned vote = __ballot_sync(0xffffffffu, eq);
      const bool all8 = ((vote >> (lane & ~7)) & 0xffu) == 0xffu;
      if (part == 0 && q < nloc && cand[q] >= 0 && !all8) cand[q] = -2;  // a chain hash collision: full walk
    }
  }
  __syncthreads();
  if (t < nloc && cand[t] == -2) slow[atomicAdd(&n_slow, 1)] = t;
  __syncthreads();
  // ---- C: the full walk for the undecided positions (lane pairs)
  for (int b = 0; b < n_slow; b += kProbe2 / kGroup) {
    const int i = b + (t >> 1);
    const bool active = i < n_slow;
    const int q = active ? slow[i] : slow[0];
    const int64_t j = j0 + q;
    const int64_t base = t0 + j * 16;
    const int len = static_cast<int>(min(static_cast<int64_t>(16), t1 - base));
    const uint64_t h = hashes[b0 + j];
    const uint64_t parent = j ? hashes[b0 + j - 1] : kRootHash;
    const int32_t id = probe_find_g<true>(P, active, h, parent, tokens + base, len, t & 1);
    if (active && (t & 1) == 0) cand[q] = id;
  }
  __syncthreads();
  if (t < nloc) {
    const int32_t id = cand[t];
    prehit[b0 + j0 + t] = id;
    if (id < 0) atomicMin(reinterpret_cast<unsigned long long*>(&fm), static_cast<unsigned long long>(j0 + t));
  }
  __syncthreads();
  if (t == 0 && first_miss && fm != INT64_MAX)
    atomicMin(reinterpret_cast<unsigned long long*>(first_miss + sq), static_cast<unsigned long long>(fm));
}

// The same three phases per WARP (32 consecutive positions, no shared memory
// and no CTA barrier, so warps of one CTA never wait for each other — ncu of
// the per-CTA version showed barrier stalls (8.2 per issue) next to the
// memory latency): A one lane per position; B four positions per round with
// eight lanes each, all rounds' loads issued before any compare; C lane pairs
// walk the undecided positions.
constexpr int kProbe3Warps = 8;
__global__ void __launch_bounds__(32 * kProbe3Warps, 4) k_probe_rows3(Pool P, const uint64_t* __restrict__ tokens,
                                                                      const int64_t* __restrict__ seq_off,
                                                                      const int64_t* __restrict__ blk_off,
                                                                      const uint64_t* __restrict__ hashes,
                                                                      int32_t* __restrict__ prehit,
                                                                      int64_t* __restrict__ first_miss,
                                                                      int full_only_check, int speculate) {
  const int sq = blockIdx.x, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t b0 = blk_off[sq], np = blk_off[sq + 1] - b0;
  const int64_t jw = (static_cast<int64_t>(blockIdx.y) * kProbe3Warps + w) * 32;  // this warp's first position
  if (jw >= np) return;  // warp-uniform
  const int64_t t0 = seq_off[sq], t1 = seq_off[sq + 1];
  const int nloc = static_cast<int>(min(static_cast<int64_t>(32), np - jw));
  // ---- A: lane 0 probes the index; the blocks of one chain are usually
  // consecutive ids (an insert allocates the lowest free ids in order), so
  // lane l first tries block anchor + l and verifies it from the block's own
  // metadata (chain hash, parent hash, ntok: coalesced reads); only lanes
  // whose guess fails probe the index (a random 32 B sector each).  The
  // verified block is the one find_chain_block returns: at most one resident
  // block matches a (chain hash, parent, tokens) — an insert that finds one
  // reuses it.
  int32_t c = -1;
  const int64_t j = jw + lane;
  const int64_t tbase = t0 + j * 16;
  const int tlen = static_cast<int>(min(static_cast<int64_t>(16), t1 - tbase));
  const bool valid = lane < nloc && !(full_only_check && tlen < 16);
  uint64_t h = 0, parent = kRootHash;
  if (valid) {
    h = hashes[b0 + j];
    if (j) parent = hashes[b0 + j - 1];
  }
  auto idx_probe = [&]() {
    uint64_t key, par;
    int32_t id, nt;
    ld_slot(P.idx + index_slot(h, P.tcap), key, par, id, nt);
    return id == -1 ? -1 : (id >= 0 && key == h && par == parent && nt == tlen) ? id : -2;
  };
  int32_t a = -1;
  if (lane == 0 && valid && speculate) a = idx_probe();
  a = __shfl_sync(0xffffffffu, a, 0);
  bool need_idx = false;
  if (lane == 0 && speculate) {
    c = a;
  } else if (valid) {
    need_idx = true;
    if (a >= 0 && a + lane < P.cap) {
      const int32_t g = a + lane;
      if (P.ntok[g] == tlen && P.chain[g] == h && P.parent[g] == parent) {
        c = g;
        need_idx = false;
      }
    }
  }
  if (need_idx) c = idx_probe();
  // ---- B: round r covers positions 4r .. 4r+3 of the warp (q = 4r + lane / 8), lane part p = lane % 8
  const int part = lane & 7, sub = lane >> 3;
  uint32_t bad = 0;  // bit q: position q's block tokens differ (a chain hash collision)
#pragma unroll
  for (int r0 = 0; r0 < 8; r0 += 4) {
    uint64_t x[4][2], y[4][2];
    int lens[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = 4 * (r0 + u) + sub;
      const int32_t id = __shfl_sync(0xffffffffu, c, q);
      const int64_t base = t0 + (jw + q) * 16;
      const int len = q < nloc ? static_cast<int>(min(static_cast<int64_t>(16), t1 - base)) : 0;
      lens[u] = id >= 0 ? len : 0;
      x[u][0] = x[u][1] = y[u][0] = y[u][1] = 0;
      if (id >= 0) {
        ld_v2(P.tok + static_cast<int64_t>(id) * 16 + 2 * part, x[u][0], x[u][1]);
        if (2 * part + 1 < len && ((base + 2 * part) & 1) == 0) {
          const ulonglong2 v = __ldg(reinterpret_cast<const ulonglong2*>(tokens + base + 2 * part));
          y[u][0] = v.x;
          y[u][1] = v.y;
        } else {
          if (2 * part < len) y[u][0] = __ldg(reinterpret_cast<const unsigned long long*>(tokens + base + 2 * part));
          if (2 * part + 1 < len) y[u][1] = __ldg(reinterpret_cast<const unsigned long long*>(tokens + base + 2 * part + 1));
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const bool eq = (2 * part >= lens[u] || x[u][0] == y[u][0]) && (2 * part + 1 >= lens[u] || x[u][1] == y[u][1]);
      const unsigned vote = __ballot_sync(0xffffffffu, !eq);  // lanes whose 2 tokens differ
#pragma unroll
      for (int k = 0; k < 4; ++k)
        if ((vote >> (8 * k)) & 0xffu) bad |= 1u << (4 * (r0 + u) + k);
    }
  }
  if (c >= 0 && ((bad >> lane) & 1u)) c = -2;
  // ---- C: lane pairs walk the undecided positions, 16 at a time
  unsigned slow = __ballot_sync(0xffffffffu, lane < nloc && c == -2);
  while (slow) {
    // the pair's position: the (lane / 2)-th set bit of slow
    unsigned m = slow;
    for (int k = 0; k < (lane >> 1) && m; ++k) m &= m - 1u;
    const bool active = m != 0;
    const int q = active ? __ffs(m) - 1 : __ffs(slow) - 1;
    const int64_t j = jw + q;
    const int64_t base = t0 + j * 16;
    const int len = static_cast<int>(min(static_cast<int64_t>(16), t1 - base));
    const uint64_t h = hashes[b0 + j];
    const uint64_t parent = j ? hashes[b0 + j - 1] : kRootHash;
    __syncwarp();
    const int32_t id = probe_find_g<true>(P, active, h, parent, tokens + base, len, lane & 1);
    // hand the result to the position's own lane
    const unsigned got = __ballot_sync(0xffffffffu, active && (lane & 1) == 0);
    for (int pr = 0; pr < 16; ++pr) {
      if (!((got >> (2 * pr)) & 1u)) continue;  // warp-uniform
      const int qq = __shfl_sync(0xffffffffu, q, 2 * pr);
      const int32_t v = __shfl_sync(0xffffffffu, id, 2 * pr);
      if (lane == qq) c = v;
      slow &= ~(1u << qq);
    }
  }
  if (lane < nloc) prehit[b0 + jw + lane] = c;
  const unsigned miss = __ballot_sync(0xffffffffu, lane < nloc && c < 0);
  if (lane == 0 && miss && first_miss)
    atomicMin(reinterpret_cast<unsigned long long*>(first_miss + sq), static_cast<unsigned long long>(jw + __ffs(miss) - 1));
}

static void launch_probe_rows(const Pool& P, const uint64_t* tokens, const int64_t* seq_off, const int64_t* blk_off,
                              const uint64_t* hashes, int32_t* prehit, int64_t* first_miss, int full_only_check,
                              int n_seqs, int64_t max_np, cudaStream_t st) {
  static int per = -1;
  if (per < 0) {
    const char* e = getenv("SB_PROBE_PER");
    per = e ? atoi(e) : 0;  // 0: the warp-granular k_probe_rows3 (16-token blocks)
  }
  if (per == 0 && P.bs == 16) {  // warp-granular two-phase probe
    const int64_t runs = (max_np + 32 * kProbe3Warps - 1) / (32 * kProbe3Warps);
    if (runs > 65535) throw Error(SB_ERR_UNSUPPORTED, "sequence too long for one lookup launch");
    static int spec = -1;  // SB_PROBE_SPEC=0: every position probes the index (no consecutive-id guess)
    if (spec < 0) {
      const char* e = getenv("SB_PROBE_SPEC");
      spec = e && e[0] == '0' ? 0 : 1;
    }
    k_probe_rows3<<<dim3(n_seqs, static_cast<unsigned>(runs)), 32 * kProbe3Warps, 0, st>>>(
        P, tokens, seq_off, blk_off, hashes, prehit, first_miss, full_only_check, spec);
    return;
  }
  if (per == 3 && P.bs == 16) {  // the per-CTA two-phase probe
    const int64_t runs = (max_np + kProbe2 - 1) / kProbe2;
    if (runs > 65535) throw Error(SB_ERR_UNSUPPORTED, "sequence too long for one lookup launch");
    k_probe_rows2<<<dim3(n_seqs, static_cast<unsigned>(runs)), kProbe2, 0, st>>>(P, tokens, seq_off, blk_off, hashes,
                                                                                 prehit, first_miss, full_only_check);
    return;
  }
  if (per == 0) per = 2;
  const int run = kProbePairs * per;
  const int64_t runs = (max_np + run - 1) / run;
  if (runs > 65535) throw Error(SB_ERR_UNSUPPORTED, "sequence too long for one lookup launch");
  const dim3 grid(n_seqs, static_cast<unsigned>(runs));
  if (per == 1)
    k_probe_rows<1><<<grid, kProbePairs * kGroup, 0, st>>>(P, tokens, seq_off, blk_off, hashes, prehit, first_miss,
                                                            full_only_check);
  else if (per == 2)
    k_probe_rows<2><<<grid, kProbePairs * kGroup, 0, st>>>(P, tokens, seq_off, blk_off, hashes, prehit, first_miss,
                                                            full_only_check);
  else
    k_probe_rows<4><<<grid, kProbePairs * kGroup, 0, st>>>(P, tokens, seq_off, blk_off, hashes, prehit, first_miss,
                                                            full_only_check);
}

// SB_LEGACY_INSERT=1: the per-sequence insert pipeline (probe, select, walk,
// commit per sequence) instead of the op program — kept for A/B checks.
static bool legacy_insert() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SB_LEGACY_INSERT");
    v = e && atoi(e) ? 1 : 0;
  }
  return v == 1;
}

static int grid_for(int64_t n, int threads = 256) {
  int64_t g = (n + threads - 1) / threads;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(g, int64_t(1) << 30)));
}

}  // namespace sb

using namespace sb;

struct sb_kv_cache {
  Pool P{};
  Scratch S{};
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t tomb_bound = 0;  // upper bound on index tombstones
  std::mutex mu;
  // device staging for the per-op API
  uint64_t* d_tok = nullptr;
  int64_t tok_cap = 0;
  sb_tag_range* d_tags = nullptr;
  int64_t tags_cap = 0;
  int64_t* d_meta = nullptr;  // seq_off[2], blk_off[2], tag_off[2], misc
  int32_t* d_ids = nullptr;
  int64_t ids_cap = 0;
  int32_t* d_status = nullptr;
  int64_t* d_first = nullptr;
  int64_t* d_hit = nullptr;
  uint64_t* d_hash_all = nullptr;
  int64_t hash_cap = 0;
  int32_t* d_prehit_all = nullptr;
  int64_t prehit_cap = 0;
  int64_t* d_batch_blk = nullptr;
  int64_t* d_batch_first = nullptr;
  int64_t batch_cap = 0;
  // cooperative scorer (large pools)
  CoopBuf G{};
  int coop_grid = 0;
  size_t coop_smem = 0;
  size_t fused_smem = 0;  // k_evict_fused's dynamic shared memory (0: not launchable, three kernels instead)
  static bool fused_enabled() {  // SB_EVICT_FUSED=0 selects k_plan + k_score + k_select_coop
    static int on = -1;
    if (on < 0) {
      const char* e = getenv("SB_EVICT_FUSED");
      on = e ? atoi(e) != 0 : 1;
    }
    return on;
  }

  // op program (pool_program.cuh)
  ProgOp* d_ops = nullptr;
  int64_t ops_cap = 0;
  ProgRes* d_res = nullptr;
  uint64_t* d_runk = nullptr;
  int64_t runk_cap = 0;
  int64_t* d_pout = nullptr;
  int64_t* h_pout = nullptr;  // pinned
  int32_t* d_pre_all = nullptr;  // pre-program probe of every insert position
  int64_t pre_all_cap = 0;
  unsigned long long* d_created = nullptr;  // chain hashes created by a program
  int64_t created_cap = 0;
  int prog_device_attr = -1;
  // parallel op-program path (pool_batch.cuh)
  FastBuf FB{};
  int64_t fb_ops_cap = 0, fb_pos_cap = 0, fb_ev_cap = 0, fb_dup_cap = 0;
  unsigned long long fast_runs = 0, fast_taken = 0;
  uint64_t launches = 0;  // kernels the op programs / lookups launched (sb_batch_run reports them)
  std::vector<int32_t> last_evicted;  // ids evicted by the last per-op insert / evict (sb_kv_last_evicted)

  // k_score + k_select_coop (all SMs, three launches incl. a cooperative one)
  // vs the one-CTA k_select (one launch).  Op programs (mode 2) run between
  // host synchronisations, where launch count is latency, so they keep the
  // one-CTA select up to kProgCoopMinCap blocks (the configs[1] engine step,
  // 27K-block pool: 1.61 vs 1.88 ms per step of pool work).
  bool use_coop(int mode) const {
    static int64_t min_cap = -1, prog_min_cap = -1;  // SB_COOP_MIN_CAP / SB_PROG_COOP_MIN_CAP override
    if (min_cap < 0) {
      const char* e = getenv("SB_COOP_MIN_CAP");
      min_cap = e ? atoll(e) : kCoopMinCap;
      const char* f = getenv("SB_PROG_COOP_MIN_CAP");
      prog_min_cap = f ? atoll(f) : kProgCoopMinCap;
    }
    return P.cap >= (mode == 2 ? std::max(min_cap, prog_min_cap) : min_cap) && coop_grid > 0;
  }

  // SB_PROG_PROFILE=1: per-phase cycle counters of the op program, printed
  // to stderr at destruction (phases: 0 setup, 1 hints, 2 re-probe, 3 flags,
  // 4 victim window, 5 walk, 6 evictions, 7 commit, 8 late runs, 9 op
  // dispatch, 10 op follow-ups: pins / unpins / releases)
  unsigned long long* d_prof = nullptr;
  unsigned long long* prof_buf() {
    static int on = -1;
    if (on < 0) {
      const char* e = getenv("SB_PROG_PROFILE");
      on = e && atoi(e) ? 1 : 0;
    }
    if (!on) return nullptr;
    if (!d_prof) {
      d_prof = dalloc<unsigned long long>(64);
      SB_CUDA(cudaMemset(d_prof, 0, 64 * sizeof(unsigned long long)));
    }
    return d_prof;
  }

  // Ordering between the pool's own stream (per-op calls) and a caller's
  // stream (batched calls): work on `st` starts after everything issued on
  // the pool stream, and later pool-stream work starts after what `st` got.
  cudaEvent_t ev_pool = nullptr, ev_user = nullptr;
  void join_in(cudaStream_t st) {
    if (st == stream) return;
    if (!ev_pool) SB_CUDA(cudaEventCreateWithFlags(&ev_pool, cudaEventDisableTiming));
    SB_CUDA(cudaEventRecord(ev_pool, stream));
    SB_CUDA(cudaStreamWaitEvent(st, ev_pool, 0));
  }
  void join_out(cudaStream_t st) {
    if (st == stream) return;
    if (!ev_user) SB_CUDA(cudaEventCreateWithFlags(&ev_user, cudaEventDisableTiming));
    SB_CUDA(cudaEventRecord(ev_user, st));
    SB_CUDA(cudaStreamWaitEvent(stream, ev_user, 0));
  }

  void ensure_ops(int64_t n) {
    if (n <= ops_cap) return;
    cudaFree(d_ops);
    cudaFree(d_res);
    ops_cap = std::max<int64_t>(n, 2 * ops_cap + 8);
    d_ops = dalloc<ProgOp>(ops_cap);
    d_res = dalloc<ProgRes>(ops_cap);
  }
  void ensure_runk(int64_t n) {
    if (n <= runk_cap) return;
    cudaFree(d_runk);
    runk_cap = std::max<int64_t>(n, 2 * runk_cap);
    d_runk = dalloc<uint64_t>(runk_cap);
  }

  // Runs ops [0, n_ops) already in d_ops on stream st: per launch, the
  // pre-state bound, one hint-aware scoring pass + select of K victims /
  // F free ids (mode 2), then the program; repeated from the op the program
  // stopped before (resources it could not see past) until all ops ran or
  // an op failed.  max_pos / total_pos: block positions of the largest
  // insert / of all inserts; pushes: worst-case candidate pushes.  Returns
  // the number of ops applied (all of them unless one failed).
  int32_t* d_first_op = nullptr;  // miss-free pin batches: first op pinning each block (INT_MAX = none)

  static bool fast_enabled() {
    static int on = -1;
    if (on < 0) {
      const char* e = getenv("SB_PROG_FAST");
      on = e && e[0] == '0' ? 0 : 1;
    }
    return on == 1;
  }
  // scratch of the parallel path; per-block arrays start neutral and are
  // restored by k_fast_reset after every use
  void ensure_fast(int64_t n_ops, int64_t total_pos, int64_t events) {
    if (!FB.hit_op) {
      FB.hit_op = dalloc<int32_t>(P.cap);
      FB.hit_max = dalloc<int32_t>(P.cap);
      FB.dref = dalloc<int32_t>(P.cap);
      FB.ev_max = dalloc<int32_t>(P.cap);
      FB.nrel = dalloc<int32_t>(P.cap);
      FB.nunp = dalloc<int32_t>(P.cap);
      FB.flags = dalloc<int32_t>(P.cap);
      FB.ctl = dalloc<int64_t>(FC_N);
      k_fill_i32<<<grid_for(P.cap), 256>>>(FB.hit_op, P.cap, kNoOp);
      k_fill_i32<<<grid_for(P.cap), 256>>>(FB.hit_max, P.cap, -1);
      k_fill_i32<<<grid_for(P.cap), 256>>>(FB.ev_max, P.cap, -1);
      SB_CUDA(cudaMemset(FB.dref, 0, sizeof(int32_t) * P.cap));
      SB_CUDA(cudaMemset(FB.nrel, 0, sizeof(int32_t) * P.cap));
      SB_CUDA(cudaMemset(FB.nunp, 0, sizeof(int32_t) * P.cap));
      SB_CUDA(cudaMemset(FB.flags, 0, sizeof(int32_t) * P.cap));
      SB_CUDA(cudaDeviceSynchronize());
    }
    if (n_ops + 1 > fb_ops_cap) {
      cudaFree(FB.miss_cnt);
      cudaFree(FB.miss_base);
      fb_ops_cap = std::max<int64_t>(n_ops + 1, 2 * fb_ops_cap);
      FB.miss_cnt = dalloc<int32_t>(fb_ops_cap);
      FB.miss_base = dalloc<int32_t>(fb_ops_cap);
    }
    if (total_pos + 1 > fb_pos_cap) {
      cudaFree(FB.mrank);
      cudaFree(FB.mpos);
      cudaFree(FB.miss_id);
      cudaFree(FB.mflag);
      fb_pos_cap = std::max<int64_t>(total_pos + 1, 2 * fb_pos_cap);
      FB.mrank = dalloc<int32_t>(fb_pos_cap);
      FB.mpos = dalloc<int32_t>(fb_pos_cap);
      FB.miss_id = dalloc<int32_t>(fb_pos_cap);
      FB.mflag = dalloc<uint8_t>(fb_pos_cap);
    }
    if (events + 1 > fb_ev_cap) {
      cudaFree(FB.pend_raw_key);
      cudaFree(FB.pend_raw_op);
      cudaFree(FB.pend_key);
      fb_ev_cap = std::max<int64_t>(events + 1, 2 * fb_ev_cap);
      FB.pend_raw_key = dalloc<uint64_t>(fb_ev_cap);
      FB.pend_raw_op = dalloc<int32_t>(fb_ev_cap);
      FB.pend_key = dalloc<uint64_t>(fb_ev_cap);
    }
    int64_t dc = 1024;
    while (dc < 2 * total_pos + 64) dc <<= 1;
    if (dc > fb_dup_cap) {
      cudaFree(FB.dup);
      fb_dup_cap = dc;
      FB.dup = dalloc<unsigned long long>(fb_dup_cap);
    }
    FB.dup_mask = dc - 1;
  }
  // the parallel path for ops [0, n_ops); stream-ordered, decides on the device
  void launch_fast(int64_t n_ops, int64_t max_pos, int64_t total_pos, int64_t pushes, int32_t* pin_cnt,
                   int8_t* real_tag, int64_t now, cudaStream_t st, bool has_pin) {
    ensure_fast(n_ops, total_pos, std::max(pushes, total_pos) + total_pos + 64);
    SB_CUDA(cudaMemsetAsync(FB.ctl, 0, sizeof(int64_t) * FC_N, st));
    SB_CUDA(cudaMemsetAsync(FB.dup, 0, sizeof(unsigned long long) * (FB.dup_mask + 1), st));
    const unsigned no = static_cast<unsigned>(n_ops);
    const dim3 g2(no, static_cast<unsigned>(std::min<int64_t>(64, std::max<int64_t>(1, (max_pos + 255) / 256))));
    launches += 7 + ((pin_cnt && has_pin) ? 3 : 0);
    k_fast_events<<<no, kFastThreads, 0, st>>>(P, d_ops, d_pre_all, pin_cnt, FB);
    k_fast_blocks<<<no, 256, 0, st>>>(P, d_ops, d_pre_all, pin_cnt, real_tag, now, FB);
    k_fast_plan<<<1, kFastThreads, kPlanSmem, st>>>(P, S, d_ops, static_cast<int>(n_ops), now, FB, prof_buf());
    k_fast_touch<<<g2, 256, 0, st>>>(P, d_ops, d_pre_all, pin_cnt, real_tag, now, FB);
    k_fast_evict<<<grid_for(std::max<int64_t>(total_pos, 1)), 256, 0, st>>>(P, S, FB);
    k_fast_create<<<g2, 256, 0, st>>>(P, d_ops, d_pre_all, now, FB);
    if (pin_cnt && has_pin) {
      if (!d_first_op) {
        d_first_op = dalloc<int32_t>(P.cap);
        k_fill_i32<<<grid_for(P.cap), 256, 0, st>>>(d_first_op, P.cap, kNoOp);
      }
      k_fast_pin_a<<<g2, 256, 0, st>>>(P, d_ops, d_first_op, FB);
      k_fast_pin_b<<<g2, 256, 0, st>>>(P, d_ops, pin_cnt, d_first_op, real_tag, FB);
      k_fast_pin_c<<<g2, 256, 0, st>>>(P, d_ops, pin_cnt, d_first_op, FB);
    }
    k_fast_finish<<<no, 256, 0, st>>>(P, S, d_ops, d_pre_all, d_res, static_cast<int>(n_ops), d_pout, FB);
    SB_CHECK_LAUNCH();
  }

  int64_t run_program(int64_t n_ops, int64_t max_pos, int64_t total_pos, int64_t pushes, int32_t* pin_cnt,
                      int8_t* real_tag, int64_t now, cudaStream_t st, int64_t* evictions = nullptr,
                      bool all_pin = false, bool has_pin = true) {
    if (max_pos > kProgMaxPos)
      throw Error(SB_ERR_UNSUPPORTED, "insert longer than " + std::to_string(kProgMaxPos) + " blocks");
    ensure_positions(std::max<int64_t>({max_pos, 2 * total_pos + 64, 64}));
    ensure_prehit_all(std::max<int64_t>(max_pos, 64));
    ensure_runk(pushes + 64 * (n_ops + 1) + 4 * kRunBuf);
    if (total_pos + 1 > pre_all_cap) {
      cudaFree(d_pre_all);
      pre_all_cap = std::max<int64_t>(total_pos + 1, 2 * pre_all_cap);
      d_pre_all = dalloc<int32_t>(pre_all_cap);
    }
    int64_t ccap = 1024;
    while (ccap < 2 * total_pos + 64) ccap <<= 1;
    if (ccap > created_cap) {
      cudaFree(d_created);
      created_cap = ccap;
      d_created = dalloc<unsigned long long>(created_cap);
    }
    if (!d_pout) {
      d_pout = dalloc<int64_t>(8);
      SB_CUDA(cudaMallocHost(&h_pout, 8 * sizeof(int64_t)));
    }
    if (prog_device_attr != device) {
      SB_CUDA(cudaFuncSetAttribute(k_program, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kProgSmem)));
      SB_CUDA(cudaFuncSetAttribute(k_fast_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kPlanSmem)));
      prog_device_attr = device;
    }
    int64_t first = 0, evs = 0;
    bool force = false;
    const unsigned gy = static_cast<unsigned>(std::max<int64_t>(1, (max_pos + 127) / 128));
    while (first < n_ops) {
      SB_CUDA(cudaMemsetAsync(d_pout, 0, 8 * sizeof(int64_t), st));
      SB_CUDA(cudaMemsetAsync(d_created, 0, sizeof(unsigned long long) * ccap, st));
      k_init_bound<<<1, 32, 0, st>>>(S.scal);
      launches += 2;
      k_prog_bound<<<dim3(static_cast<unsigned>(n_ops - first), gy), 256, 0, st>>>(
          P, d_ops, static_cast<int>(first), static_cast<int>(n_ops), S.scal, d_pre_all);
      if (force) {  // the bound left the program short once: list every candidate
        launches += 2;
        k_set_scal<<<1, 1, 0, st>>>(S.scal, S_NMISS, 1);
        k_set_scal<<<1, 1, 0, st>>>(S.scal, S_BOUND, 2 * total_pos + 64);
      }
      if (all_pin && first == 0 && !force) {
        // pin batch with no miss and no ref -1 hit: the ops commute (k_pin_nomiss_*)
        SB_CUDA(cudaMemcpyAsync(h_pout + 4, S.scal + S_NMISS, 2 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        SB_CUDA(cudaStreamSynchronize(st));
        if (h_pout[4] == 0 && h_pout[5] == 0) {
          if (!d_first_op) {
            d_first_op = dalloc<int32_t>(P.cap);
            SB_CUDA(cudaMemsetAsync(d_first_op, 0x7f, sizeof(int32_t) * P.cap, st));
          }
          const dim3 g(static_cast<unsigned>(n_ops), static_cast<unsigned>(std::min<int64_t>(gy * 128 / 256 + 1, 64)));
          launches += 3;
          k_pin_nomiss_a<<<g, 256, 0, st>>>(P, d_ops, 0, d_pre_all, d_first_op, now);
          k_pin_nomiss_b<<<g, 256, 0, st>>>(P, d_ops, 0, pin_cnt, d_first_op, real_tag);
          k_pin_nomiss_c<<<g, 256, 0, st>>>(P, d_ops, 0, pin_cnt, d_first_op, d_res);
          SB_CHECK_LAUNCH();
          if (evictions) *evictions = 0;
          return n_ops;
        }
      }
      cudaStream_t saved = stream;
      stream = st;
      InsertArgs A{};
      try {
        launch_select(A, 0, 2, 0);
      } catch (...) {
        stream = saved;
        throw;
      }
      stream = saved;
      const bool fast = first == 0 && !force && fast_enabled();
      if (fast) launch_fast(n_ops, max_pos, total_pos, pushes, pin_cnt, real_tag, now, st, has_pin);
      ProgState G{d_ops, d_res, static_cast<int32_t>(n_ops), static_cast<int32_t>(first), pin_cnt, real_tag,
                  d_runk, runk_cap, d_pout, now, d_pre_all, d_created, ccap - 1, prof_buf(),
                  fast ? FB.ctl + FC_DONE : nullptr};
      k_program<<<1, kProgThreads, kProgSmem, st>>>(P, S, G);
      ++launches;
      SB_CHECK_LAUNCH();
      SB_CUDA(cudaMemcpyAsync(h_pout, d_pout, 4 * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      if (fast) SB_CUDA(cudaMemcpyAsync(h_pout + 6, FB.ctl + FC_DONE, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
      SB_CUDA(cudaStreamSynchronize(st));
      if (fast) {
        ++fast_runs;
        fast_taken += h_pout[6] ? 1 : 0;
      }
      const int64_t next = h_pout[0];
      evs += h_pout[2];
      tomb_bound += h_pout[2];
      if (next <= first) {
        if (force) throw Error(SB_ERR_CACHE, "op program made no progress");
        force = true;
        continue;
      }
      force = false;
      first = next;
      if (h_pout[1] == PS_ERROR) break;  // a release error ends the batch (the reference throws)
    }
    if (evictions) *evictions = evs;
    if (tomb_bound > P.cap) {
      k_index_clear<<<grid_for(P.tcap), 256, 0, st>>>(P);
      k_index_fill<<<grid_for(P.cap), 256, 0, st>>>(P);
      SB_CHECK_LAUNCH();
      tomb_bound = 0;
    }
    return first;
  }

  void launch_select(const InsertArgs& A, int s, int mode, int64_t needed) {
    if (!use_coop(mode)) {
      k_select<<<1, kSelectThreads, select_smem(), stream>>>(P, S, A, s, mode, needed);
      ++launches;
      return;
    }
    Pool p_ = P;
    Scratch s_ = S;
    InsertArgs a_ = A;
    int sv = s, mv = mode;
    int64_t nv = needed;
    CoopBuf g_ = G;
    void* args[] = {&p_, &s_, &a_, &sv, &mv, &nv, &g_};
    if (fused_smem > 0 && fused_enabled()) {
      if (mode == 0) {
        k_plan<<<1, kSelectThreads, 0, stream>>>(P, S, A, s, mode, G);
        ++launches;
      }
      ++launches;
      SB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_evict_fused), dim3(coop_grid),
                                          dim3(kSelectThreads), args, fused_smem, stream));
    } else {
      launches += 3;
      k_plan<<<1, kSelectThreads, 0, stream>>>(P, S, A, s, mode, G);
      k_score<<<coop_grid, kScoreThreads, kScoreSmem, stream>>>(P, S, G);
      SB_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_select_coop), dim3(coop_grid),
                                          dim3(kSelectThreads), args, coop_smem, stream));
    }
    if (G.tprof) {  // SB_SELECT_PROF=1: phase times of this evict, relative to k_plan's start (us)
      unsigned long long h[32] = {};
      SB_CUDA(cudaStreamSynchronize(stream));
      SB_CUDA(cudaMemcpy(h, G.tprof, sizeof(h), cudaMemcpyDeviceToHost));
      auto us = [&](int i) { return h[i] ? (static_cast<double>(h[i]) - static_cast<double>(h[0])) * 1e-3 : -1.0; };
      fprintf(stderr, "SB_SELECT_PROF mode %d plan_end %.2f score_entry %.2f..%.2f score_exit %.2f select_entry %.2f..%.2f "
              "prologue %.2f", mode, us(1), us(2), us(3), us(4), us(5), us(6), us(7));
      for (int p = 0; p < 6; ++p)
        if (h[8 + 2 * p]) fprintf(stderr, " sync%d %.2f->%.2f", p, us(8 + 2 * p), us(9 + 2 * p));
      fprintf(stderr, " sort %.2f end %.2f | hist0 %.2f hist1 %.2f compact %.2f gather %.2f | cta0 %.2f %.2f %.2f"
              " | rank: keys_loaded %.2f ranked %.2f M %llu\n",
              us(20), us(21), us(22), us(23), us(24), us(25), us(26), us(27), us(28), us(29), us(30), h[31]);
      {
        unsigned long long hc[2 * 160 + 33] = {};
        SB_CUDA(cudaMemcpy(hc, G.tprof + 32, sizeof(hc), cudaMemcpyDeviceToHost));
        for (int w = 0; w < 2; ++w) {
          fprintf(stderr, "SB_SELECT_PROF_CTA %s:", w ? "compact" : "pass0");
          for (int c = 0; c < coop_grid; ++c)
            fprintf(stderr, " %.1f", hc[w * 160 + c] ? (static_cast<double>(hc[w * 160 + c]) - static_cast<double>(h[0])) * 1e-3 : -1.0);
          fprintf(stderr, "\n");
        }
        fprintf(stderr, "SB_SELECT_PROF_WARPS cta5 start %.2f:", hc[320 + 32] ? (double(hc[320 + 32]) - double(h[0])) * 1e-3 : -1.0);
        for (int w = 0; w < 32; ++w) fprintf(stderr, " %.2f", hc[320 + w] ? (double(hc[320 + w]) - double(h[0])) * 1e-3 : -1.0);
        fprintf(stderr, "\n");
      }
    }
  }

  void ensure_batch(int64_t n) {
    if (n <= batch_cap) return;
    cudaFree(d_batch_blk);
    cudaFree(d_batch_first);
    batch_cap = std::max<int64_t>(n, 2 * batch_cap);
    d_batch_blk = dalloc<int64_t>(batch_cap + 1);
    d_batch_first = dalloc<int64_t>(batch_cap + 1);
  }

  ~sb_kv_cache() {
    cudaSetDevice(device);
    // S.prehit aliases d_prehit_all: freed once below
    void* ptrs[] = {P.tok, P.ntok, P.chain, P.parent, P.tag, P.ref, P.pinned, P.last, P.idx, P.slot, P.ctr,
                    S.hashes, S.chain_out, S.kind, S.freel, S.evicted, S.victims, S.taken, S.rank_of, S.keys,
                    S.sortbuf, S.scal, S.late, d_ops, d_res, d_runk, d_pout, d_pre_all, d_created, d_first_op, d_tok, d_tags, d_meta, d_ids, d_status, d_first, d_hit, d_hash_all, d_prehit_all, d_batch_blk, d_batch_first, G.hist, G.ctr, G.keys, G.fcnt, G.ncnt, G.kmin, G.kmax, G.tprof};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    void* fptrs[] = {FB.hit_op, FB.hit_max, FB.dref, FB.ev_max, FB.nrel, FB.nunp, FB.flags, FB.miss_cnt, FB.miss_base,
                     FB.mrank, FB.mpos, FB.miss_id, FB.mflag, FB.pend_raw_key, FB.pend_raw_op, FB.pend_key,
                     FB.dup, FB.ctl};
    for (void* p : fptrs)
      if (p) cudaFree(p);
    if (d_prof) {
      unsigned long long hp[64] = {};
      cudaMemcpy(hp, d_prof, sizeof(hp), cudaMemcpyDeviceToHost);
      fprintf(stderr, "SB_PROG_PROFILE parallel path: %llu of %llu programs; k_fast_plan walks %llu: prelude %llu walk %llu cycles\n",
              fast_taken, fast_runs, hp[62], hp[60], hp[61]);
    }
    if (d_prof) {
      unsigned long long h[64] = {};
      cudaMemcpy(h, d_prof, sizeof(h), cudaMemcpyDeviceToHost);
      for (int k = 0; k < 5; ++k) {
        fprintf(stderr, "SB_PROG_PROFILE kind %d cycles:", k);
        for (int i = 0; i < 11; ++i) fprintf(stderr, " %d:%llu", i, h[k * 11 + i]);
        fprintf(stderr, "\n");
      }
      cudaFree(d_prof);
    }
    if (h_pout) cudaFreeHost(h_pout);
    if (ev_pool) cudaEventDestroy(ev_pool);
    if (ev_user) cudaEventDestroy(ev_user);
    if (stream) cudaStreamDestroy(stream);
  }

  void ensure_positions(int64_t pmax) {
    if (pmax <= S.pmax) return;
    int64_t n = std::max<int64_t>(pmax, 2 * S.pmax);
    cudaFree(S.hashes);
    cudaFree(S.chain_out);
    cudaFree(S.kind);
    cudaFree(S.freel);
    cudaFree(S.victims);
    cudaFree(S.taken);
    cudaFree(S.sortbuf);
    S.hashes = dalloc<uint64_t>(n);
    S.chain_out = dalloc<int32_t>(n);
    S.kind = dalloc<int8_t>(n);
    S.freel = dalloc<int32_t>(n);
    S.kmax = 2 * n + P.cap;
    S.victims = dalloc<uint64_t>(S.kmax);
    S.taken = dalloc<uint8_t>(S.kmax);
    int64_t pw = 1;
    while (pw < S.kmax) pw <<= 1;
    S.sortbuf = dalloc<uint64_t>(pw);
    S.pmax = n;
  }
  void ensure_tokens(int64_t n) {
    if (n <= tok_cap) return;
    cudaFree(d_tok);
    tok_cap = std::max<int64_t>(n, 2 * tok_cap);
    d_tok = dalloc<uint64_t>(tok_cap);
  }
  void ensure_tags(int64_t n) {
    if (n <= tags_cap) return;
    cudaFree(d_tags);
    tags_cap = std::max<int64_t>(n, 2 * tags_cap + 4);
    d_tags = dalloc<sb_tag_range>(tags_cap);
  }
  void ensure_ids(int64_t n) {
    if (n <= ids_cap) return;
    cudaFree(d_ids);
    ids_cap = std::max<int64_t>(n, 2 * ids_cap + 16);
    d_ids = dalloc<int32_t>(ids_cap);
  }
  void ensure_hash_all(int64_t n) {
    if (n <= hash_cap) return;
    cudaFree(d_hash_all);
    hash_cap = std::max<int64_t>(n, 2 * hash_cap);
    d_hash_all = dalloc<uint64_t>(hash_cap);
  }
  void ensure_prehit_all(int64_t n) {
    if (n <= prehit_cap) return;
    cudaFree(d_prehit_all);
    prehit_cap = std::max<int64_t>(n, 2 * prehit_cap);
    d_prehit_all = dalloc<int32_t>(prehit_cap);
    S.prehit = d_prehit_all;
  }

  void maybe_rebuild_index(int64_t added_tombs) {
    tomb_bound += added_tombs;
    if (tomb_bound <= P.cap) return;
    k_index_clear<<<grid_for(P.tcap), 256, 0, stream>>>(P);
    k_index_fill<<<grid_for(P.cap), 256, 0, stream>>>(P);
    SB_CHECK_LAUNCH();
    tomb_bound = 0;
  }

  int64_t read_scal(int idx) {
    int64_t v = 0;
    SB_CUDA(cudaMemcpyAsync(&v, S.scal + idx, sizeof(v), cudaMemcpyDeviceToHost, stream));
    SB_CUDA(cudaStreamSynchronize(stream));
    return v;
  }
  unsigned long long read_ctr(int idx) const {
    unsigned long long v = 0;
    cudaMemcpyAsync(&v, P.ctr + idx, sizeof(v), cudaMemcpyDeviceToHost, stream);
    cudaStreamSynchronize(stream);
    return v;
  }

  size_t select_smem() const { return (kCandSmem + kSortSmemKeys) * sizeof(uint64_t); }

  // Inserts sequences [0, n_seqs) described by device arrays, sequentially.
  void insert_device(const uint64_t* tokens, const int64_t* seq_off, const sb_tag_range* tags, const int64_t* tag_off,
                     const int64_t* blk_off, const uint64_t* hashes_in, int n_seqs, int64_t now, int32_t* out_ids,
                     int32_t* status, const std::vector<int64_t>& h_blk_off) {
    const int64_t total_blocks = h_blk_off[n_seqs];
    int64_t pmax = 1;
    for (int s = 0; s < n_seqs; ++s) pmax = std::max(pmax, h_blk_off[s + 1] - h_blk_off[s]);
    ensure_positions(pmax);
    ensure_prehit_all(std::max<int64_t>(total_blocks, 1));
    const uint64_t* hashes = hashes_in;
    if (!hashes) {
      ensure_hash_all(std::max<int64_t>(total_blocks, 1));
      launch_chain_hash(tokens, seq_off, blk_off, nullptr, n_seqs, P.bs, 0, d_hash_all, stream);
      SB_CHECK_LAUNCH();
      hashes = d_hash_all;
    }
    InsertArgs A{tokens, seq_off, tags, tag_off, blk_off, hashes, out_ids, status, now};
    for (int s = 0; s < n_seqs; ++s) {
      const int64_t np = h_blk_off[s + 1] - h_blk_off[s];
      if (np > 0)
        k_probe_seq<<<grid_for(np * kGroup), 256, 0, stream>>>(P, tokens, seq_off, blk_off, hashes, s, S.prehit);
      launch_select(A, s, 0, 0);
      k_walk<<<1, 32, 0, stream>>>(P, S, A, s);
      k_commit_evict<<<grid_for(np), 256, 0, stream>>>(P, S);
      k_commit_apply<<<grid_for(std::max<int64_t>(np, 1) + 2 * np), 256, 0, stream>>>(P, S, A, s);
      SB_CHECK_LAUNCH();
      maybe_rebuild_index(np);
    }
  }
};

namespace sb {
int64_t pool_run_ops(sb_kv_cache* c, const ProgOp* h_ops, int64_t n, int32_t* d_pin_cnt, int8_t* d_real_tag,
                     int64_t now, cudaStream_t st, ProgRes* h_res) {
  if (n <= 0) return 0;
  std::lock_guard<std::mutex> lk(c->mu);
  SB_CUDA(cudaSetDevice(c->device));
  check_now(c->P, now);
  int64_t max_pos = 0, total = 0, pushes = 0;
  std::vector<ProgOp> ops(h_ops, h_ops + n);
  for (int64_t i = 0; i < n; ++i) {
    const int64_t pn = (h_ops[i].n + c->P.bs - 1) / c->P.bs;
    ops[static_cast<size_t>(i)].pos_off = total;
    max_pos = std::max(max_pos, pn);
    total += pn;
    pushes += pn + h_ops[i].n_chain + h_ops[i].n_pinned;
  }
  c->ensure_ops(n);
  c->join_in(st);
  SB_CUDA(cudaMemcpyAsync(c->d_ops, ops.data(), sizeof(ProgOp) * n, cudaMemcpyHostToDevice, st));
  bool all_pin = d_pin_cnt != nullptr, has_pin = false;
  for (int64_t i = 0; i < n; ++i) {
    all_pin = all_pin && h_ops[i].kind == PK_PIN;
    has_pin = has_pin || h_ops[i].kind == PK_PIN;
  }
  const int64_t done =
      c->run_program(n, max_pos, total, pushes, d_pin_cnt, d_real_tag, now, st, nullptr, all_pin, has_pin);
  c->join_out(st);
  SB_CUDA(cudaMemcpyAsync(h_res, c->d_res, sizeof(ProgRes) * n, cudaMemcpyDeviceToHost, st));
  SB_CUDA(cudaStreamSynchronize(st));
  return done;
}

void pool_lookup(sb_kv_cache* c, const ProgOp* h_ops, int64_t n, int64_t now, int64_t* d_hits, cudaStream_t st) {
  if (n <= 0) return;
  std::lock_guard<std::mutex> lk(c->mu);
  SB_CUDA(cudaSetDevice(c->device));
  check_now(c->P, now);
  int64_t max_full = 0;
  for (int64_t i = 0; i < n; ++i) max_full = std::max(max_full, h_ops[i].n / c->P.bs);
  c->ensure_ops(n);
  c->ensure_batch(n);
  c->join_in(st);
  SB_CUDA(cudaMemcpyAsync(c->d_ops, h_ops, sizeof(ProgOp) * n, cudaMemcpyHostToDevice, st));
  c->launches += max_full > 0 ? 3 : 2;
  k_lookup_ops_init<<<static_cast<unsigned>((n + 127) / 128), 128, 0, st>>>(c->P, c->d_ops, static_cast<int>(n),
                                                                             c->d_batch_first);
  if (max_full > 0)
    k_lookup_ops_probe<<<dim3(static_cast<unsigned>(n), static_cast<unsigned>((max_full + 127) / 128)), 256, 0, st>>>(
        c->P, c->d_ops, c->d_batch_first);
  k_lookup_ops_finish<<<dim3(static_cast<unsigned>(n), static_cast<unsigned>(std::max<int64_t>(1, (max_full + 255) / 256))),
                        256, 0, st>>>(c->P, c->d_ops, c->d_batch_first, now, d_hits);
  SB_CHECK_LAUNCH();
  c->join_out(st);
}

cudaStream_t pool_stream(sb_kv_cache* c) { return c->stream; }
uint64_t pool_launches(const sb_kv_cache* c) { return c->launches; }
int pool_device(sb_kv_cache* c) { return c->device; }
}  // namespace sb

static thread_local std::string g_last_error;
void sb::set_last_error(const std::string& m) { g_last_error = m; }

extern "C" {

const char* sb_last_error(void) { return g_last_error.c_str(); }
const char* sb_version(void) { return "sutradhara_b200 0.1 (sm_100a)"; }

uint64_t sb_kv_root_hash(void) { return kRootHash; }
uint64_t sb_kv_chain_hash_host(uint64_t parent, const uint64_t* t, int64_t n) {
  uint64_t h = parent;
  for (int64_t i = 0; i < n; ++i) h = hash_combine(h, t[i]);
  return h;
}

int sb_chain_hash_batch(const uint64_t* d_tokens, const int64_t* d_seq_offsets, const int64_t* d_block_offsets,
                        const uint64_t* d_parent, int32_t n_seqs, int64_t block_size, uint64_t* d_block_hashes,
                        void* stream) {
  return guard([&] {
    if (n_seqs <= 0) return int(SB_OK);
    if (block_size < 1) throw Error(SB_ERR_INVALID, "block_size must be >= 1");
    launch_chain_hash(d_tokens, d_seq_offsets, d_block_offsets, d_parent, n_seqs, block_size, 0, d_block_hashes,
                      static_cast<cudaStream_t>(stream));
    SB_CHECK_LAUNCH();
    return int(SB_OK);
  });
}

int sb_chain_hash_segments(const uint64_t* d_tokens, const int64_t* d_seg_bounds, const int64_t* d_seg_blocks,
                           const uint64_t* d_parent, int32_t n_segs, int64_t block_size, uint64_t* d_block_hashes,
                           void* stream) {
  return guard([&] {
    if (block_size < 1) throw Error(SB_ERR_INVALID, "block_size");
    launch_chain_hash(d_tokens, d_seg_bounds, d_seg_blocks, d_parent, n_segs, block_size, 0, d_block_hashes,
                      static_cast<cudaStream_t>(stream), 1);
    SB_CHECK_LAUNCH();
    return int(SB_OK);
  });
}

int sb_kv_gather_chain_hashes(sb_kv_cache* c, const int32_t* d_ids, const int64_t* d_pos, int64_t n,
                              uint64_t* d_out, void* stream) {
  return guard([&] {
    if (n <= 0) return int(SB_OK);
    SB_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    c->join_in(st);
    k_gather_chain<<<grid_for(n), 256, 0, st>>>(c->P, d_ids, d_pos, n, d_out);
    SB_CHECK_LAUNCH();
    return int(SB_OK);
  });
}

int sb_kv_create(int64_t block_size, int64_t capacity_blocks, int32_t policy, int32_t device, sb_kv_cache** out) {
  return guard([&] {
    if (block_size < 1) throw Error(SB_ERR_CONFIG, "cache block_size must be >= 1");
    if (capacity_blocks < 1) throw Error(SB_ERR_CONFIG, "cache capacity_blocks must be >= 1");
    if (capacity_blocks > (int64_t(1) << kMaxIdBits)) throw Error(SB_ERR_UNSUPPORTED, "capacity above 2^24 blocks");
    if (policy != SB_POLICY_LRU && policy != SB_POLICY_TIERED) throw Error(SB_ERR_CONFIG, "unknown policy");
    SB_CUDA(cudaSetDevice(device));
    auto* c = new sb_kv_cache();
    try {
      c->device = device;
      // blocking stream: per-op calls order after outstanding work on the legacy stream
      SB_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamDefault));
      Pool& P = c->P;
      P.bs = block_size;
      P.cap = capacity_blocks;
      P.policy = policy;
      P.idb = kMinIdBits;
      while ((int64_t(1) << P.idb) < capacity_blocks) ++P.idb;
      P.idmask = (uint64_t(1) << P.idb) - 1;
      P.lbias = int64_t(1) << (60 - P.idb);
      P.tcap = 16;
      while (P.tcap < 4 * capacity_blocks) P.tcap <<= 1;
      // metadata arrays padded to whole 16 B vectors (k_score's bulk copies)
      const int64_t cap_pad = (capacity_blocks + 3) & ~int64_t(3);
      P.tok = dalloc<uint64_t>(static_cast<size_t>(block_size * capacity_blocks));
      P.ntok = dalloc<int32_t>(cap_pad);
      P.chain = dalloc<uint64_t>(capacity_blocks);
      P.parent = dalloc<uint64_t>(capacity_blocks);
      P.tag = dalloc<int32_t>(cap_pad);
      P.ref = dalloc<int32_t>(cap_pad);
      P.pinned = dalloc<int32_t>(cap_pad);
      P.last = dalloc<int64_t>(cap_pad);
      P.idx = dalloc<IdxEntry>(P.tcap);
      P.slot = dalloc<int32_t>(capacity_blocks);
      P.ctr = dalloc<unsigned long long>(C_N);
      SB_CUDA(cudaMemsetAsync(P.ntok, 0, sizeof(int32_t) * cap_pad, c->stream));
      SB_CUDA(cudaMemsetAsync(P.ref, 0, sizeof(int32_t) * cap_pad, c->stream));
      SB_CUDA(cudaMemsetAsync(P.pinned, 0, sizeof(int32_t) * cap_pad, c->stream));
      SB_CUDA(cudaMemsetAsync(P.ctr, 0, sizeof(unsigned long long) * C_N, c->stream));
      k_index_clear<<<grid_for(P.tcap), 256, 0, c->stream>>>(P);
      Scratch& S = c->S;
      S.rank_of = dalloc<int32_t>(capacity_blocks);
      k_fill_i32<<<grid_for(capacity_blocks), 256, 0, c->stream>>>(S.rank_of, capacity_blocks, -1);
      S.keys = dalloc<uint64_t>(capacity_blocks);
      S.evicted = dalloc<int32_t>(capacity_blocks + 16);
      S.scal = dalloc<int64_t>(S_N);
      S.late = dalloc<int32_t>(2 * kLateMax);
      SB_CUDA(cudaMemsetAsync(S.scal, 0, sizeof(int64_t) * S_N, c->stream));
      c->ensure_positions(64);
      c->ensure_prehit_all(64);
      c->d_meta = dalloc<int64_t>(16);
      c->d_status = dalloc<int32_t>(4);
      c->d_first = dalloc<int64_t>(4);
      c->d_hit = dalloc<int64_t>(4);
      SB_CUDA(cudaFuncSetAttribute(k_select, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(c->select_smem())));
      if (capacity_blocks >= kCoopMinCap) {
        int n_sm = 0, per_sm = 0;
        SB_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, device));
        const int n_slices = kSlicesPerSm * n_sm;  // k_score partition; k_select_coop CTA c owns slices c, c + n_sm, ...
        const int64_t slice = ((capacity_blocks + n_slices - 1) / n_slices + 3) & ~int64_t(3);
        cudaFuncAttributes fa{};
        SB_CUDA(cudaFuncGetAttributes(&fa, k_select_coop));
        int smem_optin = 0;
        SB_CUDA(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device));
        // the final sort: merge sort of up to kSortSmemKeys keys (2x scratch) when it fits
        const size_t sort_b = 2 * kSortSmemKeys * sizeof(uint64_t);
        const size_t sort_min = sort_b + fa.sharedSizeBytes <= static_cast<size_t>(smem_optin) ? sort_b
                                                                                               : kSortSmemKeys * sizeof(uint64_t);
        // dynamic shared memory: the final ranks / sort, and the CTA's candidate keys when every CTA's fit
        // (a CTA's full slices plus one pad key each), as much as the part allows
        const size_t full = static_cast<size_t>(kSlicesPerSm * (slice + 1)) * sizeof(uint64_t);
        const size_t avail = (static_cast<size_t>(smem_optin) - fa.sharedSizeBytes) & ~size_t(15);
        c->coop_smem = std::min(avail, std::max(full, sort_min));
        c->G.sort_keys = static_cast<int64_t>(c->coop_smem / sizeof(uint64_t));
        {
          const char* re = getenv("SB_RANK_EARLY");
          c->G.rank_early_max = re ? std::max<int64_t>(64, std::atoll(re)) : kRankEarlyMax;
        }
        SB_CUDA(cudaFuncSetAttribute(k_score, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kScoreSmem)));
        {
          SB_CUDA(cudaFuncSetAttribute(k_select_coop, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(c->coop_smem)));
          SB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_select_coop, kSelectThreads, c->coop_smem));
          if (per_sm >= 1 && n_slices <= kMaxLiveSlices) c->coop_grid = n_sm;
          {  // the fused kernel: the scoring ring and the select's buffers share its dynamic shared memory
            cudaFuncAttributes ff{};
            SB_CUDA(cudaFuncGetAttributes(&ff, k_evict_fused));
            const size_t fs = std::max(kScoreSmem, c->coop_smem);
            int per_sm_f = 0;
            if (ff.sharedSizeBytes + fs <= static_cast<size_t>(smem_optin)) {
              SB_CUDA(cudaFuncSetAttribute(k_evict_fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(fs)));
              SB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_f, k_evict_fused, kSelectThreads, fs));
            }
            if (per_sm_f >= 1 && per_sm >= 1) c->fused_smem = fs;
            if (c->fused_smem && sb_kv_cache::fused_enabled()) c->G.sort_keys = static_cast<int64_t>(fs / sizeof(uint64_t));
          }
          c->G.hist = dalloc<uint32_t>(6 * 2048);
          c->G.ctr = dalloc<unsigned long long>(8);
          c->G.n_slices = n_slices;
          c->G.slice = slice;
          c->G.keys = dalloc<uint64_t>(n_slices * slice);
          c->G.fcnt = dalloc<uint32_t>(n_slices);
          c->G.ncnt = dalloc<uint32_t>(n_slices);
          c->G.kmin = dalloc<uint64_t>(n_slices);
          c->G.kmax = dalloc<uint64_t>(n_slices);
          const char* tp = getenv("SB_SELECT_PROF");
          if (tp && atoi(tp)) c->G.tprof = dalloc<unsigned long long>(32 + 2 * 160 + 33);
        }
      }
      SB_CHECK_LAUNCH();
      SB_CUDA(cudaStreamSynchronize(c->stream));
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
    return int(SB_OK);
  });
}

void sb_kv_destroy(sb_kv_cache* c) { delete c; }

int sb_kv_lookup_prefix(sb_kv_cache* c, const uint64_t* tokens, int64_t n, int64_t now, int64_t* hit_tokens) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(c->mu);
    SB_CUDA(cudaSetDevice(c->device));
    check_now(c->P, now);
    const int64_t nblk = n / c->P.bs;
    *hit_tokens = 0;
    if (nblk == 0) return int(SB_OK);
    c->ensure_tokens(n);
    c->ensure_hash_all(nblk);
    c->ensure_prehit_all(nblk);
    int64_t meta[4] = {0, n, 0, nblk};
    SB_CUDA(cudaMemcpyAsync(c->d_tok, tokens, sizeof(uint64_t) * n, cudaMemcpyHostToDevice, c->stream));
    SB_CUDA(cudaMemcpyAsync(c->d_meta, meta, sizeof(meta), cudaMemcpyHostToDevice, c->stream));
    const int64_t* seq_off = c->d_meta;
    const int64_t* blk_off = c->d_meta + 2;
    launch_chain_hash(c->d_tok, seq_off, blk_off, nullptr, 1, c->P.bs, 1, c->d_hash_all, c->stream);
    k_lookup_init<<<1, 32, 0, c->stream>>>(blk_off, 1, c->d_first);
    launch_probe_rows(c->P, c->d_tok, seq_off, blk_off, c->d_hash_all, c->d_prehit_all, c->d_first, 0, 1, nblk,
                      c->stream);
    k_lookup_finish<<<grid_for(nblk + 1), 256, 0, c->stream>>>(c->P, seq_off, blk_off, 1, nblk, c->d_prehit_all,
                                                               c->d_first, now, c->d_hit);
    SB_CHECK_LAUNCH();
    SB_CUDA(cudaMemcpyAsync(hit_tokens, c->d_hit, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    SB_CUDA(cudaStreamSynchronize(c->stream));
    return int(SB_OK);
  });
}

int sb_kv_lookup_prefix_batch(sb_kv_cache* c, const uint64_t* d_tokens, const int64_t* d_seq_offsets,
                              const int64_t* d_block_offsets, const int64_t* h_block_offsets,
                              const uint64_t* d_block_hashes, int32_t n_seqs, int64_t now, int64_t* d_hit_tokens,
                              void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(c->mu);
    SB_CUDA(cudaSetDevice(c->device));
    if (n_seqs <= 0) return int(SB_OK);
    check_now(c->P, now);
    cudaStream_t st = static_cast<cudaStream_t>(stream);  // NULL = legacy default stream
    c->join_in(st);
    std::vector<int64_t> off(n_seqs + 1), blk(n_seqs + 1);
    const bool pre = d_block_hashes && d_block_offsets;
    if (pre && h_block_offsets) {
      std::memcpy(off.data(), h_block_offsets, sizeof(int64_t) * (n_seqs + 1));
    } else {
      SB_CUDA(cudaMemcpyAsync(off.data(), pre ? d_block_offsets : d_seq_offsets, sizeof(int64_t) * (n_seqs + 1),
                              cudaMemcpyDeviceToHost, st));
      SB_CUDA(cudaStreamSynchronize(st));
    }
    int64_t total;
    if (pre) {
      total = off[n_seqs];
    } else {
      blk[0] = 0;
      for (int s = 0; s < n_seqs; ++s) blk[s + 1] = blk[s] + (off[s + 1] - off[s]) / c->P.bs;
      total = blk[n_seqs];
    }
    c->ensure_prehit_all(total + 1);
    c->ensure_batch(n_seqs);
    const uint64_t* hashes = d_block_hashes;
    const int64_t* d_blk = d_block_offsets;
    if (!pre) {
      c->ensure_hash_all(total + 1);
      SB_CUDA(cudaMemcpyAsync(c->d_batch_blk, blk.data(), sizeof(int64_t) * (n_seqs + 1), cudaMemcpyHostToDevice, st));
      d_blk = c->d_batch_blk;
      launch_chain_hash(d_tokens, d_seq_offsets, d_blk, nullptr, n_seqs, c->P.bs, 1, c->d_hash_all, st);
      hashes = c->d_hash_all;
    }
    k_lookup_init<<<(n_seqs + 127) / 128, 128, 0, st>>>(d_blk, n_seqs, c->d_batch_first);
    if (total > 0) {
      const std::vector<int64_t>& bo = pre ? off : blk;
      int64_t max_np = 0;
      for (int i = 0; i < n_seqs; ++i) max_np = std::max(max_np, bo[i + 1] - bo[i]);
      launch_probe_rows(c->P, d_tokens, d_seq_offsets, d_blk, hashes, c->d_prehit_all, c->d_batch_first, pre ? 1 : 0,
                        n_seqs, max_np, st);
    }
    k_lookup_finish<<<grid_for(std::max<int64_t>(total, n_seqs)), 256, 0, st>>>(
        c->P, d_seq_offsets, d_blk, n_seqs, total, c->d_prehit_all, c->d_batch_first, now, d_hit_tokens);
    SB_CHECK_LAUNCH();
    c->join_out(st);
    return int(SB_OK);
  });
}

int sb_kv_insert(sb_kv_cache* c, const uint64_t* tokens, int64_t n, const sb_tag_range* tags, int64_t n_tags,
                 int64_t now, int32_t* out_ids, int64_t* n_out) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(c->mu);
    SB_CUDA(cudaSetDevice(c->device));
    *n_out = 0;
    check_now(c->P, now);
    const int64_t nblk = (n + c->P.bs - 1) / c->P.bs;
    c->ensure_tokens(std::max<int64_t>(n, 1));
    c->ensure_tags(std::max<int64_t>(n_tags, 1));
    c->ensure_ids(std::max<int64_t>(nblk, 1));
    int64_t meta[6] = {0, n, 0, n_tags, 0, nblk};
    if (n) SB_CUDA(cudaMemcpyAsync(c->d_tok, tokens, sizeof(uint64_t) * n, cudaMemcpyHostToDevice, c->stream));
    if (n_tags)
      SB_CUDA(cudaMemcpyAsync(c->d_tags, tags, sizeof(sb_tag_range) * n_tags, cudaMemcpyHostToDevice, c->stream));
    SB_CUDA(cudaMemcpyAsync(c->d_meta, meta, sizeof(meta), cudaMemcpyHostToDevice, c->stream));
    std::vector<int64_t> hb = {0, nblk};
    int32_t st = 0;
    if (legacy_insert()) {
      c->insert_device(c->d_tok, c->d_meta, c->d_tags, c->d_meta + 2, c->d_meta + 4, nullptr, 1, now, c->d_ids,
                       c->d_status, hb);
      SB_CUDA(cudaMemcpyAsync(&st, c->d_status, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
      SB_CUDA(cudaStreamSynchronize(c->stream));
    } else {
      // one PK_INSERT op through the op program
      c->ensure_hash_all(std::max<int64_t>(nblk, 1));
      if (nblk) launch_chain_hash(c->d_tok, c->d_meta, c->d_meta + 4, nullptr, 1, c->P.bs, 0, c->d_hash_all, c->stream);
      ProgOp op{};
      op.kind = PK_INSERT;
      op.n = n;
      op.tokens = c->d_tok;
      op.hashes = c->d_hash_all;
      op.ins_tags = c->d_tags;
      op.n_ins_tags = static_cast<int32_t>(n_tags);
      op.ids = c->d_ids;
      op.pos_off = 0;
      c->ensure_ops(1);
      SB_CUDA(cudaMemcpyAsync(c->d_ops, &op, sizeof(op), cudaMemcpyHostToDevice, c->stream));
      int64_t evs = 0;
      c->run_program(1, nblk, nblk, 0, nullptr, nullptr, now, c->stream, &evs);
      ProgRes r{};
      SB_CUDA(cudaMemcpyAsync(&r, c->d_res, sizeof(r), cudaMemcpyDeviceToHost, c->stream));
      c->last_evicted.resize(static_cast<size_t>(evs));
      if (evs)
        SB_CUDA(cudaMemcpyAsync(c->last_evicted.data(), c->S.evicted, sizeof(int32_t) * evs, cudaMemcpyDeviceToHost,
                                c->stream));
      SB_CUDA(cudaStreamSynchronize(c->stream));
      st = r.status;
    }
    if (st == 0 && nblk) {
      SB_CUDA(cudaMemcpy(out_ids, c->d_ids, sizeof(int32_t) * nblk, cudaMemcpyDeviceToHost));
      *n_out = nblk;
    }
    if (st == SB_ERR_CACHE_FULL) set_last_error("insert: cannot free a block (all pinned or referenced)");
    if (st == SB_ERR_CACHE) set_last_error("insert: tag ranges must cover the full token range without gaps");
    return int(st);
  });
}

int sb_kv_insert_batch(sb_kv_cache* c, const uint64_t* d_tokens, const int64_t* d_seq_offsets,
                       const sb_tag_range* d_tags, const int64_t* d_tag_offsets, const int64_t* d_block_offsets,
                       const int64_t* h_block_offsets, const uint64_t* d_block_hashes, int32_t n_seqs, int64_t now,
                       int32_t* d_out_ids, int32_t* d_status, void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(c->mu);
    SB_CUDA(cudaSetDevice(c->device));
    if (n_seqs <= 0) return int(SB_OK);
    check_now(c->P, now);
    std::vector<int64_t> hb(n_seqs + 1);
    if (h_block_offsets)
      std::memcpy(hb.data(), h_block_offsets, sizeof(int64_t) * (n_seqs + 1));
    else
      SB_CUDA(cudaMemcpy(hb.data(), d_block_offsets, sizeof(int64_t) * (n_seqs + 1), cudaMemcpyDeviceToHost));
    // the caller's stream, taken literally (NULL = legacy default stream)
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    c->join_in(st);
    if (legacy_insert()) {
      cudaStream_t saved = c->stream;
      c->stream = st;
      try {
        c->insert_device(d_tokens, d_seq_offsets, d_tags, d_tag_offsets, d_block_offsets, d_block_hashes, n_seqs, now,
                         d_out_ids, d_status, hb);
      } catch (...) {
        c->stream = saved;
        throw;
      }
      c->stream = saved;
      c->join_out(st);
      return int(SB_OK);
    }
    // the batch as PK_INSERT ops of one op program: pre-state bound, one
    // scoring pass + select for the whole batch, one program launch
    int64_t max_pos = 0;
    for (int s = 0; s < n_seqs; ++s) max_pos = std::max(max_pos, hb[s + 1] - hb[s]);
    const uint64_t* hashes = d_block_hashes;
    if (!hashes) {
      c->ensure_hash_all(std::max<int64_t>(hb[n_seqs], 1));
      launch_chain_hash(d_tokens, d_seq_offsets, d_block_offsets, nullptr, n_seqs, c->P.bs, 0, c->d_hash_all, st);
      hashes = c->d_hash_all;
    }
    c->ensure_ops(n_seqs);
    k_build_insert_ops<<<(n_seqs + 127) / 128, 128, 0, st>>>(c->d_ops, d_tokens, d_seq_offsets, d_tags, d_tag_offsets,
                                                            d_block_offsets, hashes, d_out_ids, n_seqs);
    SB_CHECK_LAUNCH();
    c->run_program(n_seqs, max_pos, hb[n_seqs], 0, nullptr, nullptr, now, st);
    k_prog_status<<<(n_seqs + 127) / 128, 128, 0, st>>>(c->d_res, n_seqs, d_status);
    SB_CHECK_LAUNCH();
    c->join_out(st);
    return int(SB_OK);
  });
}

int sb_kv_evict(sb_kv_cache* c, int64_t needed, int32_t* out_ids, int64_t* n_out) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(c->mu);
    SB_CUDA(cudaSetDevice(c->device));
    *n_out = 0;
    if (needed <= 0) return int(SB_OK);
    c->ensure_positions(std::min<int64_t>(needed, c->P.cap));
    c->ensure_ids(std::min<int64_t>(needed, c->P.cap) + 1);
    InsertArgs A{};
    c->launch_select(A, 0, 1, needed);
    k_evict_out<<<grid_for(c->P.cap), 256, 0, c->stream>>>(c->P, c->S, c->d_ids, c->d_first);
    k_commit_evict<<<grid_for(c->P.cap), 256, 0, c->stream>>>(c->P, c->S);
    SB_CHECK_LAUNCH();
    int64_t k = 0;
    SB_CUDA(cudaMemcpyAsync(&k, c->d_first, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    SB_CUDA(cudaStreamSynchronize(c->stream));
    if (k) SB_CUDA(cudaMemcpy(out_ids, c->d_ids, sizeof(int32_t) * k, cudaMemcpyDeviceToHost));
    *n_out = k;
    c->last_evicted.assign(out_ids, out_ids + k);
    c->maybe_rebuild_index(k);
    return int(SB_OK);
  });
}

static int run_validated(sb_kv_cache* c, const int32_t* ids, int64_t n, int check_ref, int kind, int a0, int a1,
                         int64_t now) {
  c->ensure_ids(std::max<int64_t>(n, 1));
  if (n) SB_CUDA(cudaMemcpyAsync(c->d_ids, ids, sizeof(int32_t) * n, cudaMemcpyHostToDevice, c->stream));
  k_set_scal<<<1, 1, 0, c->stream>>>(c->S.scal, S_ERRIDX, INT64_MAX);
  if (n) k_validate_ids<<<grid_for(n), 256, 0, c->stream>>>(c->P, c->d_ids, n, check_ref, c->S.scal);
  if (n) {
    if (kind == 0) k_release_apply<<<grid_for(n), 256, 0, c->stream>>>(c->P, c->d_ids, n, c->S.scal);
    if (kind == 1) k_touch_apply<<<grid_for(n), 256, 0, c->stream>>>(c->P, c->d_ids, n, now, c->S.scal);
    if (kind == 2) k_priority_apply<<<grid_for(n), 256, 0, c->stream>>>(c->P, c->d_ids, n, a0, a1, c->S.scal);
  }
  SB_CHECK_LAUNCH();
  const int64_t err = c->read_scal(S_ERRIDX);
  if (err >= n) return SB_OK;
  // classify the first failing id exactly as the reference's in-order loop
  int32_t id = ids[err];
  if (id < 0 || id >= c->P.cap) {
    set_last_error("block " + std::to_string(id) + " not resident");
    return SB_ERR_UNKNOWN_BLOCK;
  }
  int32_t nt = 0;
  SB_CUDA(cudaMemcpy(&nt, c->P.ntok + id, sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (nt == 0) {
    set_last_error("block " + std::to_string(id) + " not resident");
    return SB_ERR_UNKNOWN_BLOCK;
  }
  set_last_error("release of block " + std::to_string(id) + " with ref_count 0");
  return SB_ERR_ZERO_REF_RELEASE;
}

int sb_kv_release(sb_kv_cache* c, const int32_t* ids, int64_t n) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(c->mu);
    SB_CUDA(cudaSetDevice(c->device));
    return run_validated(c, ids, n, 1, 0, 0, 0, 0);
  });
}

int sb_kv_release_batch(sb_kv_cache* c, const int32_t* d_ids, int64_t n, int32_t* d_status, void* stream) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(c->mu);
    SB_CUDA(cudaSetDevice(c->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);  // NULL = legacy default stream
    c->join_in(st);
    k_set_scal<<<1, 1, 0, st>>>(c->S.scal, S_ERRIDX, INT64_MAX);
    if (n > 0) {
      k_validate_ids<<<grid_for(n), 256, 0, st>>>(c->P, d_ids, n, 1, c->S.scal, 1);
      k_release_apply<<<grid_for(n), 256, 0, st>>>(c->P, d_ids, n, c->S.scal);
    }
    // all-or-nothing outcome (kv_cache.cpp:228-236): the first failing id in
    // order decides UnknownBlock / ZeroRefRelease
    if (d_status) k_release_status<<<1, 32, 0, st>>>(c->P, d_ids, n, c->S.scal, d_status);
    SB_CHECK_LAUNCH();
    c->join_out(st);
    return int(SB_OK);
  });
}

int sb_kv_touch(sb_kv_cache* c, const int32_t* ids, int64_t n, int64_t now) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(c->mu);
    SB_CUDA(cudaSetDevice(c->device));
    check_now(c->P, now);
    return run_validated(c, ids, n, 0, 1, 0, 0, now);
  });
}

int sb_kv_set_reuse_priority(sb_kv_cache* c, const int32_t* ids, int64_t n, int32_t pinned, int32_t tier_override) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(c->mu);
    SB_CUDA(cudaSetDevice(c->device));
    if (tier_override > SB_TAG_HISTORY) throw Error(SB_ERR_INVALID, "bad tag");
    return run_validated(c, ids, n, 0, 2, pinned, tier_override, 0);
  });
}

int sb_kv_set_tag(sb_kv_cache* c, int32_t id, int32_t tag) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(c->mu);
    SB_CUDA(cudaSetDevice(c->device));
    if (tag < 0 || tag > SB_TAG_HISTORY) throw Error(SB_ERR_INVALID, "bad tag");
    return run_validated(c, &id, 1, 0, 2, -1, tag, 0);
  });
}

int64_t sb_kv_block_size(const sb_kv_cache* c) { return c->P.bs; }
int64_t sb_kv_capacity_blocks(const sb_kv_cache* c) { return c->P.cap; }
int64_t sb_kv_resident_blocks(const sb_kv_cache* c) { return static_cast<int64_t>(c->read_ctr(C_NRES)); }
int64_t sb_kv_free_blocks(const sb_kv_cache* c) { return c->P.cap - sb_kv_resident_blocks(c); }
uint64_t sb_kv_total_evicted(const sb_kv_cache* c) { return c->read_ctr(C_EVICTED); }
int32_t sb_kv_policy(const sb_kv_cache* c) { return c->P.policy; }

int sb_kv_last_evicted(const sb_kv_cache* c, int32_t* out, int64_t cap, int64_t* n_out) {
  *n_out = static_cast<int64_t>(c->last_evicted.size());
  const int64_t m = std::min<int64_t>(cap, *n_out);
  if (out && m > 0) std::memcpy(out, c->last_evicted.data(), sizeof(int32_t) * m);
  return SB_OK;
}

int sb_kv_contains(const sb_kv_cache* c, int32_t id) {
  if (id < 0 || id >= c->P.cap) return 0;
  int32_t nt = 0;
  cudaMemcpy(&nt, c->P.ntok + id, sizeof(int32_t), cudaMemcpyDeviceToHost);
  return nt > 0 ? 1 : 0;
}

int sb_kv_resident_ids(const sb_kv_cache* c, int32_t* out, int64_t* n_out) {
  return guard([&] {
    SB_CUDA(cudaStreamSynchronize(c->stream));
    std::vector<int32_t> nt(c->P.cap);
    SB_CUDA(cudaMemcpy(nt.data(), c->P.ntok, 4 * c->P.cap, cudaMemcpyDeviceToHost));
    int64_t n = 0;
    for (int64_t i = 0; i < c->P.cap; ++i)
      if (nt[i] > 0) out[n++] = static_cast<int32_t>(i);
    *n_out = n;
    return int(SB_OK);
  });
}

int sb_kv_block(const sb_kv_cache* c, int32_t id, sb_block_info* info, uint64_t* tokens_out) {
  // logical constness: the read-back only uses the pool's staging buffers
  sb_kv_cache* m = const_cast<sb_kv_cache*>(c);
  const int st = sb_kv_blocks(m, &id, 1, info);
  if (st != SB_OK) return st;
  return guard([&] {
    if (info->n_tokens == 0) {
      set_last_error("block " + std::to_string(id) + " not resident");
      return int(SB_ERR_UNKNOWN_BLOCK);
    }
    if (tokens_out)
      SB_CUDA(cudaMemcpy(tokens_out, c->P.tok + int64_t(id) * c->P.bs, sizeof(uint64_t) * info->n_tokens,
                         cudaMemcpyDeviceToHost));
    return int(SB_OK);
  });
}

int sb_kv_blocks(sb_kv_cache* c, const int32_t* ids, int64_t n, sb_block_info* infos) {
  return guard([&] {
    std::lock_guard<std::mutex> lk(c->mu);
    SB_CUDA(cudaSetDevice(c->device));
    if (n <= 0) return int(SB_OK);
    c->ensure_ids(n);
    // the token staging buffer holds the records (48 B = 6 u64 each)
    static_assert(sizeof(sb_block_info) == 6 * sizeof(uint64_t), "sb_block_info layout");
    c->ensure_tokens(6 * n);
    sb_block_info* d_out = reinterpret_cast<sb_block_info*>(c->d_tok);
    SB_CUDA(cudaMemcpyAsync(c->d_ids, ids, sizeof(int32_t) * n, cudaMemcpyHostToDevice, c->stream));
    k_block_info<<<grid_for(n), 256, 0, c->stream>>>(c->P, c->d_ids, n, d_out);
    SB_CHECK_LAUNCH();
    SB_CUDA(cudaMemcpyAsync(infos, d_out, sizeof(sb_block_info) * n, cudaMemcpyDeviceToHost, c->stream));
    SB_CUDA(cudaStreamSynchronize(c->stream));
    return int(SB_OK);
  });
}

namespace {
struct HostView {
  std::vector<int32_t> ntok, tag, ref, pinned;
  std::vector<int64_t> last;
  std::vector<uint64_t> chain, parent;
  std::vector<IdxEntry> idx;
  unsigned long long nres = 0;
};
HostView read_view(const sb_kv_cache* c, bool with_index) {
  const Pool& P = c->P;
  HostView v;
  v.ntok.resize(P.cap);
  v.tag.resize(P.cap);
  v.ref.resize(P.cap);
  v.pinned.resize(P.cap);
  v.last.resize(P.cap);
  SB_CUDA(cudaMemcpy(v.ntok.data(), P.ntok, 4 * P.cap, cudaMemcpyDeviceToHost));
  SB_CUDA(cudaMemcpy(v.tag.data(), P.tag, 4 * P.cap, cudaMemcpyDeviceToHost));
  SB_CUDA(cudaMemcpy(v.ref.data(), P.ref, 4 * P.cap, cudaMemcpyDeviceToHost));
  SB_CUDA(cudaMemcpy(v.pinned.data(), P.pinned, 4 * P.cap, cudaMemcpyDeviceToHost));
  SB_CUDA(cudaMemcpy(v.last.data(), P.last, 8 * P.cap, cudaMemcpyDeviceToHost));
  SB_CUDA(cudaMemcpy(&v.nres, P.ctr + C_NRES, 8, cudaMemcpyDeviceToHost));
  if (with_index) {
    v.chain.resize(P.cap);
    v.parent.resize(P.cap);
    v.idx.resize(P.tcap);
    SB_CUDA(cudaMemcpy(v.chain.data(), P.chain, 8 * P.cap, cudaMemcpyDeviceToHost));
    SB_CUDA(cudaMemcpy(v.parent.data(), P.parent, 8 * P.cap, cudaMemcpyDeviceToHost));
    SB_CUDA(cudaMemcpy(v.idx.data(), P.idx, sizeof(IdxEntry) * P.tcap, cudaMemcpyDeviceToHost));
  }
  return v;
}
const char* tag_name(int t) {
  static const char* n[6] = {"response", "tool_output", "user_query", "system_prompt", "partial_prefill", "history"};
  return t >= 0 && t < 6 ? n[t] : "unknown";
}
}  // namespace

int sb_kv_audit(const sb_kv_cache* c) {
  return guard([&] {
    SB_CUDA(cudaStreamSynchronize(c->stream));
    HostView v = read_view(c, true);
    int64_t res = 0;
    for (int64_t i = 0; i < c->P.cap; ++i) {
      if (v.ntok[i] == 0) continue;
      ++res;
      if (v.ref[i] < 0) throw Error(SB_ERR_CACHE, "audit: negative ref_count");
      if (v.ntok[i] < 1 || v.ntok[i] > c->P.bs) throw Error(SB_ERR_CACHE, "audit: bad block token count");
    }
    if (res != static_cast<int64_t>(v.nres) || res > c->P.cap) throw Error(SB_ERR_CACHE, "audit: block accounting mismatch");
    int64_t indexed = 0;
    for (int64_t s = 0; s < c->P.tcap; ++s) {
      const IdxEntry& e = v.idx[s];
      const int32_t id = e.id;
      if (id < 0) continue;
      if (v.ntok[id] == 0 || v.chain[id] != e.key || v.parent[id] != e.parent || v.ntok[id] != e.ntok)
        throw Error(SB_ERR_CACHE, "audit: hash index out of sync");
      ++indexed;
    }
    if (indexed != res) throw Error(SB_ERR_CACHE, "audit: hash index size mismatch");
    return int(SB_OK);
  });
}

int sb_kv_dump(const sb_kv_cache* c, char* buf, int64_t cap, int64_t* len) {
  return guard([&] {
    SB_CUDA(cudaStreamSynchronize(c->stream));
    HostView v = read_view(c, false);
    std::string out;
    out.reserve(64 * v.nres);
    char line[256];
    for (int64_t i = 0; i < c->P.cap; ++i) {
      if (v.ntok[i] == 0) continue;
      int m = snprintf(line, sizeof line, "block=%lld tag=%s tier=%d ref=%d pinned=%d last_used=%lld tokens=%d\n",
                       (long long)i, tag_name(v.tag[i]), tier_of(v.tag[i]), v.ref[i], v.pinned[i] ? 1 : 0,
                       (long long)v.last[i], v.ntok[i]);
      out.append(line, m);
    }
    *len = static_cast<int64_t>(out.size());
    if (buf && cap > 0) {
      int64_t m = std::min<int64_t>(cap - 1, *len);
      std::memcpy(buf, out.data(), m);
      buf[m] = 0;
    }
    return int(SB_OK);
  });
}

int sb_kv_program_stats(const sb_kv_cache* c, uint64_t out[2]) {
  return guard([&] {
    out[0] = c->fast_runs;
    out[1] = c->fast_taken;
    return int(SB_OK);
  });
}

int sb_kv_stats(const sb_kv_cache* c, uint64_t out[6]) {
  return guard([&] {
    unsigned long long v[C_N];
    SB_CUDA(cudaMemcpy(v, c->P.ctr, sizeof(v), cudaMemcpyDeviceToHost));
    out[0] = v[C_LOOKUPS];
    out[1] = v[C_HIT_TOK];
    out[2] = v[C_LOOK_TOK];
    out[3] = v[C_INS_BLOCKS];
    out[4] = v[C_EV_BLOCKS];
    out[5] = v[C_FULL];
    return int(SB_OK);
  });
}

}  // extern "C"
