// attention.cu — continuation-prefill attention over the paged KV pool
// (sm_100a: TMA + tcgen05/TMEM), plus the KV append of the suffix tokens.
//
// Replaces the reference engine's prefill cost model (CostModel::chunk_ms,
// /root/reference/proj/src/engine.cpp:35-39) for Engine::extend_prefill
// (engine.cpp:184-223): the suffix (tool-output) tokens of each sequence
// attend to the already-cached prefix pages plus causally to themselves.
//
// Work item = (sequence, kv head, pair of 128-row query tiles).  A query tile
// packs tokens x GQA heads of one kv head into the 128 MMA rows
// (row = token * group + head), so every K/V page is read once for the whole
// group.  One CTA per SM (192 KB smem, 512 TMEM columns):
//   warp 0      TMA producer: Q tiles once, then K/V pages (16 tokens x 64
//               dims boxes, SWIZZLE_128B) into a 4-stage ring
//   warp 1      MMA issuer (one thread): S_t = Q_t K^T  (SS, K-major),
//               O_t += P_t V (TS: P from TMEM, V MN-major), issued in four
//               32-key parts as the softmax releases them
//   warp 2      TMEM allocator
//   warps 4-7   softmax for tile 0, warps 8-11 softmax for tile 1: one TMEM
//               lane (= one query row) per thread; online softmax with a
//               lazy rescale (O is rescaled in TMEM only when the running
//               max grows by more than 2^8)
// TMEM columns: S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512); P_t is
// written as packed bf16 over the first 64 columns of S_t.
#include <cuda.h>
#include <cuda_runtime.h>

#include <mutex>

#include <cmath>
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <vector>

#include "common.h"
#include "sm100.cuh"
#include "tma_host.h"

namespace sb {
namespace attn {

constexpr int kThreads = 384;
constexpr int kStages = 4;
constexpr int kTileBytes = 32768;  // 128 rows x 128 dims bf16 (two 64-col SW128 atoms)
constexpr int kAtomBytes = 16384;
constexpr int kSmemBytes = 2 * kTileBytes + kStages * kTileBytes + 1024;

struct Params {
  const int32_t* q_off;
  const int32_t* kv_len;
  const int32_t* table;
  __nv_bfloat16* out;
  int32_t n_seqs, max_blocks, n_q_heads, n_kv_heads, group, tpt, pairs_per_seq;
  int32_t oob_row;  // a K/V row coordinate past the end: zero-filled loads
  float scale_log2;
  const int32_t* work;  // optional {seq, kvh << 16 | pair} items
};

struct Smem {
  uint64_t q_full;
  uint64_t kv_full[kStages];
  uint64_t kv_empty[kStages];
  uint64_t s_full[2];
  uint64_t p_part[2][4];  // P of keys [32i, 32i + 32) written (i < kPSplit)
  uint64_t o_done[2];
  uint32_t tmem_base;
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
// packed pair helpers (FFMA2 / FADD2 on sm_100a)
__device__ __forceinline__ void ffma2(float& d0, float& d1, float a0, float a1, float b, float c) {
  uint64_t r, pa, pb, pc;
  asm("mov.b64 %0, {%1, %2};" : "=l"(pa) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %1};" : "=l"(pb) : "f"(b));
  asm("mov.b64 %0, {%1, %1};" : "=l"(pc) : "f"(c));
  asm("fma.rn.ftz.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pa), "l"(pb), "l"(pc));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(d0), "=f"(d1) : "l"(r));
}
// 2^x for a pair on the FMA/ALU pipes (offloads MUFU): x = r + f with
// r = rint(x) (magic-number rounding), 2^f by a degree-3 minimax polynomial on
// [-0.5, 0.5] (max rel. error 7.5e-5, below bf16 rounding of P), and r added
// to the exponent field.  x is clamped to >= -120 (masked -inf -> ~1e-36).
__device__ __forceinline__ void ex2_poly2(float x0, float x1, float& y0, float& y1) {
  constexpr float kMagic = 12582912.f;  // 1.5 * 2^23
  x0 = fmaxf(x0, -120.f);  // keeps the result's exponent field normal
  x1 = fmaxf(x1, -120.f);
  uint64_t px, pm, pt, pr, pf, pc, pp;
  asm("mov.b64 %0, {%1, %2};" : "=l"(px) : "f"(x0), "f"(x1));
  asm("mov.b64 %0, {%1, %1};" : "=l"(pm) : "f"(kMagic));
  asm("add.rn.ftz.f32x2 %0, %1, %2;" : "=l"(pt) : "l"(px), "l"(pm));  // t = x + M
  asm("sub.rn.ftz.f32x2 %0, %1, %2;" : "=l"(pr) : "l"(pt), "l"(pm));  // r = t - M
  asm("sub.rn.ftz.f32x2 %0, %1, %2;" : "=l"(pf) : "l"(px), "l"(pr));  // f = x - r
  asm("mov.b64 %0, {%1, %1};" : "=l"(pc) : "f"(0.055170975625514984f));
  uint64_t c2, c1, c0;
  asm("mov.b64 %0, {%1, %1};" : "=l"(c2) : "f"(0.24260970950126648f));
  asm("mov.b64 %0, {%1, %1};" : "=l"(c1) : "f"(0.6932609677314758f));
  asm("mov.b64 %0, {%1, %1};" : "=l"(c0) : "f"(0.9999281764030457f));
  asm("fma.rn.ftz.f32x2 %0, %1, %2, %3;" : "=l"(pp) : "l"(pc), "l"(pf), "l"(c2));
  asm("fma.rn.ftz.f32x2 %0, %1, %2, %3;" : "=l"(pp) : "l"(pp), "l"(pf), "l"(c1));
  asm("fma.rn.ftz.f32x2 %0, %1, %2, %3;" : "=l"(pp) : "l"(pp), "l"(pf), "l"(c0));
  float q0, q1, t0, t1;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(q0), "=f"(q1) : "l"(pp));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(t0), "=f"(t1) : "l"(pt));
  // exponent add: the integer r sits in the low mantissa bits of t
  y0 = __uint_as_float(__float_as_uint(q0) + (__float_as_uint(t0) << 23));
  y1 = __uint_as_float(__float_as_uint(q1) + (__float_as_uint(t1) << 23));
}

__device__ __forceinline__ void fadd2(float& a0, float& a1, float b0, float b1) {
  uint64_t r, pa, pb;
  asm("mov.b64 %0, {%1, %2};" : "=l"(pa) : "f"(a0), "f"(a1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(pb) : "f"(b0), "f"(b1));
  asm("add.rn.ftz.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pa), "l"(pb));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(r));
}

// The softmax warpgroups of both kernels: warps 4-7 own query tile 0, warps
// 8-11 tile 1, one TMEM lane (= one query row) per thread.  Online softmax with
// a lazy rescale (O is rescaled in TMEM only when the running max grows by
// more than 2^8), P written as packed bf16 over the first 64 columns of S and
// released to the MMA issuer in kPSplit parts through `release(tile, part)`
// (after tcgen05.wait::st + fence::before_thread_sync), then O / l -> bf16.
template <int kPSplit, class SmemT, class Release>
__device__ __forceinline__ void softmax_warpgroup(const Params& p, SmemT& ss, uint32_t tmem, int tid, int warp,
                                                  int first_q, int prefix, int q_len, int q0, int kvh, int n_kv,
                                                  Release&& release) {
  const int t = (warp - 4) >> 2;  // tile of this warpgroup
  const int r = tid - 128 - t * 128;
  const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
  const uint32_t s_col = tmem + lane_off + t * 128;
  const uint32_t o_col = tmem + lane_off + 256 + t * 128;
  const int qidx = first_q + t * p.tpt + r / p.group;
  const int qpos = prefix + qidx;  // absolute key position of this query
  float m_used = -INFINITY, l = 0.f;
  for (int j = 0; j < n_kv; ++j) {
    mbar_wait_suspend(&ss.s_full[t], j & 1);
    tc_fence_after();
    // raw scores: four TMEM loads in flight, one wait
    uint32_t sv[128];
    tmem_ld32(s_col + 0, *reinterpret_cast<uint32_t(*)[32]>(sv + 0));
    tmem_ld32(s_col + 32, *reinterpret_cast<uint32_t(*)[32]>(sv + 32));
    tmem_ld32(s_col + 64, *reinterpret_cast<uint32_t(*)[32]>(sv + 64));
    tmem_ld32(s_col + 96, *reinterpret_cast<uint32_t(*)[32]>(sv + 96));
    tmem_wait_ld();
    float* s = reinterpret_cast<float*>(sv);
    const int kbase = j * 128;
    if (kbase + 127 > qpos) {
#pragma unroll
      for (int k = 0; k < 128; ++k)
        if (kbase + k > qpos) s[k] = -INFINITY;
    }
    // row max: 8 independent 3-input max chains, then a short tree
    float mk[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) mk[i] = fmax3(s[i], s[8 + i], s[16 + i]);
#pragma unroll
    for (int k = 24; k + 16 <= 120; k += 16)
#pragma unroll
      for (int i = 0; i < 8; ++i) mk[i] = fmax3(mk[i], s[k + i], s[k + 8 + i]);
#pragma unroll
    for (int i = 0; i < 8; ++i) mk[i] = fmaxf(mk[i], s[120 + i]);
    const float mx = fmaxf(fmax3(mk[0], mk[1], mk[2]), fmax3(fmax3(mk[3], mk[4], mk[5]), mk[6], mk[7])) *
                     p.scale_log2;
    const float m_new = fmaxf(m_used, mx);
    const bool need = m_new > m_used + 8.f;
    float factor = 1.f;
    if (need) {
      factor = ex2(m_used - m_new);  // 0 on the first tile (m_used = -inf)
      m_used = m_new;
    }
    if (j > 0 && __any_sync(0xffffffffu, need)) {
      // rescale this warp's rows of O in TMEM once PV_{j-1} has landed
      mbar_wait_suspend(&ss.o_done[t], (j - 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        uint32_t v[16];
        tmem_ld16(o_col + c * 16, v);
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = __float_as_uint(__uint_as_float(v[k]) * factor);
        tmem_st16(o_col + c * 16, v);
      }
    }
    l *= factor;
    // p = 2^(s*scale - m): one FFMA2 per pair, MUFU ex2, 4 packed partial sums
    const float neg_m = -m_used;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t w[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        float a0, a1;
        ffma2(a0, a1, s[32 * c + 2 * k], s[32 * c + 2 * k + 1], p.scale_log2, neg_m);
        float e0, e1;
        if ((k & 3) == 3) {  // a quarter of the pairs on the FMA pipes
          ex2_poly2(a0, a1, e0, e1);
        } else {
          e0 = ex2(a0);
          e1 = ex2(a1);
        }
        fadd2(acc[2 * (k & 3)], acc[2 * (k & 3) + 1], e0, e1);
        w[k] = pack_bf16x2(e0, e1);
      }
      tmem_st16(s_col + c * 16, w);
      if ((c + 1) % (4 / kPSplit) == 0) {  // release this part of P to the MMA issuer
        tmem_wait_st();
        tc_fence_before();
        release(t, c / (4 / kPSplit));
      }
    }
    fadd2(acc[0], acc[1], acc[2], acc[3]);
    fadd2(acc[4], acc[5], acc[6], acc[7]);
    fadd2(acc[0], acc[1], acc[4], acc[5]);
    l += acc[0] + acc[1];
  }
  // ---- epilogue: O / l -> bf16 -> global
  mbar_wait_suspend(&ss.o_done[t], (n_kv - 1) & 1);
  tc_fence_after();
  const bool valid = qidx < q_len;
  const float inv = (valid && l > 0.f) ? 1.f / l : 0.f;
  __nv_bfloat16* orow =
      p.out + (static_cast<int64_t>(q0 + qidx) * p.n_q_heads + kvh * p.group + (r % p.group)) * 128;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t v[32];
    tmem_ld32(o_col + c * 32, v);
    tmem_wait_ld();
    if (valid) {
      uint4* dst = reinterpret_cast<uint4*>(orow + c * 32);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint4 w;
        w.x = pack_bf16x2(__uint_as_float(v[8 * k + 0]) * inv, __uint_as_float(v[8 * k + 1]) * inv);
        w.y = pack_bf16x2(__uint_as_float(v[8 * k + 2]) * inv, __uint_as_float(v[8 * k + 3]) * inv);
        w.z = pack_bf16x2(__uint_as_float(v[8 * k + 4]) * inv, __uint_as_float(v[8 * k + 5]) * inv);
        w.w = pack_bf16x2(__uint_as_float(v[8 * k + 6]) * inv, __uint_as_float(v[8 * k + 7]) * inv);
        dst[k] = w;
      }
    }
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    k_continuation_attention(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                             const __grid_constant__ CUtensorMap tm_v, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = base;                    // [2 tiles][2 atoms][16 KB]
  uint8_t* sKV = base + 2 * kTileBytes;  // [kStages][2 atoms][16 KB]
  __shared__ Smem ss;

  const int tid = threadIdx.x, warp = tid >> 5;
  // ---- work item
  int pair, kvh, seq;
  if (p.work) {
    seq = p.work[2 * blockIdx.x];
    kvh = p.work[2 * blockIdx.x + 1] >> 16;
    pair = p.work[2 * blockIdx.x + 1] & 0xFFFF;
  } else {
    const int item = blockIdx.x;
    pair = item % p.pairs_per_seq;
    kvh = (item / p.pairs_per_seq) % p.n_kv_heads;
    seq = item / (p.pairs_per_seq * p.n_kv_heads);
  }
  const int q0 = p.q_off[seq];
  const int q_len = p.q_off[seq + 1] - q0;
  const int kv_len = p.kv_len[seq];
  const int first_q = pair * 2 * p.tpt;  // query index (within sequence) of row 0 of tile 0
  if (first_q >= q_len) return;
  const int prefix = kv_len - q_len;
  const int kv_limit = prefix + min(q_len, first_q + 2 * p.tpt);
  const int n_kv = (kv_limit + 127) / 128;

  if (tid == 0) {
    mbar_init(&ss.q_full, 1);
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&ss.kv_full[i], 1);
      mbar_init(&ss.kv_empty[i], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&ss.s_full[t], 1);
      for (int i = 0; i < 4; ++i) mbar_init(&ss.p_part[t][i], 128);
      mbar_init(&ss.o_done[t], 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(&ss.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = ss.tmem_base;
  // P is released to the MMA warp in kPSplit parts of 128 / kPSplit keys
  // (measured: 4 parts +8-10 % over one release per tile)
  constexpr int kPSplit = 4;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (elect_one()) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      mbar_arrive_expect_tx(&ss.q_full, 2 * kTileBytes);
      for (int t = 0; t < 2; ++t)
        for (int a = 0; a < 2; ++a)
          tma_load_3d(sQ + t * kTileBytes + a * kAtomBytes, &tm_q, &ss.q_full, a * 64, kvh * p.group,
                      q0 + first_q + t * p.tpt);
      const int32_t* trow = p.table + static_cast<int64_t>(seq) * p.max_blocks;
      int rows[8], next_rows[8];
      auto fetch_rows = [&](int j, int (&r)[8]) {
#pragma unroll
        for (int pg = 0; pg < 8; ++pg) {
          const int jb = j * 8 + pg;
          const int page = (jb * 16 < kv_limit) ? __ldg(trow + jb) : -1;  // -1: no page (failed insert)
          r[pg] = page >= 0 ? (page * p.n_kv_heads + kvh) * 16 : p.oob_row;
        }
      };
      fetch_rows(0, rows);
      for (int i = 0; i < 2 * n_kv; ++i) {
        const int j = i >> 1, which = i & 1, stage = i % kStages;
        if (which == 0 && j + 1 < n_kv) fetch_rows(j + 1, next_rows);  // page ids one tile ahead
        mbar_wait_suspend(&ss.kv_empty[stage], ((i / kStages) & 1) ^ 1);
        mbar_arrive_expect_tx(&ss.kv_full[stage], kTileBytes);
        uint8_t* dst = sKV + stage * kTileBytes;
        const void* tm = which ? static_cast<const void*>(&tm_v) : static_cast<const void*>(&tm_k);
#pragma unroll
        for (int pg = 0; pg < 8; ++pg)
#pragma unroll
          for (int a = 0; a < 2; ++a)
            tma_load_2d(dst + a * kAtomBytes + pg * 2048, tm, &ss.kv_full[stage], a * 64, rows[pg]);
        if (which == 1 && j + 1 < n_kv)
#pragma unroll
          for (int pg = 0; pg < 8; ++pg) rows[pg] = next_rows[pg];
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (elect_one()) {
      const uint32_t idesc_qk = idesc_bf16_f32(128, 128, 0, 0);
      const uint32_t idesc_pv = idesc_bf16_f32(128, 128, 0, 1);
      const uint32_t sq = smem_u32(sQ), skv = smem_u32(sKV);
      mbar_wait_suspend(&ss.q_full, 0);
      auto wait_stage = [&](int i) { mbar_wait_suspend(&ss.kv_full[i % kStages], (i / kStages) & 1); };
      auto qk = [&](int t, int j) {
        const uint32_t kb = skv + ((2 * j) % kStages) * kTileBytes;
        const uint32_t qb = sq + t * kTileBytes;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * kAtomBytes + (kk & 3) * 32;
          mma_ss(tmem + t * 128, smem_desc_sw128(qb + off, 16, 1024), smem_desc_sw128(kb + off, 16, 1024), idesc_qk,
                 kk > 0);
        }
        mma_commit(&ss.s_full[t]);
      };
      // PV in kPSplit parts: the MMAs of a block of keys are issued as soon
      // as the softmax has written their P, so PV overlaps the rest of the
      // exp phase
      auto pv = [&](int t, int j) {
        const uint32_t vb = skv + ((2 * j + 1) % kStages) * kTileBytes;
#pragma unroll
        for (int part = 0; part < kPSplit; ++part) {
          mbar_wait_suspend(&ss.p_part[t][part], j & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = part * (8 / kPSplit); kk < (part + 1) * (8 / kPSplit); ++kk)
            mma_ts(tmem + 256 + t * 128, tmem + t * 128 + kk * 8, smem_desc_sw128(vb + kk * 2048, kAtomBytes, 1024),
                   idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit(&ss.o_done[t]);
      };
      wait_stage(0);
      tc_fence_after();
      qk(0, 0);
      qk(1, 0);
      mma_commit(&ss.kv_empty[0]);
      for (int j = 0; j < n_kv; ++j) {
        wait_stage(2 * j + 1);
        tc_fence_after();
        pv(0, j);
        if (j + 1 < n_kv) {
          wait_stage(2 * j + 2);
          tc_fence_after();
          qk(0, j + 1);
        }
        pv(1, j);
        mma_commit(&ss.kv_empty[(2 * j + 1) % kStages]);
        if (j + 1 < n_kv) {
          qk(1, j + 1);
          mma_commit(&ss.kv_empty[(2 * j + 2) % kStages]);
        }
      }
    }
  } else if (warp >= 4) {
    // ===================== softmax (one query row per thread) =====================
    softmax_warpgroup<kPSplit>(p, ss, tmem, tid, warp, first_q, prefix, q_len, q0, kvh, n_kv,
                               [&](int tile, int part) { mbar_arrive(&ss.p_part[tile][part]); });
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// ---------------------------------------------------------------------------
// CTA-pair variant (cta_group::2, SB_ATTN_PAIR=1): a cluster of two CTAs takes a
// quad of query tiles — CTA r the pair 2*quad + r — and the leader issues
// every MMA with M = 256 over both CTAs' rows.  The K/V tiles are split
// across the pair: for S = Q K^T (N = 128 keys) CTA r stages keys
// [64r, 64r + 64) of the tile; for O += P V (N = 128 dims) CTA r stages dims
// [64r, 64r + 64) of every key.  Each SM so moves half the K/V bytes from L2
// and reads a third fewer operand bytes from shared memory per FLOP than the
// 1-CTA kernel above (the GEMM's pair kernel measured +13 % over its 1-CTA
// form under the same power cap).  The softmax is unchanged and local: each
// CTA's TMEM holds S, P and O of its own 128-row tiles.  Barriers: Q and K/V
// TMA completions of both CTAs count on the leader's q_full / kv_full; the
// leader's commits multicast to both CTAs' kv_empty / s_full / o_done; P
// parts are released on the leader's p_part by one lane per softmax warp of
// both CTAs (8 arrivals).  Both CTAs run the quad's key range (the larger of
// the two causal limits); a CTA past the sequence's last query computes
// discarded rows.
// SB_ATTN_PAIR=1: the CTA-pair kernel below instead of the 1-CTA kernel
// (A/B switch, read once per process).  Measured on the configs[1] step
// (profiles/r02/attn_pair_ab.txt): the pair runs ~4.5 % higher clocks under
// the 1 kW cap (less operand traffic per FLOP) but ~6 % less work per clock
// (the pair's MMAs wait on both CTAs' softmax; a quad's second pair may be
// empty; the quad's causal limit covers both CTAs): 261.4-261.9K vs
// 265.1-265.9K tokens/s, so the 1-CTA kernel stays the default.
inline bool pair_mode() {
  static const bool on = [] {
    const char* e = std::getenv("SB_ATTN_PAIR");
    return e && e[0] == '1';
  }();
  return on;
}

namespace pairk {

constexpr int kStages = 8;
constexpr int kHalf = 16384;       // one CTA's share of a K or V tile
constexpr int kHalfAtom = 8192;    // 64 key rows x 128 B (K half, one 64-dim atom)
constexpr int kSmemBytes = 2 * kTileBytes + kStages * kHalf + 1024;

struct Smem {
  uint64_t q_full;
  uint64_t kv_full[kStages];
  uint64_t kv_empty[kStages];
  uint64_t s_full[2];
  uint64_t p_part[2][4];
  uint64_t o_done[2];
  uint32_t tmem_base;
};

// kPSplit: P released to the issuer in this many parts per tile (2 measured
// best for the pair: each release is a remote arrive); kSpin: the issuer
// spins on those arrivals instead of a suspended wait (measured faster).
template <int kPSplit, bool kSpin>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_continuation_attention_pair(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                                  const __grid_constant__ CUtensorMap tm_v, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = base;                    // [2 tiles][2 atoms][16 KB]
  uint8_t* sKV = base + 2 * kTileBytes;  // [kStages][16 KB]
  __shared__ Smem ss;

  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t rank = cluster_rank();
  const int item = blockIdx.x >> 1;
  int quad, kvh, seq;
  if (p.work) {
    seq = p.work[2 * item];
    kvh = p.work[2 * item + 1] >> 16;
    quad = p.work[2 * item + 1] & 0xFFFF;
  } else {
    const int quads = (p.pairs_per_seq + 1) >> 1;
    quad = item % quads;
    kvh = (item / quads) % p.n_kv_heads;
    seq = item / (quads * p.n_kv_heads);
  }
  const int q0 = p.q_off[seq];
  const int q_len = p.q_off[seq + 1] - q0;
  const int kv_len = p.kv_len[seq];
  const int first_q = (2 * quad + static_cast<int>(rank)) * 2 * p.tpt;  // this CTA's row 0 of tile 0
  const int quad_q = quad * 4 * p.tpt;
  // the item exists only if the quad has queries: both CTAs run (the MMAs span the pair)
  if (quad_q >= q_len) return;
  const int prefix = kv_len - q_len;
  const int kv_limit = prefix + min(q_len, quad_q + 4 * p.tpt);
  const int n_kv = (kv_limit + 127) / 128;

  if (tid == 0) {
    mbar_init(&ss.q_full, 1);
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&ss.kv_full[i], 1);
      mbar_init(&ss.kv_empty[i], 1);
    }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&ss.s_full[t], 1);
      for (int i = 0; i < 4; ++i) mbar_init(&ss.p_part[t][i], 8);
      mbar_init(&ss.o_done[t], 1);
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc2(&ss.tmem_base);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = ss.tmem_base;

  if (warp == 0) {
    // ===================== TMA producer (both CTAs: their halves) =====================
    if (elect_one()) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      const uint32_t q_full0 = mapa(&ss.q_full, 0);
      if (rank == 0) mbar_arrive_expect_tx(&ss.q_full, 4 * kTileBytes);
      for (int t = 0; t < 2; ++t)
        for (int a = 0; a < 2; ++a)
          tma_load_3d_pair(sQ + t * kTileBytes + a * kAtomBytes, &tm_q, q_full0, a * 64, kvh * p.group,
                           q0 + first_q + t * p.tpt);
      const int32_t* trow = p.table + static_cast<int64_t>(seq) * p.max_blocks;
      int rows[8], next_rows[8];
      auto fetch_rows = [&](int j, int (&r)[8]) {
#pragma unroll
        for (int pg = 0; pg < 8; ++pg) {
          const int jb = j * 8 + pg;
          const int page = (jb * 16 < kv_limit) ? __ldg(trow + jb) : -1;
          r[pg] = page >= 0 ? (page * p.n_kv_heads + kvh) * 16 : p.oob_row;
        }
      };
      fetch_rows(0, rows);
      for (int i = 0; i < 2 * n_kv; ++i) {
        const int j = i >> 1, which = i & 1, stage = i % kStages;
        if (which == 0 && j + 1 < n_kv) fetch_rows(j + 1, next_rows);
        mbar_wait_suspend(&ss.kv_empty[stage], ((i / kStages) & 1) ^ 1);
        const uint32_t full0 = mapa(&ss.kv_full[stage], 0);
        if (rank == 0) mbar_arrive_expect_tx(&ss.kv_full[stage], 2 * kHalf);
        uint8_t* dst = sKV + stage * kHalf;
        if (which == 0) {
          // K: keys [64 rank, 64 rank + 64) = pages 4 rank .. 4 rank + 3, both 64-dim atoms
#pragma unroll
          for (int pp = 0; pp < 4; ++pp)
#pragma unroll
            for (int a = 0; a < 2; ++a)
              tma_load_2d_pair(dst + a * kHalfAtom + pp * 2048, &tm_k, full0, a * 64, rank ? rows[4 + pp] : rows[pp]);
        } else {
          // V: dims [64 rank, 64 rank + 64) of all 128 keys
#pragma unroll
          for (int pg = 0; pg < 8; ++pg)
            tma_load_2d_pair(dst + pg * 2048, &tm_v, full0, static_cast<int>(rank) * 64, rows[pg]);
          if (j + 1 < n_kv)
#pragma unroll
            for (int pg = 0; pg < 8; ++pg) rows[pg] = next_rows[pg];
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader only) =====================
    if (rank == 0 && elect_one()) {
      const uint32_t idesc_qk = idesc_bf16_f32(256, 128, 0, 0);
      const uint32_t idesc_pv = idesc_bf16_f32(256, 128, 0, 1);
      const uint32_t sq = smem_u32(sQ), skv = smem_u32(sKV);
      mbar_wait_suspend(&ss.q_full, 0);
      auto wait_stage = [&](int i) { mbar_wait_suspend(&ss.kv_full[i % kStages], (i / kStages) & 1); };
      auto qk = [&](int t, int j) {
        const uint32_t kb = skv + ((2 * j) % kStages) * kHalf;
        const uint32_t qb = sq + t * kTileBytes;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t qoff = (kk >> 2) * kAtomBytes + (kk & 3) * 32;
          const uint32_t koff = (kk >> 2) * kHalfAtom + (kk & 3) * 32;
          mma_ss2(tmem + t * 128, smem_desc_sw128(qb + qoff, 16, 1024), smem_desc_sw128(kb + koff, 16, 1024),
                  idesc_qk, kk > 0);
        }
        mma_commit2(&ss.s_full[t]);
      };
      auto pv = [&](int t, int j) {
        const uint32_t vb = skv + ((2 * j + 1) % kStages) * kHalf;
#pragma unroll
        for (int part = 0; part < kPSplit; ++part) {
          if (kSpin)
            mbar_wait(&ss.p_part[t][part], j & 1);
          else
            mbar_wait_suspend(&ss.p_part[t][part], j & 1);
          tc_fence_after();
#pragma unroll
          for (int kk = part * (8 / kPSplit); kk < (part + 1) * (8 / kPSplit); ++kk)
            mma_ts2(tmem + 256 + t * 128, tmem + t * 128 + kk * 8, smem_desc_sw128(vb + kk * 2048, kAtomBytes, 1024),
                    idesc_pv, (j > 0 || kk > 0) ? 1u : 0u);
        }
        mma_commit2(&ss.o_done[t]);
      };
      wait_stage(0);
      tc_fence_after();
      qk(0, 0);
      qk(1, 0);
      mma_commit2(&ss.kv_empty[0]);
      for (int j = 0; j < n_kv; ++j) {
        wait_stage(2 * j + 1);
        tc_fence_after();
        pv(0, j);
        if (j + 1 < n_kv) {
          wait_stage(2 * j + 2);
          tc_fence_after();
          qk(0, j + 1);
        }
        pv(1, j);
        mma_commit2(&ss.kv_empty[(2 * j + 1) % kStages]);
        if (j + 1 < n_kv) {
          qk(1, j + 1);
          mma_commit2(&ss.kv_empty[(2 * j + 2) % kStages]);
        }
      }
    }
  } else if (warp >= 4) {
    // ===================== softmax (one query row per thread; as the 1-CTA kernel) =====================
    const int lane = tid & 31;
    softmax_warpgroup<kPSplit>(p, ss, tmem, tid, warp, first_q, prefix, q_len, q0, kvh, n_kv, [&](int tile, int part) {
      __syncwarp();  // one arrival per warp, on the leader
      if (lane == 0) mbar_arrive_remote_relaxed(mapa(&ss.p_part[tile][part], 0));
    });
  }
  tc_fence_before();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc2(tmem);
  }
}

}  // namespace pairk

// fp32 continuation attention (CUDA cores): the same op on fp32 pages, for
// the fp32 precision contract (outputs within 1e-5 of an fp32 reference) —
// e.g. the toy 2-layer model of BASELINE configs[0] whose reference path is
// fp32.  One warp per (query token, q head); 32 keys per step, one per lane:
// lane l folds q . k_l over the 128 dims (q broadcast from shared memory),
// the warp runs the online softmax, and each lane accumulates 4 of the 128
// output dims (coalesced V rows).
constexpr int kF32Warps = 8;
__global__ void __launch_bounds__(32 * kF32Warps) k_continuation_attention_f32(
    const float* __restrict__ q, const float* __restrict__ k_pool, const float* __restrict__ v_pool,
    float* __restrict__ out, const int32_t* __restrict__ q_off, const int32_t* __restrict__ kv_len,
    const int32_t* __restrict__ table, int32_t n_seqs, int32_t max_blocks, int32_t n_q_heads, int32_t n_kv_heads,
    float scale) {
  __shared__ float4 qs[kF32Warps][32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row = blockIdx.x * static_cast<int64_t>(kF32Warps) + w;  // (token, head)
  const int64_t total = static_cast<int64_t>(q_off[n_seqs]) * n_q_heads;
  if (row >= total) return;
  const int64_t tok = row / n_q_heads;
  const int hq = static_cast<int>(row % n_q_heads), kvh = hq / (n_q_heads / n_kv_heads);
  int lo = 0, hi = n_seqs;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (q_off[mid] <= tok) lo = mid; else hi = mid;
  }
  const int sq = lo;
  const int q_len = q_off[sq + 1] - q_off[sq];
  const int n_keys = kv_len[sq] - q_len + static_cast<int>(tok - q_off[sq]) + 1;  // causal
  qs[w][lane] = reinterpret_cast<const float4*>(q + row * 128)[lane];
  __syncwarp();
  const int32_t* trow = table + static_cast<int64_t>(sq) * max_blocks;
  float m = -INFINITY, l = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int k0 = 0; k0 < n_keys; k0 += 32) {
    const int key = k0 + lane;
    float sc = -INFINITY;
    if (key < n_keys) {
      const int64_t page = trow[key / 16];
      const float4* kr = reinterpret_cast<const float4*>(k_pool + ((page * n_kv_heads + kvh) * 16 + key % 16) * 128);
      float d = 0.f;
#pragma unroll 8
      for (int c = 0; c < 32; ++c) {
        const float4 kv = kr[c], qv = qs[w][c];
        d = fmaf(qv.x, kv.x, fmaf(qv.y, kv.y, fmaf(qv.z, kv.z, fmaf(qv.w, kv.w, d))));
      }
      sc = d * scale;
    }
    float mx = sc;
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float m_new = fmaxf(m, mx);
    const float corr = expf(m - m_new);  // 0 on the first step
    const float pr = key < n_keys ? expf(sc - m_new) : 0.f;
    float ps = pr;
#pragma unroll
    for (int o = 16; o; o >>= 1) ps += __shfl_xor_sync(0xffffffffu, ps, o);
    l = l * corr + ps;
    acc.x *= corr;
    acc.y *= corr;
    acc.z *= corr;
    acc.w *= corr;
    const int n_here = min(32, n_keys - k0);
    for (int i = 0; i < n_here; ++i) {
      const float pi = __shfl_sync(0xffffffffu, pr, i);
      const int ki = k0 + i;
      const int64_t page = trow[ki / 16];
      const float4 vv =
          reinterpret_cast<const float4*>(v_pool + ((page * n_kv_heads + kvh) * 16 + ki % 16) * 128)[lane];
      acc.x = fmaf(pi, vv.x, acc.x);
      acc.y = fmaf(pi, vv.y, acc.y);
      acc.z = fmaf(pi, vv.z, acc.z);
      acc.w = fmaf(pi, vv.w, acc.w);
    }
    m = m_new;
  }
  const float inv = 1.f / l;
  reinterpret_cast<float4*>(out + row * 128)[lane] = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
}

// KV append: write the suffix K/V rows into their pool pages.
__global__ void k_kv_append(const __nv_bfloat16* __restrict__ k_new, const __nv_bfloat16* __restrict__ v_new,
                            __nv_bfloat16* __restrict__ k_pool, __nv_bfloat16* __restrict__ v_pool,
                            const int32_t* __restrict__ q_off, const int32_t* __restrict__ kv_len,
                            const int32_t* __restrict__ table, int32_t n_seqs, int32_t max_blocks, int32_t n_kv_heads,
                            int32_t page) {
  // one thread per (token, kv head, 16-byte chunk): 16 chunks per 128-dim row
  const int64_t total_tok = q_off[n_seqs];
  const int64_t n = total_tok * n_kv_heads * 16;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int chunk = static_cast<int>(i & 15);
    const int64_t th = i >> 4;
    const int kvh = static_cast<int>(th % n_kv_heads);
    const int64_t tok = th / n_kv_heads;
    int lo = 0, hi = n_seqs;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (q_off[mid] <= tok) lo = mid; else hi = mid;
    }
    const int s = lo;
    const int64_t pos = kv_len[s] - (q_off[s + 1] - q_off[s]) + (tok - q_off[s]);
    const int64_t blk = table[static_cast<int64_t>(s) * max_blocks + pos / page];
    if (blk < 0) continue;  // sequence without pages (its insert failed)
    const int64_t dst = ((blk * n_kv_heads + kvh) * page + pos % page) * 128 + chunk * 8;
    const int64_t src = (tok * n_kv_heads + kvh) * 128 + chunk * 8;
    *reinterpret_cast<uint4*>(k_pool + dst) = __ldg(reinterpret_cast<const uint4*>(k_new + src));
    *reinterpret_cast<uint4*>(v_pool + dst) = __ldg(reinterpret_cast<const uint4*>(v_new + src));
  }
}

}  // namespace attn
}  // namespace sb

using namespace sb;

extern "C" int sb_continuation_attention(const void* q, const void* k_pool, const void* v_pool, void* out,
                                         const int32_t* d_q_offsets, const int32_t* d_kv_lens,
                                         const int32_t* d_block_table, int32_t n_seqs, int32_t max_blocks_per_seq,
                                         int32_t max_q_len, int32_t total_q, int32_t n_q_heads, int32_t n_kv_heads,
                                         int32_t head_dim,
                                         int32_t page_size, int64_t n_pool_blocks, float softmax_scale,
                                         const int32_t* d_work, int32_t n_work, void* stream) {
  return guard([&] {
    if (head_dim != 128 || page_size != 16) throw Error(SB_ERR_UNSUPPORTED, "head_dim must be 128 and page_size 16");
    if (n_kv_heads <= 0 || n_q_heads % n_kv_heads) throw Error(SB_ERR_INVALID, "n_q_heads % n_kv_heads != 0");
    const int group = n_q_heads / n_kv_heads;
    if (group > 128 || 128 % group) throw Error(SB_ERR_UNSUPPORTED, "GQA group must divide 128");
    if (n_seqs <= 0 || max_q_len <= 0) return int(SB_OK);
    const int64_t kv_rows = n_pool_blocks * n_kv_heads * page_size;
    if (kv_rows + 16 >= (int64_t(1) << 31)) throw Error(SB_ERR_UNSUPPORTED, "KV pool too large for 32-bit TMA rows");
    const int tpt = 128 / group;
    if (total_q <= 0) return int(SB_OK);
    uint64_t qdims[3] = {128, static_cast<uint64_t>(n_q_heads), static_cast<uint64_t>(total_q)};
    uint64_t qstr[2] = {128 * 2, static_cast<uint64_t>(n_q_heads) * 128 * 2};
    uint32_t qbox[3] = {64, static_cast<uint32_t>(group), static_cast<uint32_t>(tpt)};
    CUtensorMap tm_q = make_tmap_bf16(q, 3, qdims, qstr, qbox);
    uint64_t kdims[2] = {128, static_cast<uint64_t>(kv_rows)};
    uint64_t kstr[1] = {128 * 2};
    uint32_t kbox[2] = {64, 16};
    CUtensorMap tm_k = make_tmap_bf16(k_pool, 2, kdims, kstr, kbox);
    CUtensorMap tm_v = make_tmap_bf16(v_pool, 2, kdims, kstr, kbox);
    attn::Params prm;
    prm.q_off = d_q_offsets;
    prm.kv_len = d_kv_lens;
    prm.table = d_block_table;
    prm.out = static_cast<__nv_bfloat16*>(out);
    prm.n_seqs = n_seqs;
    prm.max_blocks = max_blocks_per_seq;
    prm.n_q_heads = n_q_heads;
    prm.n_kv_heads = n_kv_heads;
    prm.group = group;
    prm.tpt = tpt;
    prm.pairs_per_seq = (max_q_len + 2 * tpt - 1) / (2 * tpt);
    prm.oob_row = static_cast<int32_t>(kv_rows);
    prm.scale_log2 = softmax_scale * 1.4426950408889634f;
    prm.work = d_work;
    // the attribute is per device context: set once per device, thread-safe
    static std::once_flag attr_once[64];
    int dev = 0;
    SB_CUDA(cudaGetDevice(&dev));
    cudaError_t attr_err = cudaSuccess;
    std::call_once(attr_once[dev & 63], [&] {
      attr_err = cudaFuncSetAttribute(attn::k_continuation_attention, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      attn::kSmemBytes);
    });
    SB_CUDA(attr_err);
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (attn::pair_mode()) {  // work items are quads of query tiles, two CTAs each
      const int64_t quads = (prm.pairs_per_seq + 1) / 2;
      const int64_t items = d_work ? static_cast<int64_t>(n_work) : static_cast<int64_t>(n_seqs) * n_kv_heads * quads;
      if (items <= 0) return int(SB_OK);
      auto kern = attn::pairk::k_continuation_attention_pair<2, true>;
      static std::once_flag pair_once[64];
      std::call_once(pair_once[dev & 63], [&] {
        attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, attn::pairk::kSmemBytes);
      });
      SB_CUDA(attr_err);
      kern<<<static_cast<unsigned>(2 * items), attn::kThreads, attn::pairk::kSmemBytes, st>>>(tm_q, tm_k, tm_v, prm);
      SB_CHECK_LAUNCH();
      return int(SB_OK);
    }
    const int64_t grid = d_work ? static_cast<int64_t>(n_work) : static_cast<int64_t>(n_seqs) * n_kv_heads * prm.pairs_per_seq;
    if (grid <= 0) return int(SB_OK);
    attn::k_continuation_attention<<<static_cast<unsigned>(grid), attn::kThreads, attn::kSmemBytes, st>>>(
        tm_q, tm_k, tm_v, prm);
    SB_CHECK_LAUNCH();
    return int(SB_OK);
  });
}

extern "C" int sb_continuation_attention_f32(const float* q, const float* k_pool, const float* v_pool, float* out,
                                             const int32_t* d_q_offsets, const int32_t* d_kv_lens,
                                             const int32_t* d_block_table, int32_t n_seqs, int32_t max_blocks_per_seq,
                                             int32_t total_q, int32_t n_q_heads, int32_t n_kv_heads, int32_t head_dim,
                                             int32_t page_size, float softmax_scale, void* stream) {
  return guard([&] {
    if (head_dim != 128 || page_size != 16) throw Error(SB_ERR_UNSUPPORTED, "head_dim must be 128 and page_size 16");
    if (n_kv_heads <= 0 || n_q_heads % n_kv_heads) throw Error(SB_ERR_INVALID, "n_q_heads % n_kv_heads != 0");
    if (n_seqs <= 0 || total_q <= 0) return int(SB_OK);
    const int64_t rows = static_cast<int64_t>(total_q) * n_q_heads;
    attn::k_continuation_attention_f32<<<static_cast<unsigned>((rows + attn::kF32Warps - 1) / attn::kF32Warps),
                                         32 * attn::kF32Warps, 0, static_cast<cudaStream_t>(stream)>>>(
        q, k_pool, v_pool, out, d_q_offsets, d_kv_lens, d_block_table, n_seqs, max_blocks_per_seq, n_q_heads,
        n_kv_heads, softmax_scale);
    SB_CHECK_LAUNCH();
    return int(SB_OK);
  });
}

extern "C" int sb_attention_work_list(const int32_t* h_q_offsets, const int32_t* h_kv_lens, int32_t n_seqs,
                                      int32_t n_q_heads, int32_t n_kv_heads, int32_t* out, int32_t cap, int32_t* n_out) {
  return guard([&] {
    if (n_kv_heads <= 0 || n_q_heads % n_kv_heads) throw Error(SB_ERR_INVALID, "n_q_heads % n_kv_heads != 0");
    // pair mode: one item per quad of query tiles (CTA pair), else per pair of tiles
    const int tpt = (128 / (n_q_heads / n_kv_heads)) * (attn::pair_mode() ? 2 : 1);
    // LPT over (sequence, kv head) groups, each group's tiles adjacent so the
    // CTAs running together share the group's K/V pages in L2; inside a
    // group the longest tiles (largest causal key range) go first.
    struct It { int64_t group_work, work; int32_t seq, kvh, pair; };
    std::vector<It> items;
    for (int s = 0; s < n_seqs; ++s) {
      const int q_len = h_q_offsets[s + 1] - h_q_offsets[s];
      const int prefix = h_kv_lens[s] - q_len;
      int64_t gw = 0;
      for (int pr = 0; pr * 2 * tpt < q_len; ++pr) gw += prefix + std::min(q_len, (pr + 1) * 2 * tpt);
      for (int h = 0; h < n_kv_heads; ++h)
        for (int pr = 0; pr * 2 * tpt < q_len; ++pr) {
          const int64_t kv_limit = prefix + std::min(q_len, (pr + 1) * 2 * tpt);
          items.push_back({gw, kv_limit, s, h, pr});
        }
    }
    std::stable_sort(items.begin(), items.end(), [](const It& a, const It& b) {
      if (a.group_work != b.group_work) return a.group_work > b.group_work;
      if (a.seq != b.seq) return a.seq < b.seq;
      if (a.kvh != b.kvh) return a.kvh < b.kvh;
      return a.work > b.work;
    });
    if (static_cast<int64_t>(items.size()) > cap) throw Error(SB_ERR_INVALID, "work list capacity too small");
    for (size_t i = 0; i < items.size(); ++i) {
      out[2 * i] = items[i].seq;
      out[2 * i + 1] = (items[i].kvh << 16) | items[i].pair;
    }
    *n_out = static_cast<int32_t>(items.size());
    return int(SB_OK);
  });
}

extern "C" int sb_kv_append(const void* k_new, const void* v_new, void* k_pool, void* v_pool,
                            const int32_t* d_q_offsets, const int32_t* d_kv_lens, const int32_t* d_block_table,
                            int32_t n_seqs, int32_t max_blocks_per_seq, int32_t n_kv_heads, int32_t head_dim,
                            int32_t page_size, void* stream) {
  return guard([&] {
    if (head_dim != 128) throw Error(SB_ERR_UNSUPPORTED, "head_dim must be 128");
    if (n_seqs <= 0) return int(SB_OK);
    attn::k_kv_append<<<148 * 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const __nv_bfloat16*>(k_new), static_cast<const __nv_bfloat16*>(v_new),
        static_cast<__nv_bfloat16*>(k_pool), static_cast<__nv_bfloat16*>(v_pool), d_q_offsets, d_kv_lens,
        d_block_table, n_seqs, max_blocks_per_seq, n_kv_heads, page_size);
    SB_CHECK_LAUNCH();
    return int(SB_OK);
  });
}
