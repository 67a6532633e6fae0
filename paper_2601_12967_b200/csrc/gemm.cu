// gemm.cu — the dense projections of the continuation prefill (configs[2]:
// QKV, O, gate/up, down, LM head) as one hand-written sm_100a GEMM:
//   Y[rows, n] (op)= X[rows, k] · W[n, k]^T      (bf16 in, fp32 accumulate)
// X and W are row-major (nn.Linear layout), i.e. both operands K-major.
//
// Two persistent kernels: k_gemm_pair (CTA pairs, 256 x 256 tiles; every
// launch with more than 128 rows, see the pair section below) and k_gemm
// (1 CTA, 128 x 256 tiles; few rows, e.g. the LM head over the last tokens).
// Both are warp-specialised, one 192-thread CTA per SM:
//   warp 4      TMA producer: 128x64 X tile + 256x64 W tile per stage
//               (SWIZZLE_128B, 4-stage ring, mbarrier transaction counts)
//   warp 5      one elected lane issues tcgen05.mma (M=128, N=256, K=16; four
//               per stage) into a TMEM accumulator; two accumulators of 256
//               fp32 columns (all 512 TMEM columns) so the epilogue of tile i
//               overlaps the main loop of tile i+1
//   warps 0-3   epilogue: tcgen05.ld (one TMEM lane = one output row per
//               thread), the fused op, 16 B stores
// Epilogue ops (the elementwise kernels they replace):
//   kStoreBf16  Y = acc                       (QKV)
//   kAddBf16    Y = Y + acc                   (O / down projection + residual)
//   kStoreF32   Y = acc in fp32               (LM head logits)
//   kSwiGLU     Y[:, j] = silu(acc_gate[:, j]) * acc_up[:, j]; W holds the
//               gate rows [0, n) then the up rows [n, 2n) (the [gate | up]
//               layout of model.cu); a 256-wide tile loads gate rows
//               [128t, 128t+128) and up rows [n+128t, ...) into the two halves
//               of its W stage, so one tile yields 128 output features.
// Out-of-range rows / columns / k are zero-filled by TMA and masked in the
// epilogue, so rows, n and k need only be multiples of 8 (16 B rows).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "common.h"
#include "gemm.h"
#include "sm100.cuh"
#include "tma_host.h"

namespace sb {
namespace gemm {

constexpr int kBM = 128, kBN = 256, kBK = 64;
constexpr int kStages = 4;
constexpr uint32_t kABytes = kBM * kBK * 2;  // 16 KB
constexpr uint32_t kBBytes = kBN * kBK * 2;  // 32 KB
constexpr uint32_t kStageBytes = kABytes + kBBytes;
constexpr int kThreads = 192;
constexpr int kSmemBytes = kStages * kStageBytes + 1024;

struct Smem {
  uint64_t full[kStages];
  uint64_t empty[kStages];
  uint64_t acc_full[2];
  uint64_t acc_empty[2];
  uint32_t tmem_base;
};

struct Params {
  void* y;
  int64_t rows, n, k;  // n = output columns (SwiGLU: output features)
  int64_t ldy;         // elements per output row
  int mode;
  int m_tiles, n_tiles, k_blocks;
};

// Tile order: bands of kGroupM row tiles, n fastest inside a band, so one
// wave of 148 CTAs covers ~16 row tiles x ~9 column tiles (~34 MB of unique
// X + W at K = 4096) instead of every row tile of X against 2-3 W tiles, and
// a band's X stays in L2 while the band's column tiles are swept.
constexpr int kGroupM = 16;
__device__ __forceinline__ void tile_coords(const Params& p, int t, int& mt, int& nt) {
  const int band = t / (kGroupM * p.n_tiles);
  const int first = band * kGroupM;
  const int rows_in_band = min(kGroupM, p.m_tiles - first);
  const int r = t - band * kGroupM * p.n_tiles;
  mt = first + r % rows_in_band;
  nt = r / rows_in_band;
}

__device__ __forceinline__ float silu_mul(float g, float u) { return g / (1.f + __expf(-g)) * u; }

// One output tile from TMEM: this thread's row `row` (one TMEM lane), the
// tile's 256 accumulator columns at tbase; column tile nt (SwiGLU: 128
// output features, gate in columns [0, 128), up in [128, 256)).
__device__ __forceinline__ void epilogue_tile(const Params& p, uint32_t tbase, int64_t row, int nt) {
  const bool row_ok = row < p.rows;
  const bool swiglu = p.mode == kSwiGLU;
  if (swiglu) {
    __nv_bfloat16* y = static_cast<__nv_bfloat16*>(p.y) + row * p.ldy;
#pragma unroll 1
    for (int c = 0; c < 4; ++c) {
      uint32_t gv[32], uv[32];
      tmem_ld32(tbase + c * 32, gv);
      tmem_ld32(tbase + 128 + c * 32, uv);
      tmem_wait_ld();
      const int64_t col0 = static_cast<int64_t>(nt) * 128 + c * 32;
      if (row_ok) {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          if (col0 + v * 8 >= p.n) break;
          uint4 o;
          uint32_t* ow = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int i = v * 8 + 2 * e;
            ow[e] = pack_bf16x2(silu_mul(__uint_as_float(gv[i]), __uint_as_float(uv[i])),
                                silu_mul(__uint_as_float(gv[i + 1]), __uint_as_float(uv[i + 1])));
          }
          *reinterpret_cast<uint4*>(y + col0 + v * 8) = o;
        }
      }
    }
  } else {
#pragma unroll 1
    for (int c = 0; c < kBN / 32; ++c) {
      uint32_t v32[32];
      tmem_ld32(tbase + c * 32, v32);
      tmem_wait_ld();
      const int64_t col0 = static_cast<int64_t>(nt) * kBN + c * 32;
      if (!row_ok || col0 >= p.n) continue;
      if (p.mode == kStoreF32) {
        float* y = static_cast<float*>(p.y) + row * p.ldy + col0;
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          if (col0 + v * 4 >= p.n) break;
          *reinterpret_cast<uint4*>(y + v * 4) = make_uint4(v32[4 * v], v32[4 * v + 1], v32[4 * v + 2], v32[4 * v + 3]);
        }
      } else {
        __nv_bfloat16* y = static_cast<__nv_bfloat16*>(p.y) + row * p.ldy + col0;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          if (col0 + v * 8 >= p.n) break;
          float f[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(v32[v * 8 + e]);
          if (p.mode == kAddBf16) {
            const uint4 old = *reinterpret_cast<const uint4*>(y + v * 8);
            const __nv_bfloat162* oh = reinterpret_cast<const __nv_bfloat162*>(&old);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 r = __bfloat1622float2(oh[e]);
              f[2 * e] += r.x;
              f[2 * e + 1] += r.y;
            }
          }
          uint4 o;
          o.x = pack_bf16x2(f[0], f[1]);
          o.y = pack_bf16x2(f[2], f[3]);
          o.z = pack_bf16x2(f[4], f[5]);
          o.w = pack_bf16x2(f[6], f[7]);
          *reinterpret_cast<uint4*>(y + v * 8) = o;
        }
      }
    }
  }}

__global__ void __launch_bounds__(kThreads, 1)
    k_gemm(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ Smem ss;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int n_tiles_total = p.m_tiles * p.n_tiles;

  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&ss.full[i], 1);
      mbar_init(&ss.empty[i], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&ss.acc_full[a], 1);
      mbar_init(&ss.acc_empty[a], 4);
    }
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc<512>(&ss.tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = ss.tmem_base;
  const bool swiglu = p.mode == kSwiGLU;

  if (warp == 4) {
    // ============================ TMA producer ============================
    if (elect_one()) {
      tma_prefetch_desc(&tm_x);
      tma_prefetch_desc(&tm_w);
      uint32_t g = 0;
      for (int t = blockIdx.x; t < n_tiles_total; t += gridDim.x) {
        int mt, nt;
        tile_coords(p, t, mt, nt);
        for (int kb = 0; kb < p.k_blocks; ++kb, ++g) {
          const int s = g % kStages;
          mbar_wait_suspend(&ss.empty[s], ((g / kStages) & 1) ^ 1);
          uint8_t* sa = base + s * kStageBytes;
          uint8_t* sb_ = sa + kABytes;
          mbar_arrive_expect_tx(&ss.full[s], kStageBytes);
          tma_load_2d(sa, &tm_x, &ss.full[s], kb * kBK, mt * kBM);
          if (swiglu) {
            tma_load_2d(sb_, &tm_w, &ss.full[s], kb * kBK, nt * 128);
            tma_load_2d(sb_ + kBBytes / 2, &tm_w, &ss.full[s], kb * kBK, static_cast<int>(p.n) + nt * 128);
          } else {
            tma_load_2d(sb_, &tm_w, &ss.full[s], kb * kBK, nt * kBN);
          }
        }
      }
    }
  } else if (warp == 5) {
    // ============================ MMA issuer ==============================
    const uint32_t idesc = idesc_bf16_f32(kBM, kBN, 0, 0);
    const uint32_t s0 = smem_u32(base);
    uint32_t g = 0, it = 0;
    for (int t = blockIdx.x; t < n_tiles_total; t += gridDim.x, ++it) {
      const uint32_t a = it & 1;
      mbar_wait_suspend(&ss.acc_empty[a], ((it >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t d = tmem + a * kBN;
      for (int kb = 0; kb < p.k_blocks; ++kb, ++g) {
        const int s = g % kStages;
        mbar_wait_suspend(&ss.full[s], (g / kStages) & 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sa = s0 + s * kStageBytes, sbw = sa + kABytes;
#pragma unroll
          for (int kk = 0; kk < kBK / 16; ++kk)
            mma_ss(d, smem_desc_sw128(sa + kk * 32, 16, 1024), smem_desc_sw128(sbw + kk * 32, 16, 1024), idesc,
                   (kb > 0 || kk > 0) ? 1u : 0u);
          mma_commit(&ss.empty[s]);
          if (kb == p.k_blocks - 1) mma_commit(&ss.acc_full[a]);
        }
        __syncwarp();
      }
    }
  } else {
    // ============================== epilogue ==============================
    uint32_t it = 0;
    const int lane = tid & 31;
    for (int t = blockIdx.x; t < n_tiles_total; t += gridDim.x, ++it) {
      const uint32_t a = it & 1;
      int mt, nt;
      tile_coords(p, t, mt, nt);
      mbar_wait_suspend(&ss.acc_full[a], (it >> 1) & 1);
      tc_fence_after();
      const int64_t row = static_cast<int64_t>(mt) * kBM + warp * 32 + lane;
      const uint32_t tbase = tmem + a * kBN + (static_cast<uint32_t>(warp * 32) << 16);
      epilogue_tile(p, tbase, row, nt);
      // this warp's TMEM reads of accumulator a are complete: release it
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&ss.acc_empty[a]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}


// ---------------------------------------------------------------------------
// CTA-pair variant (cta_group::2): a cluster of two CTAs on one TPC computes a
// 256 x 256 tile with M=256 MMAs issued by the leader CTA only.  Each CTA
// stages its own 128 rows of X and one half of the 256 W rows (rank 0 the
// first 128 — SwiGLU: the gate rows — rank 1 the second 128 — the up rows);
// the pair's tensor cores read B from both CTAs' shared memory, so per
// FLOP each SM reads half the W bytes of the 1-CTA kernel (from L2 and from
// shared memory).  Both CTAs' TMA completions count on the leader's `full`
// barrier; the leader's MMA commits multicast to both CTAs' `empty` /
// `acc_full`; both CTAs' epilogue warps release an accumulator on the
// leader's `acc_empty` (8 arrivals).  Each CTA's TMEM holds its own 128 rows.
namespace pair {

constexpr int kStages = 6;
constexpr uint32_t kHalfBytes = 128 * kBK * 2;  // 16 KB: X rows or W rows of one CTA per stage
constexpr uint32_t kStageBytes = 2 * kHalfBytes;
constexpr int kSmemBytes = kStages * kStageBytes + 1024;
constexpr int kGroupM2 = 8;

struct Smem {
  uint64_t full[kStages];
  uint64_t empty[kStages];
  uint64_t acc_full[2];
  uint64_t acc_empty[2];
  uint32_t tmem_base;
};

__device__ __forceinline__ void tile_coords2(const Params& p, int t, int& mt, int& nt) {
  const int band = t / (kGroupM2 * p.n_tiles);
  const int first = band * kGroupM2;
  const int rows_in_band = min(kGroupM2, p.m_tiles - first);
  const int r = t - band * kGroupM2 * p.n_tiles;
  mt = first + r % rows_in_band;
  nt = r / rows_in_band;
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_gemm_pair(const __grid_constant__ CUtensorMap tm_x, const __grid_constant__ CUtensorMap tm_w, const Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ Smem ss;
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t rank = cluster_rank();
  const int cluster = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;
  const int n_tiles_total = p.m_tiles * p.n_tiles;

  if (tid == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&ss.full[i], 1);
      mbar_init(&ss.empty[i], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&ss.acc_full[a], 1);
      mbar_init(&ss.acc_empty[a], 8);
    }
    fence_barrier_init();
  }
  if (warp == 5) tmem_alloc2(&ss.tmem_base);
  tc_fence_before();
  cluster_sync();  // both CTAs' barriers initialised before any remote arrive / TMA completion
  tc_fence_after();
  const uint32_t tmem = ss.tmem_base;
  const bool swiglu = p.mode == kSwiGLU;

  if (warp == 4) {
    // ====================== TMA producer (both CTAs) ======================
    if (elect_one()) {
      tma_prefetch_desc(&tm_x);
      tma_prefetch_desc(&tm_w);
      uint32_t g = 0;
      for (int t = cluster; t < n_tiles_total; t += n_clusters) {
        int mt, nt;
        tile_coords2(p, t, mt, nt);
        const int xrow = mt * 256 + static_cast<int>(rank) * 128;
        const int wrow = swiglu ? (rank ? static_cast<int>(p.n) : 0) + nt * 128 : nt * 256 + static_cast<int>(rank) * 128;
        for (int kb = 0; kb < p.k_blocks; ++kb, ++g) {
          const int s = g % kStages;
          mbar_wait_suspend(&ss.empty[s], ((g / kStages) & 1) ^ 1);
          uint8_t* sa = base + s * kStageBytes;
          const uint32_t full0 = mapa(&ss.full[s], 0);
          if (rank == 0) mbar_arrive_expect_tx(&ss.full[s], 2 * kStageBytes);
          tma_load_2d_pair(sa, &tm_x, full0, kb * kBK, xrow);
          tma_load_2d_pair(sa + kHalfBytes, &tm_w, full0, kb * kBK, wrow);
        }
      }
    }
  } else if (warp == 5) {
    // ===================== MMA issuer (leader CTA only) ====================
    if (rank == 0) {
      const uint32_t idesc = idesc_bf16_f32(256, kBN, 0, 0);
      const uint32_t s0 = smem_u32(base);
      uint32_t g = 0, it = 0;
      for (int t = cluster; t < n_tiles_total; t += n_clusters, ++it) {
        const uint32_t a = it & 1;
        mbar_wait_suspend(&ss.acc_empty[a], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + a * kBN;
        for (int kb = 0; kb < p.k_blocks; ++kb, ++g) {
          const int s = g % kStages;
          mbar_wait_suspend(&ss.full[s], (g / kStages) & 1);
          tc_fence_after();
          if (elect_one()) {
            const uint32_t sa = s0 + s * kStageBytes, sbw = sa + kHalfBytes;
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk)
              mma_ss2(d, smem_desc_sw128(sa + kk * 32, 16, 1024), smem_desc_sw128(sbw + kk * 32, 16, 1024), idesc,
                      (kb > 0 || kk > 0) ? 1u : 0u);
            mma_commit2(&ss.empty[s]);
            if (kb == p.k_blocks - 1) mma_commit2(&ss.acc_full[a]);
          }
          __syncwarp();
        }
      }
    }
  } else {
    // ====================== epilogue (both CTAs) ======================
    uint32_t it = 0;
    const int lane = tid & 31;
    for (int t = cluster; t < n_tiles_total; t += n_clusters, ++it) {
      const uint32_t a = it & 1;
      int mt, nt;
      tile_coords2(p, t, mt, nt);
      mbar_wait_suspend(&ss.acc_full[a], (it >> 1) & 1);
      tc_fence_after();
      const int64_t row = static_cast<int64_t>(mt) * 256 + rank * 128 + warp * 32 + lane;
      const uint32_t tbase = tmem + a * kBN + (static_cast<uint32_t>(warp * 32) << 16);
      epilogue_tile(p, tbase, row, nt);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote_relaxed(mapa(&ss.acc_empty[a], 0));
    }
  }
  tc_fence_before();
  cluster_sync();  // both CTAs done with TMEM; no remote arrive in flight
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc2(tmem);
  }
}

}  // namespace pair
}  // namespace gemm

void gemm_bf16(const void* x, const void* w, void* y, int64_t rows, int64_t n, int64_t k, int mode,
               cudaStream_t stream) {
  if (rows <= 0 || n <= 0) return;
  if (k <= 0 || (k % 8) || (n % 8)) throw Error(SB_ERR_UNSUPPORTED, "gemm: k and n must be positive multiples of 8");
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(y)) & 15)
    throw Error(SB_ERR_UNSUPPORTED, "gemm: x, w and y must be 16-byte aligned (TMA / vector stores)");
  if (rows >= (int64_t(1) << 31) || n >= (int64_t(1) << 30) || k >= (int64_t(1) << 31))
    throw Error(SB_ERR_UNSUPPORTED, "gemm: dimensions exceed 32-bit TMA coordinates");
  const int64_t w_rows = mode == kSwiGLU ? 2 * n : n;
  uint64_t xdims[2] = {static_cast<uint64_t>(k), static_cast<uint64_t>(rows)};
  uint64_t wdims[2] = {static_cast<uint64_t>(k), static_cast<uint64_t>(w_rows)};
  uint64_t str[1] = {static_cast<uint64_t>(k) * 2};
  uint32_t xbox[2] = {gemm::kBK, gemm::kBM};
  uint32_t wbox[2] = {gemm::kBK, mode == kSwiGLU ? 128u : static_cast<uint32_t>(gemm::kBN)};
  CUtensorMap tm_x = make_tmap_bf16(x, 2, xdims, str, xbox);
  CUtensorMap tm_w = make_tmap_bf16(w, 2, wdims, str, wbox);
  gemm::Params p;
  p.y = y;
  p.rows = rows;
  p.n = n;
  p.k = k;
  p.ldy = n;
  p.mode = mode;
  p.m_tiles = static_cast<int>((rows + gemm::kBM - 1) / gemm::kBM);
  p.n_tiles = static_cast<int>(mode == kSwiGLU ? (n + 127) / 128 : (n + gemm::kBN - 1) / gemm::kBN);
  p.k_blocks = static_cast<int>((k + gemm::kBK - 1) / gemm::kBK);
  static std::once_flag attr_once[64];
  int dev = 0, sms = 148;
  SB_CUDA(cudaGetDevice(&dev));
  cudaError_t attr_err = cudaSuccess;
  std::call_once(attr_once[dev & 63], [&] {
    attr_err = cudaFuncSetAttribute(gemm::k_gemm, cudaFuncAttributeMaxDynamicSharedMemorySize, gemm::kSmemBytes);
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(gemm::pair::k_gemm_pair, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      gemm::pair::kSmemBytes);
  });
  SB_CUDA(attr_err);
  SB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // CTA pairs (M = 256 per tile) once there are rows for both CTAs; the
  // 1-CTA kernel for few rows (the LM head over the last tokens).
  // SB_GEMM_PAIR=0: always the 1-CTA kernel (A/B switch).
  static const bool pair_ok = [] {
    const char* e = std::getenv("SB_GEMM_PAIR");
    return !(e && e[0] == '0');
  }();
  if (pair_ok && rows > gemm::kBM) {
    const int64_t w_rows_box = 128;
    uint32_t wbox2[2] = {gemm::kBK, static_cast<uint32_t>(w_rows_box)};
    CUtensorMap tm_w2 = make_tmap_bf16(w, 2, wdims, str, wbox2);
    p.m_tiles = static_cast<int>((rows + 255) / 256);
    const int64_t tiles = static_cast<int64_t>(p.m_tiles) * p.n_tiles;
    const int64_t clusters = tiles < sms / 2 ? tiles : sms / 2;
    gemm::pair::k_gemm_pair<<<static_cast<unsigned>(2 * clusters), gemm::kThreads, gemm::pair::kSmemBytes, stream>>>(
        tm_x, tm_w2, p);
    SB_CHECK_LAUNCH();
    return;
  }
  const int64_t tiles = static_cast<int64_t>(p.m_tiles) * p.n_tiles;
  const unsigned grid = static_cast<unsigned>(tiles < sms ? tiles : sms);
  gemm::k_gemm<<<grid, gemm::kThreads, gemm::kSmemBytes, stream>>>(tm_x, tm_w, p);
  SB_CHECK_LAUNCH();
}

}  // namespace sb

extern "C" int sb_gemm_bf16(const void* x, const void* w, void* y, int64_t rows, int64_t n, int64_t k, int32_t mode,
                            void* stream) {
  return sb::guard([&] {
    if (mode < sb::kStoreBf16 || mode > sb::kSwiGLU) throw sb::Error(SB_ERR_INVALID, "gemm: unknown epilogue mode");
    sb::gemm_bf16(x, w, y, rows, n, k, mode, static_cast<cudaStream_t>(stream));
    return int(SB_OK);
  });
}
