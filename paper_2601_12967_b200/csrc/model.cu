// model.cu — the dense layers around the continuation-prefill attention:
// a Llama-3-shaped decoder (random-init bf16 weights) so a continuation
// step is a real prefill of the tool-output tokens, not a stand-in.
//
// The reference models prefill compute with a cost (CostModel::chunk_ms,
// /root/reference/proj/src/engine.cpp:35-39); BASELINE configs[2] names the
// shape: Llama-3-8B (32 layers, d 4096, 32 q / 8 kv heads x 128, d_ff 14336,
// vocab 128256, rope theta 5e5).  Per layer, for the T suffix tokens of a
// batch (rows packed in batch order):
//   xn = rmsnorm(x) ; qkv = xn Wqkv^T                       (cuBLAS bf16, fp32 acc)
//   q = rope(q) -> [T, Hq, 128]; rope(k), v -> the layer's paged KV pool
//   a = continuation_attention(q, pages)                     (csrc/attention.cu)
//   x += a Wo^T ; xn = rmsnorm(x) ; gu = xn Wgu^T            (cuBLAS, residual as beta = 1)
//   h = silu(gate) * up ; x += h Wd^T
// then the last token of every sequence: logits = rmsnorm(x) Wlm^T, argmax
// = the first decoded token.  GEMMs are plain library GEMMs (cuBLAS); the
// elementwise work is fused into four small kernels here.
#include <cublas_v2.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

#include "common.h"
#include "gemm.h"
#include "hash.cuh"

namespace sb {
namespace model {

// one warp per row: y = x * rsqrt(mean(x^2) + eps) * w   (d % 256 == 0)
__global__ void k_rmsnorm(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ w,
                          __nv_bfloat16* __restrict__ y, int64_t rows, int d, float eps,
                          const int32_t* __restrict__ row_map) {
  const int64_t row = blockIdx.x * static_cast<int64_t>(blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int64_t src = row_map ? row_map[row] : row;
  const uint4* xr = reinterpret_cast<const uint4*>(x + src * d);
  float ss = 0.f;
  for (int c = lane; c < d / 8; c += 32) {
    const uint4 v = xr[c];
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __bfloat1622float2(h[k]);
      ss += f.x * f.x + f.y * f.y;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float inv = rsqrtf(ss / d + eps);
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  uint4* yr = reinterpret_cast<uint4*>(y + row * d);
  for (int c = lane; c < d / 8; c += 32) {
    const uint4 v = xr[c], g = wr[c];
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
    const __nv_bfloat162* gw = reinterpret_cast<const __nv_bfloat162*>(&g);
    uint4 o;
    __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __bfloat1622float2(h[k]), gg = __bfloat1622float2(gw[k]);
      oh[k] = __floats2bfloat162_rn(f.x * inv * gg.x, f.y * inv * gg.y);
    }
    yr[c] = o;
  }
}

// token embedding: row = token id mod vocab (token ids are the reference's
// 64-bit synthetic ids, trace.cpp:70-83)
__global__ void k_embed(const uint64_t* __restrict__ tok, const __nv_bfloat16* __restrict__ emb,
                        __nv_bfloat16* __restrict__ x, int64_t rows, int d, int64_t vocab) {
  const int64_t chunks = static_cast<int64_t>(d) / 8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < rows * chunks;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / chunks, c = i % chunks;
    const int64_t v = static_cast<int64_t>(tok[r] % static_cast<uint64_t>(vocab));
    reinterpret_cast<uint4*>(x + r * d)[c] = reinterpret_cast<const uint4*>(emb + v * d)[c];
  }
}

// RoPE (rotate-half form, HF Llama) of q and k from the fused qkv rows, q to
// a packed [T, Hq, 128] buffer (the attention's TMA layout), rotated k and v
// straight into the layer's KV pages at the token's absolute position.
// One thread per (token, head, 8-dim chunk of the first half); cos/sin of
// every (token, frequency) precomputed per batch: rope[t][i] = {cos, sin}.
__global__ void k_rope_scatter(const __nv_bfloat16* __restrict__ qkv, const float2* __restrict__ rope,
                               __nv_bfloat16* __restrict__ q_out, __nv_bfloat16* __restrict__ k_pool,
                               __nv_bfloat16* __restrict__ v_pool, const int32_t* __restrict__ q_off,
                               const int32_t* __restrict__ kv_len, const int32_t* __restrict__ table,
                               int32_t n_seqs, int32_t max_blocks, int32_t hq, int32_t hkv) {
  const int64_t total = q_off[n_seqs];
  const int heads = hq + 2 * hkv;
  const int64_t n = total * heads * 8;  // 8 chunks of 8 dims in the first half
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i & 7);
    const int h = static_cast<int>((i >> 3) % heads);
    const int64_t t = (i >> 3) / heads;
    const __nv_bfloat16* src = qkv + (t * heads + h) * 128;
    const uint4 a = reinterpret_cast<const uint4*>(src)[c];      // dims 8c .. 8c+7
    const uint4 b = reinterpret_cast<const uint4*>(src + 64)[c]; // dims 64+8c ..
    uint4 oa = a, ob = b;
    if (h < hq + hkv) {  // q or k: rotate
      const __nv_bfloat162* ah = reinterpret_cast<const __nv_bfloat162*>(&a);
      const __nv_bfloat162* bh = reinterpret_cast<const __nv_bfloat162*>(&b);
      __nv_bfloat162* oah = reinterpret_cast<__nv_bfloat162*>(&oa);
      __nv_bfloat162* obh = reinterpret_cast<__nv_bfloat162*>(&ob);
      const float2* cs = rope + t * 64 + 8 * c;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 x1 = __bfloat1622float2(ah[k]), x2 = __bfloat1622float2(bh[k]);
        const float2 c0 = cs[2 * k], c1 = cs[2 * k + 1];
        oah[k] = __floats2bfloat162_rn(x1.x * c0.x - x2.x * c0.y, x1.y * c1.x - x2.y * c1.y);
        obh[k] = __floats2bfloat162_rn(x2.x * c0.x + x1.x * c0.y, x2.y * c1.x + x1.y * c1.y);
      }
    }
    if (h < hq) {
      __nv_bfloat16* dst = q_out + (t * hq + h) * 128;
      reinterpret_cast<uint4*>(dst)[c] = oa;
      reinterpret_cast<uint4*>(dst + 64)[c] = ob;
      continue;
    }
    int lo = 0, hi = n_seqs;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (q_off[mid] <= t) lo = mid; else hi = mid;
    }
    const int64_t pos = kv_len[lo] - (q_off[lo + 1] - q_off[lo]) + (t - q_off[lo]);
    const int64_t blk = table[static_cast<int64_t>(lo) * max_blocks + pos / 16];
    if (blk < 0) continue;  // sequence without pages (its insert failed)
    const bool is_k = h < hq + hkv;
    const int kvh = is_k ? h - hq : h - hq - hkv;
    __nv_bfloat16* dst = (is_k ? k_pool : v_pool) + ((blk * hkv + kvh) * 16 + pos % 16) * 128;
    reinterpret_cast<uint4*>(dst)[c] = oa;
    reinterpret_cast<uint4*>(dst + 64)[c] = ob;
  }
}

// h = silu(gate) * up from gu = [gate | up] rows of 2 * dff
__global__ void k_swiglu(const __nv_bfloat16* __restrict__ gu, __nv_bfloat16* __restrict__ h, int64_t rows, int dff) {
  const int64_t chunks = dff / 8;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < rows * chunks;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / chunks, c = i % chunks;
    const uint4 g = reinterpret_cast<const uint4*>(gu + r * 2 * dff)[c];
    const uint4 u = reinterpret_cast<const uint4*>(gu + r * 2 * dff + dff)[c];
    const __nv_bfloat162* gh = reinterpret_cast<const __nv_bfloat162*>(&g);
    const __nv_bfloat162* uh = reinterpret_cast<const __nv_bfloat162*>(&u);
    uint4 o;
    __nv_bfloat162* oh = reinterpret_cast<__nv_bfloat162*>(&o);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 a = __bfloat1622float2(gh[k]), b = __bfloat1622float2(uh[k]);
      oh[k] = __floats2bfloat162_rn(a.x / (1.f + __expf(-a.x)) * b.x, a.y / (1.f + __expf(-a.y)) * b.y);
    }
    reinterpret_cast<uint4*>(h + r * dff)[c] = o;
  }
}

// argmax over each row of logits (first index on ties): one CTA per row
__global__ void k_argmax(const float* __restrict__ logits, int64_t vocab, int32_t* __restrict__ out) {
  __shared__ float bv[32];
  __shared__ int64_t bi[32];
  const float* row = logits + blockIdx.x * vocab;
  float best = -INFINITY;
  int64_t arg = 0;
  for (int64_t i = threadIdx.x; i < vocab; i += blockDim.x)
    if (row[i] > best) {
      best = row[i];
      arg = i;
    }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float v = __shfl_xor_sync(0xffffffffu, best, o);
    const int64_t j = __shfl_xor_sync(0xffffffffu, arg, o);
    if (v > best || (v == best && j < arg)) {
      best = v;
      arg = j;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    bv[threadIdx.x >> 5] = best;
    bi[threadIdx.x >> 5] = arg;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w)
      if (bv[w] > best || (bv[w] == best && bi[w] < arg)) {
        best = bv[w];
        arg = bi[w];
      }
    out[blockIdx.x] = static_cast<int32_t>(arg);
  }
}

__global__ void k_fill_const_bf16(__nv_bfloat16* p, int64_t n, float v) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] = __float2bfloat16(v);
}

}  // namespace model
}  // namespace sb

using namespace sb;

#define SB_BLAS(x)                                                                                  \
  do {                                                                                              \
    cublasStatus_t s_ = (x);                                                                        \
    if (s_ != CUBLAS_STATUS_SUCCESS) throw Error(SB_ERR_CUDA, std::string(#x) + ": cublas status " + \
                                                             std::to_string(static_cast<int>(s_))); \
  } while (0)

struct sb_model {
  int32_t n_layers = 0, d = 0, hq = 0, hkv = 0, dff = 0, device = 0;
  int64_t vocab = 0;
  float theta = 500000.f, eps = 1e-5f;
  struct Layer {
    __nv_bfloat16 *wqkv = nullptr, *wo = nullptr, *wgu = nullptr, *wd = nullptr, *n1 = nullptr, *n2 = nullptr;
  };
  std::vector<Layer> layers;
  __nv_bfloat16 *emb = nullptr, *lm_head = nullptr, *final_norm = nullptr;
  // A/B switch only (SB_GEMM_CUBLAS=1): the projections on cuBLAS instead of
  // the hand-written tcgen05 GEMM (gemm.cu), for the measured comparison
  bool use_cublas = false;
  cublasHandle_t blas = nullptr;
  ~sb_model() {
    cudaSetDevice(device);
    for (auto& l : layers)
      for (void* p : {l.wqkv, l.wo, l.wgu, l.wd, l.n1, l.n2})
        if (p) cudaFree(p);
    for (void* p : {static_cast<void*>(emb), static_cast<void*>(lm_head), static_cast<void*>(final_norm)})
      if (p) cudaFree(p);
    if (blas) cublasDestroy(blas);
  }
};

namespace {

__nv_bfloat16* alloc_random(int64_t n, uint64_t seed, float amp) {
  __nv_bfloat16* p = nullptr;
  SB_CUDA(cudaMalloc(&p, sizeof(__nv_bfloat16) * n));
  const int st = sb_fill_random_bf16(p, n, seed, amp, nullptr);
  if (st) throw Error(st, sb_last_error());
  return p;
}

__nv_bfloat16* alloc_const(int64_t n, float v) {
  __nv_bfloat16* p = nullptr;
  SB_CUDA(cudaMalloc(&p, sizeof(__nv_bfloat16) * n));
  model::k_fill_const_bf16<<<256, 256>>>(p, n, v);
  SB_CHECK_LAUNCH();
  return p;
}

int grid_n(int64_t n) { return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16))); }

// Y[rows, n] (+)= X[rows, k] W[n, k]^T, row-major bf16 (nn.Linear layout):
// the tcgen05 GEMM of gemm.cu with its fused epilogue (`mode`); cuBLAS only
// under the SB_GEMM_CUBLAS=1 A/B switch (kSwiGLU then writes [gate | up] to
// gu and k_swiglu follows, as before the fused epilogue)
void linear(sb_model* m, cudaStream_t st, const __nv_bfloat16* x, const __nv_bfloat16* w, void* y, int64_t rows,
            int64_t n, int64_t k, int mode) {
  if (!m->use_cublas) {
    gemm_bf16(x, w, y, rows, n, k, mode, st);
    return;
  }
  SB_BLAS(cublasSetStream(m->blas, st));
  const float alpha = 1.f, beta = mode == kAddBf16 ? 1.f : 0.f;
  const int64_t cols = mode == kSwiGLU ? 2 * n : n;
  SB_BLAS(cublasGemmEx(m->blas, CUBLAS_OP_T, CUBLAS_OP_N, static_cast<int>(cols), static_cast<int>(rows),
                       static_cast<int>(k), &alpha, w, CUDA_R_16BF, static_cast<int>(k), x, CUDA_R_16BF,
                       static_cast<int>(k), &beta, y, mode == kStoreF32 ? CUDA_R_32F : CUDA_R_16BF,
                       static_cast<int>(cols), CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT));
}

}  // namespace

extern "C" {

int sb_model_create(int32_t n_layers, int32_t d_model, int32_t n_q_heads, int32_t n_kv_heads, int32_t d_ff,
                    int64_t vocab, float rope_theta, uint64_t seed, int32_t device, sb_model** out) {
  return guard([&] {
    if (n_layers < 1 || n_q_heads < 1 || n_kv_heads < 1 || n_q_heads % n_kv_heads || d_model != n_q_heads * 128 ||
        d_model % 256 || d_ff % 8 || vocab < 1)
      throw Error(SB_ERR_INVALID, "model shape: d_model = 128 * n_q_heads, multiple of 256; d_ff % 8 == 0");
    SB_CUDA(cudaSetDevice(device));
    auto* m = new sb_model();
    try {
      m->n_layers = n_layers;
      m->d = d_model;
      m->hq = n_q_heads;
      m->hkv = n_kv_heads;
      m->dff = d_ff;
      m->vocab = vocab;
      m->theta = rope_theta;
      m->device = device;
      const int64_t d = d_model, qkv = static_cast<int64_t>(n_q_heads + 2 * n_kv_heads) * 128;
      // random-init weights, uniform with std ~0.02 (HF initializer_range)
      const float amp = 0.02f * 1.7320508f;
      uint64_t s = seed * 0x9e3779b97f4a7c15ull + 17;
      m->emb = alloc_random(vocab * d, s++, amp);
      m->lm_head = alloc_random(vocab * d, s++, amp);
      m->final_norm = alloc_const(d, 1.f);
      for (int l = 0; l < n_layers; ++l) {
        sb_model::Layer L;
        L.wqkv = alloc_random(qkv * d, s++, amp);
        L.wo = alloc_random(d * d, s++, amp);
        L.wgu = alloc_random(2 * static_cast<int64_t>(d_ff) * d, s++, amp);
        L.wd = alloc_random(d * d_ff, s++, amp);
        L.n1 = alloc_const(d, 1.f);
        L.n2 = alloc_const(d, 1.f);
        m->layers.push_back(L);
      }
      const char* ab = std::getenv("SB_GEMM_CUBLAS");
      m->use_cublas = ab && ab[0] == '1';
      if (m->use_cublas) SB_BLAS(cublasCreate(&m->blas));
      SB_CUDA(cudaDeviceSynchronize());
    } catch (...) {
      delete m;
      throw;
    }
    *out = m;
    return int(SB_OK);
  });
}

void sb_model_destroy(sb_model* m) { delete m; }

void sb_model_shape(const sb_model* m, int32_t* n_layers, int32_t* n_q_heads, int32_t* n_kv_heads) {
  *n_layers = m->n_layers;
  *n_q_heads = m->hq;
  *n_kv_heads = m->hkv;
}
void sb_model_vocab(const sb_model* m, int64_t* vocab) { *vocab = m->vocab; }

int sb_model_weight(sb_model* m, int32_t layer, int32_t which, void** ptr, int64_t* n_elems) {
  return guard([&] {
    const int64_t d = m->d, qkv = static_cast<int64_t>(m->hq + 2 * m->hkv) * 128;
    if (layer < 0) {
      if (which == 0) { *ptr = m->emb; *n_elems = m->vocab * d; }
      else if (which == 1) { *ptr = m->lm_head; *n_elems = m->vocab * d; }
      else if (which == 2) { *ptr = m->final_norm; *n_elems = d; }
      else throw Error(SB_ERR_INVALID, "weight selector");
      return int(SB_OK);
    }
    if (layer >= m->n_layers) throw Error(SB_ERR_INVALID, "layer");
    const auto& L = m->layers[layer];
    switch (which) {
      case 0: *ptr = L.wqkv; *n_elems = qkv * d; break;
      case 1: *ptr = L.wo; *n_elems = d * d; break;
      case 2: *ptr = L.wgu; *n_elems = 2 * static_cast<int64_t>(m->dff) * d; break;
      case 3: *ptr = L.wd; *n_elems = d * m->dff; break;
      case 4: *ptr = L.n1; *n_elems = d; break;
      case 5: *ptr = L.n2; *n_elems = d; break;
      default: throw Error(SB_ERR_INVALID, "weight selector");
    }
    return int(SB_OK);
  });
}

}  // extern "C"

// ---------------------------------------------------------------- forward
// Used by the continuation engine (engine.cu); the attention call is passed
// in so the engine keeps its work list / timing around it.
namespace sb {

struct ModelWorkspace {
  int64_t rows = 0;
  __nv_bfloat16 *x = nullptr, *xn = nullptr, *qkv = nullptr, *q = nullptr, *a = nullptr, *gu = nullptr, *h = nullptr;
  float2* rope = nullptr;
  int32_t* last_rows = nullptr;
  __nv_bfloat16* xl = nullptr;
  float* logits = nullptr;
  int32_t* next_tok = nullptr;
  int32_t n_seqs = 0;
  void release() {
    for (void* p : {static_cast<void*>(x), static_cast<void*>(xn), static_cast<void*>(qkv), static_cast<void*>(q),
                    static_cast<void*>(a), static_cast<void*>(gu), static_cast<void*>(h), static_cast<void*>(rope),
                    static_cast<void*>(last_rows), static_cast<void*>(xl), static_cast<void*>(logits),
                    static_cast<void*>(next_tok)})
      if (p) cudaFree(p);
    *this = ModelWorkspace{};
  }
};

ModelWorkspace* model_workspace_create(sb_model* m, const std::vector<int64_t>& prefix_len,
                                       const std::vector<int64_t>& suffix_len) {
  auto* w = new ModelWorkspace();
  try {
    int64_t T = 0;
    for (auto s : suffix_len) T += s;
    w->rows = T;
    w->n_seqs = static_cast<int32_t>(suffix_len.size());
    const int64_t d = m->d, qkv = static_cast<int64_t>(m->hq + 2 * m->hkv) * 128;
    auto al = [](auto*& p, int64_t n) { SB_CUDA(cudaMalloc(&p, sizeof(*p) * std::max<int64_t>(n, 1))); };
    al(w->x, T * d);
    al(w->xn, T * d);
    al(w->qkv, T * qkv);
    al(w->q, T * m->hq * 128);
    al(w->a, T * d);
    al(w->gu, T * 2 * m->dff);
    al(w->h, T * m->dff);
    al(w->rope, T * 64);
    al(w->last_rows, w->n_seqs);
    al(w->xl, static_cast<int64_t>(w->n_seqs) * d);
    al(w->logits, static_cast<int64_t>(w->n_seqs) * m->vocab);
    al(w->next_tok, w->n_seqs);
    // cos/sin of every (suffix token, frequency): absolute position = prefix + i
    std::vector<float2> cs(static_cast<size_t>(T) * 64);
    std::vector<int32_t> last(suffix_len.size());
    int64_t r = 0;
    for (size_t s = 0; s < suffix_len.size(); ++s) {
      for (int64_t i = 0; i < suffix_len[s]; ++i, ++r) {
        const double pos = static_cast<double>(prefix_len[s] + i);
        for (int f = 0; f < 64; ++f) {
          const double ang = pos * std::pow(static_cast<double>(m->theta), -2.0 * f / 128.0);
          cs[r * 64 + f] = make_float2(static_cast<float>(std::cos(ang)), static_cast<float>(std::sin(ang)));
        }
      }
      last[s] = static_cast<int32_t>(r - 1);
    }
    SB_CUDA(cudaMemcpy(w->rope, cs.data(), sizeof(float2) * cs.size(), cudaMemcpyHostToDevice));
    SB_CUDA(cudaMemcpy(w->last_rows, last.data(), sizeof(int32_t) * last.size(), cudaMemcpyHostToDevice));
  } catch (...) {
    w->release();
    delete w;
    throw;
  }
  return w;
}

struct ModelIO {
  __nv_bfloat16 *q, *a;
  float* logits;
  int32_t* next_tok;
};
ModelIO model_io(ModelWorkspace* w) { return ModelIO{w->q, w->a, w->logits, w->next_tok}; }

void model_workspace_destroy(ModelWorkspace* w) {
  if (w) {
    w->release();
    delete w;
  }
}

// Embedding of the step's suffix tokens (packed in batch order).
void model_embed(sb_model* m, ModelWorkspace* w, const uint64_t* d_suffix, cudaStream_t st) {
  model::k_embed<<<grid_n(w->rows * m->d / 8), 256, 0, st>>>(d_suffix, m->emb, w->x, w->rows, m->d, m->vocab);
  SB_CHECK_LAUNCH();
}

// Layer l up to the attention input: rmsnorm, QKV GEMM, RoPE + KV scatter.
void model_layer_pre(sb_model* m, ModelWorkspace* w, int l, void* k_pool, void* v_pool, const int32_t* q_off,
                     const int32_t* kv_len, const int32_t* table, int32_t n_seqs, int32_t max_blocks,
                     cudaStream_t st) {
  const auto& L = m->layers[l];
  const int64_t T = w->rows, d = m->d, qkv = static_cast<int64_t>(m->hq + 2 * m->hkv) * 128;
  model::k_rmsnorm<<<static_cast<unsigned>((T + 7) / 8), 256, 0, st>>>(w->x, L.n1, w->xn, T, m->d, m->eps, nullptr);
  linear(m, st, w->xn, L.wqkv, w->qkv, T, qkv, d, kStoreBf16);
  model::k_rope_scatter<<<grid_n(T * (m->hq + 2 * m->hkv) * 8), 256, 0, st>>>(
      w->qkv, w->rope, w->q, static_cast<__nv_bfloat16*>(k_pool), static_cast<__nv_bfloat16*>(v_pool), q_off, kv_len,
      table, n_seqs, max_blocks, m->hq, m->hkv);
  SB_CHECK_LAUNCH();
}

// Layer l after the attention (output in w->a): O projection + residual, MLP.
void model_layer_post(sb_model* m, ModelWorkspace* w, int l, cudaStream_t st) {
  const auto& L = m->layers[l];
  const int64_t T = w->rows, d = m->d;
  linear(m, st, w->a, L.wo, w->x, T, d, d, kAddBf16);
  model::k_rmsnorm<<<static_cast<unsigned>((T + 7) / 8), 256, 0, st>>>(w->x, L.n2, w->xn, T, m->d, m->eps, nullptr);
  if (m->use_cublas) {
    linear(m, st, w->xn, L.wgu, w->gu, T, m->dff, d, kSwiGLU);
    model::k_swiglu<<<grid_n(T * m->dff / 8), 256, 0, st>>>(w->gu, w->h, T, m->dff);
    SB_CHECK_LAUNCH();
  } else {
    linear(m, st, w->xn, L.wgu, w->h, T, m->dff, d, kSwiGLU);  // gate/up GEMM + SwiGLU in one kernel
  }
  linear(m, st, w->h, L.wd, w->x, T, d, m->dff, kAddBf16);
}

// Final norm of every sequence's last token, LM head (fp32 logits), argmax.
void model_head(sb_model* m, ModelWorkspace* w, cudaStream_t st) {
  model::k_rmsnorm<<<static_cast<unsigned>((w->n_seqs + 7) / 8), 256, 0, st>>>(w->x, m->final_norm, w->xl, w->n_seqs,
                                                                              m->d, m->eps, w->last_rows);
  linear(m, st, w->xl, m->lm_head, w->logits, w->n_seqs, m->vocab, m->d, kStoreF32);
  model::k_argmax<<<w->n_seqs, 256, 0, st>>>(w->logits, m->vocab, w->next_tok);
  SB_CHECK_LAUNCH();
}

double model_flops(const sb_model* m, int64_t rows) {
  const double d = m->d, qkv = (m->hq + 2.0 * m->hkv) * 128, ff = m->dff;
  return 2.0 * rows * m->n_layers * (d * qkv + d * d + 2 * d * ff + ff * d);
}

}  // namespace sb
