// probe_umma.cu — hardware check of the UMMA layouts the attention kernel uses:
//   S = Q K^T   (tcgen05.mma SS, both operands K-major SWIZZLE_128B via TMA)
//   P = bf16(S) written to TMEM with tcgen05.st
//   O = P V     (tcgen05.mma TS: A from TMEM, B = V MN-major SWIZZLE_128B)
// Built by tests/test_umma_probe.py into tests/cuda/_build/libprobe_umma.so.
#include <cuda.h>
#include <cuda_runtime.h>

#include "../../paper_2601_12967_b200/csrc/sm100.cuh"
#include "../../paper_2601_12967_b200/csrc/tma_host.h"

using namespace sb;

__global__ void __launch_bounds__(128, 1)
    probe_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                 const __grid_constant__ CUtensorMap tv, float* s_out, float* o_out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sq = smem;                // 2 atoms x 16 KB
  uint8_t* sk = smem + 32768;        // 2 atoms x 16 KB
  uint8_t* sv = smem + 65536;        // 2 atoms x 16 KB
  __shared__ uint64_t bar_load, bar_mma;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;

  if (tid == 0) {
    mbar_init(&bar_load, 1);
    mbar_init(&bar_mma, 1);
    fence_barrier_init();
  }
  if (warp == 0) tmem_alloc<512>(&tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tmem_base;

  if (tid == 0) {
    mbar_arrive_expect_tx(&bar_load, 3 * 32768);
    for (int a = 0; a < 2; ++a) {
      tma_load_2d(sq + a * 16384, &tq, &bar_load, a * 64, 0);
      tma_load_2d(sk + a * 16384, &tk, &bar_load, a * 64, 0);
      tma_load_2d(sv + a * 16384, &tv, &bar_load, a * 64, 0);
    }
  }
  mbar_wait(&bar_load, 0);

  const uint32_t idesc_s = idesc_bf16_f32(128, 128, 0, 0);
  const uint32_t idesc_o = idesc_bf16_f32(128, 128, 0, 1);
  if (tid == 0) {
    tc_fence_after();
    for (int kk = 0; kk < 8; ++kk) {
      uint32_t off = (kk / 4) * 16384 + (kk % 4) * 32;
      uint64_t ad = smem_desc_sw128(smem_u32(sq) + off, 16, 1024);
      uint64_t bd = smem_desc_sw128(smem_u32(sk) + off, 16, 1024);
      mma_ss(tb + 0, ad, bd, idesc_s, kk > 0);
    }
    mma_commit(&bar_mma);
  }
  mbar_wait(&bar_mma, 0);
  tc_fence_after();

  // each thread owns one row (TMEM lane) of S
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  uint32_t pk[64];
  for (int c = 0; c < 4; ++c) {
    uint32_t v[32];
    tmem_ld32(tb + lane_base + c * 32, v);
    tmem_wait_ld();
    for (int j = 0; j < 32; ++j) s_out[tid * 128 + c * 32 + j] = __uint_as_float(v[j]);
    for (int j = 0; j < 16; ++j) pk[c * 16 + j] = pack_bf16x2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
  }
  for (int c = 0; c < 4; ++c) {
    uint32_t w[16];
    for (int j = 0; j < 16; ++j) w[j] = pk[c * 16 + j];
    tmem_st16(tb + lane_base + 128 + c * 16, w);
  }
  tmem_wait_st();
  tc_fence_before();
  __syncthreads();
  if (tid == 0) {
    tc_fence_after();
    for (int kk = 0; kk < 8; ++kk) {
      uint64_t bd = smem_desc_sw128(smem_u32(sv) + kk * 2048, 16384, 1024);
      mma_ts(tb + 256, tb + 128 + kk * 8, bd, idesc_o, kk > 0);
    }
    mma_commit(&bar_mma);
  }
  mbar_wait(&bar_mma, 1);
  tc_fence_after();
  for (int c = 0; c < 4; ++c) {
    uint32_t v[32];
    tmem_ld32(tb + lane_base + 256 + c * 32, v);
    tmem_wait_ld();
    for (int j = 0; j < 32; ++j) o_out[tid * 128 + c * 32 + j] = __uint_as_float(v[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tb);
}

extern "C" int probe_umma(const void* q, const void* k, const void* v, float* s_out, float* o_out) {
  try {
    uint64_t dims[2] = {128, 128};
    uint64_t strides[1] = {128 * 2};
    uint32_t box[2] = {64, 128};
    CUtensorMap tq = make_tmap_bf16(q, 2, dims, strides, box);
    CUtensorMap tk = make_tmap_bf16(k, 2, dims, strides, box);
    CUtensorMap tv = make_tmap_bf16(v, 2, dims, strides, box);
    size_t smem = 3 * 32768 + 1024;
    cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    probe_kernel<<<1, 128, smem>>>(tq, tk, tv, s_out, o_out);
    cudaError_t e = cudaDeviceSynchronize();
    return e == cudaSuccess ? 0 : (int)e;
  } catch (...) {
    return -1;
  }
}
