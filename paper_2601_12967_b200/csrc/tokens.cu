// tokens.cu — device-side synthetic token streams (the reference's
// materialize_tokens, src/trace.cpp:70-78, and decode_token, trace.cpp:80-83):
// each token is an independent splitmix64 of (section seed + position), so the
// kernel is a pure HBM write stream.
#include <cuda_runtime.h>

#include "common.h"
#include "hash.cuh"
#include <cuda_bf16.h>

namespace sb {

__global__ void k_materialize(uint64_t seed, int64_t first, int64_t n, uint64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = splitmix64(seed + static_cast<uint64_t>(first + i));
}

static int grid_of(int64_t n) {
  int64_t g = (n + 255) / 256;
  return static_cast<int>(g < 1 ? 1 : (g > 148 * 32 ? 148 * 32 : g));
}

}  // namespace sb

using namespace sb;

extern "C" int sb_materialize_tokens(int32_t section_tag, int64_t length, uint64_t content_key, int32_t src_iteration,
                                     uint64_t* d_out, void* stream) {
  return guard([&] {
    if (length <= 0) return int(SB_OK);
    k_materialize<<<grid_of(length), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        section_seed(section_tag, content_key, src_iteration), 0, length, d_out);
    SB_CHECK_LAUNCH();
    return int(SB_OK);
  });
}

extern "C" int sb_decode_tokens(uint64_t stream_key, int64_t first_index, int64_t count, uint64_t* d_out,
                                void* stream) {
  return guard([&] {
    if (count <= 0) return int(SB_OK);
    k_materialize<<<grid_of(count), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        splitmix64(stream_key ^ 0xdec0de0000000001ULL), first_index, count, d_out);
    SB_CHECK_LAUNCH();
    return int(SB_OK);
  });
}

namespace sb {

__global__ void k_build_table(const int32_t* __restrict__ ids, const int64_t* __restrict__ blk_off, int32_t n_seqs,
                              int32_t max_blocks, int32_t* __restrict__ table) {
  const int64_t n = static_cast<int64_t>(n_seqs) * max_blocks;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t s = i / max_blocks, j = i % max_blocks;
    const int64_t b0 = blk_off[s], nb = blk_off[s + 1] - b0;
    table[i] = j < nb ? ids[b0 + j] : -1;
  }
}

// counter-based bf16 noise: one splitmix64 per 4 elements
__global__ void k_fill_random_bf16(__nv_bfloat16* __restrict__ out, int64_t n, uint64_t seed, float amp) {
  const int64_t n4 = (n + 3) / 4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint64_t r = splitmix64(seed + static_cast<uint64_t>(i));
    float v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = (static_cast<float>((r >> (16 * k)) & 0xFFFF) * (1.f / 32768.f) - 1.f) * amp;
    if (4 * i + 3 < n) {
      __nv_bfloat162 a = __floats2bfloat162_rn(v[0], v[1]), b = __floats2bfloat162_rn(v[2], v[3]);
      uint2 w;
      w.x = *reinterpret_cast<uint32_t*>(&a);
      w.y = *reinterpret_cast<uint32_t*>(&b);
      *reinterpret_cast<uint2*>(out + 4 * i) = w;
    } else {
      for (int k = 0; k < 4 && 4 * i + k < n; ++k) out[4 * i + k] = __float2bfloat16(v[k]);
    }
  }
}

}  // namespace sb

extern "C" int sb_build_block_table(const int32_t* d_ids, const int64_t* d_block_offsets, int32_t n_seqs,
                                    int32_t max_blocks, int32_t* d_table, void* stream) {
  return guard([&] {
    if (n_seqs <= 0 || max_blocks <= 0) return int(SB_OK);
    const int64_t n = static_cast<int64_t>(n_seqs) * max_blocks;
    k_build_table<<<grid_of(n), 256, 0, static_cast<cudaStream_t>(stream)>>>(d_ids, d_block_offsets, n_seqs,
                                                                            max_blocks, d_table);
    SB_CHECK_LAUNCH();
    return int(SB_OK);
  });
}

extern "C" int sb_fill_random_bf16(void* d_out, int64_t n_elems, uint64_t seed, float amp, void* stream) {
  return guard([&] {
    if (n_elems <= 0) return int(SB_OK);
    k_fill_random_bf16<<<grid_of((n_elems + 3) / 4), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<__nv_bfloat16*>(d_out), n_elems, seed, amp);
    SB_CHECK_LAUNCH();
    return int(SB_OK);
  });
}
