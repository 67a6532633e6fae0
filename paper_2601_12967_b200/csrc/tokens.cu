// tokens.cu — device-side synthetic token streams (the reference's
// materialize_tokens, src/trace.cpp:70-78, and decode_token, trace.cpp:80-83):
// each token is an independent splitmix64 of (section seed + position), so the
// kernel is a pure HBM write stream.
#include <cuda_runtime.h>

#include "common.h"
#include "hash.cuh"

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
