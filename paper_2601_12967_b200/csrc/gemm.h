// gemm.h — the hand-written sm_100a GEMM of the dense projections (gemm.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace sb {

// epilogue ops; the values are the C-ABI `mode` of sb_gemm_bf16
enum GemmMode : int { kStoreBf16 = 0, kAddBf16 = 1, kStoreF32 = 2, kSwiGLU = 3 };

// Y[rows, n] (op)= X[rows, k] W[n, k]^T, row-major bf16 (kSwiGLU: W is
// [2n, k], gate rows then up rows, Y[rows, n] = silu(gate) * up).  Throws
// sb::Error on unsupported shapes.
void gemm_bf16(const void* x, const void* w, void* y, int64_t rows, int64_t n, int64_t k, int mode,
               cudaStream_t stream);

}  // namespace sb
