// Streaming-read calibration on one B200 (not product code): how fast can a
// single pass read N bytes with (a) 16 B vector loads from many CTAs,
// (b) 1-D bulk copies (cp.async.bulk) into a staged shared-memory ring.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_probe stream_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void k_ldg(const int4* __restrict__ p, int64_t n16, unsigned* out) {
  unsigned acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
    int4 v = __ldg(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) *out = acc;
}

template <int U>
__global__ void k_ldg_u(const int4* __restrict__ p, int64_t n16, unsigned* out) {
  unsigned acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += U * stride) {
    int4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = i + u * stride < n16 ? __ldg(p + i + u * stride) : make_int4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  if (acc == 0x12345678u) *out = acc;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int STAGES>
__global__ void k_bulk(const uint8_t* __restrict__ p, int64_t nbytes, int chunk, unsigned* out) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar[STAGES];
  const int64_t per = (nbytes / gridDim.x) & ~int64_t(15);
  const uint8_t* src = p + blockIdx.x * per;
  const int64_t nch = per / chunk;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int64_t c) {
    uint64_t* b = &bar[c % STAGES];
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(chunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(sm + (c % STAGES) * chunk)),
                 "l"(src + c * chunk), "r"(chunk), "r"(smem_u32(b))
                 : "memory");
  };
  if (threadIdx.x == 0)
    for (int64_t c = 0; c < nch && c < STAGES; ++c) issue(c);
  unsigned acc = 0;
  for (int64_t c = 0; c < nch; ++c) {
    uint32_t ok = 0, par = (c / STAGES) & 1;
    while (!ok)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0,1,0,p;\n}"
                   : "=r"(ok) : "r"(smem_u32(&bar[c % STAGES])), "r"(par) : "memory");
    const int4* s4 = reinterpret_cast<const int4*>(sm + (c % STAGES) * chunk);
    for (int i = threadIdx.x; i < chunk / 16; i += blockDim.x) { int4 v = s4[i]; acc ^= v.x ^ v.w; }
    __syncthreads();
    if (threadIdx.x == 0 && c + STAGES < nch) issue(c + STAGES);
  }
  if (acc == 0x12345678u) *out = acc;
}

// random access: each group of G lanes reads one random aligned line of
// 16*G bytes (G = 2: 32 B sector, G = 8: 128 B line) from a region.
template <int G>
__global__ void k_rand(const int4* __restrict__ p, int64_t region16, int64_t n_reads, unsigned* out) {
  unsigned acc = 0;
  const int64_t gid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x);
  const int part = threadIdx.x % G;
  for (int64_t r = gid / G; r < n_reads; r += (int64_t)gridDim.x * blockDim.x / G) {
    uint64_t h = (uint64_t)r * 0x9e3779b97f4a7c15ull;
    h ^= h >> 29;
    const int64_t line = (int64_t)(h % (uint64_t)(region16 / G));
    int4 v = __ldg(p + line * G + part);
    acc ^= v.x ^ v.w;
  }
  if (acc == 0x12345678u) *out = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint8_t* buf;
  const int64_t maxb = int64_t(1) << 31;
  cudaMalloc(&buf, maxb);
  cudaMemset(buf, 1, maxb);
  uint8_t* fl;
  cudaMalloc(&fl, 256 << 20);
  unsigned* out;
  cudaMalloc(&out, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto f) {
    float best = 1e9;
    for (int r = 0; r < 7; ++r) {
      cudaMemset(fl, r, 256 << 20);  // flush L2
      cudaEventRecord(a);
      f();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (r > 1 && ms < best) best = ms;
    }
    return best;
  };
  for (int64_t nb : {int64_t(25) << 20, int64_t(100) << 20, int64_t(400) << 20, int64_t(1600) << 20}) {
    for (int per_sm : {4, 8, 16}) {
      float ms = timeit([&] { k_ldg<<<sms * per_sm, 256>>>((const int4*)buf, nb / 16, out); });
      printf("{\"kind\":\"ldg\",\"mb\":%lld,\"ctas_per_sm\":%d,\"us\":%.2f,\"gbs\":%.0f}\n", (long long)(nb >> 20), per_sm, ms * 1e3, nb / (ms * 1e-3) / 1e9);
    }
    {
      float ms = timeit([&] { k_ldg_u<4><<<sms * 8, 256>>>((const int4*)buf, nb / 16, out); });
      printf("{\"kind\":\"ldg_u4\",\"mb\":%lld,\"ctas_per_sm\":8,\"us\":%.2f,\"gbs\":%.0f}\n", (long long)(nb >> 20), ms * 1e3, nb / (ms * 1e-3) / 1e9);
    }
    for (int chunk : {16384, 32768}) {
      for (int ctas : {1, 2}) {
        const int stages = 4;
        const int smem = stages * chunk;
        if (smem * ctas > 220 * 1024) continue;
        cudaFuncSetAttribute(k_bulk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        float ms = timeit([&] { k_bulk<4><<<sms * ctas, 256, smem>>>(buf, nb, chunk, out); });
        printf("{\"kind\":\"bulk\",\"mb\":%lld,\"chunk\":%d,\"stages\":4,\"ctas_per_sm\":%d,\"us\":%.2f,\"gbs\":%.0f}\n", (long long)(nb >> 20), chunk, ctas, ms * 1e3, nb / (ms * 1e-3) / 1e9);
      }
    }
    {
      const int chunk = 8192, smem = 8 * chunk;
      cudaFuncSetAttribute(k_bulk<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      for (int ctas : {2, 3}) {
        float ms = timeit([&] { k_bulk<8><<<sms * ctas, 256, smem>>>(buf, nb, chunk, out); });
        printf("{\"kind\":\"bulk\",\"mb\":%lld,\"chunk\":%d,\"stages\":8,\"ctas_per_sm\":%d,\"us\":%.2f,\"gbs\":%.0f}\n", (long long)(nb >> 20), chunk, ctas, ms * 1e3, nb / (ms * 1e-3) / 1e9);
      }
    }
  }
  for (int64_t nb : {int64_t(100) << 20, int64_t(400) << 20}) {
    const int64_t region = int64_t(1) << 31;
    for (int per_sm : {8, 16}) {
      float ms = timeit([&] { k_rand<2><<<sms * per_sm, 256>>>((const int4*)buf, region / 16, nb / 32, out); });
      printf("{\"kind\":\"rand32\",\"mb\":%lld,\"ctas_per_sm\":%d,\"us\":%.2f,\"gbs\":%.0f}\n", (long long)(nb >> 20), per_sm, ms * 1e3, nb / (ms * 1e-3) / 1e9);
      ms = timeit([&] { k_rand<8><<<sms * per_sm, 256>>>((const int4*)buf, region / 16, nb / 128, out); });
      printf("{\"kind\":\"rand128\",\"mb\":%lld,\"ctas_per_sm\":%d,\"us\":%.2f,\"gbs\":%.0f}\n", (long long)(nb >> 20), per_sm, ms * 1e3, nb / (ms * 1e-3) / 1e9);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("{\"status\":\"%s\"}\n", cudaGetErrorString(e));
  return 0;
}
