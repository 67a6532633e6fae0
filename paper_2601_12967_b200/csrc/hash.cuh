// hash.cuh — the reference's token/block hashing, restated for host and device.
//   splitmix64 / hash_combine   include/agentsim/common.hpp:136-145
//   kv_root_hash / kv_chain_hash src/kv_cache.cpp:35-41
//   materialize_tokens           src/trace.cpp:50-78
//   decode_token                 src/trace.cpp:80-83
#pragma once
#include <cstdint>

#ifndef SB_HD
#define SB_HD __host__ __device__ __forceinline__
#endif

namespace sb {

constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;
constexpr uint64_t kRootHash = 0x6b76726f6f740001ULL;

SB_HD uint64_t splitmix64(uint64_t x) {
  x += kGolden;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

// One chain step.  `vk` = token + kGolden is independent of the chain and is
// computed ahead of the dependent path.
SB_HD uint64_t chain_step(uint64_t h, uint64_t vk) { return splitmix64(h ^ (vk + (h << 6) + (h >> 2))); }

SB_HD uint64_t hash_combine(uint64_t seed, uint64_t value) { return chain_step(seed, value + kGolden); }

SB_HD uint64_t section_salt(int tag) {
  return tag == 0 ? 0x53595354454d5052ULL
                  : tag == 1 ? 0x555345525155455aULL
                             : tag == 2 ? 0x544f4f4c4f555450ULL : tag == 3 ? 0x48495354f52590aaULL : 0ULL;
}

SB_HD uint64_t section_seed(int tag, uint64_t key, int32_t src_iter) {
  uint64_t seed = splitmix64(key ^ section_salt(tag));
  if (tag == 2) seed = hash_combine(seed, static_cast<uint64_t>(static_cast<int64_t>(src_iter)));
  return seed;
}

SB_HD uint64_t decode_token(uint64_t stream_key, int64_t index) {
  return splitmix64(splitmix64(stream_key ^ 0xdec0de0000000001ULL) + static_cast<uint64_t>(index));
}

// Eviction tier of a tag (kv_cache.cpp:23-33).
SB_HD int tier_of(int tag) {
  return tag == 0 ? 0 : tag == 1 ? 1 : (tag == 2 || tag == 5) ? 2 : tag == 3 ? 3 : tag == 4 ? 4 : 0;
}

}  // namespace sb
