// keys.cuh -- packed 64-bit (score, id) keys.
//
// Result order is (fp32 score descending, id ascending) with -0.0 == +0.0
// (readings R5).  A key is
//     key = (ordered(score) << 32) | (0xFFFFFFFF - id)
// where ordered() is the usual monotone bijection fp32 -> uint32, so "larger
// key" == "ranks earlier" and every (score, id) pair maps to a distinct key.
// key 0 is the empty slot (it would need score = -NaN, excluded by R7).
#pragma once
#include <cstdint>

namespace sa {

__host__ __device__ __forceinline__ uint32_t ordered_from_float(float s) {
  if (s == 0.0f) s = 0.0f;  // canonicalise -0.0
#ifdef __CUDA_ARCH__
  uint32_t u = __float_as_uint(s);
#else
  uint32_t u;
  __builtin_memcpy(&u, &s, 4);
#endif
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

__host__ __device__ __forceinline__ float float_from_ordered(uint32_t o) {
  uint32_t u = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
#ifdef __CUDA_ARCH__
  return __uint_as_float(u);
#else
  float f;
  __builtin_memcpy(&f, &u, 4);
  return f;
#endif
}

__host__ __device__ __forceinline__ uint64_t make_key(float s, uint32_t id) {
  return ((uint64_t)ordered_from_float(s) << 32) | (uint64_t)(0xFFFFFFFFu - id);
}
__host__ __device__ __forceinline__ float key_score(uint64_t key) {
  return float_from_ordered((uint32_t)(key >> 32));
}
__host__ __device__ __forceinline__ uint32_t key_id(uint64_t key) {
  return 0xFFFFFFFFu - (uint32_t)key;
}

}  // namespace sa
