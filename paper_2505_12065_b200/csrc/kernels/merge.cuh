// merge.cuh -- launcher interfaces for the merge and staging kernels.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace sa {

// Candidate j of group g for query q is cand[g*gstride + q*qstride + j], j < k.
// Alternative candidate layouts (checked in this order):
//   slot_off != nullptr: query q's candidates are cand[slot_off[q*slot_stride]*slot_keys,
//                        slot_off[(q+1)*slot_stride]*slot_keys)   (IVF: variable per query)
//   m_flat > 0:          cand[q*qstride + i], i < m_flat
struct MergeArgs {
  const uint64_t* cand;
  int32_t groups;
  int32_t k;
  int64_t qstride;
  int64_t gstride;
  const int64_t* slot_off = nullptr;
  int32_t slot_stride = 0;
  int32_t slot_keys = 0;
  int64_t m_flat = 0;
  const float* cand_scores = nullptr;  // with m_flat: candidate i = key(cand_scores[q*qstride+i], i)
  int64_t* out_ids;     // [nq, k] (when out_keys == nullptr)
  float* out_scores;    // [nq, k]
  uint64_t* out_keys;   // [nq, k] packed keys, sorted (for another merge level)
  int64_t id_offset;    // added to the 32-bit key id on unpack
};

cudaError_t launch_merge(const MergeArgs& a, int64_t nq, cudaStream_t stream);

cudaError_t launch_cast_pad(const void* src, bool src_f32, int64_t rows, int d, __nv_bfloat16* dst,
                            int64_t rows_pad, int d_pad, int num_sms, cudaStream_t stream);

}  // namespace sa
