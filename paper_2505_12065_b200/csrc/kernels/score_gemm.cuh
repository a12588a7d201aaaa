// score_gemm.cuh -- dense score dump on the tensor cores (score_gemm.cu; the IVF probe and the
// graph search's entry points).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace sa {

struct ScoreGemmArgs {
  int64_t nq;       // query rows (the query tensor map covers them; rows past nq are not written)
  int64_t n_rows;   // corpus rows (the corpus tensor map covers exactly these)
  int32_t d_pad;    // multiple of 64
  float* out;       // [nq, ldo] fp32 scores, out[q * ldo + r] = <Q[q], X[r]>
  int64_t ldo;      // >= n_rows
};

// true when d_pad suits the kernel (a multiple of 64)
bool score_gemm_applies(int d_pad);
// tmap_q: staged bf16 queries, box 128 rows x 64; tmap_x: bf16 corpus rows, box 128 rows x 64
// (the flat scan's cta_group-1 map), both SWIZZLE_128B.  One CTA per SM (<= num_sms).
cudaError_t launch_score_gemm(const CUtensorMap& tmap_q, const CUtensorMap& tmap_x,
                              const ScoreGemmArgs& a, int num_sms, cudaStream_t stream);

}  // namespace sa
