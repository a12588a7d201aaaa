// fp8.cuh -- e4m3 corpus for the flat scan + bf16 re-rank (DESIGN.md §4.8,
// readings R30-R33).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace sa {

constexpr int F8_MAX_CAND = 256;  // re-ranked candidates per query

// out_bits (zeroed by the caller) = fp32 bits of max |X[r][c]| over rows [0, n), cols [0, d_pad)
cudaError_t launch_absmax_bf16(const __nv_bfloat16* X, int64_t n, int32_t d_pad,
                               uint32_t* out_bits, int num_sms, cudaStream_t s);

// R30/R31: X8[r][c] = e4m3_rne_satfinite(X[r][c] * 2^e) for c < d_pad, 0 for d_pad <= c < d8_pad,
// with e = the largest integer such that m * 2^e <= 448 (m = max |.|; m = 0 -> e = 0).
// absmax_bits != nullptr: one m for every row (the corpus, R30); nullptr: m = the row's own
// max (queries, R31).  exp_out (optional): e per row ([n]) or, with absmax_bits, one value.
cudaError_t launch_quant_e4m3(const __nv_bfloat16* X, int64_t n, int32_t d_pad,
                              const uint32_t* absmax_bits, uint8_t* X8, int32_t d8_pad,
                              int32_t* exp_out, int num_sms, cudaStream_t s);

// R32: re-rank.  For query q: every candidate key cand[q][0, n_cand) (id field = stored row
// position; key 0 = empty) is re-scored as the fp32 dot product of the bf16 rows Qs[q] and
// X[pos] and re-keyed with its global id (row_ids[pos], or row_offset + pos); the k best keys
// (score desc, id asc) go to out_keys [nq, k] or to (out_ids, out_scores) [nq, k], padded
// (0 / -1, -INF).
struct RerankArgs {
  const __nv_bfloat16* X;
  int32_t d_pad;
  const int32_t* row_ids;
  int64_t row_offset;
  const __nv_bfloat16* Qs;   // staged bf16 queries [nq, d_pad]
  const uint64_t* cand;      // [nq, n_cand]
  int32_t n_cand, k;
  uint64_t* out_keys;
  int64_t* out_ids;
  float* out_scores;
};
cudaError_t launch_rerank(const RerankArgs& a, int64_t nq, cudaStream_t s);

}  // namespace sa
