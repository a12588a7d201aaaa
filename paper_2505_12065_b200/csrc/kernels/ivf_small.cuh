// ivf_small.cuh -- one-launch IVF search for agent-step batches (ivf_small.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace sa {

constexpr int IVSM_MAX_NQ = 8;     // queries per launch (agent-step batches)
constexpr int IVSM_MAX_K = 32;
constexpr int IVSM_MAX_NPROBE = 256;
constexpr int IVSM_THREADS = 512;

struct IvfSmallArgs {
  const void* Q;              // queries [nq, d] row-major, bf16 or fp32 (q_f32)
  int32_t q_f32;
  int32_t nq;                 // 1..IVSM_MAX_NQ
  int32_t d, d_pad;           // d_pad multiple of 64, <= 768
  const __nv_bfloat16* C;     // bf16 centroids [nlist, d_pad]
  int32_t nlist;
  int32_t nprobe;             // 1..min(nlist, IVSM_MAX_NPROBE)
  const __nv_bfloat16* X;     // list-major rows [n_local, d_pad]
  const int64_t* list_off;    // [nlist + 1]
  const int32_t* row_ids;     // stored row -> global id
  int32_t k;                  // 1..IVSM_MAX_K
  float* psc;                 // scratch [nq, nlist]
  int32_t* probes;            // scratch [nq, nprobe] (the probe set, unordered)
  uint64_t* cand;             // scratch [grid, nq, k] per-CTA top-k lists
  uint64_t* out_keys;         // [nq, k] sorted packed keys, or
  int64_t* out_ids;           // [nq, k] ids (-1 padded) +
  float* out_scores;          // [nq, k] scores (-inf padded)
};

// Dynamic shared memory of one CTA.
size_t ivf_small_smem_bytes(int nlist, int grid, int k);
// Cooperative launch, grid = one CTA per SM.
cudaError_t launch_ivf_small(const IvfSmallArgs& a, int grid, cudaStream_t s);

}  // namespace sa
