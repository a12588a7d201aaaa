// ivf_small.cuh -- one-launch IVF search for agent-step batches (ivf_small.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace sa {

constexpr int IVSM_MAX_NQ = 8;     // queries per launch (agent-step batches)
constexpr int IVSM_MAX_K = 32;
constexpr int IVSM_MAX_NPROBE = 256;
constexpr int IVSM_THREADS = 544;  // 16 scoring warps + 1 copy-issuing warp
constexpr int IVSM_MAX_LOCAL = 256;  // centroids per CTA: nlist <= 256 * grid
constexpr int IVSM_MAX_NLIST = 18176;  // probe candidates + selection in the smem ring
constexpr int IVSM_EXTRA = 7;      // keys published per CTA beyond the m of the probe threshold
constexpr int IVSM_MAX_STAGE = 64; // maturity path: nq * check_every entries per stage
constexpr int IVSM_MAX_G = 32;     // maturity path: check_every (one lane per list of a stage)

struct IvfSmallArgs {
  const void* Q;              // queries [nq, d] row-major, bf16 or fp32 (q_f32)
  int32_t q_f32;
  int32_t nq;                 // 1..IVSM_MAX_NQ
  int32_t d, d_pad;           // d_pad multiple of 64, <= 768
  const __nv_bfloat16* C;     // bf16 centroids [nlist, d_pad]
  int32_t nlist;              // <= min(IVSM_MAX_NLIST, IVSM_MAX_LOCAL * grid)
  int32_t nprobe;             // 1..min(nlist, IVSM_MAX_NPROBE)
  const __nv_bfloat16* X;     // list-major rows [n_local, d_pad]
  const int64_t* list_off;    // [nlist + 1]
  const int32_t* row_ids;     // stored row -> global id
  int32_t k;                  // 1..IVSM_MAX_K
  // scratch (no initialisation needed: the kernel zeroes what it counts with)
  uint64_t* top;              // [nq, grid, m + IVSM_EXTRA] per-CTA best centroid keys
  uint64_t* pcand;            // [nq, nlist] probe candidates
  int32_t* counters;          // [nq + 1]: candidates per query, CTAs done
  uint64_t* cand;             // [grid, nq, k] per-CTA top-k lists
  int64_t* debug_ns;          // optional [grid, 8] %globaltimer at the phase ends (tests)
  const void* Q_host;         // optional pinned host queries (layout of Q): CTA 0 reads them
  int32_t* q_ready;           // and stores them to Q (device), then *q_ready = *seq + 1
  int32_t* seq;               // optional completion signal: the last CTA increments *seq
  int32_t* done_host;         // (device memory) and stores it to *done_host (pinned host)
                              // after the results, so a host thread can spin on it
                              // (seq and q_ready live in persistent, zeroed scratch)
  uint64_t* out_keys;         // [nq, k] sorted packed keys, or
  int64_t* out_ids;           // [nq, k] ids (-1 padded) +
  float* out_scores;          // [nq, k] scores (-inf padded)
};

// Non-stall maturity exit in the same launch (§3.3; R14-R19): stages of g
// lists per active query; state in device memory, initialised by the kernel.
struct SmallMatureArgs {
  int32_t g = 0;              // lists per stage (exit test after each stage), nq * g <= 64
  double tau = 0, alpha = 0;  // EMA threshold, EMA weight 2 / (W + 1)
  const int32_t* ready = nullptr;   // engine-ready flag (host pinned or device), null = ready
  uint64_t* R = nullptr;      // [nq, k] running top-k keys
  double* ema = nullptr;      // [nq]
  int32_t* active = nullptr;  // [nq]
  int32_t* t_done = nullptr;  // [nq] lists scanned at the exit
  double* trace_rq = nullptr; // optional [nq, nprobe] (NaN past the exit)
  double* trace_ema = nullptr;
  int32_t* out_t = nullptr;   // optional [nq]: lists scanned, written at the end
  int64_t* stage_ns = nullptr;   // optional debug [64][4] %globaltimer per stage: CTA 0 start,
                                 // CTA 0 scan done, last CTA arrival, release
};

// Per-CTA best centroid keys that set the probe threshold: m * grid >= nprobe.
__host__ __device__ inline int ivf_small_m(int nprobe, int grid) { return (nprobe + grid - 1) / grid; }
// Whether the kernel's smem ring holds the probe step's working set for this shape.
bool ivf_small_fits(int nq, int nprobe, int nlist, int grid);
// Dynamic shared memory of one CTA.
size_t ivf_small_smem_bytes();
// Cooperative launch, grid = one CTA per SM.
cudaError_t launch_ivf_small(const IvfSmallArgs& a, int grid, cudaStream_t s);
// The same search with the maturity exit: nprobe = nprobe_max; a.cand holds
// [2][grid, nq * g, k] (stage parity); a.counters [nq + 3].
cudaError_t launch_ivf_small_mature(const IvfSmallArgs& a, const SmallMatureArgs& mo, int grid,
                                    cudaStream_t s);

}  // namespace sa
