// mature.cuh -- device side of the non-stall maturity exit on IVF list order
// (§3.3, App. B.2).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

namespace sa {

// Device state of one progressive search (all buffers owned by the plan).
struct MatureArgs {
  int32_t nq, k, nprobe_max, g;  // g = lists per stage (checkpoint every g lists)
  double tau;                    // EMA threshold
  double alpha;                  // EMA weight 2 / (window + 1)
  const volatile int32_t* ready; // engine-ready flag (pinned host or device), nullptr = ready
  const int64_t* probes;         // [nq, nprobe_max] probe order, best first
  int64_t* stage_probes;         // [nq, g] lists of the current stage, -1 = none
  const int64_t* q_slot;         // [nq * g + 1] first output slot of (query, stage rank)
  const uint64_t* part;          // [slot][parts][k] partial lists of the stage's scan
  int32_t parts;                 // partial lists per slot
  uint64_t* R;                   // [nq, k] running result (sorted keys, 0 = empty)
  double* ema;                   // [nq]
  int32_t* active;               // [nq] 1 while the query is still searching
  int32_t* t_done;               // [nq] lists scanned when the query finished
  int32_t* ctrl;                 // [0] stage, [1] active queries, [2] ivf_scan item counter,
                                 // [3] update CTAs done
  double* trace_rq;              // optional [nq, nprobe_max] RQ_t (NaN when not scanned)
  double* trace_ema;             // optional [nq, nprobe_max] EMA_t
};

cudaError_t launch_mature_init(const MatureArgs& a, cudaStream_t s);
// merge the stage's partial lists into R list by list, RQ/EMA, exit decisions; the last CTA
// advances the stage and sets the WHILE condition h (0 = every query finished)
cudaError_t launch_mature_update(const MatureArgs& a, cudaGraphConditionalHandle h,
                                 cudaStream_t s);
// R -> out_ids int64 [nq, k] / out_scores fp32 [nq, k] (padded -1 / -inf), t_done -> out_t
cudaError_t launch_mature_final(const MatureArgs& a, int64_t* out_ids, float* out_scores,
                                int32_t* out_t, cudaStream_t s);

}  // namespace sa
