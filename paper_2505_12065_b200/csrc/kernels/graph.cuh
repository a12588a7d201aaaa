// graph.cuh -- proximity-graph ANN kernels (R22-R27).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace sa {

constexpr int GR_MAX_K = 64;       // kNN list length (build)
constexpr int GR_MAX_R = 64;       // graph degree
constexpr int GR_MAX_L = 256;      // search list (search range)
constexpr int GR_MAX_NEW = 256;    // w * R per iteration
constexpr int GR_HASH_LOG = 13;
constexpr int GR_HASH = 1 << GR_HASH_LOG;  // visited-set slots per query (smem, 32 KB)
constexpr int GR_VISIT_CAP = GR_HASH * 3 / 4;  // visited nodes per query (load <= 3/4)

// kNN ids from the IVF search (global ids [nb, kk], best first, -1 padded) -> stored positions
// [nb, K] without the row itself (R22).  row p0 + b is row b of the batch.
cudaError_t launch_knn_to_pos(const int64_t* ids, int64_t nb, int kk, int64_t p0,
                              const int32_t* pos_of, int64_t row_offset, int K, int32_t* knn,
                              cudaStream_t s);
// pos_of[row_ids[p] - row_offset] = p
cudaError_t launch_inverse_ids(const int32_t* row_ids, int64_t n, int64_t row_offset,
                               int32_t* pos_of, cudaStream_t s);
// R23 + R24: detour counts, fwd [n, R]
cudaError_t launch_graph_prune(const int32_t* knn, int64_t n, int K, int R, int32_t* fwd,
                               cudaStream_t s);
// R25: the R smallest (p, global id of i) reverse keys of every node (rev [n, R] u64,
// pre-filled ~0)
cudaError_t launch_graph_reverse(const int32_t* fwd, int64_t n, int R, const int32_t* row_ids,
                                 uint64_t* rev, cudaStream_t s);
// R26: final lists [n, R] (stored positions; pos_of maps global id - row_offset -> position)
cudaError_t launch_graph_merge(const int32_t* fwd, const uint64_t* rev, int64_t n, int R,
                               const int32_t* pos_of, int64_t row_offset, int32_t* nbr,
                               cudaStream_t s);

struct GraphSearchArgs {
  const __nv_bfloat16* X;   // stored rows [n, d_pad]
  const int32_t* row_ids;   // stored row -> global id
  const int32_t* nbr;       // [n, R] stored positions, -1 padded
  const __nv_bfloat16* Q;   // staged queries [nq, d_pad]
  const uint64_t* entry_keys;  // [nq, E] probe keys (list id in the key, 0 = none)
  const int64_t* list_off;  // [nlist + 1]
  int32_t d_pad, R, L, w, E, T, k;
  int64_t* out_ids;         // [nq, k]
  float* out_scores;        // [nq, k]
  int32_t* out_expanded;    // optional [2, nq]: entries expanded, rows scored
  int32_t nq;
  // fp8 navigation (reading R34): rows scored on the e4m3 copy X8 [n, d8_pad] against the
  // staged e4m3 queries Q8 [nq, d8_pad]; the final list (L entries, keys with STORED
  // positions, 0-padded) goes to out_keys [nq, L] for the bf16 re-rank (fp8.cu)
  const uint8_t* X8;
  const uint8_t* Q8;
  int32_t d8_pad;
  uint64_t* out_keys;
  // L2 prefetch (bit 0: a row's bytes when it is first discovered, so the warps' register
  // gathers hit L2; bit 1: the neighbour list of a row scored above the list's floor, read
  // when it is expanded)
  int32_t prefetch;
  // tuning builds only (SA_GRAPH_DBG): per query [8] u64 -- globaltimer at start / end, clock64
  // cycles thread 0 spent in merge, pick, expand, score (each up to its closing barrier),
  // iterations, 0
  unsigned long long* dbg;
};
// non-stall maturity exit on the beam search (§3.3; readings R28-R29): a step is one
// iteration; RQ_t / EMA_t in fp64; after every g-th step the query stops if EMA_t >= tau and
// *ready != 0 (NULL = always ready).  A separate kernel argument, so the plain search's
// argument block (and its register allocation) is unchanged.
struct GraphMatureArgs {
  double tau, alpha;
  int32_t g, trace_cols;
  const int32_t* ready;
  int32_t* out_steps;       // optional [nq]: iterations run
  double* out_rq;           // optional [nq, trace_cols] (NaN past the exit)
  double* out_ema;
};
size_t graph_search_smem(int L);
// m == nullptr: plain beam search; fp8: navigation on the e4m3 copy (no maturity exit)
cudaError_t launch_graph_search(const GraphSearchArgs& a, const GraphMatureArgs* m, int64_t nq,
                                cudaStream_t s, bool fp8 = false);

}  // namespace sa
