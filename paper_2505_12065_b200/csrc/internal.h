// internal.h -- library-private declarations shared by the C-ABI translation units.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/sa.h"

struct sa_comm_group;   // in-process rank group (comm.cu)
struct sa_comm {
  void* nccl = nullptr;            // ncclComm_t (NCCL transport)
  sa_comm_group* group = nullptr;  // in-process transport (sa_comm_init_local)
  int32_t rank = 0, world = 1, device = 0;
  bool check_args = false;         // sa_comm_set_checks: cross-rank argument check
  bool collectives_at_one = false; // sa_comm_set_collectives: sharded path even at world 1
};
// the sharded code path (collectives + merge) applies to indexes built with this communicator
inline bool comm_sharded(const sa_comm* c) {
  return c != nullptr && (c->world > 1 || c->collectives_at_one);
}

// One captured search (sa_search_host fast path): H2D from a pinned staging buffer, the whole
// search, D2H into pinned staging -- replayed with a single cudaGraphLaunch.
struct sa_graph_entry {
  int64_t nq = 0;
  int32_t k = 0, nprobe = 0, qdtype = 0;
  cudaGraphExec_t exec = nullptr;
  void* h_q = nullptr;
  int64_t* h_ids = nullptr;
  float* h_sc = nullptr;
  void* d_q = nullptr;
  int64_t* d_ids = nullptr;
  float* d_sc = nullptr;
  void* small_scratch = nullptr;            // agent-step path: persistent kernel scratch,
  int32_t* h_done = nullptr;                // pinned completion flag the kernel stores,
  int32_t seq = 0;                          // and the number of replays so far
  int64_t launches[SA_KERNEL_KINDS] = {};   // per-kind kernel launches of one replay
  uint64_t last_use = 0;                    // LRU stamp (sa_index::use_clock)
};
// Bound on the captured-graph caches of one index (sa_search_host shapes, maturity plans):
// an agent loop whose batch size changes every step must not grow memory without limit.
constexpr size_t kMaxCapturedSearches = 32;

namespace sa {
struct MaturePlan;
void free_mature_plan(MaturePlan* p);
}  // namespace sa

struct sa_index {
  int device = 0;
  int num_sms = 148;
  int64_t n_local = 0;
  int32_t d = 0, d_pad = 0;
  int32_t nlist = 0;
  int64_t row_offset = 0, n_total = 0;
  int32_t list_world = 0, list_rank = 0;   // list sharding (sa_build_opts.list_shard_*)
  __nv_bfloat16* X = nullptr;  // [n_local, d_pad] (list-major when nlist > 0)
  CUtensorMap tmap_x;   // box 128 rows (cta_group 1)
  CUtensorMap tmap_x2;  // box 64 rows (cta_group 2: each CTA of a pair stages half a tile)
  CUtensorMap tmap_xt;  // box 32 rows (IVF list tails)
  int32_t* row_ids = nullptr;  // nlist > 0: stored row -> global id (fits 32 bits)
  // IVF coarse quantiser
  float* centroids = nullptr;                // [nlist, d_pad] fp32 (unit norm)
  __nv_bfloat16* centroids_bf16 = nullptr;   // [nlist, d_pad]
  CUtensorMap tmap_c;    // centroids, box 128 rows (cta_group 1)
  CUtensorMap tmap_c2;   // centroids, box 64 rows (cta_group 2)
  int64_t* list_off = nullptr;               // device [nlist + 1]
  std::vector<int64_t> h_list_off;           // host copy
  int64_t max_list = 0;
  const sa_comm* comm = nullptr;
  // captured small-batch searches (host-buffer path), guarded by graph_mu
  std::mutex graph_mu;
  std::vector<sa_graph_entry> graphs;
  uint64_t use_clock = 0;   // LRU clock of both caches
  // proximity graph (graph_api.cu): neighbour lists in stored positions [n_local, graph_R]
  int32_t graph_R = 0, graph_K = 0;
  int32_t* graph = nullptr;
  int32_t* graph_knn = nullptr;  // kept kNN lists [n_local, graph_K] (build flag bit 0)
  // e4m3 copy of the stored rows for the fp8 flat scan (fp8_api.cu; sa_index_build_fp8)
  uint8_t* X8 = nullptr;       // [n_local, d8_pad], stored order, scaled by 2^x8_exp
  int32_t d8_pad = 0;          // multiple of 128 (one 128-byte K-block)
  int32_t x8_exp = 0;
  CUtensorMap tmap_x8;         // as 16-bit pairs [n_local, d8_pad / 2], box 128 rows
  CUtensorMap tmap_x8_2;       // box 64 rows (cta_group 2)
  CUtensorMap tmap_x8t;        // box 32 rows (IVF list tails)
  // captured progressive (maturity-exit) searches, guarded by graph_mu (mature.cu)
  std::vector<std::unique_ptr<sa::MaturePlan, void (*)(sa::MaturePlan*)>> mature_plans;
};

namespace sa {

sa_status set_error(sa_status s, const std::string& msg);
// getenv for timing-experiment switches; always NULL unless built with -DSA_TUNING_BUILD
const char* tuning_env(const char* name);
sa_status cuda_status(cudaError_t e, const char* what);

// TMA descriptor for a row-major bf16 [rows, cols] matrix with box [box_rows, 64 cols], SW128.
sa_status make_tmap_bf16(CUtensorMap* m, const void* base, int64_t rows, int32_t cols,
                         int32_t box_rows);

// Collectives (comm.cu; NCCL or the in-process group): every rank r contributes bytes [off[r], off[r]+len[r]) of buf; all ranks end with all.
sa_status comm_broadcast_parts(const sa_comm* c, void* buf, const int64_t* off, const int64_t* len,
                               cudaStream_t s);
// all-gather of `bytes` per rank: recv holds world * bytes, rank-major
sa_status comm_allgather_bytes(const sa_comm* c, const void* send, void* recv, size_t bytes,
                               cudaStream_t s);
// Cross-rank argument check before a sharded call (sa_comm_set_checks; a no-op when off):
// every rank all-gathers its kCommArgs arguments and its local validation status; any failure
// or mismatch -> SA_ERR_INVALID_ARG on every rank (no rank left waiting in a collective).
constexpr int kCommArgs = 6;
sa_status comm_check_args(const sa_comm* c, const int64_t (&args)[kCommArgs], sa_status local,
                          cudaStream_t s);
// balanced contiguous split
inline void shard_range(int64_t n, int world, int rank, int64_t* off, int64_t* len) {
  const int64_t base = n / world, rem = n % world;
  *off = rank * base + (rank < rem ? rank : rem);
  *len = base + (rank < rem ? 1 : 0);
}

// Kernel accounting (sa_api.cu).  A region attributes every launch made while it is the
// calling thread's outermost open region (note_launch(), kernels/launch.cuh) to `kind`, and
// times itself with CUDA events on `s` when profiling is on.  Inner regions are absorbed.
class ProfRegion {
 public:
  ProfRegion(int kind, cudaStream_t s);
  ~ProfRegion();
  ProfRegion(const ProfRegion&) = delete;
  ProfRegion& operator=(const ProfRegion&) = delete;

 private:
  bool owner_;
  cudaStream_t s_;
  cudaEvent_t begin_ = nullptr;
};
// While a graph is captured no events are recorded and launches go to a per-kind tally
// (capture_tally); a replay adds the tally back with prof_add_launches.
void set_capturing(bool on);
void capture_tally(int64_t out[SA_KERNEL_KINDS]);
void prof_add_launches(const int64_t counts[SA_KERNEL_KINDS]);

// Query padding / kernel variant: cta_group 2 (M=256 pairs) when more than one
// 128-query block is searched, else cta_group 1.
inline int flat_cta_group(int64_t nq) { return nq > 128 ? 2 : 1; }
inline int64_t padded_nq(int64_t nq) {
  const int64_t m = 128 * flat_cta_group(nq);
  return (nq + m - 1) / m * m;
}

// Where a search writes its [nq, k] result: packed keys (for a cross-rank
// merge) or unpacked (id, score) pairs.
struct SearchOut {
  uint64_t* keys = nullptr;
  int64_t* ids = nullptr;
  float* scores = nullptr;
};

// A matrix scanned by the flat kernel: the index corpus, or the IVF centroids.
struct CorpusView {
  const CUtensorMap* tmap1;  // box 128 rows (cta_group 1)
  const CUtensorMap* tmap2;  // box 64 rows (cta_group 2)
  int64_t n_rows;
  int32_t d_pad;
  const int32_t* row_ids;    // stored row -> global id, or nullptr (id = id_base + row)
  uint32_t id_base;
  bool fp8 = false;          // e4m3 corpus and queries; d_pad counts 16-bit pairs (bytes / 2)
};

// a9 for sharded indexes: rank-local sorted [nq, k] keys -> ncclAllGather -> k-way merge
// into (out_ids, out_scores) (sa_api.cu)
sa_status gather_merge_keys(const sa_index* idx, const uint64_t* keys_local, int64_t nq, int32_t k,
                            int64_t* out_ids, float* out_scores, cudaStream_t s);

// exact scan of `cv` for nq staged queries (bf16 [>= nq, d_pad]) + intra-GPU merge (sa_api.cu)
// prepass: seed the shared pruning bound with the k-th best score of a sub-scan (exact: a lower
// bound of the final k-th score)
sa_status flat_search_view(const CorpusView& cv, int num_sms, const __nv_bfloat16* Qs, int64_t nq,
                           int32_t k, const SearchOut& out, cudaStream_t s, bool prepass = true);
// raw fp32 score matrix out[q, row] = <Q_q, X_row> for q < nq (tensor cores, no selection)
sa_status flat_scores_view(const CorpusView& cv, int num_sms, const __nv_bfloat16* Qs, int64_t nq,
                           float* out, cudaStream_t s);
sa_status flat_search(const sa_index* idx, const __nv_bfloat16* Qs, int64_t nq, int64_t nq_pad,
                      int32_t k, const SearchOut& out, cudaStream_t s);

template <typename T>
sa_status dalloc(T** p, size_t count, cudaStream_t s, const char* what) {
  *p = nullptr;
  if (count == 0) return SA_OK;
  return cuda_status(cudaMallocAsync(reinterpret_cast<void**>(p), count * sizeof(T), s), what);
}

// Stream-ordered scratch that is released (cudaFreeAsync on s) when the scope ends, on every
// return path.
struct StreamFreer {
  cudaStream_t s;
  std::vector<void*> ptrs;
  StreamFreer(const StreamFreer&) = delete;
  StreamFreer& operator=(const StreamFreer&) = delete;
  ~StreamFreer() {
    for (void* p : ptrs)
      if (p) cudaFreeAsync(p, s);
  }
  template <typename T>
  T* add(T* p) {
    ptrs.push_back(p);
    return p;
  }
  template <typename T>
  sa_status alloc(T** p, size_t count, const char* what) {
    sa_status st = dalloc(p, count, s, what);
    if (st == SA_OK) ptrs.push_back(*p);
    return st;
  }
};

#define SA_TRY(expr)                   \
  do {                                 \
    sa_status _st = (expr);            \
    if (_st != SA_OK) return _st;      \
  } while (0)
#define SA_CUDA(expr, what) SA_TRY(::sa::cuda_status((expr), (what)))

// IVF (ivf.cu)
sa_status ivf_build(sa_index* idx, const sa_build_opts& o, cudaStream_t s);
// Q8: optional staged e4m3 queries [nq, d8_pad] -> the list scan runs on the e4m3 copy and
// `out.keys` receive keys with STORED positions (for the bf16 re-rank, fp8_api.cu); the probe
// still uses the bf16 queries Qs
sa_status ivf_search(const sa_index* idx, const __nv_bfloat16* Qs, int64_t nq, int64_t nq_pad,
                     int32_t k, int32_t nprobe, const SearchOut& out, cudaStream_t s,
                     const uint8_t* Q8 = nullptr);
sa_status ivf_probe(const sa_index* idx, const __nv_bfloat16* Qs, int64_t nq, int64_t nq_pad,
                    int32_t nprobe, int32_t* out_lists, cudaStream_t s);
// Agent-step batches (nq <= 8, k <= 32, nprobe <= 256): the one-launch IVF search straight
// from the caller's bf16 / fp32 queries (kernels/ivf_small.cu)
bool ivf_small_applies(const sa_index* idx, int64_t nq, int32_t k, int32_t nprobe);
// scratch: nullptr = stream-ordered allocations per call, else a block from
// ivf_small_scratch_alloc for this (nq, k, nprobe) (sa_search_host's captured graphs), which
// may also pass done_host (pinned completion flag) and queries_host (pinned queries, read by
// the kernel; `queries` is then the device buffer it stages them in).
sa_status ivf_small_search(const sa_index* idx, const void* queries, bool q_f32, int64_t nq,
                           int32_t k, int32_t nprobe, const SearchOut& out, cudaStream_t s,
                           int64_t* debug_ns = nullptr, void* scratch = nullptr,
                           int32_t* done_host = nullptr, const void* queries_host = nullptr);
sa_status ivf_small_scratch_alloc(const sa_index* idx, int64_t nq, int32_t k, int32_t nprobe,
                                  void** scratch);

}  // namespace sa
