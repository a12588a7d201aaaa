/*
 * sa.h -- C ABI of the B200-native retrieval library (libsa.so).
 *
 * The operation is the retrieval step SearchAgent-X interleaves with LLM
 * reasoning (§3.1: "the system checks for special tags
 * that trigger the Retriever"; Alg. 1 LaunchAsyncRetrievalTask):
 * top-k search of query embeddings against a dense passage-embedding
 * knowledge base (§2.1: queries "encoded into dense vector
 * representations"; top-k documents concatenated into the context, P:44,
 * P:216).  Similarity is the inner product (maximum inner-product
 * search, BASELINE.json north_star; reading R1).  Modes:
 *   - exact flat scan ("exact nearest neighbor (ENN) search");
 *   - IVF approximate search whose nprobe knob plays the role of the HNSW
 *     "search range": more effort, higher recall;
 *   - proximity-graph beam search (the paper's own ANN family, HNSW-like; its
 *     search range is the paper's knob), optionally with the non-stall
 *     maturity exit of §3.3 (sa_search_graph*, below);
 *   - fp8 (e4m3) flat scan with bf16 re-rank (a compressed exact mode;
 *     sa_search_fp8, below).
 * Plus the agent-side support of Alg. 1: the maturity exit on IVF list order
 * (sa_search_mature), the priority scheduler (sa_priority_order) and an
 * asynchronous retrieval executor (sa_retriever_*).
 *
 * Conventions (all entry points):
 *   - Every call returns sa_status; nothing else crosses the boundary.  On
 *     error, sa_last_error() returns a thread-local message.
 *   - Argument validation is synchronous and side-effect free: an invalid
 *     call returns SA_ERR_INVALID_ARG (or SA_ERR_STATE) and leaves every
 *     output untouched.
 *   - "DEVICE" pointers are CUDA global-memory pointers on the index's
 *     device; "HOST" pointers are ordinary (pinned or pageable) host memory.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Result order (R5): fp32 score descending, then global id
 *     ascending; -0.0 ranks as +0.0.  If fewer than k candidates exist the
 *     tail is padded with id -1 and score -INFINITY (R6).
 *   - Limits: 1 <= k <= 256; d <= 768 (d is zero-padded to a multiple of 64
 *     internally); nlist <= 32768; global ids < 2^32; n_local < 2^31.
 *   - Requires an sm_100 device (B200); other devices -> SA_ERR_UNSUPPORTED.
 */
#ifndef SA_H_
#define SA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SA_OK = 0,
  SA_ERR_INVALID_ARG = 1, /* bad argument; nothing was done */
  SA_ERR_STATE = 2,       /* call not valid for this object (e.g. nprobe>0 on a flat index) */
  SA_ERR_OOM = 3,         /* device allocation failed */
  SA_ERR_CUDA = 4,        /* CUDA runtime / launch error */
  SA_ERR_NCCL = 5,        /* NCCL error (sharded indexes) */
  SA_ERR_UNSUPPORTED = 6  /* not an sm_100 device, or a size beyond the limits above */
} sa_status;

typedef enum { SA_BF16 = 0, SA_F32 = 1 } sa_dtype;

typedef struct sa_index sa_index; /* opaque; owns all device memory of one rank's shard */
typedef struct sa_comm sa_comm;   /* opaque; an NCCL communicator or an in-process rank */

typedef struct {
  sa_dtype dtype;          /* dtype of `corpus` (default SA_BF16) */
  int32_t kmeans_iters;    /* Lloyd iterations for the IVF quantiser (default 20) */
  int32_t train_per_list;  /* training rows per list: n_train = min(n_total, this*nlist) (256) */
  uint64_t seed;           /* k-means initialisation seed (default 0x5A2505) */
  int64_t row_offset;      /* global id of local row 0 (default 0) */
  int64_t n_total;         /* total rows over all shards (default: n) */
  const sa_comm* comm;     /* NULL = unsharded; else the communicator this shard belongs to */
  void* stream;            /* stream used for the build (default NULL) */
  const float* centroids;  /* optional DEVICE fp32 [nlist, d]: use these IVF centroids instead
                              of training (e.g. a quantiser trained once for all shards) */
  int32_t list_shard_world; /* 0 (default): row sharding as above.  >= 1: LIST sharding --
                              `corpus` is the FULL corpus on every rank (row_offset 0, n_total
                              n or 0), the quantiser is trained identically on every rank from
                              it (no training collective), and this index keeps the whole IVF
                              lists l with l % list_shard_world == list_shard_rank (global ids).
                              A rank's search work then depends only on its lists; a sharded
                              search (comm of the same world and rank) all-gathers and merges
                              exactly as for row shards.  Needs nlist >= 1; SA_ERR_UNSUPPORTED
                              if the rank owns no rows. */
  int32_t list_shard_rank;
} sa_build_opts;

/* Fill *o with the defaults listed above. */
void sa_build_opts_default(sa_build_opts* o);

/*
 * Build an index over `corpus` (DEVICE, [n, d] row-major contiguous, bf16).
 * nlist = 0 -> flat-only index (exact search); nlist >= 1 -> also trains an
 * IVF coarse quantiser with nlist lists (requires nlist <= n_total) and
 * permutes the rows list-major.  Synchronous: returns after the index is
 * complete; the caller may free `corpus` afterwards.  The index copies the
 * rows into its own bf16 [n, d_pad] buffer (fp32 inputs are rounded to
 * nearest-even, R3).
 */
sa_status sa_index_build(const void* corpus, int64_t n, int32_t d, int32_t nlist, sa_index** out);
sa_status sa_index_build_ex(const void* corpus, int64_t n, int32_t d, int32_t nlist,
                            const sa_build_opts* opts, sa_index** out);

/*
 * Top-k search.  queries: DEVICE bf16 [nq, d]; out_ids: DEVICE int64 [nq, k];
 * out_scores: DEVICE fp32 [nq, k].  nprobe = 0 -> exact flat scan;
 * 1 <= nprobe <= nlist -> IVF search over the nprobe best lists.
 * Stream-ordered and asynchronous: returns after enqueue; inputs must stay
 * valid and outputs must not be read until `stream` reaches this point.
 * For a sharded index every rank must call with identical (nq, k, nprobe) in
 * the same order; every rank receives the global result.
 */
sa_status sa_search(const sa_index* idx, const void* queries, int64_t nq, int32_t k, int32_t nprobe,
                    int64_t* out_ids, float* out_scores, void* stream);
sa_status sa_search_ex(const sa_index* idx, const void* queries, sa_dtype qdtype, int64_t nq,
                       int32_t k, int32_t nprobe, int64_t* out_ids, float* out_scores,
                       void* stream);
/*
 * Same search with HOST buffers (queries HOST [nq, d] of qdtype, out_ids HOST
 * int64 [nq, k], out_scores HOST fp32 [nq, k]).  The host->device copy of the
 * queries, the search and the device->host copy of the results are enqueued
 * on `stream`; the call returns after the results are in host memory.
 */
sa_status sa_search_host(const sa_index* idx, const void* queries_host, sa_dtype qdtype,
                         int64_t nq, int32_t k, int32_t nprobe, int64_t* out_ids_host,
                         float* out_scores_host, void* stream);

/*
 * The two halves of a row-sharded search, exposed so the cross-rank step
 * can be driven (and tested) by the caller:
 *   sa_search_keys: this shard's top-k as packed 64-bit keys, DEVICE uint64 [nq, k], sorted
 *                   best first; key = (order-preserving fp32 bits << 32) | (0xFFFFFFFF - id)
 *                   with the GLOBAL id (row_offset + local row); empty slots are 0.
 *   sa_merge_keys:  the final k-way merge of w such lists, DEVICE uint64 [w, nq, k]
 *                   (rank-major, as ncclAllGather lays them out) -> DEVICE out_ids int64
 *                   [nq, k] / out_scores fp32 [nq, k], padded (-1, -INF).
 * sa_search on a sharded index is exactly sa_search_keys + ncclAllGather + sa_merge_keys.
 */
sa_status sa_search_keys(const sa_index* idx, const void* queries, sa_dtype qdtype, int64_t nq,
                         int32_t k, int32_t nprobe, uint64_t* out_keys, void* stream);
sa_status sa_merge_keys(const uint64_t* keys, int32_t w, int64_t nq, int32_t k, int64_t* out_ids,
                        float* out_scores, void* stream);

sa_status sa_index_free(sa_index* idx);

/* NCCL plumbing for row-sharded indexes.  The 128-byte unique
 * id is created on rank 0 with sa_comm_unique_id and broadcast by the caller
 * (e.g. torch.distributed).  libnccl is resolved at run time (the copy the
 * process already loaded, else libnccl.so.2). */
sa_status sa_comm_unique_id(void* out_128_bytes);
sa_status sa_comm_init(const void* nccl_unique_id, int32_t rank, int32_t world, int32_t cuda_device,
                       sa_comm** out);
sa_status sa_comm_free(sa_comm* c);

/*
 * In-process communicator group: `world` ranks that live in
 * ONE process, each driven by its own host thread, on one or several GPUs.  The library's
 * sharded code paths run unchanged on top of it -- the row-sharded search (a9: per-rank keys
 * -> all-gather -> merge), the sharded IVF build (the training sample assembled from every
 * rank's part), the fp8 build (global scale).  Collectives are stream-synchronous
 * device-to-device copies between the ranks' buffers under a group barrier, so every rank of
 * the group must make the same sequence of sharded calls concurrently (from its own thread);
 * a rank missing for 300 s makes the waiting ranks fail with SA_ERR_STATE instead of hanging.
 * (NCCL refuses two ranks on one device; this transport is how one GPU exercises the sharded
 * branch, and it serves single-process multi-GPU drivers.)
 *   sa_comm_group_create: world in [1, 1024].  The group outlives its communicators:
 *                         sa_comm_group_free returns SA_ERR_STATE while any is alive.
 *   sa_comm_init_local:   the communicator of `rank` in group `g` on CUDA device
 *                         `cuda_device`; owned by the caller (sa_comm_free).
 */
typedef struct sa_comm_group sa_comm_group;
sa_status sa_comm_group_create(int32_t world, sa_comm_group** out);
sa_status sa_comm_group_free(sa_comm_group* g);
sa_status sa_comm_init_local(sa_comm_group* g, int32_t rank, int32_t cuda_device, sa_comm** out);

/*
 * Cross-rank argument check (SURVEY.md §8(b) "Errors").  When on, every sharded sa_search /
 * sa_search_ex / sa_search_host / sa_search_fp8 first all-gathers a fixed-size header of its
 * arguments (nq, k, nprobe, qdtype, n_cand) and its local validation status; if any rank
 * failed validation or passed different arguments, EVERY rank returns SA_ERR_INVALID_ARG
 * (outputs untouched) instead of some ranks waiting in a collective the others never enter.
 * Costs one small all-gather and a host synchronisation per call; off by default.
 * All ranks must set the same value.
 */
sa_status sa_comm_set_checks(sa_comm* c, int32_t on);
/*
 * Sharded code path at world 1 (tests and one-GPU validation).  When on, an
 * index built with this communicator takes the sharded path even if world == 1: the sharded
 * IVF build assembles its training sample with the communicator's broadcasts, and every search
 * runs rank-local keys -> all-gather -> k-way merge (and the argument check when enabled) --
 * with an NCCL communicator of one rank these are real NCCL calls, so a one-GPU job executes
 * exactly the collective code a multi-GPU job does (the results equal the unsharded search).
 * Set before building the index; off by default.  c NULL -> SA_ERR_INVALID_ARG.
 */
sa_status sa_comm_set_collectives(sa_comm* c, int32_t on);
/* rank / world of this communicator; nccl_nranks = ncclCommCount for an NCCL communicator
 * (world for the in-process transport).  Any output pointer may be NULL. */
sa_status sa_comm_info(const sa_comm* c, int32_t* rank, int32_t* world, int32_t* nccl_nranks);

const char* sa_status_string(sa_status s);
const char* sa_last_error(void);

/* ---- non-stall retrieval: IVF search with the maturity exit ----
 * PAPER.md §3.3 "Non-Stall Retrieval" and App. B.2: the search
 * watches RQ_t = (d_t - d_best)/(d_worst - d_best) of the newly discovered candidates,
 * smooths it with an EMA and halts once the EMA exceeds tau AND the LLM engine is ready;
 * otherwise it stops naturally.  Carried to IVF (readings R14-R19):
 *   - a step t is one probed list, in probe-rank order (best centroid first);
 *   - s_t = the best score of list t; after inserting the list into the running top-k R,
 *     RQ_t = (s_best - s_t) / (s_best - s_worst) over R's first / last entries (1.0 when
 *     s_best == s_worst or the list is empty; not clamped);
 *   - EMA_1 = RQ_1, EMA_t = a*RQ_t + (1-a)*EMA_{t-1}, a = 2/(window+1) (fp64);
 *   - after every check_every lists the device reads *engine_ready; the query stops there
 *     if EMA_t >= tau and the flag is nonzero, else it goes on, up to nprobe_max lists;
 *   - the result is R after the last scanned list (score desc, id asc; padded -1/-INF).
 * The device makes every decision; no host round trip sits between stages.  Agent-step
 * batches (nq * min(check_every, nprobe_max) <= 64, k <= 32) run as ONE cooperative kernel
 * whose stages are closed on the device; larger ones as one captured graph with a conditional
 * WHILE node per shape. */
typedef struct {
  double tau;              /* EMA threshold (the paper's HNSW value is 0.9) */
  int32_t window;          /* EMA window in lists, >= 1 (the paper's is 500 candidates) */
  int32_t check_every;     /* g >= 1: exit test after every g lists (values > nprobe_max are
                              clamped to nprobe_max) */
  const int32_t* engine_ready; /* readiness flag, read by the device at every checkpoint:
                              pinned HOST memory (cudaHostAlloc / torch pin_memory) or DEVICE
                              memory; nonzero = the LLM engine is ready for its next step
                              (P:177).  The caller may change it while the search runs.
                              NULL = always ready. */
} sa_maturity_opts;
/*
 * queries: DEVICE [nq, d] of qdtype.  out_ids DEVICE int64 [nq, k], out_scores DEVICE fp32
 * [nq, k], out_lists_scanned DEVICE int32 [nq] (lists scanned per query; may be NULL),
 * out_rq / out_ema DEVICE fp64 [nq, nprobe_max] per-step signal (NaN past the exit; both
 * NULL or both set).  Stream-ordered and asynchronous like sa_search.
 * Limits: unsharded IVF index (SA_ERR_STATE on a flat-only index, SA_ERR_UNSUPPORTED on a
 * sharded one); nq * min(check_every, nprobe_max) <= 4096 (agent-step batches), else
 * SA_ERR_UNSUPPORTED.  Per (shape, opts, stream) the library keeps the captured graph and
 * its buffers (freed with the index); concurrent calls must use different streams.
 */
sa_status sa_search_mature(const sa_index* idx, const void* queries, sa_dtype qdtype, int64_t nq,
                           int32_t k, int32_t nprobe_max, const sa_maturity_opts* opts,
                           int64_t* out_ids, float* out_scores, int32_t* out_lists_scanned,
                           double* out_rq, double* out_ema, void* stream);

/* ---- proximity-graph index (readings R22-R27) ----
 * The paper's retriever is a graph index (HNSW, App. B.3) whose
 * "search range" (efSearch) trades recall for effort.  Built on an IVF index:
 *   R22 knn(i): the knn_k best rows (score desc, id asc) over the union of the nprobe_build
 *       lists row i probes, excluding i (the IVF search with each stored row as a query);
 *   R23/R24 fwd(i): knn(i) reordered by (detour count, rank), first `degree`, where the
 *       detour count of the rank-j neighbour c_j is #{k < j : c_j is in knn(c_k) at rank < j};
 *   R25/R26 final list: the first degree/2 of fwd(c), then reverse edges (p, i) with
 *       fwd(i)[p] == c in (p, i) order, then the rest of fwd(c), without repeats.
 * sa_index_build_graph: idx must be an unsharded IVF index; 1 <= degree <= 64,
 * degree <= knn_k <= 64, knn_k < n, 1 <= nprobe_build <= nlist; flags bit 0 keeps the kNN
 * lists for sa_index_export_graph.  Synchronous.  Memory: n*degree*4 bytes kept (+ transient
 * n*(knn_k*4 + degree*12)).
 * sa_search_graph (R27): beam search per query over a list of search_range (L) entries,
 * expanding the search_width (w) best unexpanded entries per iteration, at most max_iters
 * iterations (the visited table is 8192 slots per query; when it would pass 3/4 load it is
 * cleared down to the list's rows -- the list evolves exactly as with an unbounded visited
 * set, forgotten rows may be scored again);
 * entry points = the first stored row (lowest id) of each of the n_entries (E) best IVF
 * lists of the query.  queries DEVICE [nq, d] of qdtype; out_ids DEVICE int64 [nq, k],
 * out_scores DEVICE fp32 [nq, k] (score desc, id asc; padded -1 / -INF), out_expanded
 * DEVICE int32 [2, nq] (row 0: list entries expanded, row 1: rows scored; may be NULL).  1 <= k <= L <= 256,
 * w*degree <= 256, 1 <= E <= min(nlist, 256).  Stream-ordered, asynchronous.
 * sa_index_export_graph: *degree, host_nbr HOST int64 [n_local, degree] (row = global id -
 * row_offset, entries global ids, -1 padded), host_knn HOST int64 [n_local, knn_k] likewise
 * (NULL, or the kept kNN lists), *knn_k.
 */
sa_status sa_index_build_graph(sa_index* idx, int32_t knn_k, int32_t degree, int32_t nprobe_build,
                               int32_t flags, void* stream);
sa_status sa_search_graph(const sa_index* idx, const void* queries, sa_dtype qdtype, int64_t nq,
                          int32_t k, int32_t search_range, int32_t search_width,
                          int32_t n_entries, int32_t max_iters, int64_t* out_ids,
                          float* out_scores, int32_t* out_expanded, void* stream);
sa_status sa_index_export_graph(const sa_index* idx, int32_t* degree, int32_t* knn_k,
                                int64_t* host_nbr, int64_t* host_knn);
/* sa_search_graph_ex: sa_search_graph with flags.  SA_GRAPH_FP8 (reading R34): the beam
 * search scores rows on the index's e4m3 copy (sa_index_build_fp8; R30/R31 quantisation,
 * scores = fp32 sums of e4m3 products) -- half the gathered bytes -- and the final list of
 * search_range entries is re-scored on the bf16 rows (fp32 dot products), the k best returned
 * (score desc, id asc).  SA_ERR_STATE without the e4m3 copy; other flags SA_ERR_INVALID_ARG. */
#define SA_GRAPH_FP8 1
sa_status sa_search_graph_ex(const sa_index* idx, const void* queries, sa_dtype qdtype,
                             int64_t nq, int32_t k, int32_t search_range, int32_t search_width,
                             int32_t n_entries, int32_t max_iters, int32_t flags,
                             int64_t* out_ids, float* out_scores, int32_t* out_expanded,
                             void* stream);
/* sa_search_graph_host: sa_search_graph_ex (no iteration cap) with HOST buffers (queries HOST
 * [nq, d] of qdtype, out_ids HOST int64 [nq, k], out_scores HOST fp32 [nq, k]); the
 * host->device copy, the search and the device->host copy are enqueued on `stream` and the
 * call returns when the results are in host memory (the end-to-end API of the graph mode). */
sa_status sa_search_graph_host(const sa_index* idx, const void* queries_host, sa_dtype qdtype,
                               int64_t nq, int32_t k, int32_t search_range, int32_t search_width,
                               int32_t n_entries, int32_t flags, int64_t* out_ids_host,
                               float* out_scores_host, void* stream);
/* sa_index_import_graph: replace idx's graph by host_nbr HOST int64 [n_local, degree] in
 * sa_index_export_graph's layout (row = global id - row_offset, entries global ids of this
 * index, -1 padded); the inverse of export (a saved graph, or a hand-built one in tests).
 * Synchronous; the caller keeps host_nbr.  SA_ERR_STATE on a flat-only index,
 * SA_ERR_INVALID_ARG on degree outside [1, 64] or an id outside the index. */
sa_status sa_index_import_graph(sa_index* idx, int32_t degree, const int64_t* host_nbr);

/* sa_search_graph_mature: the beam search of sa_search_graph with the non-stall maturity
 * exit of PAPER.md §3.3 (App. B.2) in the paper's own setting, a graph
 * search (readings R28-R29):
 *   - a step t is one iteration (search_width expansions);
 *   - s_t = the best score among the rows scored in step t; after they are merged into the
 *     list, RQ_t = (s_best - s_t) / (s_best - s_worst) over the list's first / last entries
 *     (1.0 when the step scored nothing or s_best == s_worst; not clamped);
 *   - EMA_1 = RQ_1, EMA_t = a*RQ_t + (1-a)*EMA_{t-1}, a = 2/(opts->window+1), fp64;
 *   - after every opts->check_every steps the query stops if EMA_t >= opts->tau and
 *     *opts->engine_ready is nonzero (read by the device at that moment; NULL = always);
 *     otherwise it runs until no entry is left to expand or max_iters;
 *   - after a visited-table reset (see sa_search_graph) a re-scored forgotten row counts in
 *     s_t; it lies below the list's last entry, so it can change s_t only in a step whose
 *     genuinely new rows are all below that entry too (RQ_t > 1 either way);
 *   - the result is the list's first k entries at that point (R19).
 * One launch; each query's CTA decides on its own.  out_steps DEVICE int32 [nq] (iterations
 * run; may be NULL); out_rq / out_ema DEVICE fp64 [nq, trace_cols] per-step signal for steps
 * 1..trace_cols (NaN past the exit; both NULL, or both set with trace_cols >= 1).  Other
 * arguments, limits and errors as sa_search_graph; SA_ERR_INVALID_ARG on opts NULL, tau NaN,
 * window < 1 or check_every < 1. */
sa_status sa_search_graph_mature(const sa_index* idx, const void* queries, sa_dtype qdtype,
                                 int64_t nq, int32_t k, int32_t search_range,
                                 int32_t search_width, int32_t n_entries, int32_t max_iters,
                                 const sa_maturity_opts* opts, int64_t* out_ids,
                                 float* out_scores, int32_t* out_steps, double* out_rq,
                                 double* out_ema, int32_t trace_cols, void* stream);

/* ---- fp8 flat scan with bf16 re-rank (readings R30-R33) ----
 * Not in the paper: a compressed variant of the exact mode (ENN).  The
 * corpus scan reads an e4m3 copy of the rows (half the bytes, twice the bf16 tensor rate) to
 * pick candidates; the candidates are re-scored on the bf16 rows, so returned scores and order
 * are the bf16 data's, and the result is the exact top-k whenever the true top-k lie among the
 * candidates.
 *   R30 corpus: X8 = e4m3_rne_satfinite(x * 2^e), e = the largest integer with
 *       max|x| * 2^e <= 448 over the whole corpus (every rank: the global maximum);
 *   R31 queries: the same per query row with the row's own maximum;
 *   R32 candidates: the n_cand best stored rows by the fp32 sum of the e4m3 products (score
 *       desc, stored position asc); re-scored as the fp32 dot product of the bf16 query and row;
 *   R33 result: the k best re-scored candidates (score desc, global id asc), padded (-1, -INF).
 * sa_index_build_fp8: builds the copy (n_local * ceil(d/128)*128 bytes kept).  Synchronous;
 * collective on a sharded index (every rank must call).
 * sa_search_fp8: queries DEVICE [nq, d] of qdtype; out_ids DEVICE int64 [nq, k], out_scores
 * DEVICE fp32 [nq, k]; 1 <= k <= n_cand <= 256.  nprobe = 0: the candidates come from every
 * row (exact mode, compressed); 1 <= nprobe <= nlist: from the rows of the nprobe best IVF
 * lists (probed with the bf16 query exactly as sa_search, R11), the list scan on the e4m3 copy
 * (IVF mode, compressed: half the list bytes).  Stream-ordered, asynchronous; sharded indexes
 * as sa_search (every rank calls, every rank receives the global result).  SA_ERR_STATE
 * without sa_index_build_fp8 or with nprobe > 0 on a flat-only index.
 * sa_index_export_fp8: *scale_exp = e; host_out (may be NULL) HOST uint8 [n_local, d] e4m3
 * bytes, row = global id - row_offset. */
sa_status sa_index_build_fp8(sa_index* idx, void* stream);
sa_status sa_search_fp8(const sa_index* idx, const void* queries, sa_dtype qdtype, int64_t nq,
                        int32_t k, int32_t nprobe, int32_t n_cand, int64_t* out_ids,
                        float* out_scores, void* stream);
sa_status sa_index_export_fp8(const sa_index* idx, uint8_t* host_out, int32_t* scale_exp);

/* ---- agent loop support (Alg. 1, App. A.1) ---- */

/*
 * Priority scheduling (§3.2, Eq. 1-2): orders the engine's n waiting
 * sequences.  Per sequence i (HOST arrays, length n): R[i] = retrievals completed, W_us[i] =
 * microseconds since the request first arrived, C[i] = context length in tokens, Wcur_us[i] =
 * microseconds since the current sequence became ready, ids[i] = request id.  With min/max
 * over these n sequences (reading R20), Eq. 1 thresholds T_{M,k} = min(M) + (k/G)(max(M) -
 * min(M)) and Eq. 2 level_i = the largest k with R_i > T_{R,k} or W_i > T_{W,k} or C_i >
 * T_{C,k} (0 if none; evaluated exactly in integers).  out_order (HOST int64 [n]) receives
 * the input positions in execution order: level descending, Wcur descending, id ascending
 * (R21); out_level (HOST int32 [n], may be NULL) the levels.  Metrics must lie in [0, 2^50]
 * and G >= 1 (the paper uses G = 6), else SA_ERR_INVALID_ARG.  Host only, synchronous.
 */
sa_status sa_priority_order(int64_t n, const int64_t* R, const int64_t* W_us, const int64_t* C,
                            const int64_t* Wcur_us, const int64_t* ids, int32_t G,
                            int32_t* out_level, int64_t* out_order);

/*
 * Asynchronous retrieval tasks (Alg. 1: LaunchAsyncRetrievalTask, ActiveSearchTasks,
 * CheckExternalNonStallSignal, getResult).  A retriever owns `streams` CUDA
 * streams, a pinned engine-ready flag and `slots` task slots with pinned staging buffers for
 * up to max_nq queries of d = the index's d.  submit copies fp32 HOST queries [nq, d] into a
 * slot and enqueues H2D + search + D2H on the next stream without blocking: nprobe_max = 0 ->
 * exact search; mature = 0 -> fixed-nprobe IVF (sa_search); mature = 1 -> maturity exit
 * (sa_search_mature with *opts and the retriever's flag).  poll never blocks; result copies
 * a finished task's ids int64 [nq, k] / scores fp32 [nq, k] / lists scanned int32 [nq] (may
 * be NULL) to HOST memory and frees the slot.  set_engine_ready writes the flag every running
 * maturity search reads at its checkpoints.  Errors: SA_ERR_STATE when no slot is free
 * (submit) or the task is unknown / not finished (result); SA_ERR_INVALID_ARG on bad sizes.
 */
typedef struct sa_retriever sa_retriever;
sa_status sa_retriever_create(const sa_index* idx, int32_t streams, int32_t slots, int32_t max_nq,
                              int32_t max_k, sa_retriever** out);
sa_status sa_retriever_submit(sa_retriever* r, const float* queries_host, int32_t nq, int32_t k,
                              int32_t nprobe_max, int32_t mature, const sa_maturity_opts* opts,
                              int64_t* task_id);
/* The same task over the proximity graph (the paper's own retriever family): mature = 0 ->
 * sa_search_graph, mature = 1 -> sa_search_graph_mature with *opts and the retriever's flag.
 * result's per-query count is the beam-search iterations run (maturity exit) or -1 (plain).
 * Errors as sa_retriever_submit and sa_search_graph. */
sa_status sa_retriever_submit_graph(sa_retriever* r, const float* queries_host, int32_t nq,
                                    int32_t k, int32_t search_range, int32_t search_width,
                                    int32_t n_entries, int32_t mature,
                                    const sa_maturity_opts* opts, int64_t* task_id);
sa_status sa_retriever_poll(sa_retriever* r, int64_t task_id, int32_t* done);
sa_status sa_retriever_result(sa_retriever* r, int64_t task_id, int64_t* ids_host,
                              float* scores_host, int32_t* lists_host);
sa_status sa_retriever_set_engine_ready(sa_retriever* r, int32_t ready);
sa_status sa_retriever_free(sa_retriever* r);

/* ---- introspection (tests); HOST outputs, synchronous ---- */
sa_status sa_index_info(const sa_index* idx, int64_t* n_local, int32_t* d, int32_t* nlist,
                        int64_t* row_offset);
/* IVF centroids as fp32 [nlist, d] (HOST). */
sa_status sa_index_export_centroids(const sa_index* idx, float* host_out);
/* IVF layout: offsets int64 [nlist+1] and the global id of every stored row,
 * int64 [n_local], list-major (HOST). */
sa_status sa_index_export_lists(const sa_index* idx, int64_t* host_offsets, int64_t* host_ids);
/* The probe step alone: out_lists DEVICE int32 [nq, nprobe], best list first. */
sa_status sa_search_probes(const sa_index* idx, const void* queries, int64_t nq, int32_t nprobe,
                           int32_t* out_lists, void* stream);
/* Debug: the raw fp32 score matrix S = Q . X^T of the flat kernel, DEVICE
 * [nq, n_local], columns in stored-row order (tests of the tensor-core path only). */
sa_status sa_debug_scores(const sa_index* idx, const void* queries, int64_t nq, float* out_scores,
                          void* stream);
/* Debug: sa_search_mature on the one-launch path with per-stage timestamps: host_ns HOST
 * int64 [64 * 4] receives %globaltimer (ns) per stage: CTA 0 stage start, CTA 0 scan done,
 * last CTA arrival, stage release.  Synchronous.  SA_ERR_UNSUPPORTED when the one-launch path
 * does not apply. */
sa_status sa_debug_mature_stages(const sa_index* idx, const void* queries, int64_t nq, int32_t k,
                                 int32_t nprobe_max, const sa_maturity_opts* opts,
                                 int64_t* out_ids, float* out_scores, int32_t* out_lists_scanned,
                                 int64_t* host_ns, void* stream);
/* Debug: the one-launch agent-step IVF search (nq <= 8; DESIGN.md §4.2 "small batches") with
 * per-CTA phase timestamps.  queries DEVICE bf16 [nq, d]; out_ids / out_scores DEVICE as in
 * sa_search; host_ns HOST int64 [grid * 8] receives %globaltimer (ns) per CTA at: 0 start,
 * 1 centroid keys done, 2 probe candidates appended, 3 probe sets known, 4 list scan done,
 * 5 final merge done (last CTA only; 0 elsewhere), 6 first centroid piece scored, 7 first list
 * piece arrived; *host_grid = grid (<= 1024).  Synchronous.
 * SA_ERR_UNSUPPORTED when the one-launch path does not apply to (nq, k, nprobe). */
sa_status sa_debug_small_phases(const sa_index* idx, const void* queries, int64_t nq, int32_t k,
                                int32_t nprobe, int64_t* out_ids, float* out_scores,
                                int64_t* host_ns, int32_t* host_grid, void* stream);

/* ---- kernel accounting (bench.py) ----
 * When enabled, every kernel launch is counted per kind and the dominant
 * kernels are bracketed by CUDA events on the stream they run on. */
typedef enum {
  SA_KERNEL_FLAT_SCAN = 0, /* fused tcgen05 scan + top-k */
  SA_KERNEL_MERGE = 1,     /* partial-list merge / final merge */
  SA_KERNEL_STAGE = 2,     /* query/corpus cast + pad */
  SA_KERNEL_IVF_PROBE = 3, /* centroid scoring + top-nprobe */
  SA_KERNEL_IVF_SCAN = 4,  /* inverted-list scan + partial top-k */
  SA_KERNEL_OTHER = 5,
  SA_KERNEL_GRAPH_SEARCH = 6, /* proximity-graph beam search */
  SA_KERNEL_KINDS = 7
} sa_kernel_kind;
sa_status sa_profile_enable(int32_t on); /* also resets the counters */
/* Synchronises the recorded events; ms_total = summed event time of that kind,
 * launches = kernels launched of that kind since the last reset. */
sa_status sa_profile_read(int32_t kind, double* ms_total, int64_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* SA_H_ */
