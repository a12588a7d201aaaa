// graph_api.cu -- proximity-graph index build + search entry points (
// DESIGN.md §4.7; include/sa.h for the contract).
//
// Build: the kNN lists come from the IVF search itself -- every stored row, in list-major
// order, is a query of ivf_search (tcgen05 list scan; consecutive stored rows probe nearly the
// same lists, so a batch reads few distinct lists); then the rank-only prune / reverse / merge
// kernels of graph.cu.  Search: stage queries, probe the IVF centroids for entry points
// (tensor-core scores + exact top-E select), beam search (graph.cu).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "internal.h"
#include "kernels/fp8.cuh"
#include "kernels/graph.cuh"
#include "kernels/merge.cuh"

using namespace sa;

namespace {


struct DevFree {
  std::vector<void*> p;
  ~DevFree() {
    for (void* x : p) cudaFree(x);
  }
};

template <typename T>
sa_status galloc(DevFree& f, T** ptr, size_t count, const char* what) {
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(ptr), std::max<size_t>(count, 1) * sizeof(T));
  if (e != cudaSuccess) return cuda_status(e, what);
  f.p.push_back(*ptr);
  return SA_OK;
}

}  // namespace

extern "C" {

sa_status sa_index_build_graph(sa_index* idx, int32_t knn_k, int32_t degree, int32_t nprobe_build,
                               int32_t flags, void* stream) {
  if (!idx) return set_error(SA_ERR_INVALID_ARG, "null index");
  if (idx->nlist == 0) return set_error(SA_ERR_STATE, "the graph is built on an IVF index");
  if (comm_sharded(idx->comm))
    return set_error(SA_ERR_UNSUPPORTED, "graph index on a sharded index");
  const int64_t n = idx->n_local;
  if (degree < 1 || degree > GR_MAX_R || knn_k < degree || knn_k > GR_MAX_K || knn_k >= n)
    return set_error(SA_ERR_INVALID_ARG, "need 1 <= degree <= knn_k <= 64 and knn_k < n");
  if (nprobe_build < 1 || nprobe_build > idx->nlist)
    return set_error(SA_ERR_INVALID_ARG, "nprobe_build must be in [1, nlist]");
  cudaStream_t s = (cudaStream_t)stream;
  const int K = knn_k, R = degree, kk = K + 1;
  DevFree f;
  int32_t *pos_of, *knn, *fwd, *nbr = nullptr;
  uint64_t* rev;
  int64_t* ids;
  float* sc;
  const int64_t B = 16384;
  SA_TRY(galloc(f, &pos_of, n, "graph build"));
  SA_TRY(galloc(f, &knn, (size_t)n * K, "graph kNN lists"));
  SA_TRY(galloc(f, &fwd, (size_t)n * R, "graph build"));
  SA_TRY(galloc(f, &rev, (size_t)n * R, "graph build"));
  SA_TRY(galloc(f, &ids, (size_t)B * kk, "graph build"));
  SA_TRY(galloc(f, &sc, (size_t)B * kk, "graph build"));
  SA_TRY(cuda_status(cudaMalloc(&nbr, (size_t)n * R * sizeof(int32_t)), "graph"));
  auto fail = [&](sa_status st) {
    cudaFree(nbr);
    return st;
  };
  // SA_VERBOSE=1: phase timings on stderr (synchronises between phases)
  static const bool verbose = [] {
    const char* e = getenv("SA_VERBOSE");
    return e && e[0] == '1';
  }();
  auto t_last = std::chrono::steady_clock::now();
  auto phase = [&](const char* name) {
    if (!verbose) return;
    cudaStreamSynchronize(s);
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[sa] graph build %s: %.3f s\n", name,
            std::chrono::duration<double>(t - t_last).count());
    t_last = t;
  };
  sa_status st = cuda_status(launch_inverse_ids(idx->row_ids, n, idx->row_offset, pos_of, s),
                             "inverse ids");
  // R22: kNN lists, batch by batch of consecutive stored rows
  for (int64_t p0 = 0; st == SA_OK && p0 < n; p0 += B) {
    const int64_t nb = std::min(B, n - p0);
    SearchOut out;
    out.ids = ids;
    out.scores = sc;
    st = ivf_search(idx, idx->X + (size_t)p0 * idx->d_pad, nb, nb, kk, nprobe_build, out, s);
    if (st == SA_OK)
      st = cuda_status(launch_knn_to_pos(ids, nb, kk, p0, pos_of, idx->row_offset, K, knn, s),
                       "kNN lists");
  }
  phase("kNN lists (IVF search)");
  if (st == SA_OK) st = cuda_status(launch_graph_prune(knn, n, K, R, fwd, s), "graph prune");
  phase("prune");
  if (st == SA_OK)
    st = cuda_status(cudaMemsetAsync(rev, 0xff, (size_t)n * R * sizeof(uint64_t), s), "memset");
  if (st == SA_OK) st = cuda_status(launch_graph_reverse(fwd, n, R, idx->row_ids, rev, s), "graph reverse");
  phase("reverse");
  if (st == SA_OK) st = cuda_status(launch_graph_merge(fwd, rev, n, R, pos_of, idx->row_offset, nbr, s), "graph merge");
  phase("merge");
  if (st == SA_OK) st = cuda_status(cudaStreamSynchronize(s), "graph build sync");
  if (st != SA_OK) return fail(st);
  cudaFree(idx->graph);
  cudaFree(idx->graph_knn);
  idx->graph = nbr;
  idx->graph_knn = nullptr;
  if (flags & 1) {
    // keep the kNN lists (tests): hand the buffer over instead of freeing it
    f.p.erase(std::find(f.p.begin(), f.p.end(), (void*)knn));
    idx->graph_knn = knn;
  }
  idx->graph_R = R;
  idx->graph_K = K;
  return SA_OK;
}

}  // extern "C"

namespace {

// sa_search_graph(_ex) and sa_search_graph_mature: `mo` NULL = plain beam search (R27);
// fp8 = navigation on the e4m3 copy + bf16 re-rank of the final list (R34)
sa_status graph_search(const sa_index* idx, const void* queries, sa_dtype qdtype, int64_t nq,
                       int32_t k, int32_t search_range, int32_t search_width, int32_t n_entries,
                       int32_t max_iters, const sa_maturity_opts* mo, int64_t* out_ids,
                       float* out_scores, int32_t* out_expanded, int32_t* out_steps,
                       double* out_rq, double* out_ema, int32_t trace_cols, void* stream,
                       bool fp8 = false) {
  if (!idx || !queries || !out_ids || !out_scores)
    return set_error(SA_ERR_INVALID_ARG, "null pointer");
  if (!idx->graph) return set_error(SA_ERR_STATE, "no graph: call sa_index_build_graph");
  if (qdtype != SA_BF16 && qdtype != SA_F32) return set_error(SA_ERR_INVALID_ARG, "bad qdtype");
  if (nq < 1 || nq > (1ll << 31) - 1) return set_error(SA_ERR_INVALID_ARG, "bad nq");
  const int L = search_range, w = search_width, E = n_entries, R = idx->graph_R;
  if (k < 1 || k > L || L > GR_MAX_L)
    return set_error(SA_ERR_INVALID_ARG, "need 1 <= k <= search_range <= 256");
  if (w < 1 || w * R > GR_MAX_NEW || w > 8)
    return set_error(SA_ERR_INVALID_ARG, "need 1 <= search_width <= 8, search_width*degree <= 256");
  if (E < 1 || E > std::min(idx->nlist, 256))
    return set_error(SA_ERR_INVALID_ARG, "need 1 <= n_entries <= min(nlist, 256)");
  if (max_iters < 0) return set_error(SA_ERR_INVALID_ARG, "max_iters must be >= 0");
  if (fp8 && !idx->X8) return set_error(SA_ERR_STATE, "fp8 navigation: call sa_index_build_fp8");
  if (fp8 && mo) return set_error(SA_ERR_UNSUPPORTED, "maturity exit with fp8 navigation");
  if (mo) {
    if (!(mo->tau == mo->tau)) return set_error(SA_ERR_INVALID_ARG, "tau is NaN");
    if (mo->window < 1 || mo->check_every < 1)
      return set_error(SA_ERR_INVALID_ARG, "need window >= 1 and check_every >= 1");
    if ((out_rq == nullptr) != (out_ema == nullptr) || trace_cols < 0 ||
        (out_rq && trace_cols < 1))
      return set_error(SA_ERR_INVALID_ARG, "out_rq / out_ema: both NULL or both [nq, trace_cols >= 1]");
  }
  const int T = max_iters;   // the visited table forgets (graph.cu), so no capacity cap
  cudaStream_t s = (cudaStream_t)stream;
  // queries in chunks: the probe's dense score buffer is chunk x nlist fp32
  const int64_t C = 4096;
  const size_t qsize = (size_t)idx->d * (qdtype == SA_F32 ? 4 : 2);
  sa_status st = SA_OK;
  for (int64_t q0 = 0; st == SA_OK && q0 < nq; q0 += C) {
    const int64_t nc = std::min(C, nq - q0);
    const int64_t nq_pad = padded_nq(nc);
    __nv_bfloat16* Qbuf = nullptr;   // staged copy (fp32 input, padding or fp8 navigation)
    const __nv_bfloat16* Qs = nullptr;
    float* psc = nullptr;
    uint64_t* pkeys = nullptr;
    uint8_t* Q8 = nullptr;
    uint64_t* cand = nullptr;
    if (fp8) {
      st = dalloc(&Q8, (size_t)nq_pad * idx->d8_pad, s, "graph search");
      if (st == SA_OK) st = dalloc(&cand, (size_t)nc * L, s, "graph search");
    }
    // bf16 queries whose rows need no padding are read in place (every reader stays below row
    // nc: the probe GEMM's tensor map covers nc rows, the search reads rows < nc)
    const uint8_t* qsrc = static_cast<const uint8_t*>(queries) + q0 * qsize;
    const bool in_place = !fp8 && qdtype == SA_BF16 && idx->d == idx->d_pad &&
                          (reinterpret_cast<uintptr_t>(qsrc) & 15) == 0;
    if (st == SA_OK && !in_place) st = dalloc(&Qbuf, (size_t)nq_pad * idx->d_pad, s, "graph search");
    Qs = in_place ? reinterpret_cast<const __nv_bfloat16*>(qsrc) : Qbuf;
    if (st == SA_OK) st = dalloc(&psc, (size_t)nc * idx->nlist, s, "graph search");
    if (st == SA_OK) st = dalloc(&pkeys, (size_t)nc * E, s, "graph search");
    if (st == SA_OK && !in_place) {
      ProfRegion prof_region(SA_KERNEL_STAGE, s);
      st = cuda_status(launch_cast_pad(qsrc, qdtype == SA_F32, nc, idx->d, Qbuf, nq_pad,
                                       idx->d_pad, idx->num_sms, s),
                       "stage queries");
      if (st == SA_OK && fp8)
        st = cuda_status(launch_quant_e4m3(Qbuf, nq_pad, idx->d_pad, nullptr, Q8, idx->d8_pad,
                                           nullptr, idx->num_sms, s),
                         "stage fp8 queries");
    }
    if (st == SA_OK) {
      // entry points: the E best IVF lists (tensor-core centroid scores + exact select)
      ProfRegion prof_region(SA_KERNEL_IVF_PROBE, s);
      const CorpusView cvc{&idx->tmap_c, &idx->tmap_c2, idx->nlist, idx->d_pad, nullptr, 0u};
      // score dump + exact select (a fused top-E scan was measured slower: 0.19 vs 0.07 ms at
      // nq = 512, the per-unit query staging dominates a 16384-row scan)
      st = flat_scores_view(cvc, idx->num_sms, Qs, nc, psc, s);
      if (st == SA_OK) {
        MergeArgs m{};
        m.cand_scores = psc;
        m.m_flat = idx->nlist;
        m.qstride = idx->nlist;
        m.k = E;
        m.out_keys = pkeys;
        st = cuda_status(launch_merge(m, nc, s), "entry select");
      }
    }
    if (st == SA_OK) {
      GraphSearchArgs a{};
      a.X = idx->X;
      a.row_ids = idx->row_ids;
      a.nbr = idx->graph;
      a.Q = Qs;
      a.entry_keys = pkeys;
      a.list_off = idx->list_off;
      a.d_pad = idx->d_pad;
      a.R = R;
      a.L = L;
      a.w = w;
      a.E = E;
      a.T = T;
      a.k = k;
      a.out_ids = out_ids + q0 * k;
      a.out_scores = out_scores + q0 * k;
      a.out_expanded = out_expanded ? out_expanded + q0 : nullptr;
      a.nq = (int32_t)nq;   // row stride of out_expanded
      // bits: 1 row prefetch (0.85x), 2 list prefetch (1.00x), 4 rows evict-first, 8 ids
      // evict-last (4+8: 1.00-1.03x; meant to keep the 84 MB of row ids in L2 across the row
      // stream)
      a.prefetch = 12;
      if (const char* e = tuning_env("SA_GRAPH_PF")) a.prefetch = atoi(e);
      if (R % 4 != 0) a.prefetch &= ~2;   // bulk prefetch needs 16-byte aligned list rows
      if (const char* e = tuning_env("SA_GRAPH_DBG"))   // device pointer, [nq, 8] u64
        a.dbg = reinterpret_cast<unsigned long long*>(strtoull(e, nullptr, 0)) + q0 * 8;
      GraphMatureArgs m{};
      if (mo) {
        m.tau = mo->tau;
        m.alpha = 2.0 / (mo->window + 1.0);
        m.g = mo->check_every;
        m.ready = mo->engine_ready;
        m.out_steps = out_steps ? out_steps + q0 : nullptr;
        m.trace_cols = out_rq ? trace_cols : 0;
        m.out_rq = out_rq ? out_rq + q0 * trace_cols : nullptr;
        m.out_ema = out_rq ? out_ema + q0 * trace_cols : nullptr;
      }
      if (fp8) {
        a.X8 = idx->X8;
        a.Q8 = Q8;
        a.d8_pad = idx->d8_pad;
        a.out_keys = cand;
      }
      ProfRegion prof_region(SA_KERNEL_GRAPH_SEARCH, s);
      st = cuda_status(launch_graph_search(a, mo ? &m : nullptr, nc, s, fp8), "graph search");
    }
    if (st == SA_OK && fp8) {
      // R34: the final list re-scored on the bf16 rows, the k best
      RerankArgs r{};
      r.X = idx->X;
      r.d_pad = idx->d_pad;
      r.row_ids = idx->row_ids;
      r.row_offset = idx->row_offset;
      r.Qs = Qs;
      r.cand = cand;
      r.n_cand = L;
      r.k = k;
      r.out_ids = out_ids + q0 * k;
      r.out_scores = out_scores + q0 * k;
      ProfRegion prof_region(SA_KERNEL_MERGE, s);
      st = cuda_status(launch_rerank(r, nc, s), "graph re-rank");
    }
    if (Qbuf) cudaFreeAsync(Qbuf, s);
    if (psc) cudaFreeAsync(psc, s);
    if (pkeys) cudaFreeAsync(pkeys, s);
    if (Q8) cudaFreeAsync(Q8, s);
    if (cand) cudaFreeAsync(cand, s);
  }
  return st;
}

}  // namespace

extern "C" {

sa_status sa_search_graph(const sa_index* idx, const void* queries, sa_dtype qdtype, int64_t nq,
                          int32_t k, int32_t search_range, int32_t search_width,
                          int32_t n_entries, int32_t max_iters, int64_t* out_ids,
                          float* out_scores, int32_t* out_expanded, void* stream) {
  return graph_search(idx, queries, qdtype, nq, k, search_range, search_width, n_entries,
                      max_iters, nullptr, out_ids, out_scores, out_expanded, nullptr, nullptr,
                      nullptr, 0, stream);
}

sa_status sa_search_graph_ex(const sa_index* idx, const void* queries, sa_dtype qdtype,
                             int64_t nq, int32_t k, int32_t search_range, int32_t search_width,
                             int32_t n_entries, int32_t max_iters, int32_t flags,
                             int64_t* out_ids, float* out_scores, int32_t* out_expanded,
                             void* stream) {
  if (flags & ~SA_GRAPH_FP8) return set_error(SA_ERR_INVALID_ARG, "unknown flags");
  return graph_search(idx, queries, qdtype, nq, k, search_range, search_width, n_entries,
                      max_iters, nullptr, out_ids, out_scores, out_expanded, nullptr, nullptr,
                      nullptr, 0, stream, (flags & SA_GRAPH_FP8) != 0);
}

sa_status sa_search_graph_host(const sa_index* idx, const void* queries_host, sa_dtype qdtype,
                               int64_t nq, int32_t k, int32_t search_range, int32_t search_width,
                               int32_t n_entries, int32_t flags, int64_t* out_ids_host,
                               float* out_scores_host, void* stream) {
  if (flags & ~SA_GRAPH_FP8) return set_error(SA_ERR_INVALID_ARG, "unknown flags");
  if (!idx || !queries_host || !out_ids_host || !out_scores_host)
    return set_error(SA_ERR_INVALID_ARG, "null pointer");
  if (qdtype != SA_BF16 && qdtype != SA_F32) return set_error(SA_ERR_INVALID_ARG, "bad qdtype");
  if (nq < 1 || nq > (1ll << 31) - 1) return set_error(SA_ERR_INVALID_ARG, "bad nq");
  if (k < 1 || k > 256) return set_error(SA_ERR_INVALID_ARG, "k must be in [1, 256]");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t qbytes = (size_t)nq * idx->d * (qdtype == SA_F32 ? 4 : 2);
  void* dq = nullptr;
  int64_t* dids = nullptr;
  float* dsc = nullptr;
  sa_status st = cuda_status(cudaMallocAsync(&dq, qbytes, s), "alloc queries");
  if (st == SA_OK) st = dalloc(&dids, (size_t)nq * k, s, "alloc ids");
  if (st == SA_OK) st = dalloc(&dsc, (size_t)nq * k, s, "alloc scores");
  if (st == SA_OK)
    st = cuda_status(cudaMemcpyAsync(dq, queries_host, qbytes, cudaMemcpyHostToDevice, s), "H2D");
  if (st == SA_OK)
    st = graph_search(idx, dq, qdtype, nq, k, search_range, search_width, n_entries, 1 << 30,
                      nullptr, dids, dsc, nullptr, nullptr, nullptr, nullptr, 0, stream,
                      (flags & SA_GRAPH_FP8) != 0);
  if (st == SA_OK)
    st = cuda_status(cudaMemcpyAsync(out_ids_host, dids, (size_t)nq * k * 8,
                                     cudaMemcpyDeviceToHost, s), "D2H ids");
  if (st == SA_OK)
    st = cuda_status(cudaMemcpyAsync(out_scores_host, dsc, (size_t)nq * k * 4,
                                     cudaMemcpyDeviceToHost, s), "D2H scores");
  if (dq) cudaFreeAsync(dq, s);
  if (dids) cudaFreeAsync(dids, s);
  if (dsc) cudaFreeAsync(dsc, s);
  sa_status st2 = cuda_status(cudaStreamSynchronize(s), "search sync");
  return st != SA_OK ? st : st2;
}

sa_status sa_search_graph_mature(const sa_index* idx, const void* queries, sa_dtype qdtype,
                                 int64_t nq, int32_t k, int32_t search_range,
                                 int32_t search_width, int32_t n_entries, int32_t max_iters,
                                 const sa_maturity_opts* opts, int64_t* out_ids,
                                 float* out_scores, int32_t* out_steps, double* out_rq,
                                 double* out_ema, int32_t trace_cols, void* stream) {
  if (!opts) return set_error(SA_ERR_INVALID_ARG, "null maturity options");
  return graph_search(idx, queries, qdtype, nq, k, search_range, search_width, n_entries,
                      max_iters, opts, out_ids, out_scores, nullptr, out_steps, out_rq, out_ema,
                      trace_cols, stream);
}

sa_status sa_index_import_graph(sa_index* idx, int32_t degree, const int64_t* host_nbr) {
  if (!idx || !host_nbr) return set_error(SA_ERR_INVALID_ARG, "null pointer");
  if (idx->nlist == 0) return set_error(SA_ERR_STATE, "the graph is built on an IVF index");
  if (degree < 1 || degree > GR_MAX_R)
    return set_error(SA_ERR_INVALID_ARG, "need 1 <= degree <= 64");
  const int64_t n = idx->n_local;
  std::vector<int32_t> ids(n), pos_of(n), buf((size_t)n * degree);
  cudaError_t e = cudaMemcpy(ids.data(), idx->row_ids, n * 4, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_status(e, "import graph");
  for (int64_t p = 0; p < n; ++p) pos_of[(int64_t)(uint32_t)ids[p] - idx->row_offset] = (int32_t)p;
  for (int64_t p = 0; p < n; ++p) {
    const int64_t* src = host_nbr + ((int64_t)(uint32_t)ids[p] - idx->row_offset) * degree;
    for (int j = 0; j < degree; ++j) {
      const int64_t v = src[j];
      if (v >= 0 && (v < idx->row_offset || v >= idx->row_offset + n))
        return set_error(SA_ERR_INVALID_ARG, "neighbour id outside the index");
      buf[(size_t)p * degree + j] = v < 0 ? -1 : pos_of[v - idx->row_offset];
    }
  }
  int32_t* nbr = nullptr;
  e = cudaMalloc(&nbr, buf.size() * 4);
  if (e == cudaSuccess) e = cudaMemcpy(nbr, buf.data(), buf.size() * 4, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    cudaFree(nbr);
    return cuda_status(e, "import graph");
  }
  cudaFree(idx->graph);
  cudaFree(idx->graph_knn);
  idx->graph = nbr;
  idx->graph_knn = nullptr;
  idx->graph_R = degree;
  idx->graph_K = 0;
  return SA_OK;
}

sa_status sa_index_export_graph(const sa_index* idx, int32_t* degree, int32_t* knn_k,
                                int64_t* host_nbr, int64_t* host_knn) {
  if (!idx || !degree) return set_error(SA_ERR_INVALID_ARG, "null pointer");
  *degree = idx->graph_R;
  if (knn_k) *knn_k = idx->graph_K;
  if (!idx->graph) return set_error(SA_ERR_STATE, "no graph");
  const int64_t n = idx->n_local;
  std::vector<int32_t> ids(n), buf;
  cudaError_t e = cudaMemcpy(ids.data(), idx->row_ids, n * 4, cudaMemcpyDeviceToHost);
  auto conv = [&](const int32_t* dev, int cols, int64_t* out) -> cudaError_t {
    buf.resize((size_t)n * cols);
    cudaError_t e2 = cudaMemcpy(buf.data(), dev, buf.size() * 4, cudaMemcpyDeviceToHost);
    if (e2 != cudaSuccess) return e2;
    // rows in local-id order (global id - row_offset), entries as global ids
    for (int64_t p = 0; p < n; ++p) {
      int64_t* o = out + ((int64_t)(uint32_t)ids[p] - idx->row_offset) * cols;
      for (int j = 0; j < cols; ++j) {
        const int32_t v = buf[(size_t)p * cols + j];
        o[j] = v < 0 ? -1 : (int64_t)(uint32_t)ids[v];
      }
    }
    return cudaSuccess;
  };
  if (e == cudaSuccess && host_nbr) e = conv(idx->graph, idx->graph_R, host_nbr);
  if (e == cudaSuccess && host_knn) {
    if (!idx->graph_knn) return set_error(SA_ERR_STATE, "kNN lists not kept (build flag bit 0)");
    e = conv(idx->graph_knn, idx->graph_K, host_knn);
  }
  return cuda_status(e, "export graph");
}

}  // extern "C"
