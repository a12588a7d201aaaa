// mature_api.cu -- sa_search_mature: IVF search with the non-stall maturity exit
// (§3.3 "Non-Stall Retrieval"; App. B.2; SURVEY.md §8(f)1;
// DESIGN.md §4.5).
//
// The whole progressive search is ONE captured CUDA graph per shape:
//   prologue  cast/pad the queries, probe (tensor-core centroid scores + exact top-nprobe),
//             init the running results;
//   WHILE     (a conditional graph node; the device decides when to stop)
//               one-CTA stage lists + probe inversion -> ivf_scan_kernel (no shared bound,
//               grid sized to the stage) -> in-order merge + RQ/EMA + exit test (reads the
//               engine-ready flag); its last CTA advances the stage and sets the loop
//               condition to 0 once every query has finished
//   epilogue  unpack the results.
// No host round trip decides anything: a query leaves the loop at the first checkpoint where
// its EMA >= tau while the flag is set, or after nprobe_max lists.
#include <algorithm>
#include <cstring>
#include <memory>

#include "internal.h"
#include "kernels/ivf_kernels.cuh"
#include "kernels/ivf_scan.cuh"
#include "kernels/ivf_small.cuh"
#include "kernels/mature.cuh"
#include "kernels/merge.cuh"

namespace sa {

struct MaturePlan {
  // key
  int64_t nq = 0;
  int32_t k = 0, nprobe_max = 0, g = 0, window = 0, qdtype = 0;
  double tau = 0;
  const int32_t* ready = nullptr;
  bool trace = false;
  cudaStream_t stream = nullptr;
  // buffers
  void* d_q = nullptr;
  __nv_bfloat16* Qs = nullptr;
  float* psc = nullptr;
  uint64_t* pkeys = nullptr;
  int64_t* probes = nullptr;
  int64_t* stage_probes = nullptr;
  IvfSearchScratch w{};
  uint64_t* part = nullptr;
  uint64_t* heap = nullptr;
  uint64_t* R = nullptr;
  double* ema = nullptr;
  int32_t *active = nullptr, *t_done = nullptr, *ctrl = nullptr;
  double *trace_rq = nullptr, *trace_ema = nullptr;
  int64_t* out_ids = nullptr;
  float* out_sc = nullptr;
  int32_t* out_t = nullptr;
  cudaGraphExec_t exec = nullptr;
  std::vector<void*> allocs;
  // launches of one replay per kernel kind (the WHILE body counted once: the number of
  // stages is decided on the device); LRU stamp
  int64_t launches[SA_KERNEL_KINDS] = {};
  uint64_t last_use = 0;
};

void free_mature_plan(MaturePlan* p) {
  if (!p) return;
  if (p->exec) cudaGraphExecDestroy(p->exec);
  for (void* a : p->allocs) cudaFree(a);
  delete p;
}

namespace {

template <typename T>
sa_status palloc(MaturePlan& p, T** ptr, size_t count, const char* what) {
  *ptr = nullptr;
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(ptr), count * sizeof(T));
  if (e != cudaSuccess) return cuda_status(e, what);
  p.allocs.push_back(*ptr);
  return SA_OK;
}


struct CaptureFlag {
  CaptureFlag() { set_capturing(true); }
  ~CaptureFlag() { set_capturing(false); }
};

sa_status make_plan(const sa_index* idx, MaturePlan& p) {
  const int64_t nq = p.nq, P = p.nprobe_max, g = p.g;
  const int64_t np = nq * g;
  const int sms = idx->num_sms;
  const int64_t nq_pad = padded_nq(nq);
  const size_t qbytes = (size_t)nq * idx->d * (p.qdtype == SA_F32 ? 4 : 2);
  // work-item size as in ivf_search: ~4 items per SM from the rows one stage probes
  const int64_t mean_list = std::max<int64_t>(1, idx->n_local / idx->nlist);
  int64_t want = np * mean_list / (4 * (int64_t)sms);
  want = (want + IVS_BM - 1) / IVS_BM * IVS_BM;
  const int chunk_rows = (int)std::min<int64_t>(4096, std::max<int64_t>(256, want));
  const int64_t max_chunks = std::max<int64_t>(1, (idx->max_list + chunk_rows - 1) / chunk_rows);
  const size_t max_slots = (size_t)np * max_chunks;
  // a stage probes ~np lists of ~mean_list rows: a grid of ~2 CTAs per expected work item
  // (items are taken dynamically, so any grid is correct; a small one launches faster)
  const int64_t exp_items = np * ((mean_list + chunk_rows - 1) / chunk_rows);
  const int scan_grid = (int)std::max<int64_t>(8, std::min<int64_t>(sms, 2 * exp_items));

  SA_TRY(palloc(p, reinterpret_cast<uint8_t**>(&p.d_q), qbytes, "mature plan"));
  SA_TRY(palloc(p, &p.Qs, (size_t)nq_pad * idx->d_pad, "mature plan"));
  SA_TRY(palloc(p, &p.psc, (size_t)nq * idx->nlist, "mature plan"));
  SA_TRY(palloc(p, &p.pkeys, (size_t)nq * P, "mature plan"));
  SA_TRY(palloc(p, &p.probes, (size_t)nq * P, "mature plan"));
  SA_TRY(palloc(p, &p.stage_probes, (size_t)np, "mature plan"));
  SA_TRY(palloc(p, &p.w.lq_ent, (size_t)np, "mature plan"));
  SA_TRY(palloc(p, &p.w.q_slot, (size_t)np + 1, "mature plan"));
  SA_TRY(palloc(p, &p.w.items, max_slots, "mature plan"));
  SA_TRY(palloc(p, &p.w.n_items, 1, "mature plan"));
  SA_TRY(palloc(p, &p.part, max_slots * IVS_PARTS * p.k, "mature partials"));
  if (p.k > IVS_KSMEM) SA_TRY(palloc(p, &p.heap, (size_t)sms * p.k * IVS_HEAPS, "mature heaps"));
  SA_TRY(palloc(p, &p.R, (size_t)nq * p.k, "mature plan"));
  SA_TRY(palloc(p, &p.ema, (size_t)nq, "mature plan"));
  SA_TRY(palloc(p, &p.active, (size_t)nq, "mature plan"));
  SA_TRY(palloc(p, &p.t_done, (size_t)nq, "mature plan"));
  SA_TRY(palloc(p, &p.ctrl, 4, "mature plan"));  // stage, active, item counter, update CTAs
  if (p.trace) {
    SA_TRY(palloc(p, &p.trace_rq, (size_t)nq * P, "mature plan"));
    SA_TRY(palloc(p, &p.trace_ema, (size_t)nq * P, "mature plan"));
  }
  SA_TRY(palloc(p, &p.out_ids, (size_t)nq * p.k, "mature plan"));
  SA_TRY(palloc(p, &p.out_sc, (size_t)nq * p.k, "mature plan"));
  SA_TRY(palloc(p, &p.out_t, (size_t)nq, "mature plan"));

  MatureArgs m{};
  m.nq = (int32_t)nq;
  m.k = p.k;
  m.nprobe_max = p.nprobe_max;
  m.g = p.g;
  m.tau = p.tau;
  m.alpha = 2.0 / ((double)p.window + 1.0);
  m.ready = p.ready;
  m.probes = p.probes;
  m.stage_probes = p.stage_probes;
  m.q_slot = p.w.q_slot;
  m.part = p.part;
  m.parts = IVS_PARTS;
  m.R = p.R;
  m.ema = p.ema;
  m.active = p.active;
  m.t_done = p.t_done;
  m.ctrl = p.ctrl;
  m.trace_rq = p.trace_rq;
  m.trace_ema = p.trace_ema;

  IvfScanArgs v{};
  v.Q = p.Qs;
  v.d_pad = idx->d_pad;
  v.k = p.k;
  v.row_ids = idx->row_ids;
  v.part = p.part;
  v.heap_g = p.heap;
  v.items = p.w.items;
  v.n_items = p.w.n_items;
  v.list_off = idx->list_off;
  v.lq_ent = p.w.lq_ent;
  v.q_slot = p.w.q_slot;
  v.nprobe = p.g;
  v.chunk_rows = chunk_rows;
  v.q_hint = nullptr;  // exact per-(query, list) top-k: RQ needs every list's best score
  v.item_counter = p.ctrl + 2;

  cudaStream_t cs;
  SA_TRY(cuda_status(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "capture stream"));
  std::unique_ptr<CUstream_st, cudaError_t (*)(cudaStream_t)> cs_guard(cs, cudaStreamDestroy);
  cudaGraph_t graph = nullptr;
  SA_TRY(cuda_status(cudaGraphCreate(&graph, 0), "graph create"));
  std::unique_ptr<CUgraph_st, cudaError_t (*)(cudaGraph_t)> graph_guard(graph, cudaGraphDestroy);
  CaptureFlag cap;
  const cudaStreamCaptureMode mode = cudaStreamCaptureModeThreadLocal;

  // ---- prologue: stage queries, probe, init
  std::vector<cudaGraphNode_t> tail;
  {
    SA_TRY(cuda_status(cudaStreamBeginCaptureToGraph(cs, graph, nullptr, nullptr, 0, mode),
                       "begin capture"));
    sa_status st = cuda_status(launch_cast_pad(p.d_q, p.qdtype == SA_F32, nq, idx->d, p.Qs, nq_pad,
                                               idx->d_pad, sms, cs),
                               "stage queries");
    if (st == SA_OK) {
      const CorpusView cvc{&idx->tmap_c, &idx->tmap_c2, idx->nlist, idx->d_pad, nullptr, 0u};
      st = flat_scores_view(cvc, sms, p.Qs, nq, p.psc, cs);
    }
    if (st == SA_OK) {
      MergeArgs mg{};
      mg.cand_scores = p.psc;
      mg.m_flat = idx->nlist;
      mg.qstride = idx->nlist;
      mg.k = p.nprobe_max;
      mg.out_keys = p.pkeys;
      st = cuda_status(launch_merge(mg, nq, cs), "probe select");
    }
    if (st == SA_OK)
      st = cuda_status(launch_keys_to_lists(p.pkeys, nq * P, p.probes, nullptr, sms, cs),
                       "probe lists");
    if (st == SA_OK) st = cuda_status(launch_mature_init(m, cs), "mature init");
    if (st == SA_OK) {
      cudaStreamCaptureStatus cst;
      const cudaGraphNode_t* deps = nullptr;
      size_t nd = 0;
      st = cuda_status(cudaStreamGetCaptureInfo(cs, &cst, nullptr, nullptr, &deps, &nd),
                       "capture info");
      if (st == SA_OK) tail.assign(deps, deps + nd);
    }
    cudaGraph_t g2 = nullptr;
    cudaError_t e = cudaStreamEndCapture(cs, &g2);
    if (st != SA_OK) return st;
    SA_TRY(cuda_status(e, "end capture (prologue)"));
  }

  // ---- the WHILE node
  cudaGraphConditionalHandle handle;
  SA_TRY(cuda_status(cudaGraphConditionalHandleCreate(&handle, graph, 1, cudaGraphCondAssignDefault),
                     "conditional handle"));
  cudaGraphNodeParams cp{};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = handle;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cnode;
  SA_TRY(cuda_status(cudaGraphAddNode(&cnode, graph, tail.data(), tail.size(), &cp),
                     "conditional node"));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  {
    SA_TRY(cuda_status(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, mode),
                       "begin capture (body)"));
    StageSrc src;
    src.probes_full = p.probes;
    src.P = p.nprobe_max;
    src.ctrl = p.ctrl;
    src.active = p.active;
    src.item_counter = p.ctrl + 2;
    sa_status st = cuda_status(launch_invert_stage(p.stage_probes, (int)nq, p.g, src,
                                                   idx->list_off, chunk_rows, IVS_NQ, p.w, cs),
                               "stage inversion");
    if (st == SA_OK)
      st = cuda_status(launch_ivf_scan(idx->tmap_x, idx->tmap_xt, v, scan_grid, cs), "stage scan");
    if (st == SA_OK) st = cuda_status(launch_mature_update(m, handle, cs), "mature update");
    cudaGraph_t g2 = nullptr;
    cudaError_t e = cudaStreamEndCapture(cs, &g2);
    if (st != SA_OK) return st;
    SA_TRY(cuda_status(e, "end capture (body)"));
  }

  // ---- epilogue
  {
    SA_TRY(cuda_status(cudaStreamBeginCaptureToGraph(cs, graph, &cnode, nullptr, 1, mode),
                       "begin capture (epilogue)"));
    sa_status st = cuda_status(launch_mature_final(m, p.out_ids, p.out_sc, p.out_t, cs),
                               "mature final");
    cudaGraph_t g2 = nullptr;
    cudaError_t e = cudaStreamEndCapture(cs, &g2);
    if (st != SA_OK) return st;
    SA_TRY(cuda_status(e, "end capture (epilogue)"));
  }
  SA_TRY(cuda_status(cudaGraphInstantiate(&p.exec, graph, 0), "instantiate"));
  capture_tally(p.launches);
  return SA_OK;
}

// Agent-step batches (nq * g <= 64, k <= 32): the whole progressive search in ONE cooperative
// launch (ivf_small.cu) -- probe, then stages of g lists per active query, each closed by the
// last CTA to finish it (in-order merge, RQ / EMA, exit test on the engine flag), no graph.
sa_status mature_small(const sa_index* idx, const void* queries, bool q_f32, int64_t nq,
                       int32_t k, int32_t P, int32_t g, const sa_maturity_opts& o,
                       int64_t* out_ids, float* out_scores, int32_t* out_t, double* out_rq,
                       double* out_ema, cudaStream_t s, int64_t* stage_ns = nullptr) {
  const int grid = idx->num_sms;
  StreamFreer f{s};
  IvfSmallArgs a{};
  SmallMatureArgs m{};
  SA_TRY(f.alloc(&a.top, (size_t)nq * grid * (ivf_small_m(P, grid) + IVSM_EXTRA), "mature scratch"));
  SA_TRY(f.alloc(&a.pcand, (size_t)nq * idx->nlist, "mature scratch"));
  SA_TRY(f.alloc(&a.counters, (size_t)nq + 3, "mature scratch"));
  SA_TRY(f.alloc(&a.cand, (size_t)2 * grid * nq * g * k, "mature scratch"));
  SA_TRY(f.alloc(&m.R, (size_t)nq * k, "mature scratch"));
  SA_TRY(f.alloc(&m.ema, (size_t)nq, "mature scratch"));
  SA_TRY(f.alloc(&m.active, (size_t)nq, "mature scratch"));
  SA_TRY(f.alloc(&m.t_done, (size_t)nq, "mature scratch"));
  a.Q = queries;
  a.q_f32 = q_f32 ? 1 : 0;
  a.nq = (int32_t)nq;
  a.d = idx->d;
  a.d_pad = idx->d_pad;
  a.C = idx->centroids_bf16;
  a.nlist = idx->nlist;
  a.nprobe = P;
  a.X = idx->X;
  a.list_off = idx->list_off;
  a.row_ids = idx->row_ids;
  a.k = k;
  a.out_ids = out_ids;
  a.out_scores = out_scores;
  m.g = g;
  m.tau = o.tau;
  m.alpha = 2.0 / (o.window + 1.0);
  m.ready = o.engine_ready;
  m.trace_rq = out_rq;
  m.trace_ema = out_ema;
  m.out_t = out_t;
  m.stage_ns = stage_ns;
  ProfRegion prof_region(SA_KERNEL_IVF_SCAN, s);
  return cuda_status(launch_ivf_small_mature(a, m, grid, s), "maturity search (one launch)");
}

}  // namespace
}  // namespace sa

using namespace sa;

extern "C" sa_status sa_search_mature(const sa_index* idx, const void* queries, sa_dtype qdtype,
                                      int64_t nq, int32_t k, int32_t nprobe_max,
                                      const sa_maturity_opts* opts, int64_t* out_ids,
                                      float* out_scores, int32_t* out_lists_scanned,
                                      double* out_rq, double* out_ema, void* stream) {
  if (!idx || !queries || !opts || !out_ids || !out_scores)
    return set_error(SA_ERR_INVALID_ARG, "null pointer");
  if (qdtype != SA_BF16 && qdtype != SA_F32) return set_error(SA_ERR_INVALID_ARG, "bad qdtype");
  if (nq < 1) return set_error(SA_ERR_INVALID_ARG, "nq must be >= 1");
  if (k < 1 || k > 256) return set_error(SA_ERR_INVALID_ARG, "k must be in [1, 256]");
  if (idx->nlist == 0) return set_error(SA_ERR_STATE, "maturity exit needs an IVF index");
  if (nprobe_max < 1 || nprobe_max > idx->nlist)
    return set_error(SA_ERR_INVALID_ARG, "nprobe_max must be in [1, nlist]");
  if (opts->check_every < 1 || opts->window < 1)
    return set_error(SA_ERR_INVALID_ARG, "check_every and window must be >= 1");
  if (opts->tau != opts->tau) return set_error(SA_ERR_INVALID_ARG, "tau is NaN");
  if ((out_rq == nullptr) != (out_ema == nullptr))
    return set_error(SA_ERR_INVALID_ARG, "out_rq and out_ema go together");
  const int32_t g = std::min(opts->check_every, nprobe_max);
  if (nq * (int64_t)g > kInvertSmallMax)
    return set_error(SA_ERR_UNSUPPORTED, "nq * check_every > 4096 (agent-step batches)");
  if (comm_sharded(idx->comm))
    return set_error(SA_ERR_UNSUPPORTED, "maturity exit on a sharded index");
  cudaStream_t s = (cudaStream_t)stream;
  if (nq * g <= IVSM_MAX_STAGE && g <= IVSM_MAX_G && k <= IVSM_MAX_K &&
      ivf_small_applies(idx, nq, k, nprobe_max))
    return mature_small(idx, queries, qdtype == SA_F32, nq, k, nprobe_max, g, *opts, out_ids,
                        out_scores, out_lists_scanned, out_rq, out_ema, s);
  sa_index* mi = const_cast<sa_index*>(idx);
  std::lock_guard<std::mutex> lock(mi->graph_mu);
  MaturePlan* p = nullptr;
  const bool trace = out_rq != nullptr;
  for (auto& e : mi->mature_plans)
    if (e->nq == nq && e->k == k && e->nprobe_max == nprobe_max && e->g == g &&
        e->window == opts->window && e->tau == opts->tau && e->ready == opts->engine_ready &&
        e->qdtype == (int32_t)qdtype && e->trace == trace && e->stream == s)
      p = e.get();
  if (!p) {
    if (mi->mature_plans.size() >= kMaxCapturedSearches) {
      // bounded cache: drop the least recently used plan once its last replay has finished
      auto lru = std::min_element(mi->mature_plans.begin(), mi->mature_plans.end(),
                                  [](const auto& a, const auto& b) {
                                    return a->last_use < b->last_use;
                                  });
      cudaError_t e = cudaStreamSynchronize((*lru)->stream);
      if (e != cudaSuccess) return cuda_status(e, "evict maturity plan");
      mi->mature_plans.erase(lru);
    }
    std::unique_ptr<MaturePlan, void (*)(MaturePlan*)> np(new MaturePlan, free_mature_plan);
    np->nq = nq;
    np->k = k;
    np->nprobe_max = nprobe_max;
    np->g = g;
    np->window = opts->window;
    np->tau = opts->tau;
    np->ready = opts->engine_ready;
    np->qdtype = (int32_t)qdtype;
    np->trace = trace;
    np->stream = s;
    sa_status st = make_plan(idx, *np);
    if (st != SA_OK) return st;
    p = np.get();
    mi->mature_plans.push_back(std::move(np));
  }
  p->last_use = ++mi->use_clock;
  const size_t qbytes = (size_t)nq * idx->d * (qdtype == SA_F32 ? 4 : 2);
  sa_status st = cuda_status(cudaMemcpyAsync(p->d_q, queries, qbytes, cudaMemcpyDefault, s),
                             "queries in");
  if (st == SA_OK) st = cuda_status(cudaGraphLaunch(p->exec, s), "graph launch");
  const size_t nk = (size_t)nq * k;
  if (st == SA_OK)
    st = cuda_status(cudaMemcpyAsync(out_ids, p->out_ids, nk * 8, cudaMemcpyDefault, s), "ids out");
  if (st == SA_OK)
    st = cuda_status(cudaMemcpyAsync(out_scores, p->out_sc, nk * 4, cudaMemcpyDefault, s),
                     "scores out");
  if (st == SA_OK && out_lists_scanned)
    st = cuda_status(cudaMemcpyAsync(out_lists_scanned, p->out_t, (size_t)nq * 4,
                                     cudaMemcpyDefault, s),
                     "lists out");
  if (st == SA_OK && trace) {
    const size_t nt = (size_t)nq * nprobe_max * 8;
    st = cuda_status(cudaMemcpyAsync(out_rq, p->trace_rq, nt, cudaMemcpyDefault, s), "trace out");
    if (st == SA_OK)
      st = cuda_status(cudaMemcpyAsync(out_ema, p->trace_ema, nt, cudaMemcpyDefault, s),
                       "trace out");
  }
  if (st == SA_OK) prof_add_launches(p->launches);
  return st;
}

extern "C" sa_status sa_debug_mature_stages(const sa_index* idx, const void* queries, int64_t nq,
                                            int32_t k, int32_t nprobe_max,
                                            const sa_maturity_opts* opts, int64_t* out_ids,
                                            float* out_scores, int32_t* out_lists_scanned,
                                            int64_t* host_ns, void* stream) {
  if (!idx || !queries || !opts || !out_ids || !out_scores || !host_ns)
    return set_error(SA_ERR_INVALID_ARG, "null pointer");
  const int32_t g = std::min(opts->check_every, nprobe_max);
  if (g < 1 || nq * g > IVSM_MAX_STAGE || g > IVSM_MAX_G || k > IVSM_MAX_K ||
      !ivf_small_applies(idx, nq, k, nprobe_max))
    return set_error(SA_ERR_UNSUPPORTED, "the one-launch maturity path does not apply");
  cudaStream_t s = (cudaStream_t)stream;
  int64_t* dns = nullptr;
  sa_status st = dalloc(&dns, 64 * 4, s, "alloc debug timestamps");
  if (st != SA_OK) return st;
  st = cuda_status(cudaMemsetAsync(dns, 0, 64 * 4 * sizeof(int64_t), s), "memset");
  if (st == SA_OK)
    st = mature_small(idx, queries, false, nq, k, nprobe_max, g, *opts, out_ids, out_scores,
                      out_lists_scanned, nullptr, nullptr, s, dns);
  if (st == SA_OK)
    st = cuda_status(cudaMemcpyAsync(host_ns, dns, 64 * 4 * sizeof(int64_t),
                                     cudaMemcpyDeviceToHost, s), "copy timestamps");
  if (st == SA_OK) st = cuda_status(cudaStreamSynchronize(s), "sync");
  cudaFreeAsync(dns, s);
  return st;
}
