// retriever.cu -- asynchronous retrieval tasks for an agent loop (Alg. 1,
// App. A.1: LaunchAsyncRetrievalTask / ActiveSearchTasks / CheckExternalNonStallSignal /
// getResult).
//
// The LLM engine's loop must never block on retrieval ("Retrieval and generation operate
// asynchronously").  A retriever owns CUDA streams, pinned per-slot staging buffers
// and the pinned engine-ready flag that maturity searches read on the device (§4.5): submit
// enqueues H2D -> search -> D2H and returns, poll is an event query, result copies out of
// pinned memory.  All device work is the library's own kernels (sa_search / sa_search_mature).
#include <cstring>
#include <mutex>
#include <vector>

#include "internal.h"

struct sa_retriever {
  struct Slot {
    bool busy = false;
    int64_t task = -1;
    int32_t nq = 0, k = 0, nprobe = 0, mature = 0;
    float* h_q = nullptr;
    int64_t* h_ids = nullptr;
    float* h_sc = nullptr;
    int32_t* h_lists = nullptr;
    float* d_q = nullptr;
    int64_t* d_ids = nullptr;
    float* d_sc = nullptr;
    int32_t* d_lists = nullptr;
    cudaEvent_t done = nullptr;
  };
  const sa_index* idx = nullptr;
  std::vector<cudaStream_t> streams;
  size_t next_stream = 0;
  std::vector<Slot> slots;
  int32_t* flag = nullptr;  // pinned host, read by the device (ld.relaxed.sys)
  int64_t next_task = 0;
  int32_t max_nq = 0, max_k = 0;
  std::mutex mu;
};

using namespace sa;

namespace {

void destroy(sa_retriever* r) {
  for (auto& s : r->slots) {
    if (s.done) cudaEventSynchronize(s.done);
    cudaFreeHost(s.h_q);
    cudaFreeHost(s.h_ids);
    cudaFreeHost(s.h_sc);
    cudaFreeHost(s.h_lists);
    cudaFree(s.d_q);
    cudaFree(s.d_ids);
    cudaFree(s.d_sc);
    cudaFree(s.d_lists);
    if (s.done) cudaEventDestroy(s.done);
  }
  for (cudaStream_t st : r->streams) cudaStreamDestroy(st);
  cudaFreeHost(r->flag);
  delete r;
}

sa_retriever::Slot* find(sa_retriever* r, int64_t task) {
  for (auto& s : r->slots)
    if (s.busy && s.task == task) return &s;
  return nullptr;
}

}  // namespace

extern "C" {

sa_status sa_retriever_create(const sa_index* idx, int32_t streams, int32_t slots, int32_t max_nq,
                              int32_t max_k, sa_retriever** out) {
  if (!idx || !out) return set_error(SA_ERR_INVALID_ARG, "null pointer");
  if (streams < 1 || slots < 1 || max_nq < 1 || max_k < 1 || max_k > 256)
    return set_error(SA_ERR_INVALID_ARG, "streams, slots, max_nq >= 1; 1 <= max_k <= 256");
  auto* r = new sa_retriever;
  r->idx = idx;
  r->max_nq = max_nq;
  r->max_k = max_k;
  cudaError_t e = cudaHostAlloc(&r->flag, sizeof(int32_t), cudaHostAllocMapped);
  if (e == cudaSuccess) *r->flag = 0;
  for (int i = 0; e == cudaSuccess && i < streams; ++i) {
    cudaStream_t st;
    e = cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    if (e == cudaSuccess) r->streams.push_back(st);
  }
  r->slots.resize(slots);
  const size_t nq = max_nq, nk = (size_t)max_nq * max_k, d = idx->d;
  for (auto& s : r->slots) {
    if (e == cudaSuccess) e = cudaMallocHost(&s.h_q, nq * d * sizeof(float));
    if (e == cudaSuccess) e = cudaMallocHost(&s.h_ids, nk * sizeof(int64_t));
    if (e == cudaSuccess) e = cudaMallocHost(&s.h_sc, nk * sizeof(float));
    if (e == cudaSuccess) e = cudaMallocHost(&s.h_lists, nq * sizeof(int32_t));
    if (e == cudaSuccess) e = cudaMalloc(&s.d_q, nq * d * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&s.d_ids, nk * sizeof(int64_t));
    if (e == cudaSuccess) e = cudaMalloc(&s.d_sc, nk * sizeof(float));
    if (e == cudaSuccess) e = cudaMalloc(&s.d_lists, nq * sizeof(int32_t));
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming);
  }
  if (e != cudaSuccess) {
    destroy(r);
    return cuda_status(e, "retriever create");
  }
  *out = r;
  return SA_OK;
}

}  // extern "C"

namespace {

// Alg. 1 LaunchAsyncRetrievalTask: stage the queries in a free slot's pinned buffer, enqueue
// H2D -> `search(d_q, d_ids, d_sc, d_lists, stream)` -> D2H on the next stream, record the
// slot's event and return the task id.  `lists_fill` >= 0: the per-query count reported
// instead of a device-written one.
template <typename Search>
sa_status submit_task(sa_retriever* r, const float* queries_host, int32_t nq, int32_t k,
                      bool device_lists, int32_t lists_fill, int32_t nprobe, int32_t mature,
                      int64_t* task_id, Search search) {
  if (!r || !queries_host || !task_id) return set_error(SA_ERR_INVALID_ARG, "null pointer");
  if (nq < 1 || nq > r->max_nq || k < 1 || k > r->max_k)
    return set_error(SA_ERR_INVALID_ARG, "nq / k outside the retriever's limits");
  std::lock_guard<std::mutex> lock(r->mu);
  sa_retriever::Slot* s = nullptr;
  for (auto& c : r->slots)
    if (!c.busy) {
      s = &c;
      break;
    }
  if (!s) return set_error(SA_ERR_STATE, "no free retrieval slot");
  cudaStream_t st = r->streams[r->next_stream];
  const int64_t d = r->idx->d;
  std::memcpy(s->h_q, queries_host, (size_t)nq * d * sizeof(float));
  sa_status rc = cuda_status(cudaMemcpyAsync(s->d_q, s->h_q, (size_t)nq * d * sizeof(float),
                                             cudaMemcpyHostToDevice, st),
                             "retrieval H2D");
  if (rc != SA_OK) return rc;
  rc = search(s->d_q, s->d_ids, s->d_sc, s->d_lists, st);
  if (rc != SA_OK) return rc;
  const size_t nk = (size_t)nq * k;
  rc = cuda_status(cudaMemcpyAsync(s->h_ids, s->d_ids, nk * 8, cudaMemcpyDeviceToHost, st), "D2H");
  if (rc == SA_OK)
    rc = cuda_status(cudaMemcpyAsync(s->h_sc, s->d_sc, nk * 4, cudaMemcpyDeviceToHost, st), "D2H");
  if (rc == SA_OK && device_lists)
    rc = cuda_status(cudaMemcpyAsync(s->h_lists, s->d_lists, (size_t)nq * 4,
                                     cudaMemcpyDeviceToHost, st),
                     "D2H");
  if (rc == SA_OK) rc = cuda_status(cudaEventRecord(s->done, st), "event");
  if (rc != SA_OK) return rc;
  if (!device_lists)
    for (int i = 0; i < nq; ++i) s->h_lists[i] = lists_fill;
  s->busy = true;
  s->task = r->next_task++;
  s->nq = nq;
  s->k = k;
  s->nprobe = nprobe;
  s->mature = mature;
  r->next_stream = (r->next_stream + 1) % r->streams.size();
  *task_id = s->task;
  return SA_OK;
}

}  // namespace

extern "C" {

sa_status sa_retriever_submit(sa_retriever* r, const float* queries_host, int32_t nq, int32_t k,
                              int32_t nprobe_max, int32_t mature, const sa_maturity_opts* opts,
                              int64_t* task_id) {
  if (mature && (!opts || nprobe_max < 1))
    return set_error(SA_ERR_INVALID_ARG, "maturity exit needs opts and nprobe_max >= 1");
  if (!r) return set_error(SA_ERR_INVALID_ARG, "null pointer");
  return submit_task(r, queries_host, nq, k, mature != 0, nprobe_max, nprobe_max, mature, task_id,
                     [&](float* dq, int64_t* dids, float* dsc, int32_t* dlists, cudaStream_t st) {
                       if (mature) {
                         sa_maturity_opts o = *opts;
                         o.engine_ready = r->flag;
                         return sa_search_mature(r->idx, dq, SA_F32, nq, k, nprobe_max, &o, dids,
                                                 dsc, dlists, nullptr, nullptr, st);
                       }
                       return sa_search_ex(r->idx, dq, SA_F32, nq, k, nprobe_max, dids, dsc, st);
                     });
}

sa_status sa_retriever_submit_graph(sa_retriever* r, const float* queries_host, int32_t nq,
                                    int32_t k, int32_t search_range, int32_t search_width,
                                    int32_t n_entries, int32_t mature,
                                    const sa_maturity_opts* opts, int64_t* task_id) {
  if (mature && !opts) return set_error(SA_ERR_INVALID_ARG, "maturity exit needs opts");
  if (!r) return set_error(SA_ERR_INVALID_ARG, "null pointer");
  return submit_task(r, queries_host, nq, k, mature != 0, -1, 0, mature, task_id,
                     [&](float* dq, int64_t* dids, float* dsc, int32_t* dsteps, cudaStream_t st) {
                       if (mature) {
                         sa_maturity_opts o = *opts;
                         o.engine_ready = r->flag;
                         return sa_search_graph_mature(r->idx, dq, SA_F32, nq, k, search_range,
                                                       search_width, n_entries, 1 << 30, &o, dids,
                                                       dsc, dsteps, nullptr, nullptr, 0, st);
                       }
                       return sa_search_graph(r->idx, dq, SA_F32, nq, k, search_range,
                                              search_width, n_entries, 1 << 30, dids, dsc,
                                              nullptr, st);
                     });
}

sa_status sa_retriever_poll(sa_retriever* r, int64_t task_id, int32_t* done) {
  if (!r || !done) return set_error(SA_ERR_INVALID_ARG, "null pointer");
  std::lock_guard<std::mutex> lock(r->mu);
  sa_retriever::Slot* s = find(r, task_id);
  if (!s) return set_error(SA_ERR_STATE, "unknown retrieval task");
  cudaError_t e = cudaEventQuery(s->done);
  if (e == cudaErrorNotReady) {
    *done = 0;
    return SA_OK;
  }
  if (e != cudaSuccess) return cuda_status(e, "retrieval task");
  *done = 1;
  return SA_OK;
}

sa_status sa_retriever_result(sa_retriever* r, int64_t task_id, int64_t* ids_host,
                              float* scores_host, int32_t* lists_host) {
  if (!r || !ids_host || !scores_host) return set_error(SA_ERR_INVALID_ARG, "null pointer");
  std::lock_guard<std::mutex> lock(r->mu);
  sa_retriever::Slot* s = find(r, task_id);
  if (!s) return set_error(SA_ERR_STATE, "unknown retrieval task");
  cudaError_t e = cudaEventQuery(s->done);
  if (e == cudaErrorNotReady) return set_error(SA_ERR_STATE, "retrieval task not finished");
  if (e != cudaSuccess) return cuda_status(e, "retrieval task");
  const size_t nk = (size_t)s->nq * s->k;
  std::memcpy(ids_host, s->h_ids, nk * 8);
  std::memcpy(scores_host, s->h_sc, nk * 4);
  if (lists_host) std::memcpy(lists_host, s->h_lists, (size_t)s->nq * 4);
  s->busy = false;
  s->task = -1;
  return SA_OK;
}

sa_status sa_retriever_set_engine_ready(sa_retriever* r, int32_t ready) {
  if (!r) return set_error(SA_ERR_INVALID_ARG, "null pointer");
  __atomic_store_n(r->flag, ready ? 1 : 0, __ATOMIC_RELEASE);
  return SA_OK;
}

sa_status sa_retriever_free(sa_retriever* r) {
  if (!r) return set_error(SA_ERR_INVALID_ARG, "null pointer");
  destroy(r);
  return SA_OK;
}

}  // extern "C"
