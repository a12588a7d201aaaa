// fp8_api.cu -- e4m3 flat scan with bf16 re-rank (readings
// R30-R33; include/sa.h for the contract).
//
// sa_index_build_fp8 keeps an e4m3 copy of the stored rows (one power-of-two scale for the
// whole corpus, the same on every rank); sa_search_fp8 stages the queries (bf16, and e4m3 with
// a per-query power-of-two scale), runs flat_scan_topk_kernel<CG, F8 = true> for the n_cand
// best candidates per query by fp8 score, then re-scores them on the bf16 rows and keeps the
// k best (rerank_kernel).  Sharded indexes: rank-local keys, ncclAllGather, merge -- as
// sa_search.
#include <algorithm>
#include <cstring>
#include <vector>

#include "internal.h"
#include "kernels/flat_scan.cuh"
#include "kernels/fp8.cuh"
#include "kernels/merge.cuh"

using namespace sa;

namespace {

sa_status fp8_search_local(const sa_index* idx, const void* queries, sa_dtype qdtype, int64_t nq,
                           int32_t k, int32_t nprobe, int32_t n_cand, const SearchOut& out,
                           cudaStream_t s) {
  const int64_t nq_pad = padded_nq(nq);
  __nv_bfloat16* Qs = nullptr;
  uint8_t* Q8 = nullptr;
  uint64_t* cand = nullptr;
  sa_status st = dalloc(&Qs, (size_t)nq_pad * idx->d_pad, s, "alloc staged queries");
  if (st == SA_OK) st = dalloc(&Q8, (size_t)nq_pad * idx->d8_pad, s, "alloc fp8 queries");
  if (st == SA_OK) st = dalloc(&cand, (size_t)nq * n_cand, s, "alloc candidates");
  if (st == SA_OK) {
    ProfRegion prof_region(SA_KERNEL_STAGE, s);
    cudaError_t e = launch_cast_pad(queries, qdtype == SA_F32, nq, idx->d, Qs, nq_pad, idx->d_pad,
                                    idx->num_sms, s);
    // R31: each query row on its own power-of-two scale (rows >= nq are zero -> stay zero)
    if (e == cudaSuccess)
      e = launch_quant_e4m3(Qs, nq_pad, idx->d_pad, nullptr, Q8, idx->d8_pad, nullptr,
                            idx->num_sms, s);
    st = cuda_status(e, "stage queries");
  }
  if (st == SA_OK) {
    // R32: the n_cand best stored rows by e4m3 score (all rows, or the rows of the nprobe
    // best lists -- probed on the bf16 query, as the bf16 IVF mode); keys carry stored positions
    SearchOut c;
    c.keys = cand;
    if (nprobe > 0) {
      st = ivf_search(idx, Qs, nq, nq_pad, n_cand, nprobe, c, s, Q8);
    } else {
      CorpusView cv{&idx->tmap_x8, &idx->tmap_x8_2, idx->n_local, idx->d8_pad / 2, nullptr, 0u,
                    true};
      st = flat_search_view(cv, idx->num_sms, reinterpret_cast<const __nv_bfloat16*>(Q8), nq,
                            n_cand, c, s);
    }
  }
  if (st == SA_OK) {
    RerankArgs r{};
    r.X = idx->X;
    r.d_pad = idx->d_pad;
    r.row_ids = idx->row_ids;
    r.row_offset = idx->row_offset;
    r.Qs = Qs;
    r.cand = cand;
    r.n_cand = n_cand;
    r.k = k;
    r.out_keys = out.keys;
    r.out_ids = out.ids;
    r.out_scores = out.scores;
    ProfRegion prof_region(SA_KERNEL_MERGE, s);
    st = cuda_status(launch_rerank(r, nq, s), "re-rank");
  }
  if (Qs) cudaFreeAsync(Qs, s);
  if (Q8) cudaFreeAsync(Q8, s);
  if (cand) cudaFreeAsync(cand, s);
  return st;
}

}  // namespace

extern "C" {

sa_status sa_index_build_fp8(sa_index* idx, void* stream) {
  if (!idx) return set_error(SA_ERR_INVALID_ARG, "null index");
  cudaStream_t s = (cudaStream_t)stream;
  const int32_t d8_pad = (idx->d_pad + 127) / 128 * 128;
  if (d8_pad / 2 > FS_MAX_DPAD) return set_error(SA_ERR_UNSUPPORTED, "d too large");
  const int64_t n = idx->n_local;
  uint8_t* X8 = nullptr;
  uint32_t* amax = nullptr;
  sa_status st = cuda_status(cudaMalloc(&X8, (size_t)n * d8_pad), "alloc fp8 corpus");
  if (st == SA_OK) st = cuda_status(cudaMalloc(&amax, 64 * sizeof(uint32_t)), "alloc");
  if (st == SA_OK) st = cuda_status(cudaMemsetAsync(amax, 0, 64 * sizeof(uint32_t), s), "memset");
  if (st == SA_OK)
    st = cuda_status(launch_absmax_bf16(idx->X, n, idx->d_pad, amax, idx->num_sms, s), "absmax");
  if (st == SA_OK && comm_sharded(idx->comm)) {
    // R30: one scale for the whole (sharded) corpus -> max over the ranks' maxima
    const int w = idx->comm->world;
    uint32_t* all = nullptr;
    st = cuda_status(cudaMalloc(&all, (size_t)w * sizeof(uint32_t)), "alloc");
    if (st == SA_OK) st = comm_allgather_bytes(idx->comm, amax, all, sizeof(uint32_t), s);
    std::vector<uint32_t> h(w);
    if (st == SA_OK)
      st = cuda_status(cudaMemcpyAsync(h.data(), all, w * sizeof(uint32_t),
                                       cudaMemcpyDeviceToHost, s), "copy");
    if (st == SA_OK) st = cuda_status(cudaStreamSynchronize(s), "sync");
    if (st == SA_OK) {
      const uint32_t m = *std::max_element(h.begin(), h.end());
      st = cuda_status(cudaMemcpyAsync(amax, &m, sizeof(uint32_t), cudaMemcpyHostToDevice, s),
                       "copy");
      if (st == SA_OK) st = cuda_status(cudaStreamSynchronize(s), "sync");
    }
    cudaFree(all);
  }
  int32_t* e_dev = reinterpret_cast<int32_t*>(amax + 32);
  if (st == SA_OK)
    st = cuda_status(launch_quant_e4m3(idx->X, n, idx->d_pad, amax, X8, d8_pad, e_dev,
                                       idx->num_sms, s),
                     "quantise corpus");
  int32_t e_host = 0;
  if (st == SA_OK)
    st = cuda_status(cudaMemcpyAsync(&e_host, e_dev, sizeof(int32_t), cudaMemcpyDeviceToHost, s),
                     "copy");
  if (st == SA_OK) st = cuda_status(cudaStreamSynchronize(s), "fp8 build sync");
  CUtensorMap t1, t2, t3;
  if (st == SA_OK) st = make_tmap_bf16(&t1, X8, n, d8_pad / 2, FS_BN);
  if (st == SA_OK) st = make_tmap_bf16(&t2, X8, n, d8_pad / 2, FS_BN / 2);
  if (st == SA_OK) st = make_tmap_bf16(&t3, X8, n, d8_pad / 2, FS_TAIL_ROWS);
  cudaFree(amax);
  if (st != SA_OK) {
    cudaFree(X8);
    return st;
  }
  cudaFree(idx->X8);
  idx->X8 = X8;
  idx->d8_pad = d8_pad;
  idx->x8_exp = e_host;
  idx->tmap_x8 = t1;
  idx->tmap_x8_2 = t2;
  idx->tmap_x8t = t3;
  return SA_OK;
}

sa_status sa_search_fp8(const sa_index* idx, const void* queries, sa_dtype qdtype, int64_t nq,
                        int32_t k, int32_t nprobe, int32_t n_cand, int64_t* out_ids,
                        float* out_scores, void* stream) {
  if (!idx) return set_error(SA_ERR_INVALID_ARG, "null index");
  sa_status st = SA_OK;
  if (!queries || !out_ids || !out_scores)
    st = set_error(SA_ERR_INVALID_ARG, "null pointer");
  else if (!idx->X8)
    st = set_error(SA_ERR_STATE, "no fp8 copy: call sa_index_build_fp8");
  else if (qdtype != SA_BF16 && qdtype != SA_F32)
    st = set_error(SA_ERR_INVALID_ARG, "bad qdtype");
  else if (nq < 1 || nq > (1ll << 31) / 2)
    st = set_error(SA_ERR_INVALID_ARG, "bad nq");
  else if (k < 1 || n_cand < k || n_cand > F8_MAX_CAND)
    st = set_error(SA_ERR_INVALID_ARG, "need 1 <= k <= n_cand <= 256");
  else if (nprobe < 0 || nprobe > idx->nlist)
    st = set_error(nprobe > 0 && idx->nlist == 0 ? SA_ERR_STATE : SA_ERR_INVALID_ARG,
                   "need 0 <= nprobe <= nlist");
  cudaStream_t s = (cudaStream_t)stream;
  const bool sharded = comm_sharded(idx->comm);
  if (sharded) {
    const int64_t args[kCommArgs] = {0x5a58, nq, k, nprobe, (int64_t)qdtype, n_cand};
    st = comm_check_args(idx->comm, args, st, s);
  }
  if (st != SA_OK) return st;
  if (!sharded) {
    SearchOut out;
    out.ids = out_ids;
    out.scores = out_scores;
    return fp8_search_local(idx, queries, qdtype, nq, k, nprobe, n_cand, out, s);
  }
  uint64_t* keys_local = nullptr;
  st = dalloc(&keys_local, (size_t)nq * k, s, "alloc local keys");
  if (st == SA_OK) {
    SearchOut out;
    out.keys = keys_local;
    st = fp8_search_local(idx, queries, qdtype, nq, k, nprobe, n_cand, out, s);
  }
  if (st == SA_OK) st = gather_merge_keys(idx, keys_local, nq, k, out_ids, out_scores, s);
  if (keys_local) cudaFreeAsync(keys_local, s);
  return st;
}

sa_status sa_index_export_fp8(const sa_index* idx, uint8_t* host_out, int32_t* scale_exp) {
  if (!idx || !scale_exp) return set_error(SA_ERR_INVALID_ARG, "null pointer");
  if (!idx->X8) return set_error(SA_ERR_STATE, "no fp8 copy: call sa_index_build_fp8");
  *scale_exp = idx->x8_exp;
  if (!host_out) return SA_OK;
  const int64_t n = idx->n_local;
  std::vector<uint8_t> buf((size_t)n * idx->d8_pad);
  std::vector<int32_t> ids;
  cudaError_t e = cudaMemcpy(buf.data(), idx->X8, buf.size(), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && idx->row_ids) {
    ids.resize(n);
    e = cudaMemcpy(ids.data(), idx->row_ids, n * 4, cudaMemcpyDeviceToHost);
  }
  if (e != cudaSuccess) return cuda_status(e, "export fp8");
  // rows in local-id order (global id - row_offset), the first d bytes of each
  for (int64_t p = 0; p < n; ++p) {
    const int64_t r = ids.empty() ? p : (int64_t)(uint32_t)ids[p] - idx->row_offset;
    std::memcpy(host_out + r * idx->d, buf.data() + (size_t)p * idx->d8_pad, idx->d);
  }
  return SA_OK;
}

}  // extern "C"
