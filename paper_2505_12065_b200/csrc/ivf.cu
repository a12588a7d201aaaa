// ivf.cu -- IVF coarse quantiser build and IVF search (§8(a) a2, a3, a7, a8).
//
// The paper's retriever is an HNSW graph whose "search range" trades recall for
// effort (§2.2.1; App. B.3 efSearch).  BJ
// replaces it with an inverted-file index whose nprobe knob plays that role.
// Everything that is a dense contraction runs on the tcgen05 flat kernel:
//   * k-means assignment (a2) and the full assignment (a3): queries = rows,
//     corpus = the bf16 centroids, k = 1 (ties -> lowest list id, R8);
//   * the probe (a7): queries x centroids, k = nprobe (ties -> lowest id, R11);
//   * the list scan (a8): ivf_scan.cu (list rows on the MMA M side, the probing
//     queries of a list on N).
// The rest (sample gather, stable sort by list, deterministic centroid update,
// empty-list repair, probe inversion) is SIMT glue in ivf_kernels.cu.
#include <algorithm>
#include <vector>

#include "internal.h"
#include "kernels/flat_scan.cuh"
#include "kernels/ivf_kernels.cuh"
#include "kernels/ivf_scan.cuh"
#include "kernels/ivf_small.cuh"
#include "kernels/launch.cuh"
#include "kernels/merge.cuh"

namespace sa {

namespace {
// Rows per IVF work item (multiple of FS_BN), between these bounds: big batches have many
// lists to spread over the SMs; small (agent-step) batches probe only a few dozen lists, so
// lists are cut into short chunks to put every SM on the few lists there are.
constexpr int kChunkRows = 4096;
constexpr int kChunkRowsSmall = 256;

// Stable sort of rows by list id + CSR offsets: perm = rows in list-major order (ascending row
// inside a list), off[nlist + 1].
sa_status sort_by_list(const int64_t* ids, int64_t n, int nlist, int num_sms, int32_t* perm,
                       int64_t* off, cudaStream_t s) {
  StreamFreer f{s};
  int32_t *keys, *ktmp, *vtmp, *kout;
  int64_t *counts, *offs, *scratch, *hist;
  const int64_t cs = sort_counts_size(n);
  SA_TRY(dalloc(&keys, n, s, "sort keys"));
  f.add(keys);
  SA_TRY(dalloc(&ktmp, n, s, "sort tmp"));
  f.add(ktmp);
  SA_TRY(dalloc(&vtmp, n, s, "sort tmp"));
  f.add(vtmp);
  SA_TRY(dalloc(&kout, n, s, "sort out"));
  f.add(kout);
  SA_TRY(dalloc(&counts, cs, s, "sort counts"));
  f.add(counts);
  SA_TRY(dalloc(&offs, cs + 1, s, "sort offs"));
  f.add(offs);
  const int64_t sc = std::max<int64_t>(cs, nlist) / 1024 + 4;
  SA_TRY(dalloc(&scratch, sc, s, "scan scratch"));
  f.add(scratch);
  SA_TRY(dalloc(&hist, nlist, s, "hist"));
  f.add(hist);
  SA_CUDA(launch_i64_to_i32(ids, n, keys, num_sms, s), "ids->keys");
  SA_CUDA(stable_sort_by_key16(keys, n, ktmp, vtmp, kout, perm, counts, offs, scratch, s), "sort");
  SA_CUDA(cudaMemsetAsync(hist, 0, sizeof(int64_t) * nlist, s), "memset");
  SA_CUDA(launch_histogram(keys, n, hist, num_sms, s), "histogram");
  SA_CUDA(exclusive_scan_i64(hist, nlist, off, scratch, s), "scan");
  return SA_OK;
}

}  // namespace

// list sharding: dst[d0 + i] = src[s0 + i] for every kept list's segment (s0, d0, len)
static __global__ void copy_segments_kernel(const int32_t* __restrict__ src, const int64_t* __restrict__ seg,
                                     int nseg, int32_t* __restrict__ dst) {
  for (int g = blockIdx.x; g < nseg; g += gridDim.x) {
    const int64_t s0 = seg[3 * g], d0 = seg[3 * g + 1], len = seg[3 * g + 2];
    for (int64_t i = threadIdx.x; i < len; i += blockDim.x) dst[d0 + i] = src[s0 + i];
  }
}

sa_status ivf_build(sa_index* idx, const sa_build_opts& o, cudaStream_t s) {
  const int nlist = idx->nlist;
  const int dp = idx->d_pad;
  const int sms = idx->num_sms;
  const int64_t n = idx->n_local;
  if (nlist > 65536) return set_error(SA_ERR_UNSUPPORTED, "nlist > 65536");
  const int64_t n_total = idx->n_total;
  // list sharding trains on the full corpus every rank holds: no training collective
  const sa_comm* comm = comm_sharded(idx->comm) && idx->list_world == 0 ? idx->comm : nullptr;
  const int64_t n_train = std::min<int64_t>(n_total, (int64_t)o.train_per_list * nlist);
  StreamFreer f{s};

  SA_CUDA(cudaMalloc(&idx->centroids, (size_t)nlist * dp * sizeof(float)), "alloc centroids");
  SA_CUDA(cudaMalloc(&idx->centroids_bf16, (size_t)nlist * dp * sizeof(__nv_bfloat16)),
          "alloc centroids bf16");
  SA_TRY(make_tmap_bf16(&idx->tmap_c, idx->centroids_bf16, nlist, dp, FS_BN));
  SA_TRY(make_tmap_bf16(&idx->tmap_c2, idx->centroids_bf16, nlist, dp, FS_BN / 2));
  const CorpusView cvc{&idx->tmap_c, &idx->tmap_c2, nlist, dp, nullptr, 0u};
  const bool train = o.centroids == nullptr;

  // ---- a2: training sample by global id (R9).  Shards are contiguous row ranges, so rank r
  // owns the contiguous sample range t in [ceil(off_r * n_train / n_total), ...): each rank
  // gathers its part and NCCL broadcasts assemble the identical full sample everywhere.
  __nv_bfloat16* sample = nullptr;
  if (train) {
    SA_TRY(dalloc(&sample, (size_t)n_train * dp, s, "alloc sample"));
    f.add(sample);
    const int world = comm ? comm->world : 1;
    std::vector<int64_t> toff(world + 1), boff(world), blen(world);
    for (int r = 0; r <= world; ++r) {
      int64_t off_r = n_total, len_r = 0;
      if (r < world) shard_range(n_total, world, r, &off_r, &len_r);
      // smallest t with floor(t * n_total / n_train) >= off_r
      toff[r] = (off_r * n_train + n_total - 1) / n_total;
    }
    const int me = comm ? comm->rank : 0;
    if (comm) {
      int64_t off_me, len_me;
      shard_range(n_total, world, me, &off_me, &len_me);
      if (off_me != idx->row_offset || len_me != n)
        return set_error(SA_ERR_INVALID_ARG,
                         "sharded IVF build expects the balanced split off_r = r*floor(n/w) + "
                         "min(r, n mod w)");
    }
    SA_CUDA(launch_gather_rows(idx->X, dp, nullptr, n_total, idx->row_offset, toff[me], n_train,
                               toff[me + 1] - toff[me], sample + (size_t)toff[me] * dp, sms, s),
            "gather sample");
    if (comm) {
      for (int r = 0; r < world; ++r) {
        boff[r] = toff[r] * dp * (int64_t)sizeof(__nv_bfloat16);
        blen[r] = (toff[r + 1] - toff[r]) * dp * (int64_t)sizeof(__nv_bfloat16);
      }
      SA_TRY(comm_broadcast_parts(comm, sample, boff.data(), blen.data(), s));
    }
    SA_CUDA(launch_init_centroids(sample, dp, nlist, n_train, o.seed, idx->centroids, s), "init");
  } else {
    // caller-provided quantiser: fp32 [nlist, d] -> [nlist, d_pad], zero padded
    SA_CUDA(cudaMemsetAsync(idx->centroids, 0, (size_t)nlist * dp * sizeof(float), s), "memset");
    SA_CUDA(cudaMemcpy2DAsync(idx->centroids, (size_t)dp * sizeof(float), o.centroids,
                              (size_t)idx->d * sizeof(float), (size_t)idx->d * sizeof(float), nlist,
                              cudaMemcpyDeviceToDevice, s),
            "copy centroids");
  }

  int64_t* ids;
  float* scores;
  int32_t* perm;
  int64_t* off;
  int32_t *empty_flag, *n_empty;
  uint64_t *rkeys, *rsel;
  SA_TRY(dalloc(&ids, n_train, s, "alloc ids"));
  f.add(ids);
  SA_TRY(dalloc(&scores, n_train, s, "alloc scores"));
  f.add(scores);
  SA_TRY(dalloc(&perm, n_train, s, "alloc perm"));
  f.add(perm);
  SA_TRY(dalloc(&off, nlist + 1, s, "alloc off"));
  f.add(off);
  SA_TRY(dalloc(&empty_flag, nlist, s, "alloc flags"));
  f.add(empty_flag);
  SA_TRY(dalloc(&n_empty, 1, s, "alloc n_empty"));
  f.add(n_empty);
  SA_TRY(dalloc(&rkeys, n_train, s, "alloc repair keys"));
  f.add(rkeys);
  SA_TRY(dalloc(&rsel, 256, s, "alloc repair sel"));
  f.add(rsel);

  for (int it = 0; train && it < o.kmeans_iters; ++it) {
    SA_CUDA(launch_f32_to_bf16(idx->centroids, (int64_t)nlist * dp, idx->centroids_bf16, sms, s),
            "centroids->bf16");
    SearchOut so;
    so.ids = ids;
    so.scores = scores;
    SA_TRY(flat_search_view(cvc, sms, sample, n_train, 1, so, s));   // assignment (GEMM + top-1)
    SA_TRY(sort_by_list(ids, n_train, nlist, sms, perm, off, s));
    SA_CUDA(cudaMemsetAsync(n_empty, 0, sizeof(int32_t), s), "memset");
    SA_CUDA(launch_centroid_update(sample, dp, perm, off, nlist, idx->centroids, empty_flag, n_empty,
                                   s),
            "centroid update");
    int32_t h_empty = 0;
    SA_CUDA(cudaMemcpyAsync(&h_empty, n_empty, sizeof(int32_t), cudaMemcpyDeviceToHost, s), "D2H");
    SA_CUDA(cudaStreamSynchronize(s), "sync");
    if (h_empty > 0) {
      // R10: empty lists take the sample rows with the lowest assigned score
      int left = h_empty;
      if (left > 256) return set_error(SA_ERR_UNSUPPORTED, "more than 256 empty IVF lists");
      SA_CUDA(launch_repair_keys(scores, n_train, rkeys, sms, s), "repair keys");
      MergeArgs m{};
      m.cand = rkeys;
      m.k = left;
      m.qstride = 0;
      m.m_flat = n_train;
      m.out_keys = rsel;
      SA_CUDA(launch_merge(m, 1, s), "repair select");
      SA_CUDA(launch_repair_apply(sample, dp, nlist, empty_flag, rsel, idx->centroids, s),
              "repair apply");
    }
  }
  SA_CUDA(launch_f32_to_bf16(idx->centroids, (int64_t)nlist * dp, idx->centroids_bf16, sms, s),
          "centroids->bf16");

  // ---- a3: assign every local row, sort list-major, permute
  int64_t* ids_all;
  float* sc_all;
  int32_t* perm_all;
  SA_TRY(dalloc(&ids_all, n, s, "alloc ids"));
  f.add(ids_all);
  SA_TRY(dalloc(&sc_all, n, s, "alloc scores"));
  f.add(sc_all);
  SA_TRY(dalloc(&perm_all, n, s, "alloc perm"));
  f.add(perm_all);
  {
    SearchOut so;
    so.ids = ids_all;
    so.scores = sc_all;
    SA_TRY(flat_search_view(cvc, sms, idx->X, n, 1, so, s));
  }
  SA_CUDA(cudaMalloc(&idx->list_off, (nlist + 1) * sizeof(int64_t)), "alloc list offsets");
  SA_TRY(sort_by_list(ids_all, n, nlist, sms, perm_all, idx->list_off, s));
  int64_t n_keep = n;
  if (idx->list_world > 0) {
    // list sharding: keep the whole lists l % W == R (list-major order, so each is one
    // contiguous segment of the sorted permutation); the other lists become empty
    std::vector<int64_t> off(nlist + 1), noff(nlist + 1, 0), seg;
    SA_CUDA(cudaMemcpyAsync(off.data(), idx->list_off, (nlist + 1) * sizeof(int64_t),
                            cudaMemcpyDeviceToHost, s), "list offsets D2H");
    SA_CUDA(cudaStreamSynchronize(s), "list offsets");
    for (int l = 0; l < nlist; ++l) {
      const int64_t len = l % idx->list_world == idx->list_rank ? off[l + 1] - off[l] : 0;
      noff[l + 1] = noff[l] + len;
      if (len > 0) seg.insert(seg.end(), {off[l], noff[l], len});
    }
    n_keep = noff[nlist];
    if (n_keep == 0) return set_error(SA_ERR_UNSUPPORTED, "this list shard owns no rows");
    int64_t* dseg;
    int32_t* perm_keep;
    SA_TRY(dalloc(&dseg, seg.size(), s, "alloc segments"));
    f.add(dseg);
    SA_TRY(dalloc(&perm_keep, (size_t)n_keep, s, "alloc kept permutation"));
    f.add(perm_keep);
    SA_CUDA(cudaMemcpyAsync(dseg, seg.data(), seg.size() * sizeof(int64_t), cudaMemcpyHostToDevice,
                            s), "segments H2D");
    SA_CUDA(cudaMemcpyAsync(idx->list_off, noff.data(), (nlist + 1) * sizeof(int64_t),
                            cudaMemcpyHostToDevice, s), "list offsets H2D");
    const int nseg = (int)(seg.size() / 3);
    copy_segments_kernel<<<std::min(nseg, sms * 8), 256, 0, s>>>(perm_all, dseg, nseg, perm_keep);
    note_launch();
    SA_CUDA(cudaGetLastError(), "copy segments");
    SA_CUDA(cudaStreamSynchronize(s), "list shard");   // seg / noff (host) outlive the copies
    perm_all = perm_keep;
  }
  __nv_bfloat16* Xp = nullptr;
  SA_CUDA(cudaMalloc(&Xp, (size_t)n_keep * dp * sizeof(__nv_bfloat16)), "alloc list-major corpus");
  cudaError_t e = launch_gather_rows(idx->X, dp, perm_all, 0, 0, 0, 1, n_keep, Xp, sms, s);
  // +4 entries: the agent-step kernel bulk-copies 16-byte-aligned id ranges (ivf_small.cu)
  if (e == cudaSuccess) e = cudaMalloc(&idx->row_ids, ((size_t)n_keep + 4) * sizeof(int32_t));
  if (e == cudaSuccess) e = launch_perm_ids(perm_all, n_keep, idx->row_offset, idx->row_ids, sms, s);
  if (e == cudaSuccess) e = cudaMemsetAsync(idx->row_ids + n_keep, 0xff, 4 * sizeof(int32_t), s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) {
    cudaFree(Xp);
    return cuda_status(e, "permute corpus");
  }
  cudaFree(idx->X);
  idx->X = Xp;
  idx->n_local = n_keep;
  SA_TRY(make_tmap_bf16(&idx->tmap_x, idx->X, n_keep, dp, FS_BN));
  SA_TRY(make_tmap_bf16(&idx->tmap_x2, idx->X, n_keep, dp, FS_BN / 2));
  SA_TRY(make_tmap_bf16(&idx->tmap_xt, idx->X, n_keep, dp, FS_TAIL_ROWS));
  idx->h_list_off.resize(nlist + 1);
  SA_CUDA(cudaMemcpy(idx->h_list_off.data(), idx->list_off, (nlist + 1) * sizeof(int64_t),
                     cudaMemcpyDeviceToHost),
          "list offsets D2H");
  idx->max_list = 0;
  for (int l = 0; l < nlist; ++l)
    idx->max_list = std::max<int64_t>(idx->max_list, idx->h_list_off[l + 1] - idx->h_list_off[l]);
  return SA_OK;
}

// a7: centroid scores on the tensor cores (dumped, nq x nlist fp32 -- 32 MB at nq=512,
// L2-resident), then an exact per-query top-nprobe radix select (ties -> lowest id, R11).
// Sorted packed keys [nq, nprobe] (list id in the key).
static sa_status probe_keys(const sa_index* idx, const __nv_bfloat16* Qs, int64_t nq,
                            int32_t nprobe, uint64_t* pkeys, cudaStream_t s) {
  StreamFreer f{s};
  float* sc;
  SA_TRY(dalloc(&sc, (size_t)nq * idx->nlist, s, "alloc probe scores"));
  f.add(sc);
  const CorpusView cvc{&idx->tmap_c, &idx->tmap_c2, idx->nlist, idx->d_pad, nullptr, 0u};
  SA_TRY(flat_scores_view(cvc, idx->num_sms, Qs, nq, sc, s));
  MergeArgs m{};
  m.cand_scores = sc;
  m.m_flat = idx->nlist;
  m.qstride = idx->nlist;
  m.k = nprobe;
  m.out_keys = pkeys;
  SA_CUDA(launch_merge(m, nq, s), "probe select");
  return SA_OK;
}

sa_status ivf_probe(const sa_index* idx, const __nv_bfloat16* Qs, int64_t nq, int64_t nq_pad,
                    int32_t nprobe, int32_t* out_lists, cudaStream_t s) {
  (void)nq_pad;
  StreamFreer f{s};
  uint64_t* pkeys;
  SA_TRY(dalloc(&pkeys, (size_t)nq * nprobe, s, "alloc probe keys"));
  f.add(pkeys);
  SA_TRY(probe_keys(idx, Qs, nq, nprobe, pkeys, s));
  SA_CUDA(launch_keys_to_lists(pkeys, nq * nprobe, nullptr, out_lists, idx->num_sms, s), "lists");
  return SA_OK;
}

bool ivf_small_applies(const sa_index* idx, int64_t nq, int32_t k, int32_t nprobe) {
  const int G = idx->num_sms;
  return idx->nlist > 0 && idx->row_ids && idx->n_local < (1ll << 31) && nq >= 1 &&
         nq <= IVSM_MAX_NQ && k <= IVSM_MAX_K &&
         nprobe >= 1 && nprobe <= IVSM_MAX_NPROBE && G >= nq && idx->d_pad <= 768 &&
         nprobe <= idx->nlist && ivf_small_fits((int)nq, nprobe, idx->nlist, G);
}

// Scratch of one agent-step search: the sizes of its four arrays, in one block.
static void small_scratch_layout(const sa_index* idx, int64_t nq, int32_t k, int32_t nprobe,
                                 size_t off[5]) {
  const int grid = idx->num_sms;
  const size_t n_top = (size_t)nq * grid * (ivf_small_m(nprobe, grid) + IVSM_EXTRA);
  const size_t n_pc = (size_t)nq * idx->nlist, n_cand = (size_t)grid * nq * k;
  off[0] = 0;                                   // top   (u64)
  off[1] = off[0] + n_top * 8;                  // pcand (u64)
  off[2] = off[1] + n_pc * 8;                   // cand  (u64)
  off[3] = off[2] + n_cand * 8;                 // counters (i32) [nq + 1], seq, q-ready
  off[4] = off[3] + ((size_t)nq + 3) * 4;       // total
}

sa_status ivf_small_scratch_alloc(const sa_index* idx, int64_t nq, int32_t k, int32_t nprobe,
                                  void** scratch) {
  size_t off[5];
  small_scratch_layout(idx, nq, k, nprobe, off);
  sa_status st = cuda_status(cudaMalloc(scratch, off[4]), "ivf small scratch");
  if (st == SA_OK) st = cuda_status(cudaMemset(*scratch, 0, off[4]), "ivf small scratch");
  return st;
}

// Agent-step batches: probe + list scan + merge in one cooperative launch (ivf_small.cu),
// straight from the caller's queries (no staging kernel).
sa_status ivf_small_search(const sa_index* idx, const void* queries, bool q_f32, int64_t nq,
                           int32_t k, int32_t nprobe, const SearchOut& out, cudaStream_t s,
                           int64_t* debug_ns, void* scratch, int32_t* done_host,
                           const void* queries_host) {
  const int grid = idx->num_sms;
  StreamFreer f{s};
  size_t off[5];
  small_scratch_layout(idx, nq, k, nprobe, off);
  uint8_t* base = static_cast<uint8_t*>(scratch);
  if (!base) SA_TRY(f.alloc(&base, off[4], "ivf small scratch"));
  IvfSmallArgs a{};
  a.top = reinterpret_cast<uint64_t*>(base + off[0]);
  a.pcand = reinterpret_cast<uint64_t*>(base + off[1]);
  a.cand = reinterpret_cast<uint64_t*>(base + off[2]);
  a.counters = reinterpret_cast<int32_t*>(base + off[3]);
  a.Q = queries;
  a.q_f32 = q_f32 ? 1 : 0;
  a.nq = (int32_t)nq;
  a.d = idx->d;
  a.d_pad = idx->d_pad;
  a.C = idx->centroids_bf16;
  a.nlist = idx->nlist;
  a.nprobe = nprobe;
  a.X = idx->X;
  a.list_off = idx->list_off;
  a.row_ids = idx->row_ids;
  a.k = k;
  a.debug_ns = debug_ns;
  a.seq = a.counters + nq + 1;
  a.q_ready = a.counters + nq + 2;
  a.done_host = done_host;
  a.Q_host = queries_host;
  a.out_keys = out.keys;
  a.out_ids = out.ids;
  a.out_scores = out.scores;
  ProfRegion prof_region(SA_KERNEL_IVF_SCAN, s);
  return cuda_status(launch_ivf_small(a, grid, s), "ivf small-batch search");
}

sa_status ivf_search(const sa_index* idx, const __nv_bfloat16* Qs, int64_t nq, int64_t nq_pad,
                     int32_t k, int32_t nprobe, const SearchOut& out, cudaStream_t s,
                     const uint8_t* Q8) {
  (void)nq_pad;
  const int nlist = idx->nlist;
  const int sms = idx->num_sms;
  const int64_t np = nq * nprobe;
  StreamFreer f{s};
  // ---- a7: probe = top-nprobe centroids per query on the tensor cores
  uint64_t* pkeys;
  int64_t* probes;
  SA_TRY(dalloc(&pkeys, np, s, "alloc probe keys"));
  f.add(pkeys);
  SA_TRY(dalloc(&probes, np, s, "alloc probes"));
  f.add(probes);
  {
    ProfRegion prof_region(SA_KERNEL_IVF_PROBE, s);
    sa_status st = probe_keys(idx, Qs, nq, nprobe, pkeys, s);
    if (st != SA_OK) return st;
  }
  SA_CUDA(launch_keys_to_lists(pkeys, np, probes, nullptr, sms, s), "probe lists");

  // ---- invert: lists -> probing queries, output slots, work items
  // aim for ~4 work items per SM: rows probed ~= np * mean list length
  const int64_t mean_list = std::max<int64_t>(1, idx->n_local / nlist);
  int64_t want = np * mean_list / (4 * (int64_t)sms);
  want = (want + FS_BN - 1) / FS_BN * FS_BN;
  const int chunk_rows = (int)std::min<int64_t>(kChunkRows, std::max<int64_t>(kChunkRowsSmall, want));
  const int64_t max_chunks = std::max<int64_t>(1, (idx->max_list + chunk_rows - 1) / chunk_rows);
  IvfSearchScratch w{};
  SA_TRY(dalloc(&w.cnt, nlist, s, "ivf scratch"));
  f.add(w.cnt);
  SA_TRY(dalloc(&w.cursor, nlist, s, "ivf scratch"));
  f.add(w.cursor);
  SA_TRY(dalloc(&w.tmp64, nlist + 1, s, "ivf scratch"));
  f.add(w.tmp64);
  SA_TRY(dalloc(&w.tmp64b, np, s, "ivf scratch"));
  f.add(w.tmp64b);
  SA_TRY(dalloc(&w.lq_off64, nlist + 1, s, "ivf scratch"));
  f.add(w.lq_off64);
  SA_TRY(dalloc(&w.lq_ent, np, s, "ivf scratch"));
  f.add(w.lq_ent);
  SA_TRY(dalloc(&w.q_slot, np + 1, s, "ivf scratch"));
  f.add(w.q_slot);
  SA_TRY(dalloc(&w.item_off, nlist + 1, s, "ivf scratch"));
  f.add(w.item_off);
  SA_TRY(dalloc(&w.items, (size_t)np * max_chunks, s, "ivf items"));
  f.add(w.items);
  SA_TRY(dalloc(&w.n_items, 1, s, "ivf scratch"));
  f.add(w.n_items);
  SA_TRY(dalloc(&w.scratch, std::max<int64_t>(nlist, np) / 1024 + 4, s, "ivf scratch"));
  f.add(w.scratch);
  if (np <= kInvertSmallMax) {
    SA_CUDA(launch_invert_small(probes, (int)nq, nprobe, idx->list_off, chunk_rows, IVS_NQ, w, s),
            "probe inversion");
  } else {
    SA_CUDA(launch_probe_invert(probes, nq, nprobe, nlist, idx->list_off, chunk_rows, IVS_NQ, w, sms, s),
            "probe inversion");
  }

  // ---- a8: list-major scan on the tensor cores
  const size_t max_slots = (size_t)np * max_chunks;
  uint64_t *part, *heap = nullptr;
  SA_TRY(dalloc(&part, max_slots * IVS_PARTS * k, s, "ivf partials"));
  f.add(part);
  if (k > IVS_KSMEM) {
    SA_TRY(dalloc(&heap, (size_t)sms * k * IVS_HEAPS, s, "ivf heaps"));
    f.add(heap);
  }
  uint32_t* hint;   // [nq] pruning bounds + [1] dynamic item counter
  SA_TRY(dalloc(&hint, nq + 1, s, "ivf hints"));
  f.add(hint);
  SA_CUDA(cudaMemsetAsync(hint, 0, sizeof(uint32_t) * (nq + 1), s), "memset hints");
  {
    IvfScanArgs v{};
    v.Q = Q8 ? reinterpret_cast<const __nv_bfloat16*>(Q8) : Qs;
    v.d_pad = Q8 ? idx->d8_pad / 2 : idx->d_pad;
    v.fp8 = Q8 ? 1 : 0;
    v.k = k;
    v.row_ids = Q8 ? nullptr : idx->row_ids;
    v.part = part;
    v.heap_g = heap;
    v.items = w.items;
    v.n_items = w.n_items;
    v.list_off = idx->list_off;
    v.lq_ent = w.lq_ent;
    v.q_slot = w.q_slot;
    v.nprobe = nprobe;
    v.chunk_rows = chunk_rows;
    v.q_hint = hint;
    v.item_counter = reinterpret_cast<int32_t*>(hint + nq);
    ProfRegion prof_region(SA_KERNEL_IVF_SCAN, s);
    SA_CUDA(Q8 ? launch_ivf_scan(idx->tmap_x8, idx->tmap_x8t, v, sms, s)
               : launch_ivf_scan(idx->tmap_x, idx->tmap_xt, v, sms, s),
            "ivf scan");
  }

  MergeArgs m{};
  m.cand = part;
  m.k = k;
  m.slot_off = w.q_slot;
  m.slot_stride = nprobe;
  m.slot_keys = IVS_PARTS * k;
  m.out_keys = out.keys;
  m.out_ids = out.ids;
  m.out_scores = out.scores;
  ProfRegion prof_region(SA_KERNEL_MERGE, s);
  return cuda_status(launch_merge(m, nq, s), "ivf merge");
}

}  // namespace sa
