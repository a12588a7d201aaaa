// ivf_kernels.cuh -- launchers of the IVF build / search SIMT kernels (ivf_kernels.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace sa {

uint64_t host_splitmix64(uint64_t z);

// out[t] = X[idx[t]] (idx != nullptr), else the training-sample rows t0 .. t0+n_out-1 of an
// n_train-row sample strided by global id over n_total rows (local row = global - row_offset).
cudaError_t launch_gather_rows(const __nv_bfloat16* X, int d_pad, const int32_t* idx,
                               int64_t n_total, int64_t row_offset, int64_t t0, int64_t n_train,
                               int64_t n_out, __nv_bfloat16* out, int num_sms, cudaStream_t s);
cudaError_t launch_init_centroids(const __nv_bfloat16* sample, int d_pad, int nlist,
                                  int64_t n_train, uint64_t seed, float* cent, cudaStream_t s);
cudaError_t launch_f32_to_bf16(const float* in, int64_t n, __nv_bfloat16* out, int num_sms,
                               cudaStream_t s);
cudaError_t exclusive_scan_i64(const int64_t* in, int64_t n, int64_t* out, int64_t* scratch,
                               cudaStream_t s);
// Stable sort of positions 0..n-1 by 16-bit keys: keys_out = sorted keys, vals_out = positions.
// counts/offs: 256 * ceil(n / 2048) int64 each; scratch: counts / 1024 + 2 int64.
cudaError_t stable_sort_by_key16(const int32_t* keys, int64_t n, int32_t* keys_tmp,
                                 int32_t* vals_tmp, int32_t* keys_out, int32_t* vals_out,
                                 int64_t* counts, int64_t* offs, int64_t* scratch, cudaStream_t s);
inline int64_t sort_counts_size(int64_t n) { return 256 * ((n + 2047) / 2048); }
cudaError_t launch_histogram(const int32_t* keys, int64_t n, int64_t* hist, int num_sms,
                             cudaStream_t s);
cudaError_t launch_i64_to_i32(const int64_t* in, int64_t n, int32_t* out, int num_sms,
                              cudaStream_t s);
cudaError_t launch_centroid_update(const __nv_bfloat16* sample, int d_pad, const int32_t* rows,
                                   const int64_t* off, int nlist, float* cent,
                                   int32_t* empty_flag, int32_t* n_empty, cudaStream_t s);
cudaError_t launch_repair_keys(const float* scores, int64_t n, uint64_t* keys, int num_sms,
                               cudaStream_t s);
cudaError_t launch_repair_apply(const __nv_bfloat16* sample, int d_pad, int nlist,
                                const int32_t* empty_flag, const uint64_t* sel, float* cent,
                                cudaStream_t s);
cudaError_t launch_keys_to_lists(const uint64_t* keys, int64_t n, int64_t* lists, int32_t* lists32,
                                 int num_sms, cudaStream_t s);
cudaError_t launch_perm_ids(const int32_t* perm, int64_t n, int64_t row_offset, int32_t* ids,
                            int num_sms, cudaStream_t s);

// Device scratch of one IVF search (probe inversion + work items).
struct IvfSearchScratch {
  int32_t* cnt;        // [nlist] probers per list
  int32_t* cursor;     // [nlist]
  int64_t* tmp64;      // [nlist + 1]
  int64_t* tmp64b;     // [nq * nprobe]
  int64_t* lq_off64;   // [nlist + 1]
  int2* lq_ent;        // [nq * nprobe] (query, probe rank) grouped by list
  int64_t* q_slot;     // [nq * nprobe + 1] first output slot of (q, j)
  int64_t* item_off;   // [nlist + 1]
  int4* items;         // [<= nq * nprobe * max_chunks]
  int32_t* n_items;    // [1]
  int64_t* scratch;    // [ceil(max(nlist, nq*nprobe) / 1024) + 2]
};
constexpr int kInvertSmallMax = 4096;  // nq * nprobe handled by one-CTA inversion
// Work items = (list, block of <= qblock probers, chunk of chunk_rows rows).
cudaError_t launch_invert_small(const int64_t* probes, int nq, int nprobe, const int64_t* list_off,
                                int chunk_rows, int qblock, IvfSearchScratch& w, cudaStream_t s);
// Maturity stages (mature.cu): the inversion computes its own probe table -- entry (q, j) of
// stage s = ctrl[0] probes list probes_full[q, s*g + j] if active[q] and s*g + j < P, else none
// (-1) -- into `stage_probes`, and zeroes the scan's item counter.
struct StageSrc {
  const int64_t* probes_full = nullptr;  // [nq, P] probe order
  int32_t P = 0;
  const int32_t* ctrl = nullptr;         // [0] = stage
  const int32_t* active = nullptr;       // [nq]
  int32_t* item_counter = nullptr;
};
cudaError_t launch_invert_stage(int64_t* stage_probes, int nq, int g, const StageSrc& src,
                                const int64_t* list_off, int chunk_rows, int qblock,
                                IvfSearchScratch& w, cudaStream_t s);
cudaError_t launch_probe_invert(const int64_t* probes, int64_t nq, int nprobe, int nlist,
                                const int64_t* list_off, int chunk_rows, int qblock,
                                IvfSearchScratch& w, int num_sms, cudaStream_t s);

}  // namespace sa
