// ivf_kernels.cu -- SIMT kernels of the IVF build and search plumbing (§8(a) a2, a3, a7, a8).
//
// The tensor-core work of IVF (k-means assignment, full assignment, probe, list
// scan) runs in flat_scan.cu; these kernels are the HBM/latency-bound glue:
// strided training-sample gather, fp32/bf16 centroid conversion, a stable LSD
// radix sort by list id (deterministic list order = ascending row), exclusive
// scans, the deterministic centroid update (one CTA per list, members summed
// in ascending row order in fp32), empty-list repair, probe inversion and
// work-item generation.
#include <cuda_bf16.h>

#include "ivf_kernels.cuh"
#include "keys.cuh"
#include "launch.cuh"

namespace sa {

namespace {
constexpr int kScanBlock = 1024;
constexpr int kSortTile = 2048;  // elements per sort block (one warp walks it in order)

}  // namespace

uint64_t host_splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// ------------------------------------------------------------------ gathers
// out[t] = X[src(t)] with src(t) = floor((t0 + t) * n_total / n_train) - row_offset (training
// sample rows t0.., global-id strided, R9), or src(t) = idx[t] when idx != nullptr.
__global__ void gather_rows_kernel(const __nv_bfloat16* __restrict__ X, int d_pad,
                                   const int32_t* __restrict__ idx, int64_t n_total,
                                   int64_t row_offset, int64_t t0, int64_t n_train,
                                   int64_t n_out, __nv_bfloat16* __restrict__ out) {
  const int v8 = d_pad / 8;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n_out * v8;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = e / v8;
    const int c = (int)(e % v8);
    const int64_t src = idx ? (int64_t)idx[t] : ((t0 + t) * n_total) / n_train - row_offset;
    reinterpret_cast<uint4*>(out + t * d_pad)[c] =
        reinterpret_cast<const uint4*>(X + src * d_pad)[c];
  }
}

cudaError_t launch_gather_rows(const __nv_bfloat16* X, int d_pad, const int32_t* idx,
                               int64_t n_total, int64_t row_offset, int64_t t0, int64_t n_train,
                               int64_t n_out, __nv_bfloat16* out, int num_sms, cudaStream_t s) {
  if (n_out <= 0) return cudaSuccess;
  const int64_t work = n_out * (d_pad / 8);
  int64_t blocks = (work + 255) / 256;
  if (blocks > (int64_t)num_sms * 16) blocks = (int64_t)num_sms * 16;
  gather_rows_kernel<<<(unsigned)blocks, 256, 0, s>>>(X, d_pad, idx, n_total, row_offset, t0,
                                                      n_train, n_out, out);
  note_launch();
  return cudaGetLastError();
}

// Initial centroids: c_j = sample row (j * stride + o), widened to fp32 (R9).
__global__ void init_centroids_kernel(const __nv_bfloat16* __restrict__ sample, int d_pad,
                                      int nlist, int64_t stride, int64_t o,
                                      float* __restrict__ cent) {
  const int j = blockIdx.x;
  const __nv_bfloat16* src = sample + (j * stride + o) * d_pad;
  for (int c = threadIdx.x; c < d_pad; c += blockDim.x)
    cent[(size_t)j * d_pad + c] = __bfloat162float(src[c]);
}

cudaError_t launch_init_centroids(const __nv_bfloat16* sample, int d_pad, int nlist,
                                  int64_t n_train, uint64_t seed, float* cent, cudaStream_t s) {
  const int64_t stride = n_train / nlist;
  const int64_t o = (int64_t)(host_splitmix64(seed) % (uint64_t)stride);
  init_centroids_kernel<<<nlist, 256, 0, s>>>(sample, d_pad, nlist, stride, o, cent);
  note_launch();
  return cudaGetLastError();
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ in, int64_t n,
                                   __nv_bfloat16* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __float2bfloat16_rn(in[i]);
}

cudaError_t launch_f32_to_bf16(const float* in, int64_t n, __nv_bfloat16* out, int num_sms,
                               cudaStream_t s) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)num_sms * 16) blocks = (int64_t)num_sms * 16;
  if (blocks < 1) return cudaSuccess;
  f32_to_bf16_kernel<<<(unsigned)blocks, 256, 0, s>>>(in, n, out);
  note_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ scans
// Exclusive scan of int64 values (three phases; n up to ~2^31).
__global__ void scan_block_kernel(const int64_t* __restrict__ in, int64_t n,
                                  int64_t* __restrict__ out, int64_t* __restrict__ block_sums) {
  __shared__ int64_t s[kScanBlock];
  const int64_t base = (int64_t)blockIdx.x * kScanBlock;
  const int t = threadIdx.x;
  s[t] = base + t < n ? in[base + t] : 0;
  __syncthreads();
  for (int off = 1; off < kScanBlock; off <<= 1) {
    int64_t v = t >= off ? s[t - off] : 0;
    __syncthreads();
    s[t] += v;
    __syncthreads();
  }
  if (base + t < n) out[base + t] = s[t] - (base + t < n ? in[base + t] : 0);
  if (t == kScanBlock - 1) block_sums[blockIdx.x] = s[t];
}
__global__ void scan_sums_kernel(int64_t* sums, int64_t nb, int64_t* total) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int64_t acc = 0;
    for (int64_t i = 0; i < nb; ++i) {
      const int64_t v = sums[i];
      sums[i] = acc;
      acc += v;
    }
    if (total) *total = acc;
  }
}
__global__ void scan_add_kernel(int64_t* __restrict__ out, int64_t n,
                                const int64_t* __restrict__ block_off) {
  const int64_t i = (int64_t)blockIdx.x * kScanBlock + threadIdx.x;
  if (i < n) out[i] += block_off[blockIdx.x];
}

// out[i] = sum_{j<i} in[i]; out[n] = total (out has n + 1 entries).  scratch: >= nb + 1.
cudaError_t exclusive_scan_i64(const int64_t* in, int64_t n, int64_t* out, int64_t* scratch,
                               cudaStream_t s) {
  const int64_t nb = (n + kScanBlock - 1) / kScanBlock;
  if (n > 0) {
    scan_block_kernel<<<(unsigned)nb, kScanBlock, 0, s>>>(in, n, out, scratch);
    note_launch();
  }
  scan_sums_kernel<<<1, 32, 0, s>>>(scratch, nb, out + n);
  note_launch();
  if (n > 0) {
    scan_add_kernel<<<(unsigned)nb, kScanBlock, 0, s>>>(out, n, scratch);
    note_launch();
  }
  return cudaGetLastError();
}

// ------------------------------------------------------------------ stable radix sort
// Sort (key, value) pairs by key (< 2^16), stable, two LSD passes of 8 bits.  Each block
// owns a tile of kSortTile elements; one warp walks the tile in order so in-tile ranks
// preserve input order.
__global__ void radix_count_kernel(const int32_t* __restrict__ keys, int64_t n, int shift,
                                   int64_t nblocks, int64_t* __restrict__ counts) {
  __shared__ int hist[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * kSortTile;
  for (int i = threadIdx.x; i < kSortTile; i += blockDim.x) {
    const int64_t e = base + i;
    if (e < n) atomicAdd(&hist[(keys[e] >> shift) & 255], 1);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    counts[(int64_t)i * nblocks + blockIdx.x] = hist[i];  // digit-major
}

__global__ void radix_scatter_kernel(const int32_t* __restrict__ keys,
                                     const int32_t* __restrict__ vals, int64_t n, int shift,
                                     int64_t nblocks, const int64_t* __restrict__ offs,
                                     int32_t* __restrict__ keys_out,
                                     int32_t* __restrict__ vals_out) {
  __shared__ int64_t cur[256];
  const int lane = threadIdx.x;
  for (int i = lane; i < 256; i += 32) cur[i] = offs[(int64_t)i * nblocks + blockIdx.x];
  __syncwarp();
  const int64_t base = (int64_t)blockIdx.x * kSortTile;
  const unsigned lt = (1u << lane) - 1u;
  for (int c = 0; c < kSortTile; c += 32) {
    const int64_t e = base + c + lane;
    const bool ok = e < n;
    const unsigned act = __ballot_sync(0xffffffffu, ok);
    if (act == 0) break;
    int key = 0, val = 0, dig = 256 + lane;  // inactive lanes: unique dummy digit
    if (ok) {
      key = keys[e];
      val = vals ? vals[e] : (int32_t)e;
      dig = (key >> shift) & 255;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, dig);
    int64_t pos = 0;
    if (ok) pos = cur[dig] + __popc(peers & lt);
    __syncwarp();
    if (ok && (peers & lt) == 0) cur[dig] += __popc(peers);
    __syncwarp();
    if (ok) {
      keys_out[pos] = key;
      vals_out[pos] = val;
    }
  }
}

cudaError_t stable_sort_by_key16(const int32_t* keys, int64_t n, int32_t* keys_tmp,
                                 int32_t* vals_tmp, int32_t* keys_out, int32_t* vals_out,
                                 int64_t* counts, int64_t* offs, int64_t* scratch, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int64_t nb = (n + kSortTile - 1) / kSortTile;
  // pass 1: low byte, values = positions
  radix_count_kernel<<<(unsigned)nb, 256, 0, s>>>(keys, n, 0, nb, counts);
  note_launch();
  exclusive_scan_i64(counts, 256 * nb, offs, scratch, s);
  radix_scatter_kernel<<<(unsigned)nb, 32, 0, s>>>(keys, nullptr, n, 0, nb, offs, keys_tmp,
                                                   vals_tmp);
  note_launch();
  // pass 2: high byte
  radix_count_kernel<<<(unsigned)nb, 256, 0, s>>>(keys_tmp, n, 8, nb, counts);
  note_launch();
  exclusive_scan_i64(counts, 256 * nb, offs, scratch, s);
  radix_scatter_kernel<<<(unsigned)nb, 32, 0, s>>>(keys_tmp, vals_tmp, n, 8, nb, offs, keys_out,
                                                   vals_out);
  note_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ histograms
__global__ void histogram_kernel(const int32_t* __restrict__ keys, int64_t n,
                                 int64_t* __restrict__ hist) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(reinterpret_cast<unsigned long long*>(&hist[keys[i]]), 1ull);
}
cudaError_t launch_histogram(const int32_t* keys, int64_t n, int64_t* hist, int num_sms,
                             cudaStream_t s) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)num_sms * 16) blocks = (int64_t)num_sms * 16;
  if (blocks < 1) return cudaSuccess;
  histogram_kernel<<<(unsigned)blocks, 256, 0, s>>>(keys, n, hist);
  note_launch();
  return cudaGetLastError();
}

// int64 ids (assignment output) -> int32 keys
__global__ void i64_to_i32_kernel(const int64_t* __restrict__ in, int64_t n,
                                  int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)in[i];
}
cudaError_t launch_i64_to_i32(const int64_t* in, int64_t n, int32_t* out, int num_sms,
                              cudaStream_t s) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)num_sms * 16) blocks = (int64_t)num_sms * 16;
  if (blocks < 1) return cudaSuccess;
  i64_to_i32_kernel<<<(unsigned)blocks, 256, 0, s>>>(in, n, out);
  note_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ centroid update
// c_l = normalise(sum of members), members = sorted_rows[off[l], off[l+1]) in ascending row
// order, fp32 sequential per dimension (R8).  Empty lists are left for the repair step and
// counted in *n_empty.
__global__ void centroid_update_kernel(const __nv_bfloat16* __restrict__ sample, int d_pad,
                                       const int32_t* __restrict__ rows,
                                       const int64_t* __restrict__ off, float* __restrict__ cent,
                                       int32_t* __restrict__ empty_flag,
                                       int32_t* __restrict__ n_empty) {
  const int l = blockIdx.x;
  const int64_t b = off[l], e = off[l + 1];
  __shared__ float red[32];
  if (b == e) {
    if (threadIdx.x == 0) {
      empty_flag[l] = 1;
      atomicAdd(n_empty, 1);
    }
    return;
  }
  if (threadIdx.x == 0) empty_flag[l] = 0;
  constexpr int kMaxPer = 4;  // d_pad <= 768 with 256 threads -> 3 dims per thread
  float acc[kMaxPer] = {0.f, 0.f, 0.f, 0.f};
  for (int64_t m = b; m < e; ++m) {
    const __nv_bfloat16* x = sample + (int64_t)rows[m] * d_pad;
#pragma unroll
    for (int i = 0; i < kMaxPer; ++i) {
      const int c = threadIdx.x + i * blockDim.x;
      if (c < d_pad) acc[i] += __bfloat162float(x[c]);
    }
  }
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < kMaxPer; ++i) ss += acc[i] * acc[i];
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float inv = red[0] > 0.f ? rsqrtf(red[0]) : 0.f;
#pragma unroll
  for (int i = 0; i < kMaxPer; ++i) {
    const int c = threadIdx.x + i * blockDim.x;
    if (c < d_pad) cent[(size_t)l * d_pad + c] = acc[i] * inv;
  }
}

cudaError_t launch_centroid_update(const __nv_bfloat16* sample, int d_pad, const int32_t* rows,
                                   const int64_t* off, int nlist, float* cent,
                                   int32_t* empty_flag, int32_t* n_empty, cudaStream_t s) {
  centroid_update_kernel<<<nlist, 256, 0, s>>>(sample, d_pad, rows, off, cent, empty_flag,
                                                n_empty);
  note_launch();
  return cudaGetLastError();
}

// keys for the empty-list repair: larger key = lower assigned score, ties -> lower row (R10)
__global__ void repair_keys_kernel(const float* __restrict__ scores, int64_t n,
                                   uint64_t* __restrict__ keys) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    keys[i] = make_key(-scores[i], (uint32_t)i);
}
cudaError_t launch_repair_keys(const float* scores, int64_t n, uint64_t* keys, int num_sms,
                               cudaStream_t s) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)num_sms * 16) blocks = (int64_t)num_sms * 16;
  repair_keys_kernel<<<(unsigned)blocks, 256, 0, s>>>(scores, n, keys);
  note_launch();
  return cudaGetLastError();
}
// The i-th empty list (ascending id) takes sample row key_id(sel[i]).
__global__ void repair_apply_kernel(const __nv_bfloat16* __restrict__ sample, int d_pad, int nlist,
                                    const int32_t* __restrict__ empty_flag,
                                    const uint64_t* __restrict__ sel, float* __restrict__ cent) {
  // single block: walk lists in order, assign selections sequentially
  __shared__ int rank;
  if (threadIdx.x == 0) rank = 0;
  __syncthreads();
  for (int l = 0; l < nlist; ++l) {
    if (empty_flag[l]) {
      const int64_t row = (int64_t)key_id(sel[rank]);
      for (int c = threadIdx.x; c < d_pad; c += blockDim.x)
        cent[(size_t)l * d_pad + c] = __bfloat162float(sample[row * d_pad + c]);
      __syncthreads();
      if (threadIdx.x == 0) ++rank;
      __syncthreads();
    }
  }
}
cudaError_t launch_repair_apply(const __nv_bfloat16* sample, int d_pad, int nlist,
                                const int32_t* empty_flag, const uint64_t* sel, float* cent,
                                cudaStream_t s) {
  repair_apply_kernel<<<1, 256, 0, s>>>(sample, d_pad, nlist, empty_flag, sel, cent);
  note_launch();
  return cudaGetLastError();
}

// ------------------------------------------------------------------ search-side plumbing
// Count probers per list.
__global__ void probe_count_kernel(const int64_t* __restrict__ probes, int64_t n,
                                   int32_t* __restrict__ cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = probes[i];
    if (l >= 0) atomicAdd(&cnt[l], 1);
  }
}
// Per (q, j): number of chunk slots = chunks of list probes[q, j] (0 for an empty list).
__global__ void probe_slots_kernel(const int64_t* __restrict__ probes, int64_t n,
                                   const int64_t* __restrict__ list_off, int chunk_rows,
                                   int64_t* __restrict__ nslots) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = probes[i];
    int64_t c = 0;
    if (l >= 0) {
      const int64_t len = list_off[l + 1] - list_off[l];
      c = (len + chunk_rows - 1) / chunk_rows;
    }
    nslots[i] = c;
  }
}
// Per list: work items = query blocks x chunks (0 if unprobed or empty).
__global__ void list_items_kernel(const int32_t* __restrict__ cnt, int nlist,
                                  const int64_t* __restrict__ list_off, int chunk_rows,
                                  int qblock, int64_t* __restrict__ nitems) {
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nlist; l += gridDim.x * blockDim.x) {
    const int64_t len = list_off[l + 1] - list_off[l];
    const int64_t nch = (len + chunk_rows - 1) / chunk_rows;
    const int64_t nqb = (cnt[l] + qblock - 1) / qblock;
    nitems[l] = nch * nqb;
  }
}
// Fill lq_ent (any order inside a list) and the items of every list.
__global__ void probe_fill_kernel(const int64_t* __restrict__ probes, int64_t nq, int nprobe,
                                  const int64_t* __restrict__ lq_off64, int32_t* __restrict__ cursor,
                                  int2* __restrict__ lq_ent) {
  const int64_t n = nq * nprobe;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = probes[i];
    if (l < 0) continue;
    const int pos = atomicAdd(&cursor[l], 1);
    lq_ent[lq_off64[l] + pos] = make_int2((int)(i / nprobe), (int)(i % nprobe));
  }
}
__global__ void items_fill_kernel(const int32_t* __restrict__ cnt, int nlist,
                                  const int64_t* __restrict__ list_off, int chunk_rows, int qblock,
                                  const int64_t* __restrict__ lq_off64,
                                  const int64_t* __restrict__ item_off, int4* __restrict__ items,
                                  int32_t* __restrict__ n_items) {
  for (int l = blockIdx.x * blockDim.x + threadIdx.x; l < nlist; l += gridDim.x * blockDim.x) {
    const int64_t len = list_off[l + 1] - list_off[l];
    const int nch = (int)((len + chunk_rows - 1) / chunk_rows);
    const int nqb = (cnt[l] + qblock - 1) / qblock;
    int64_t o = item_off[l];
    for (int b = 0; b < nqb; ++b) {
      const int e0 = (int)lq_off64[l] + b * qblock;
      const int c_b = cnt[l] - b * qblock < qblock ? cnt[l] - b * qblock : qblock;
      for (int c = 0; c < nch; ++c) items[o++] = make_int4(l, e0, c, c_b);
    }
    if (l == nlist - 1) *n_items = (int32_t)item_off[nlist];
  }
}

// Whole inversion in one CTA for small batches (nq * nprobe <= kInvertSmallMax): sort the
// (list, query, probe rank) entries by list in smem, emit probers grouped by list, the
// per-(query, probe) output slots and the work items -- one launch instead of ~13.
// probes[i] < 0 = no list (a finished query of a maturity stage): no items, an empty slot.
constexpr uint32_t kNoList = 0xFFFFFFFFu;
__global__ void __launch_bounds__(1024)
invert_small_kernel(const int64_t* __restrict__ probes, int nq, int nprobe,
                    const int64_t* __restrict__ list_off, int chunk_rows, int qblock,
                    int2* __restrict__ lq_ent, int64_t* __restrict__ q_slot,
                    int4* __restrict__ items, int32_t* __restrict__ n_items, StageSrc src) {
  extern __shared__ uint64_t ent[];  // [P2] (list << 32 | entry index)
  __shared__ int wtot[32];
  __shared__ int s_total;
  const int n = nq * nprobe;
  int P2 = 1;
  while (P2 < n) P2 <<= 1;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int lane = tid & 31, wid = tid >> 5;
  if (src.probes_full) {
    // maturity stage: entry (q, j) probes rank stage*nprobe + j of a still-active query
    const int stage = src.ctrl[0];
    int64_t* sp = const_cast<int64_t*>(probes);
    for (int i = tid; i < n; i += nt) {
      const int q = i / nprobe, r = stage * nprobe + i % nprobe;
      sp[i] = (src.active[q] && r < src.P) ? src.probes_full[(int64_t)q * src.P + r] : -1;
    }
    if (tid == 0) *src.item_counter = 0;
    __syncthreads();
  }
  for (int i = tid; i < P2; i += nt)
    ent[i] = i < n ? (((uint64_t)(uint32_t)probes[i] << 32) | (uint32_t)i) : ~0ull;
  __syncthreads();
  for (int sz = 2; sz <= P2; sz <<= 1)
    for (int st = sz >> 1; st > 0; st >>= 1) {
      for (int i = tid; i < P2; i += nt) {
        const int j = i ^ st;
        if (j > i) {
          const bool up = (i & sz) == 0;
          const uint64_t x = ent[i], y = ent[j];
          if (up ? x > y : x < y) { ent[i] = y; ent[j] = x; }
        }
      }
      __syncthreads();
    }
  // block exclusive scan helper over one int per thread
  auto block_scan = [&](int v, int* total) -> int {
    int incl = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) wtot[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      int w = lane < (nt >> 5) ? wtot[lane] : 0;
      int wi = w;
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= o) wi += t;
      }
      if (lane < (nt >> 5)) wtot[lane] = wi - w;
      if (lane == 31) s_total = wi;
    }
    __syncthreads();
    const int base = wtot[wid];
    const int tot = s_total;
    __syncthreads();
    *total = tot;
    return base + incl - v;
  };
  // contiguous chunk per thread
  const int per = (n + nt - 1) / nt;
  const int lo = tid * per, hi = min(n, lo + per);
  // probers grouped by list (sorted order) and item counts of the runs that start here
  int my_items = 0;
  for (int i = lo; i < hi; ++i) {
    const uint32_t e = (uint32_t)ent[i];
    lq_ent[i] = make_int2((int)(e / nprobe), (int)(e % nprobe));
    const uint32_t l = (uint32_t)(ent[i] >> 32);
    if (l != kNoList && (i == 0 || (uint32_t)(ent[i - 1] >> 32) != l)) {
      int c = 1;
      while (i + c < n && (uint32_t)(ent[i + c] >> 32) == l) ++c;
      const int64_t len = list_off[l + 1] - list_off[l];
      const int nch = (int)((len + chunk_rows - 1) / chunk_rows);
      my_items += ((c + qblock - 1) / qblock) * nch;
    }
  }
  int total_items;
  int o = block_scan(my_items, &total_items);
  for (int i = lo; i < hi; ++i) {
    const uint32_t l = (uint32_t)(ent[i] >> 32);
    if (l != kNoList && (i == 0 || (uint32_t)(ent[i - 1] >> 32) != l)) {
      int c = 1;
      while (i + c < n && (uint32_t)(ent[i + c] >> 32) == l) ++c;
      const int64_t len = list_off[l + 1] - list_off[l];
      const int nch = (int)((len + chunk_rows - 1) / chunk_rows);
      for (int b = 0; b * qblock < c; ++b)
        for (int ch = 0; ch < nch; ++ch)
          items[o++] = make_int4((int)l, i + b * qblock, ch,
                                 c - b * qblock < qblock ? c - b * qblock : qblock);
    }
  }
  // output slots per (q, j), original order: chunks of the probed list
  int my_slots = 0;
  for (int i = lo; i < hi; ++i) {
    const int64_t l = probes[i];
    if (l < 0) continue;  // no list (maturity stages: finished query)
    const int64_t len = list_off[l + 1] - list_off[l];
    my_slots += (int)((len + chunk_rows - 1) / chunk_rows);
  }
  int total_slots;
  int so = block_scan(my_slots, &total_slots);
  for (int i = lo; i < hi; ++i) {
    q_slot[i] = so;
    const int64_t l = probes[i];
    if (l < 0) continue;
    const int64_t len = list_off[l + 1] - list_off[l];
    so += (int)((len + chunk_rows - 1) / chunk_rows);
  }
  if (tid == 0) {
    q_slot[n] = total_slots;
    *n_items = total_items;
  }
}

cudaError_t launch_invert_small(const int64_t* probes, int nq, int nprobe, const int64_t* list_off,
                                int chunk_rows, int qblock, IvfSearchScratch& w, cudaStream_t s) {
  int P2 = 1;
  while (P2 < nq * nprobe) P2 <<= 1;
  invert_small_kernel<<<1, 1024, P2 * sizeof(uint64_t), s>>>(probes, nq, nprobe, list_off,
                                                              chunk_rows, qblock, w.lq_ent, w.q_slot,
                                                              w.items, w.n_items, StageSrc{});
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_invert_stage(int64_t* stage_probes, int nq, int g, const StageSrc& src,
                                const int64_t* list_off, int chunk_rows, int qblock,
                                IvfSearchScratch& w, cudaStream_t s) {
  int P2 = 1;
  while (P2 < nq * g) P2 <<= 1;
  invert_small_kernel<<<1, 1024, P2 * sizeof(uint64_t), s>>>(stage_probes, nq, g, list_off,
                                                              chunk_rows, qblock, w.lq_ent, w.q_slot,
                                                              w.items, w.n_items, src);
  note_launch();
  return cudaGetLastError();
}
__global__ void i32_to_i64_kernel(const int32_t* __restrict__ in, int64_t n,
                                  int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

cudaError_t launch_probe_invert(const int64_t* probes, int64_t nq, int nprobe, int nlist,
                                const int64_t* list_off, int chunk_rows, int qblock,
                                IvfSearchScratch& w, int num_sms, cudaStream_t s) {
  const int64_t n = nq * nprobe;
  unsigned b = (unsigned)((n + 255) / 256);
  if (b > (unsigned)num_sms * 8) b = (unsigned)num_sms * 8;
  if (b < 1) b = 1;
  const unsigned bl = (unsigned)((nlist + 255) / 256);
  cudaMemsetAsync(w.cnt, 0, sizeof(int32_t) * nlist, s);
  cudaMemsetAsync(w.cursor, 0, sizeof(int32_t) * nlist, s);
  probe_count_kernel<<<b, 256, 0, s>>>(probes, n, w.cnt);
  note_launch();
  i32_to_i64_kernel<<<bl, 256, 0, s>>>(w.cnt, nlist, w.tmp64);
  note_launch();
  exclusive_scan_i64(w.tmp64, nlist, w.lq_off64, w.scratch, s);
  probe_fill_kernel<<<b, 256, 0, s>>>(probes, nq, nprobe, w.lq_off64, w.cursor, w.lq_ent);
  note_launch();
  probe_slots_kernel<<<b, 256, 0, s>>>(probes, n, list_off, chunk_rows, w.tmp64b);
  note_launch();
  exclusive_scan_i64(w.tmp64b, n, w.q_slot, w.scratch, s);
  list_items_kernel<<<bl, 256, 0, s>>>(w.cnt, nlist, list_off, chunk_rows, qblock, w.tmp64);
  note_launch();
  exclusive_scan_i64(w.tmp64, nlist, w.item_off, w.scratch, s);
  items_fill_kernel<<<bl, 256, 0, s>>>(w.cnt, nlist, list_off, chunk_rows, qblock, w.lq_off64, w.item_off,
                                       w.items, w.n_items);
  note_launch();
  return cudaGetLastError();
}

// probes from packed probe keys [nq, nprobe] (list id in the key, empty -> -1)
__global__ void keys_to_lists_kernel(const uint64_t* __restrict__ keys, int64_t n,
                                     int64_t* __restrict__ lists, int32_t* __restrict__ lists32) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
    const int64_t l = k == 0ull ? -1 : (int64_t)key_id(k);
    if (lists) lists[i] = l;
    if (lists32) lists32[i] = (int32_t)l;
  }
}
cudaError_t launch_keys_to_lists(const uint64_t* keys, int64_t n, int64_t* lists, int32_t* lists32,
                                 int num_sms, cudaStream_t s) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)num_sms * 8) blocks = (int64_t)num_sms * 8;
  if (blocks < 1) return cudaSuccess;
  keys_to_lists_kernel<<<(unsigned)blocks, 256, 0, s>>>(keys, n, lists, lists32);
  note_launch();
  return cudaGetLastError();
}

// row ids of the permuted layout: ids[i] = row_offset + perm[i]
__global__ void perm_ids_kernel(const int32_t* __restrict__ perm, int64_t n, int64_t row_offset,
                                int32_t* __restrict__ ids) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    ids[i] = (int32_t)(uint32_t)(row_offset + perm[i]);
}
cudaError_t launch_perm_ids(const int32_t* perm, int64_t n, int64_t row_offset, int32_t* ids,
                            int num_sms, cudaStream_t s) {
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)num_sms * 16) blocks = (int64_t)num_sms * 16;
  if (blocks < 1) return cudaSuccess;
  perm_ids_kernel<<<(unsigned)blocks, 256, 0, s>>>(perm, n, row_offset, ids);
  note_launch();
  return cudaGetLastError();
}

}  // namespace sa
