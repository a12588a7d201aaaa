// merge.cu -- k-way merge of partial top-k lists (§8(a) a6, a9 final merge, a10 output).
//
// One CTA per query.  The candidates of a query are G groups of k packed keys
// (groups = corpus slices of one GPU, or ranks after the all-gather).  An
// exact MSB-first radix select (8 passes x 8 bits over the 64-bit keys) finds
// the k-th largest key T; the k keys >= T are sorted with a bitonic network in
// shared memory and unpacked to (id, score), or kept packed for the next level.
#include <cuda_bf16.h>

#include "keys.cuh"
#include "merge.cuh"

namespace sa {

namespace {
constexpr int kThreads = 256;
constexpr int kMaxK = 256;
constexpr int kSmemCand = 4096;  // candidates cached in smem when G*k fits
}

__global__ void __launch_bounds__(kThreads)
merge_topk_kernel(const MergeArgs a) {
  __shared__ uint32_t hist[256];
  __shared__ uint64_t sel[kMaxK];
  __shared__ uint64_t cache[kSmemCand];
  __shared__ int s_bucket, s_above, s_pos;

  const int64_t q = blockIdx.x;
  const int k = a.k;
  int64_t base = 0;
  int64_t M;
  if (a.slot_off) {
    base = a.slot_off[q * a.slot_stride] * a.slot_keys;
    M = a.slot_off[(q + 1) * a.slot_stride] * a.slot_keys - base;
  } else if (a.m_flat > 0) {
    base = q * a.qstride;
    M = a.m_flat;
  } else {
    M = (int64_t)a.groups * k;
  }
  const bool grouped = !a.slot_off && a.m_flat <= 0;
  const int tid = threadIdx.x;
  const bool cached = M <= kSmemCand;

  auto cand_g = [&](int64_t i) -> uint64_t {
    if (a.cand_scores) return make_key(a.cand_scores[base + i], (uint32_t)i);
    if (!grouped) return a.cand[base + i];
    const int64_t g = i / k, j = i % k;
    return a.cand[(size_t)g * a.gstride + (size_t)q * a.qstride + j];
  };
  if (cached) {
    for (int i = tid; i < M; i += kThreads) cache[i] = cand_g(i);
    __syncthreads();
  }
  auto cand = [&](int64_t i) -> uint64_t { return cached ? cache[i] : cand_g(i); };

  uint64_t prefix = 0, pmask = 0;
  int kr = k;
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 56 - 8 * pass;
    for (int i = tid; i < 256; i += kThreads) hist[i] = 0;
    __syncthreads();
    for (int64_t i = tid; i < M; i += kThreads) {
      const uint64_t c = cand(i);
      if ((c & pmask) == prefix) atomicAdd(&hist[(c >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid == 0) {
      int acc = 0, b = 255;
      for (; b > 0; --b) {
        if (acc + (int)hist[b] >= kr) break;
        acc += hist[b];
      }
      s_bucket = b;
      s_above = acc;
    }
    __syncthreads();
    prefix |= (uint64_t)s_bucket << shift;
    pmask |= 255ull << shift;
    kr -= s_above;
    __syncthreads();
  }
  // prefix = T, the k-th largest key; (k - kr) keys are strictly larger.
  const uint64_t T = prefix;
  if (tid == 0) s_pos = 0;
  for (int i = tid; i < kMaxK; i += kThreads) sel[i] = 0ull;
  __syncthreads();
  for (int64_t i = tid; i < M; i += kThreads) {
    const uint64_t c = cand(i);
    if (c > T) sel[atomicAdd(&s_pos, 1)] = c;
  }
  __syncthreads();
  for (int i = (k - kr) + tid; i < k; i += kThreads) sel[i] = T;
  __syncthreads();
  // bitonic sort of sel[0..256) descending (zeros = empty sink to the end)
  for (int size = 2; size <= kMaxK; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < kMaxK; i += kThreads) {
        const int j = i ^ stride;
        if (j > i) {
          const bool desc = ((i & size) == 0);
          const uint64_t x = sel[i], y = sel[j];
          if (desc ? (x < y) : (x > y)) { sel[i] = y; sel[j] = x; }
        }
      }
      __syncthreads();
    }
  }
  for (int i = tid; i < k; i += kThreads) {
    const uint64_t key = sel[i];
    if (a.out_keys) {
      a.out_keys[(size_t)q * k + i] = key;
    } else {
      if (key == 0ull) {
        a.out_ids[(size_t)q * k + i] = -1;
        a.out_scores[(size_t)q * k + i] = -__int_as_float(0x7f800000);
      } else {
        a.out_ids[(size_t)q * k + i] = (int64_t)key_id(key) + a.id_offset;
        a.out_scores[(size_t)q * k + i] = key_score(key);
      }
    }
  }
}

// k = 1 with few grouped candidates (k-means / full assignment: millions of queries):
// one thread per query, max over its candidate keys.
__global__ void merge_top1_kernel(const MergeArgs a, int64_t nq) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nq;
       q += (int64_t)gridDim.x * blockDim.x) {
    uint64_t best = 0ull;
    for (int g = 0; g < a.groups; ++g) {
      const uint64_t c = a.cand[(size_t)g * a.gstride + (size_t)q * a.qstride];
      best = c > best ? c : best;
    }
    if (a.out_keys) {
      a.out_keys[q] = best;
    } else if (best == 0ull) {
      a.out_ids[q] = -1;
      a.out_scores[q] = -__int_as_float(0x7f800000);
    } else {
      a.out_ids[q] = (int64_t)key_id(best) + a.id_offset;
      a.out_scores[q] = key_score(best);
    }
  }
}

cudaError_t launch_merge(const MergeArgs& a, int64_t nq, cudaStream_t stream) {
  if (nq <= 0) return cudaSuccess;
  if (a.k == 1 && !a.slot_off && a.m_flat <= 0 && a.groups <= 64) {
    int64_t blocks = (nq + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    merge_top1_kernel<<<(unsigned)blocks, 256, 0, stream>>>(a, nq);
    return cudaGetLastError();
  }
  merge_topk_kernel<<<(unsigned)nq, kThreads, 0, stream>>>(a);
  return cudaGetLastError();
}

// ---------------------------------------------------------------- staging (a1, a4)
// dst[r, c] = bf16_rne(src[r, c]) for r < rows, c < d; 0 in the padding.
template <typename T>
__global__ void cast_pad_kernel(const T* __restrict__ src, int64_t rows, int d,
                                __nv_bfloat16* __restrict__ dst, int64_t rows_pad, int d_pad) {
  const int64_t total8 = rows_pad * (int64_t)(d_pad / 8);
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < total8;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = v / (d_pad / 8);
    const int c0 = (int)(v % (d_pad / 8)) * 8;
    __align__(16) __nv_bfloat16 o[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int c = c0 + i;
      float x = 0.0f;
      if (r < rows && c < d) x = (float)src[(size_t)r * d + c];
      o[i] = __float2bfloat16_rn(x);
    }
    *reinterpret_cast<uint4*>(dst + (size_t)r * d_pad + c0) = *reinterpret_cast<uint4*>(o);
  }
}
template <>
__global__ void cast_pad_kernel<__nv_bfloat16>(const __nv_bfloat16* __restrict__ src, int64_t rows,
                                               int d, __nv_bfloat16* __restrict__ dst,
                                               int64_t rows_pad, int d_pad) {
  const int64_t total8 = rows_pad * (int64_t)(d_pad / 8);
  for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < total8;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = v / (d_pad / 8);
    const int c0 = (int)(v % (d_pad / 8)) * 8;
    __align__(16) __nv_bfloat16 o[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int c = c0 + i;
      o[i] = (r < rows && c < d) ? src[(size_t)r * d + c] : __float2bfloat16_rn(0.0f);
    }
    *reinterpret_cast<uint4*>(dst + (size_t)r * d_pad + c0) = *reinterpret_cast<uint4*>(o);
  }
}

cudaError_t launch_cast_pad(const void* src, bool src_f32, int64_t rows, int d, __nv_bfloat16* dst,
                            int64_t rows_pad, int d_pad, int num_sms, cudaStream_t stream) {
  const int64_t total8 = rows_pad * (int64_t)(d_pad / 8);
  if (total8 == 0) return cudaSuccess;
  int64_t blocks = (total8 + 255) / 256;
  const int64_t cap = (int64_t)num_sms * 8;
  if (blocks > cap) blocks = cap;
  if (src_f32)
    cast_pad_kernel<float><<<(unsigned)blocks, 256, 0, stream>>>(
        static_cast<const float*>(src), rows, d, dst, rows_pad, d_pad);
  else
    cast_pad_kernel<__nv_bfloat16><<<(unsigned)blocks, 256, 0, stream>>>(
        static_cast<const __nv_bfloat16*>(src), rows, d, dst, rows_pad, d_pad);
  return cudaGetLastError();
}

}  // namespace sa
