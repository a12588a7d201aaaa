// fp8.cu -- e4m3 quantisation and bf16 re-rank for the fp8 flat scan (
// DESIGN.md §4.8, readings R30-R33).
//
// The flat scan itself is flat_scan_topk_kernel<CG, F8 = true> (kind::f8f6f4 MMAs over the
// e4m3 copy of the corpus: half the bytes and twice the tensor rate of bf16).  Its candidates
// are re-scored here against the bf16 rows the index keeps, so the returned scores and order
// are those of the bf16 data (the exact mode's values), only the candidate set comes from fp8.
#include <cuda_bf16.h>
#include <cuda_fp8.h>

#include "fp8.cuh"
#include "keys.cuh"
#include "launch.cuh"

namespace sa {

namespace {

unsigned grid_for(int64_t n, int per_block, int num_sms) {
  int64_t b = (n + per_block - 1) / per_block;
  if (b < 1) b = 1;
  const int64_t cap = (int64_t)num_sms * 16;
  return (unsigned)(b < cap ? b : cap);
}

__global__ void absmax_kernel(const __nv_bfloat16* __restrict__ X, int64_t n_elems,
                              uint32_t* __restrict__ out) {
  const uint4* X4 = reinterpret_cast<const uint4*>(X);
  const int64_t n4 = n_elems / 8;
  float m = 0.f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldg(X4 + i);
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float2 f = __bfloat1622float2(b[j]);
      m = fmaxf(m, fmaxf(fabsf(f.x), fabsf(f.y)));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  // non-negative fp32 values order like their bit patterns
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}

// largest e with m * 2^e <= 448 (R30): m = f * 2^E, f in [0.5, 1); 448 = 0.875 * 2^9
__device__ __forceinline__ int e4m3_exponent(float m) {
  if (!(m > 0.f)) return 0;
  int E;
  const float f = frexpf(m, &E);
  return f <= 0.875f ? 9 - E : 8 - E;
}

__global__ void quant_e4m3_kernel(const __nv_bfloat16* __restrict__ X, int64_t n, int32_t d_pad,
                                  const uint32_t* __restrict__ absmax_bits,
                                  uint8_t* __restrict__ X8, int32_t d8_pad,
                                  int32_t* __restrict__ exp_out) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
  const int groups = d8_pad / 16;      // 16 values per lane step
  const int in_groups = d_pad / 16;    // groups with bf16 data (d_pad is a multiple of 64)
  const int e_glob = absmax_bits ? e4m3_exponent(__uint_as_float(*absmax_bits)) : 0;
  if (absmax_bits && exp_out && blockIdx.x == 0 && threadIdx.x == 0) exp_out[0] = e_glob;
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32; r < n; r += nw) {
    const uint4* src = reinterpret_cast<const uint4*>(X + r * d_pad);
    int e = e_glob;
    if (!absmax_bits) {
      float m = 0.f;
      for (int g = lane; g < in_groups; g += 32)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint4 v = __ldg(src + 2 * g + h);
          const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 f = __bfloat1622float2(b[j]);
            m = fmaxf(m, fmaxf(fabsf(f.x), fabsf(f.y)));
          }
        }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      e = e4m3_exponent(m);
      if (exp_out && lane == 0) exp_out[r] = e;
    }
    uint4* dst = reinterpret_cast<uint4*>(X8 + r * d8_pad);
    for (int g = lane; g < groups; g += 32) {
      uint32_t w[4] = {0u, 0u, 0u, 0u};
      if (g < in_groups) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint4 v = __ldg(src + 2 * g + h);
          const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float2 f = __bfloat1622float2(b[j]);
            // x * 2^e is exact in fp32 here (bf16 values, |x| * 2^e <= 448); one RNE rounding
            const uint32_t lo = __nv_cvt_float_to_fp8(ldexpf(f.x, e), __NV_SATFINITE, __NV_E4M3);
            const uint32_t hi = __nv_cvt_float_to_fp8(ldexpf(f.y, e), __NV_SATFINITE, __NV_E4M3);
            const int idx = h * 8 + j * 2;   // value index within the group of 16
            w[idx / 4] |= (lo << (8 * (idx % 4))) | (hi << (8 * (idx % 4 + 1)));
          }
        }
      }
      dst[g] = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
}

constexpr int kRrThreads = 256;

__device__ __forceinline__ float bf16x8_dot_f(const uint4 v, const float* q) {
  const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v);
  float acc = 0.f;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 f = __bfloat1622float2(b[j]);
    acc = fmaf(f.x, q[2 * j], acc);
    acc = fmaf(f.y, q[2 * j + 1], acc);
  }
  return acc;
}

__global__ void __launch_bounds__(kRrThreads) rerank_kernel(const RerankArgs a) {
  __shared__ __align__(16) float qs[768];
  __shared__ unsigned long long key[F8_MAX_CAND];
  const int q = blockIdx.x;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  for (int i = threadIdx.x; i < a.d_pad; i += kRrThreads)
    qs[i] = __bfloat162float(a.Qs[(int64_t)q * a.d_pad + i]);
  for (int i = threadIdx.x; i < F8_MAX_CAND; i += kRrThreads) key[i] = 0ull;
  __syncthreads();
  const int nchunk = a.d_pad / 8;
  const uint4* X4 = reinterpret_cast<const uint4*>(a.X);
  // two candidates per warp step, all their 16-byte chunks in flight at once
  for (int c0 = warp * 2; c0 < a.n_cand; c0 += 2 * (kRrThreads / 32)) {
    uint64_t ck[2];
    uint4 v[2][3];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      ck[u] = c0 + u < a.n_cand ? a.cand[(int64_t)q * a.n_cand + c0 + u] : 0ull;
      const int64_t pos = (int64_t)key_id(ck[u]);
#pragma unroll
      for (int rd = 0; rd < 3; ++rd) {
        const int c = rd * 32 + lane;
        v[u][rd] = (ck[u] != 0ull && c < nchunk) ? __ldg(X4 + pos * nchunk + c)
                                                 : make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      float acc = 0.f;
#pragma unroll
      for (int rd = 0; rd < 3; ++rd)
        if (rd * 32 + lane < nchunk) acc += bf16x8_dot_f(v[u][rd], qs + (rd * 32 + lane) * 8);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0 && ck[u] != 0ull) {
        const int64_t pos = (int64_t)key_id(ck[u]);
        const uint32_t gid = a.row_ids ? (uint32_t)a.row_ids[pos] : (uint32_t)(a.row_offset + pos);
        key[c0 + u] = make_key(acc, gid);
      }
    }
  }
  __syncthreads();
  // bitonic sort of the 256 slots, descending (empty slots = 0 sort last)
  for (int size = 2; size <= F8_MAX_CAND; size <<= 1)
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const int i = threadIdx.x;
      const int j = i ^ stride;
      if (j > i) {
        const bool desc = (i & size) == 0;
        const unsigned long long x = key[i], y = key[j];
        if (desc ? x < y : x > y) {
          key[i] = y;
          key[j] = x;
        }
      }
      __syncthreads();
    }
  for (int i = threadIdx.x; i < a.k; i += kRrThreads) {
    const unsigned long long kk = key[i];
    if (a.out_keys) a.out_keys[(int64_t)q * a.k + i] = kk;
    if (a.out_ids) {
      a.out_ids[(int64_t)q * a.k + i] = kk == 0ull ? -1 : (int64_t)key_id(kk);
      a.out_scores[(int64_t)q * a.k + i] = kk == 0ull ? -INFINITY : key_score(kk);
    }
  }
}

}  // namespace

cudaError_t launch_absmax_bf16(const __nv_bfloat16* X, int64_t n, int32_t d_pad,
                               uint32_t* out_bits, int num_sms, cudaStream_t s) {
  absmax_kernel<<<grid_for(n * d_pad / 8, 256, num_sms), 256, 0, s>>>(X, n * d_pad, out_bits);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_quant_e4m3(const __nv_bfloat16* X, int64_t n, int32_t d_pad,
                              const uint32_t* absmax_bits, uint8_t* X8, int32_t d8_pad,
                              int32_t* exp_out, int num_sms, cudaStream_t s) {
  quant_e4m3_kernel<<<grid_for(n, 8, num_sms), 256, 0, s>>>(X, n, d_pad, absmax_bits, X8, d8_pad,
                                                            exp_out);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_rerank(const RerankArgs& a, int64_t nq, cudaStream_t s) {
  if (a.n_cand > F8_MAX_CAND || a.k > a.n_cand || a.d_pad > 768) return cudaErrorInvalidValue;
  rerank_kernel<<<(unsigned)nq, kRrThreads, 0, s>>>(a);
  note_launch();
  return cudaGetLastError();
}

}  // namespace sa
