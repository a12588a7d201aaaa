// merge.cu -- k-way merge of partial top-k lists (§8(a) a6, a9 final merge, a10 output).
//
// One CTA per query.  The candidates of a query are G groups of k packed keys
// (groups = corpus slices of one GPU, or ranks after the all-gather).  An
// exact MSB-first radix select (8 passes x 8 bits over the 64-bit keys) finds
// the k-th largest key T; the k keys >= T are sorted with a bitonic network in
// shared memory and unpacked to (id, score), or kept packed for the next level.
#include <cuda_bf16.h>

#include "keys.cuh"
#include "launch.cuh"
#include "merge.cuh"

namespace sa {

namespace {
constexpr int kThreads = 256;
constexpr int kMaxK = 256;
constexpr int kSmemCand = 4096;  // u64 candidates cached in smem when they fit (32 KB)
constexpr int kPrefilterCap = 2048;  // dense select: candidates surviving the prefilter

// Warp 0 finds the radix bucket holding the kr-th largest element: buckets are scanned from
// the top, 8 per lane, with one warp prefix sum (instead of a 256-step serial loop).
__device__ __forceinline__ void pick_bucket(const uint32_t* hist, int kr, int* s_bucket,
                                            int* s_above) {
  const int lane = threadIdx.x & 31;
  uint32_t c[8];
  uint32_t sum = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    c[i] = hist[255 - (lane * 8 + i)];
    sum += c[i];
  }
  uint32_t incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  const uint32_t excl = incl - sum;
  const unsigned hit = __ballot_sync(0xffffffffu, incl >= (uint32_t)kr);
  // hit != 0 whenever at least kr candidates remain; otherwise take the lowest bucket (0)
  const int owner = hit ? __ffs(hit) - 1 : 31;
  if (lane == owner) {
    uint32_t acc = excl;
    int b = 255 - lane * 8;
    for (int i = 0; i < 8; ++i, --b) {
      if (b == 0 || acc + c[i] >= (uint32_t)kr) break;
      acc += c[i];
    }
    *s_bucket = b;
    *s_above = (int)acc;
  }
}

// Bitonic sort of sel[0..size) descending; size = power of two >= k.
__device__ __forceinline__ void sort_desc(uint64_t* sel, int size) {
  for (int sz = 2; sz <= size; sz <<= 1) {
    for (int stride = sz >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < size; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const bool desc = ((i & sz) == 0);
          const uint64_t x = sel[i], y = sel[j];
          if (desc ? (x < y) : (x > y)) { sel[i] = y; sel[j] = x; }
        }
      }
      __syncthreads();
    }
  }
}

__device__ __forceinline__ int pow2_at_least(int k) {
  int s = 1;
  while (s < k) s <<= 1;
  return s < 2 ? 2 : s;
}

__device__ __forceinline__ void write_out(const MergeArgs& a, int64_t q, int i, uint64_t key) {
  const int k = a.k;
  if (a.out_keys) {
    a.out_keys[(size_t)q * k + i] = key;
  } else if (key == 0ull) {
    a.out_ids[(size_t)q * k + i] = -1;
    a.out_scores[(size_t)q * k + i] = -__int_as_float(0x7f800000);
  } else {
    a.out_ids[(size_t)q * k + i] = (int64_t)key_id(key) + a.id_offset;
    a.out_scores[(size_t)q * k + i] = key_score(key);
  }
}
}  // namespace

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
    if (!grouped) return a.cand[base + i];
    const int64_t g = i / k, j = i % k;
    return a.cand[(size_t)g * a.gstride + (size_t)q * a.qstride + j];
  };
  if (cached) {
    for (int i = tid; i < M; i += kThreads) cache[i] = cand_g(i);
    __syncthreads();
  }
  auto cand = [&](int64_t i) -> uint64_t { return cached ? cache[i] : cand_g(i); };

  // Prefilter (as in select_dense_kernel): T0 = k-th largest per-thread maximum is a lower
  // bound of the k-th largest key; sort the keys >= T0 directly when they are few.
  {
    __shared__ uint64_t tmax[kThreads];
    uint64_t mx = 0ull;
    for (int64_t i = tid; i < M; i += kThreads) {
      const uint64_t c = cand(i);
      mx = c > mx ? c : mx;
    }
    tmax[tid] = mx;
    if (tid == 0) s_pos = 0;
    __syncthreads();
    for (int sz = 2; sz <= kThreads; sz <<= 1)
      for (int st = sz >> 1; st > 0; st >>= 1) {
        const int j = tid ^ st;
        if (j > tid) {
          const bool desc = (tid & sz) == 0;
          const uint64_t x = tmax[tid], y = tmax[j];
          if (desc ? x < y : x > y) { tmax[tid] = y; tmax[j] = x; }
        }
        __syncthreads();
      }
    const uint64_t T0 = tmax[k - 1];
    uint64_t* buf = cached ? nullptr : cache;   // reuse the smem cache when it is not in use
    __shared__ uint64_t small[512];
    const int cap = cached ? 512 : kSmemCand;
    if (cached) buf = small;
    for (int64_t i = tid; i < M; i += kThreads) {
      const uint64_t c = cand(i);
      if (c >= T0 && c != 0ull) {
        const int p = atomicAdd(&s_pos, 1);
        if (p < cap) buf[p] = c;
      }
    }
    __syncthreads();
    const int nc = s_pos;
    if (nc <= cap) {
      const int size = pow2_at_least(nc < k ? k : nc);
      if (size <= cap) {
        for (int i = nc + tid; i < size; i += kThreads) buf[i] = 0ull;
        __syncthreads();
        sort_desc(buf, size);
        for (int i = tid; i < k; i += kThreads) write_out(a, q, i, i < nc ? buf[i] : 0ull);
        return;
      }
    }
    __syncthreads();
  }

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
    if (tid < 32) pick_bucket(hist, kr, &s_bucket, &s_above);
    __syncthreads();
    prefix |= (uint64_t)s_bucket << shift;
    pmask |= 255ull << shift;
    kr -= s_above;
  }
  // prefix = T, the k-th largest key; (k - kr) keys are strictly larger.
  const uint64_t T = prefix;
  const int size = pow2_at_least(k);
  if (tid == 0) s_pos = 0;
  for (int i = tid; i < size; i += kThreads) sel[i] = 0ull;
  __syncthreads();
  for (int64_t i = tid; i < M; i += kThreads) {
    const uint64_t c = cand(i);
    if (c > T) sel[atomicAdd(&s_pos, 1)] = c;
  }
  __syncthreads();
  for (int i = (k - kr) + tid; i < k; i += kThreads) sel[i] = T;
  __syncthreads();
  sort_desc(sel, size);   // zeros (empty) sink to the end
  for (int i = tid; i < k; i += kThreads) write_out(a, q, i, sel[i]);
}

// Top-k of a dense score row (probe: one row of nq x nlist centroid scores): keys
// (score desc, index asc).  Scores are cached in dynamic smem as order-preserving uint32,
// a 4-pass radix select finds the k-th value T, and the values equal to T are taken in
// index order (contiguous per-thread chunks + a block prefix sum), which reproduces the
// 64-bit key order exactly.
__global__ void __launch_bounds__(kThreads)
select_dense_kernel(const MergeArgs a) {
  extern __shared__ uint32_t vals[];
  __shared__ uint32_t hist[256];
  __shared__ uint64_t sel[kMaxK];
  __shared__ int s_bucket, s_above, s_pos;
  __shared__ int wsum[kThreads / 32];
  __shared__ uint32_t tmax[kThreads];
  __shared__ uint64_t cand[kPrefilterCap];

  const int64_t q = blockIdx.x;
  const int k = a.k;
  const int M = (int)a.m_flat;
  const float* row = a.cand_scores + (size_t)q * a.qstride;
  const int tid = threadIdx.x;
  uint32_t mx = 0u;
  if ((M & 3) == 0 && ((reinterpret_cast<uintptr_t>(row) & 15) == 0)) {
    // 16-byte loads, 4 in flight per thread: this load is the latency-critical part for
    // small batches (one CTA per query streams the whole score row)
    const float4* r4 = reinterpret_cast<const float4*>(row);
    const int M4 = M >> 2;
    for (int i0 = tid; i0 < M4; i0 += 4 * kThreads) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = (i0 + u * kThreads < M4) ? __ldg(r4 + i0 + u * kThreads)
                                                                   : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + u * kThreads;
        if (i < M4) {
          const uint32_t o0 = ordered_from_float(v[u].x), o1 = ordered_from_float(v[u].y);
          const uint32_t o2 = ordered_from_float(v[u].z), o3 = ordered_from_float(v[u].w);
          *reinterpret_cast<uint4*>(vals + 4 * i) = make_uint4(o0, o1, o2, o3);
          mx = max(mx, max(max(o0, o1), max(o2, o3)));
        }
      }
    }
  } else {
    for (int i = tid; i < M; i += kThreads) {
      const uint32_t v = ordered_from_float(row[i]);
      vals[i] = v;
      mx = v > mx ? v : mx;
    }
  }
  tmax[tid] = mx;
  if (tid == 0) s_pos = 0;
  __syncthreads();
  // Prefilter: the k-th largest of the per-thread maxima (k <= kThreads) is a lower bound
  // T0 of the k-th largest value (k threads each hold a value >= it).  Usually only a few
  // hundred values reach T0; they are sorted directly.  Too many (heavy ties) -> radix path.
  {
    // bitonic sort of the 256 maxima, descending
    for (int sz = 2; sz <= kThreads; sz <<= 1)
      for (int st = sz >> 1; st > 0; st >>= 1) {
        const int j = tid ^ st;
        if (j > tid) {
          const bool desc = (tid & sz) == 0;
          const uint32_t x = tmax[tid], y = tmax[j];
          if (desc ? x < y : x > y) { tmax[tid] = y; tmax[j] = x; }
        }
        __syncthreads();
      }
    const uint32_t T0 = k <= kThreads ? tmax[k - 1] : 0u;
    for (int i = tid; i < M; i += kThreads) {
      const uint32_t v = vals[i];
      if (v >= T0) {
        const int p = atomicAdd(&s_pos, 1);
        if (p < kPrefilterCap) cand[p] = ((uint64_t)v << 32) | (0xFFFFFFFFu - (uint32_t)i);
      }
    }
    __syncthreads();
    const int nc = s_pos;
    if (k <= kThreads && nc <= kPrefilterCap) {
      const int size = pow2_at_least(nc < k ? k : nc);
      for (int i = nc + tid; i < size; i += kThreads) cand[i] = 0ull;
      __syncthreads();
      sort_desc(cand, size);
      for (int i = tid; i < k; i += kThreads) write_out(a, q, i, i < nc ? cand[i] : 0ull);
      return;
    }
    __syncthreads();
  }

  uint32_t prefix = 0, pmask = 0;
  int kr = k;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    for (int i = tid; i < 256; i += kThreads) hist[i] = 0;
    __syncthreads();
    for (int i = tid; i < M; i += kThreads) {
      const uint32_t v = vals[i];
      if ((v & pmask) == prefix) atomicAdd(&hist[(v >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid < 32) pick_bucket(hist, kr, &s_bucket, &s_above);
    __syncthreads();
    prefix |= (uint32_t)s_bucket << shift;
    pmask |= 255u << shift;
    kr -= s_above;
  }
  const uint32_t T = prefix;            // k-th largest value; k - kr values are larger
  const int size = pow2_at_least(k);
  if (tid == 0) s_pos = 0;
  for (int i = tid; i < size; i += kThreads) sel[i] = 0ull;
  __syncthreads();
  // values > T: any order (the sort fixes it)
  for (int i = tid; i < M; i += kThreads)
    if (vals[i] > T) sel[atomicAdd(&s_pos, 1)] = ((uint64_t)vals[i] << 32) | (0xFFFFFFFFu - (uint32_t)i);
  // values == T: the kr smallest indices -- contiguous chunks, block prefix count
  const int chunk = (M + kThreads - 1) / kThreads;
  const int lo = tid * chunk, hi = min(M, lo + chunk);
  int my = 0;
  for (int i = lo; i < hi; ++i) my += vals[i] == T;
  int incl = my;
  const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  int wbase = 0;
  for (int w = 0; w < wid; ++w) wbase += wsum[w];
  int r = wbase + incl - my;           // rank among equal values of my first equal element
  const int first = k - kr;
  for (int i = lo; i < hi && r < kr; ++i)
    if (vals[i] == T) {
      sel[first + r] = ((uint64_t)T << 32) | (0xFFFFFFFFu - (uint32_t)i);
      ++r;
    }
  __syncthreads();
  sort_desc(sel, size);
  for (int i = tid; i < k; i += kThreads) write_out(a, q, i, sel[i]);
}

// Top-k (k <= 64) of a dense score row without caching the row in shared memory, so 6-8 CTAs
// fit an SM and a 512-query probe runs in one wave (select_dense_kernel's 64 KB row cache
// allows 2 per SM).  Two streaming passes over the row (L2-resident right after the score
// dump): (1) each thread keeps its two largest values; each warp sorts its 64 and T_w = their
// k-th largest is a lower bound of the row's k-th largest value (k distinct elements are
// >= T_w), T0 = max_w T_w;
// (2) the values >= T0 (usually ~100) are appended to smem as (value, index) keys and each
// key's rank among them (keys are distinct) is its output position.  More than kStreamCap
// survivors (heavy ties): the exact radix select of select_dense_kernel, reading the row from
// global memory.  Same keys and ties as select_dense_kernel (value desc, index asc).
constexpr int kStreamCap = 1024;
constexpr int kStreamMaxK = 64;
constexpr int kStreamLoads = 8;   // float4 loads in flight per thread and pass

__global__ void __launch_bounds__(kThreads)
select_dense_stream_kernel(const MergeArgs a) {
  __shared__ uint64_t cand[kStreamCap];
  __shared__ uint32_t wT[kThreads / 32];
  __shared__ uint32_t hist[256];
  __shared__ uint64_t sel[kStreamMaxK];
  __shared__ int s_pos, s_bucket, s_above;
  __shared__ int wsum[kThreads / 32];
  const int64_t q = blockIdx.x;
  const int k = a.k;
  const int M = (int)a.m_flat;
  const float* row = a.cand_scores + (size_t)q * a.qstride;
  const float4* r4 = reinterpret_cast<const float4*>(row);
  const int M4 = M >> 2;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) s_pos = 0;
  // pass 1: per-thread two largest values, kStreamLoads float4 loads in flight
  uint32_t m1 = 0u, m2 = 0u;
  for (int i0 = tid; i0 < M4; i0 += kStreamLoads * kThreads) {
    float4 v[kStreamLoads];
#pragma unroll
    for (int u = 0; u < kStreamLoads; ++u)
      v[u] = i0 + u * kThreads < M4 ? __ldcg(r4 + i0 + u * kThreads)
                                    : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
#pragma unroll
    for (int u = 0; u < kStreamLoads; ++u) {
      const float f[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint32_t o = ordered_from_float(f[c]);
        m2 = max(m2, min(m1, o));
        m1 = max(m1, o);
      }
    }
  }
  // bitonic sort of the warp's 64 values {m1, m2} (element e = j * 32 + lane of register j),
  // descending; element k-1 is the k-th largest
  uint32_t x[2] = {m1, m2};
#pragma unroll
  for (int sz = 2; sz <= 64; sz <<= 1)
#pragma unroll
    for (int st = sz >> 1; st > 0; st >>= 1) {
      if (st == 32) {   // sz == 64: partners are the lane's two registers, all descending
        const uint32_t hi = max(x[0], x[1]), lo = min(x[0], x[1]);
        x[0] = hi;
        x[1] = lo;
      } else {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int e = j * 32 + lane;
          const uint32_t y = __shfl_xor_sync(0xffffffffu, x[j], st);
          const bool desc = (e & sz) == 0 || sz == 64;
          const bool lower = (e & st) == 0;
          x[j] = (lower == desc) ? max(x[j], y) : min(x[j], y);
        }
      }
    }
  const uint32_t tw = __shfl_sync(0xffffffffu, (k - 1) < 32 ? x[0] : x[1], (k - 1) & 31);
  if (lane == 0) wT[wid] = tw;
  __syncthreads();
  uint32_t T0 = 0u;
#pragma unroll
  for (int w = 0; w < kThreads / 32; ++w) T0 = max(T0, wT[w]);
  // pass 2: the values >= T0 as keys
  for (int i0 = tid; i0 < M4; i0 += kStreamLoads * kThreads) {
    float4 v[kStreamLoads];
#pragma unroll
    for (int u = 0; u < kStreamLoads; ++u)
      v[u] = i0 + u * kThreads < M4 ? __ldcg(r4 + i0 + u * kThreads)
                                    : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
#pragma unroll
    for (int u = 0; u < kStreamLoads; ++u) {
      const float f[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const uint32_t o = ordered_from_float(f[c]);
        if (o >= T0 && i0 + u * kThreads < M4) {
          const int p = atomicAdd(&s_pos, 1);
          const uint32_t idx = (uint32_t)(4 * (i0 + u * kThreads) + c);
          if (p < kStreamCap) cand[p] = ((uint64_t)o << 32) | (0xFFFFFFFFu - idx);
        }
      }
    }
  }
  __syncthreads();
  const int nc = s_pos;
  if (nc <= kStreamCap) {
    // rank of each key among the survivors = its output position
    for (int i = tid; i < nc; i += kThreads) {
      const uint64_t key = cand[i];
      int r = 0;
      for (int j = 0; j < nc; ++j) r += cand[j] > key;
      if (r < k) write_out(a, q, r, key);
    }
    for (int i = nc + tid; i < k; i += kThreads) write_out(a, q, i, 0ull);
    return;
  }
  // heavy ties: exact radix select over the row (global reads), as select_dense_kernel
  auto val = [&](int i) { return ordered_from_float(__ldcg(row + i)); };
  uint32_t prefix = 0, pmask = 0;
  int kr = k;
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    for (int i = tid; i < 256; i += kThreads) hist[i] = 0;
    __syncthreads();
    for (int i = tid; i < M; i += kThreads) {
      const uint32_t v = val(i);
      if ((v & pmask) == prefix) atomicAdd(&hist[(v >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (tid < 32) pick_bucket(hist, kr, &s_bucket, &s_above);
    __syncthreads();
    prefix |= (uint32_t)s_bucket << shift;
    pmask |= 255u << shift;
    kr -= s_above;
  }
  const uint32_t T = prefix;            // k-th largest value; k - kr values are larger
  const int size = pow2_at_least(k);
  if (tid == 0) s_pos = 0;
  for (int i = tid; i < size; i += kThreads) sel[i] = 0ull;
  __syncthreads();
  for (int i = tid; i < M; i += kThreads) {
    const uint32_t v = val(i);
    if (v > T) sel[atomicAdd(&s_pos, 1)] = ((uint64_t)v << 32) | (0xFFFFFFFFu - (uint32_t)i);
  }
  // values == T: the kr smallest indices -- contiguous chunks, block prefix count
  const int chunk = (M + kThreads - 1) / kThreads;
  const int lo = tid * chunk, hi = min(M, lo + chunk);
  int my = 0;
  for (int i = lo; i < hi; ++i) my += val(i) == T;
  int incl = my;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  int wbase = 0;
  for (int w = 0; w < wid; ++w) wbase += wsum[w];
  int r = wbase + incl - my;
  const int first = k - kr;
  for (int i = lo; i < hi && r < kr; ++i)
    if (val(i) == T) {
      sel[first + r] = ((uint64_t)T << 32) | (0xFFFFFFFFu - (uint32_t)i);
      ++r;
    }
  __syncthreads();
  sort_desc(sel, size);
  for (int i = tid; i < k; i += kThreads) write_out(a, q, i, sel[i]);
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
    write_out(a, q, 0, best);
  }
}

cudaError_t launch_merge(const MergeArgs& a, int64_t nq, cudaStream_t stream) {
  if (nq <= 0) return cudaSuccess;
  // k <= 32: for larger k the per-warp bound (the k-th of 64 lane values) is weaker, more values
  // survive and the quadratic ranking loses to the cached radix select (measured at k = 48,
  // M = 16384: 42 vs 27 us)
  if (a.cand_scores && a.k <= 32 && (a.m_flat & 3) == 0 && (a.qstride & 3) == 0 &&
      (reinterpret_cast<uintptr_t>(a.cand_scores) & 15) == 0 && a.m_flat >= kThreads) {
    select_dense_stream_kernel<<<(unsigned)nq, kThreads, 0, stream>>>(a);
    note_launch();
    return cudaGetLastError();
  }
  if (a.cand_scores) {
    const size_t smem = (size_t)a.m_flat * sizeof(uint32_t);
    cudaError_t e = ensure_max_smem(reinterpret_cast<const void*>(select_dense_kernel), smem);
    if (e != cudaSuccess) return e;
    select_dense_kernel<<<(unsigned)nq, kThreads, smem, stream>>>(a);
    note_launch();
    return cudaGetLastError();
  }
  if (a.k == 1 && !a.slot_off && a.m_flat <= 0 && a.groups <= 64) {
    int64_t blocks = (nq + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    merge_top1_kernel<<<(unsigned)blocks, 256, 0, stream>>>(a, nq);
    note_launch();
    return cudaGetLastError();
  }
  merge_topk_kernel<<<(unsigned)nq, kThreads, 0, stream>>>(a);
  note_launch();
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
  note_launch();
  return cudaGetLastError();
}

}  // namespace sa
