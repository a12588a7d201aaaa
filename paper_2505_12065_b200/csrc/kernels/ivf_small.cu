// ivf_small.cu -- IVF search of an agent-step batch in ONE cooperative launch (SURVEY.md §8(d)
// C5; DESIGN.md §4.2 "small batches").
//
// SearchAgent-X retrieves once per <search> tag (Alg. 1), a handful of
// queries at a time, and the engine stalls until the documents arrive: an agent step
// is latency-bound.  The batch path (probe kernel + select + inversion + list scan + merge)
// costs ~10 launches of fixed overhead for ~20 us of HBM work at batch 1.  Here the whole
// search -- R11's probe and the exact scan of the probed lists with the R5 ordering -- is
// one kernel of one CTA per SM, phases separated by grid-wide barriers:
//   A  centroid scores: each CTA streams its 1/G of the bf16 centroids (the dominant read,
//      25 MB at nlist = 16384, d = 768) and writes the fp32 scores <q, c> of every query;
//   B  probe: CTA q selects query q's nprobe best lists from its nlist scores (exact MSB-first
//      radix select on the ordered fp32 bits; ties at the threshold -> lowest list id, R11);
//   C  scan: the probed lists are cut into 64-row chunks, every CTA takes an equal share;
//      16 warps x 4 rows in flight, fp32 dot products against the query in shared memory,
//      per-warp top-k lists, merged into one list per (CTA, query);
//   D  merge: CTA q keeps the k best of the G per-CTA lists of query q (R5 order) and writes
//      the result (packed keys for a cross-rank merge, or ids / scores padded -1 / -inf).
// Scores are fp32 sums of exact bf16 products on the CUDA cores (the batch path uses the
// tensor cores; the two agree up to fp32 rounding order, i.e. at near-ties, R36).
#include <cooperative_groups.h>
#include <cuda_bf16.h>

#include "ivf_small.cuh"
#include "keys.cuh"
#include "launch.cuh"

namespace sa {

namespace cg = cooperative_groups;

namespace {

constexpr int kThreads = IVSM_THREADS;
constexpr int kWarps = kThreads / 32;
constexpr int kChunk = 64;           // rows per scan work item (16 warps x 4 rows)
constexpr int kRowsPerWarp = 4;
constexpr int kMaxDPad = 768;
constexpr int kMaxNp = IVSM_MAX_NQ * IVSM_MAX_NPROBE;

struct SmallSmem {
  float q[IVSM_MAX_NQ][kMaxDPad];            // the queries, bf16-rounded, widened to fp32
  uint64_t wl[kWarps][IVSM_MAX_NQ][IVSM_MAX_K];  // per-warp top-k lists (descending)
  int32_t pre[kMaxNp + 1];                   // exclusive prefix of chunks per probe entry
  int32_t lst[kMaxNp];                       // probe entry -> list id
  uint32_t hist[256];
  uint64_t red[kWarps];
  int32_t s_int[4];
};

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t x = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += x;
  }
  return v;
}

// Block-wide max of one u64 per thread (result to every thread).
__device__ __forceinline__ uint64_t block_max(uint64_t v, SmallSmem& sm) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t x = __shfl_xor_sync(0xffffffffu, v, o);
    v = x > v ? x : v;
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sm.red[threadIdx.x >> 5] = v;
  __syncthreads();
  uint64_t m = 0ull;
#pragma unroll
  for (int w = 0; w < kWarps; ++w) m = sm.red[w] > m ? sm.red[w] : m;
  return m;
}

// Descending bitonic sort of 64 keys held by one warp, two per lane (x0 = element lane,
// x1 = element lane + 32).
__device__ __forceinline__ void warp_sort64_desc(uint64_t& x0, uint64_t& x1) {
  const int lane = threadIdx.x & 31;
  for (int size = 2; size <= 64; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride == 32) {                  // partners sit in the same lane
        const uint64_t hi = x0 > x1 ? x0 : x1, lo = x0 > x1 ? x1 : x0;
        x0 = hi;
        x1 = lo;
        continue;
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint64_t& v = h ? x1 : x0;
        const int i = lane + 32 * h;
        const uint64_t o = __shfl_xor_sync(0xffffffffu, v, stride);
        const bool keep_max = ((i & stride) == 0) == ((i & size) == 0);
        v = keep_max ? (v > o ? v : o) : (v > o ? o : v);
      }
    }
  }
}

// Descending bitonic sort of sv[0, P) in shared memory by the whole block (P a power of two).
__device__ void block_sort_desc(uint64_t* sv, int P) {
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int j = i ^ stride;
        if (j > i) {
          const uint64_t a = sv[i], b = sv[j];
          const bool desc = (i & size) == 0;
          if (desc ? a < b : a > b) {
            sv[i] = b;
            sv[j] = a;
          }
        }
      }
    }
  }
  __syncthreads();
}

// The k best keys of L descending lists of k keys (list j at lists[j * lstride], empty slots
// 0) -> out[0, k) descending (0-padded), by the whole block.  Every key of the top k is
// >= T = max_j lists[j][k-1] (k keys of one list are >= T), so only those survive to a sort.
__device__ void topk_of_lists(const uint64_t* lists, int L, int64_t lstride, int k,
                              uint64_t* sv, int sv_cap, uint64_t* out, SmallSmem& sm) {
  uint64_t t = 0ull;
  for (int j = threadIdx.x; j < L; j += blockDim.x) {
    const uint64_t x = lists[(int64_t)j * lstride + k - 1];
    t = x > t ? x : t;
  }
  const uint64_t T = block_max(t, sm);
  if (threadIdx.x == 0) sm.s_int[0] = 0;
  __syncthreads();
  for (int e = threadIdx.x; e < L * k; e += blockDim.x) {
    const uint64_t x = lists[(int64_t)(e / k) * lstride + e % k];
    if (x != 0ull && x >= T) {
      const int pos = atomicAdd(&sm.s_int[0], 1);
      if (pos < sv_cap) sv[pos] = x;
    }
  }
  __syncthreads();
  const int m = min(sm.s_int[0], sv_cap);
  if (m <= 64) {
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      uint64_t x0 = lane < m ? sv[lane] : 0ull, x1 = lane + 32 < m ? sv[lane + 32] : 0ull;
      warp_sort64_desc(x0, x1);
      if (lane < k) out[lane] = x0;
      if (lane + 32 < k) out[lane + 32] = x1;
    }
  } else {
    int P = 1;
    while (P < m) P <<= 1;
    for (int i = m + threadIdx.x; i < P; i += blockDim.x) sv[i] = 0ull;
    block_sort_desc(sv, P);
    for (int i = threadIdx.x; i < k; i += blockDim.x) out[i] = sv[i];
  }
  __syncthreads();
}

}  // namespace

// survivors capacity of the merges: a power of two >= max(grid * k, warps * IVSM_MAX_K)
__host__ __device__ inline int sv_capacity(int grid, int k) {
  int p = 1;
  while (p < grid * k || p < kWarps * IVSM_MAX_K) p <<= 1;
  return p;
}

template <int NQ>
__global__ void __launch_bounds__(kThreads, 1) ivf_small_kernel(const IvfSmallArgs a) {
  // dynamic smem: SmallSmem, then a region shared by phase B (nlist ordered scores) and the
  // merges of phases C / D (survivors + the k results)
  extern __shared__ __align__(16) uint8_t smem_raw[];
  SmallSmem& sm = *reinterpret_cast<SmallSmem*>(smem_raw);
  uint8_t* dyn = smem_raw + (sizeof(SmallSmem) + 15) / 16 * 16;
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x, b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nch = a.d_pad / 8;   // 16-byte chunks per row
  const int k = a.k;

  // queries -> smem, RNE-rounded to bf16 (R3) then widened exactly; padding is zero
  for (int i = threadIdx.x; i < NQ * a.d_pad; i += kThreads) {
    const int qi = i / a.d_pad, c = i % a.d_pad;
    float v = 0.f;
    if (qi < a.nq && c < a.d) {
      v = a.q_f32 ? __bfloat162float(__float2bfloat16_rn(
                        static_cast<const float*>(a.Q)[(int64_t)qi * a.d + c]))
                  : __bfloat162float(static_cast<const __nv_bfloat16*>(a.Q)[(int64_t)qi * a.d + c]);
    }
    sm.q[qi][c] = v;
  }
  __syncthreads();

  // ---- A: centroid scores of this CTA's share of the lists
  {
    const int c0 = (int)((int64_t)b * a.nlist / G), c1 = (int)((int64_t)(b + 1) * a.nlist / G);
    const uint4* C4 = reinterpret_cast<const uint4*>(a.C);
    for (int c = c0 + warp * 2; c < c1; c += kWarps * 2) {
      uint4 v[2][3];
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int u = 0; u < 3; ++u) {
          const int ch = lane + 32 * u;
          v[r][u] = (c + r < c1 && ch < nch) ? __ldg(C4 + (int64_t)(c + r) * nch + ch)
                                             : make_uint4(0, 0, 0, 0);
        }
      float acc[2][NQ];
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int qi = 0; qi < NQ; ++qi) acc[r][qi] = 0.f;
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        const int ch = lane + 32 * u;
        if (ch >= nch) break;
#pragma unroll
        for (int qi = 0; qi < NQ; ++qi) {
          const float4 qa = *reinterpret_cast<const float4*>(&sm.q[qi][ch * 8]);
          const float4 qb = *reinterpret_cast<const float4*>(&sm.q[qi][ch * 8 + 4]);
#pragma unroll
          for (int r = 0; r < 2; ++r) {
            const uint4 w = v[r][u];
            float x = acc[r][qi];
            x = fmaf(__uint_as_float(w.x << 16), qa.x, x);
            x = fmaf(__uint_as_float(w.x & 0xFFFF0000u), qa.y, x);
            x = fmaf(__uint_as_float(w.y << 16), qa.z, x);
            x = fmaf(__uint_as_float(w.y & 0xFFFF0000u), qa.w, x);
            x = fmaf(__uint_as_float(w.z << 16), qb.x, x);
            x = fmaf(__uint_as_float(w.z & 0xFFFF0000u), qb.y, x);
            x = fmaf(__uint_as_float(w.w << 16), qb.z, x);
            x = fmaf(__uint_as_float(w.w & 0xFFFF0000u), qb.w, x);
            acc[r][qi] = x;
          }
        }
      }
#pragma unroll
      for (int r = 0; r < 2; ++r)
#pragma unroll
        for (int qi = 0; qi < NQ; ++qi) {
          float s = acc[r][qi];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
          if (lane == 0 && qi < a.nq && c + r < c1) a.psc[(int64_t)qi * a.nlist + c + r] = s;
        }
    }
  }
  grid.sync();

  // ---- B: query b's probe set = its nprobe best lists (ties -> lowest list id)
  if (b < a.nq) {
    uint32_t* key = reinterpret_cast<uint32_t*>(dyn);
    const float* ps = a.psc + (int64_t)b * a.nlist;
    for (int c = threadIdx.x; c < a.nlist; c += kThreads) key[c] = ordered_from_float(ps[c]);
    uint32_t prefix = 0u, mask = 0u;
    int remaining = a.nprobe;
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int i = threadIdx.x; i < 256; i += kThreads) sm.hist[i] = 0u;
      __syncthreads();
      for (int c = threadIdx.x; c < a.nlist; c += kThreads) {
        const uint32_t v = key[c];
        if ((v & mask) == prefix) atomicAdd(&sm.hist[(v >> shift) & 255u], 1u);
      }
      __syncthreads();
      if (warp == 0) {
        // buckets from the top, 8 per lane: the first bucket where the count reaches
        // `remaining` holds the threshold
        uint32_t cnt[8], sum = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          cnt[i] = sm.hist[255 - (lane * 8 + i)];
          sum += cnt[i];
        }
        const uint32_t incl = warp_incl_scan(sum);
        const unsigned hit = __ballot_sync(0xffffffffu, incl >= (uint32_t)remaining);
        const int owner = hit ? __ffs(hit) - 1 : 31;
        if (lane == owner) {
          uint32_t acc = incl - sum;
          int bk = 255 - lane * 8;
          for (int i = 0; i < 8; ++i, --bk) {
            if (bk == 0 || acc + cnt[i] >= (uint32_t)remaining) break;
            acc += cnt[i];
          }
          sm.s_int[1] = bk;
          sm.s_int[2] = (int)acc;
        }
      }
      __syncthreads();
      remaining -= sm.s_int[2];
      prefix |= (uint32_t)sm.s_int[1] << shift;
      mask |= 255u << shift;
      __syncthreads();
    }
    // prefix = the nprobe-th largest value T; take every list above T, then the first
    // `remaining` lists equal to T in ascending id order
    int32_t* out = a.probes + (int64_t)b * a.nprobe;
    if (threadIdx.x == 0) sm.s_int[0] = 0;
    __syncthreads();
    for (int c = threadIdx.x; c < a.nlist; c += kThreads)
      if (key[c] > prefix) out[atomicAdd(&sm.s_int[0], 1)] = c;
    __syncthreads();
    const int above = sm.s_int[0];
    int taken = 0;
    for (int c0 = 0; c0 < a.nlist && taken < remaining; c0 += kThreads) {
      const int c = c0 + threadIdx.x;
      const bool eq = c < a.nlist && key[c] == prefix;
      const unsigned bal = __ballot_sync(0xffffffffu, eq);
      if (lane == 0) sm.red[warp] = __popc(bal);
      __syncthreads();
      int before = 0, tot = 0;
      for (int w = 0; w < kWarps; ++w) {
        const int n = (int)sm.red[w];
        if (w < warp) before += n;
        tot += n;
      }
      const int pos = taken + before + __popc(bal & ((1u << lane) - 1u));
      if (eq && pos < remaining) out[above + pos] = c;
      taken += tot;
      __syncthreads();
    }
  }
  grid.sync();

  // ---- C: scan the probed lists in 64-row chunks, an equal share of chunks per CTA
  const int np = a.nq * a.nprobe;
  for (int e = threadIdx.x; e < np; e += kThreads) sm.lst[e] = a.probes[e];
  __syncthreads();
  {
    // exclusive prefix of chunk counts (np <= 2048: 4 entries per thread)
    int loc[4], s = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = threadIdx.x * 4 + i;
      int c = 0;
      if (e < np) {
        const int l = sm.lst[e];
        c = (int)((a.list_off[l + 1] - a.list_off[l] + kChunk - 1) / kChunk);
      }
      loc[i] = s;
      s += c;
    }
    const uint32_t incl = warp_incl_scan((uint32_t)s);
    if (lane == 31) sm.red[warp] = incl;
    __syncthreads();
    int base = 0;
    for (int w = 0; w < warp; ++w) base += (int)sm.red[w];
    base += (int)incl - s;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = threadIdx.x * 4 + i;
      if (e < np) sm.pre[e] = base + loc[i];
    }
    if (threadIdx.x == kThreads - 1) sm.pre[np] = base + s;
    for (int i = threadIdx.x; i < kWarps * IVSM_MAX_NQ * IVSM_MAX_K; i += kThreads)
      (&sm.wl[0][0][0])[i] = 0ull;
    __syncthreads();
  }
  const int total = sm.pre[np];
  const int cb = (int)((int64_t)b * total / G), ce = (int)((int64_t)(b + 1) * total / G);
  const uint4* X4 = reinterpret_cast<const uint4*>(a.X);
  int e = 0;
  for (int ch = cb; ch < ce; ++ch) {
    // probe entry of chunk ch: the last e with pre[e] <= ch (entries with no rows are skipped)
    int lo = e, hi = np - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (sm.pre[mid] <= ch) lo = mid;
      else hi = mid - 1;
    }
    e = lo;
    const int qi = e / a.nprobe;
    const int l = sm.lst[e];
    const int64_t lend = a.list_off[l + 1];
    const int64_t r0 = a.list_off[l] + (int64_t)(ch - sm.pre[e]) * kChunk + warp * kRowsPerWarp;
    uint4 v[kRowsPerWarp][3];
#pragma unroll
    for (int r = 0; r < kRowsPerWarp; ++r)
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        const int cc = lane + 32 * u;
        v[r][u] = (r0 + r < lend && cc < nch) ? __ldg(X4 + (r0 + r) * nch + cc)
                                              : make_uint4(0, 0, 0, 0);
      }
    float acc[kRowsPerWarp];
#pragma unroll
    for (int r = 0; r < kRowsPerWarp; ++r) acc[r] = 0.f;
    const float* qv = sm.q[qi];
#pragma unroll
    for (int u = 0; u < 3; ++u) {
      const int cc = lane + 32 * u;
      if (cc >= nch) break;
      const float4 qa = *reinterpret_cast<const float4*>(qv + cc * 8);
      const float4 qb = *reinterpret_cast<const float4*>(qv + cc * 8 + 4);
#pragma unroll
      for (int r = 0; r < kRowsPerWarp; ++r) {
        const uint4 w = v[r][u];
        acc[r] = fmaf(__uint_as_float(w.x << 16), qa.x, acc[r]);
        acc[r] = fmaf(__uint_as_float(w.x & 0xFFFF0000u), qa.y, acc[r]);
        acc[r] = fmaf(__uint_as_float(w.y << 16), qa.z, acc[r]);
        acc[r] = fmaf(__uint_as_float(w.y & 0xFFFF0000u), qa.w, acc[r]);
        acc[r] = fmaf(__uint_as_float(w.z << 16), qb.x, acc[r]);
        acc[r] = fmaf(__uint_as_float(w.z & 0xFFFF0000u), qb.y, acc[r]);
        acc[r] = fmaf(__uint_as_float(w.w << 16), qb.z, acc[r]);
        acc[r] = fmaf(__uint_as_float(w.w & 0xFFFF0000u), qb.w, acc[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < kRowsPerWarp; ++r)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
    if (lane == 0) {
      uint64_t* wl = sm.wl[warp][qi];
#pragma unroll
      for (int r = 0; r < kRowsPerWarp; ++r) {
        if (r0 + r >= lend) break;
        uint64_t key = make_key(acc[r], (uint32_t)a.row_ids[r0 + r]);
        if (key <= wl[k - 1]) continue;
        for (int j = 0; j < k; ++j) {      // insert into the descending list
          const uint64_t x = wl[j];
          if (key > x) {
            wl[j] = key;
            key = x;
          }
        }
      }
    }
  }
  __syncthreads();
  // this CTA's k best per query (the 16 warp lists merged) -> cand[b][q]
  {
    uint64_t* sv = reinterpret_cast<uint64_t*>(dyn);
    for (int qi = 0; qi < a.nq; ++qi)
      topk_of_lists(&sm.wl[0][qi][0], kWarps, (int64_t)IVSM_MAX_NQ * IVSM_MAX_K, k, sv,
                    sv_capacity(G, k), a.cand + ((int64_t)b * a.nq + qi) * k, sm);
  }
  grid.sync();

  // ---- D: query b's k best over the G per-CTA lists -> output
  if (b < a.nq) {
    uint64_t* sv = reinterpret_cast<uint64_t*>(dyn);
    const int cap = sv_capacity(G, k);
    uint64_t* best = sv + cap;   // the k sorted keys, after the survivors
    topk_of_lists(a.cand + (int64_t)b * k, G, (int64_t)a.nq * k, k, sv, cap, best, sm);
    for (int j = threadIdx.x; j < k; j += kThreads) {
      const uint64_t key = best[j];
      const int64_t o = (int64_t)b * k + j;
      if (a.out_keys) {
        a.out_keys[o] = key;
      } else {
        a.out_ids[o] = key == 0ull ? -1 : (int64_t)key_id(key);
        a.out_scores[o] = key == 0ull ? -__int_as_float(0x7f800000) : key_score(key);
      }
    }
  }
}

size_t ivf_small_smem_bytes(int nlist, int grid, int k) {
  // phase B: nlist ordered scores; phases C / D: survivors + the k results
  const size_t cd = ((size_t)sv_capacity(grid, k) + IVSM_MAX_K) * sizeof(uint64_t);
  const size_t bsel = (size_t)nlist * sizeof(uint32_t);
  return (sizeof(SmallSmem) + 15) / 16 * 16 + (bsel > cd ? bsel : cd);
}

cudaError_t launch_ivf_small(const IvfSmallArgs& a, int grid, cudaStream_t s) {
  if (a.nq < 1 || a.nq > IVSM_MAX_NQ || a.k < 1 || a.k > IVSM_MAX_K || a.nprobe < 1 ||
      a.nprobe > IVSM_MAX_NPROBE || a.d_pad > kMaxDPad || grid < a.nq)
    return cudaErrorInvalidValue;
  const size_t smem = ivf_small_smem_bytes(a.nlist, grid, a.k);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = ensure_max_smem(reinterpret_cast<const void*>(kern), smem);
    if (e != cudaSuccess) return e;
    e = cudaLaunchKernelEx(&cfg, kern, a);
    note_launch();
    return e;
  };
  if (a.nq <= 1) return go(ivf_small_kernel<1>);
  if (a.nq <= 2) return go(ivf_small_kernel<2>);
  if (a.nq <= 4) return go(ivf_small_kernel<4>);
  return go(ivf_small_kernel<8>);
}

}  // namespace sa
