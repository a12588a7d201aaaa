// graph.cu -- proximity-graph ANN on B200.
//
// The paper's retriever is a graph index (HNSW) whose search range
// trades recall for effort.  Build (readings R22-R26): an approximate kNN graph
// from the IVF index (every stored row searched as a query on the tcgen05 list scan), then
// rank-only pruning by detour counts and a reverse-edge merge -- integer work on the kNN
// lists, no distances.  Search (R27): one CTA per query runs best-first beam search over a
// candidate list of L entries (the search range), expanding the w best unexpanded entries
// per iteration; neighbour rows (1.5 KB bf16 each) are gathered by whole warps with 16-byte
// loads, 3 rows (and their global ids) in flight per warp; the visited set is an exact open-addressing table in
// shared memory; scored rows below the list's L-th key are dropped at once and the few
// survivors are merged into the sorted list by rank counting.  Memory-latency bound: a query's
// iterations are dependent gathers, so several CTAs per SM hide each other's latency.
#include <cuda_bf16.h>

#include "graph.cuh"
#include "keys.cuh"
#include "launch.cuh"

namespace sa {

namespace {

unsigned grid_for(int64_t n, int per_block) {
  int64_t b = (n + per_block - 1) / per_block;
  if (b < 1) b = 1;
  if (b > 148 * 64) b = 148 * 64;
  return (unsigned)b;
}

__global__ void inverse_ids_kernel(const int32_t* __restrict__ row_ids, int64_t n,
                                   int64_t row_offset, int32_t* __restrict__ pos_of) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x)
    pos_of[(int64_t)(uint32_t)row_ids[p] - row_offset] = (int32_t)p;
}

__global__ void knn_to_pos_kernel(const int64_t* __restrict__ ids, int64_t nb, int kk, int64_t p0,
                                  const int32_t* __restrict__ pos_of, int64_t row_offset, int K,
                                  int32_t* __restrict__ knn) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb;
       b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t self = p0 + b;
    int32_t* out = knn + self * K;
    int cnt = 0;
    for (int j = 0; j < kk && cnt < K; ++j) {
      const int64_t id = ids[b * kk + j];
      if (id < 0) break;
      const int32_t pos = pos_of[id - row_offset];
      if (pos == self) continue;
      out[cnt++] = pos;
    }
    for (; cnt < K; ++cnt) out[cnt] = -1;
  }
}

constexpr int kHashW = 128;  // per-warp rank table slots (>= 2 * GR_MAX_K)

__device__ __forceinline__ uint32_t hslot(int32_t y) {
  return ((uint32_t)y * 2654435761u) >> (32 - 7);
}

// R23 + R24.  One warp per node; lanes own ranks j = lane and lane + 32.
__global__ void __launch_bounds__(256) graph_prune_kernel(const int32_t* __restrict__ knn,
                                                          int64_t n, int K, int R,
                                                          int32_t* __restrict__ fwd) {
  __shared__ int32_t hkey[8][kHashW];
  __shared__ int32_t hval[8][kHashW];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  int32_t* hk = hkey[warp];
  int32_t* hv = hval[warp];
  const int64_t nw = (int64_t)gridDim.x * 8;
  for (int64_t i = blockIdx.x * 8 + warp; i < n; i += nw) {
    const int j0 = lane, j1 = lane + 32;
    const int32_t c0 = j0 < K ? knn[i * K + j0] : -1;
    const int32_t c1 = j1 < K ? knn[i * K + j1] : -1;
    int det0 = 0, det1 = 0;
    for (int k = 0; k < K - 1; ++k) {
      const int32_t ck = __shfl_sync(0xffffffffu, k < 32 ? c0 : c1, k & 31);
      if (ck < 0) break;
      for (int s = lane; s < kHashW; s += 32) hk[s] = -1;
      __syncwarp();
      const int32_t y0 = j0 < K ? knn[(int64_t)ck * K + j0] : -1;
      const int32_t y1 = j1 < K ? knn[(int64_t)ck * K + j1] : -1;
      if (y0 >= 0) {
        uint32_t h = hslot(y0);
        while (atomicCAS(&hk[h], -1, y0) != -1) h = (h + 1) & (kHashW - 1);
        hv[h] = j0;
      }
      if (y1 >= 0) {
        uint32_t h = hslot(y1);
        while (atomicCAS(&hk[h], -1, y1) != -1) h = (h + 1) & (kHashW - 1);
        hv[h] = j1;
      }
      __syncwarp();
      // c_j occurs in knn(c_k) at rank r < j, with k < j
      if (c0 >= 0 && k < j0) {
        uint32_t h = hslot(c0);
        while (hk[h] != -1) {
          if (hk[h] == c0) {
            if (hv[h] < j0) ++det0;
            break;
          }
          h = (h + 1) & (kHashW - 1);
        }
      }
      if (c1 >= 0 && k < j1) {
        uint32_t h = hslot(c1);
        while (hk[h] != -1) {
          if (hk[h] == c1) {
            if (hv[h] < j1) ++det1;
            break;
          }
          h = (h + 1) & (kHashW - 1);
        }
      }
      __syncwarp();
    }
    // order by (detour, rank): rank of each own entry among the valid ones
    const uint32_t key0 = c0 >= 0 ? ((uint32_t)det0 << 8) | (uint32_t)j0 : 0xffffffffu;
    const uint32_t key1 = c1 >= 0 ? ((uint32_t)det1 << 8) | (uint32_t)j1 : 0xffffffffu;
    int r0 = 0, r1 = 0, valid = 0;
    for (int m = 0; m < K; ++m) {
      const uint32_t km = __shfl_sync(0xffffffffu, m < 32 ? key0 : key1, m & 31);
      if (km == 0xffffffffu) continue;
      ++valid;
      r0 += km < key0;
      r1 += km < key1;
    }
    if (c0 >= 0 && r0 < R) fwd[i * R + r0] = c0;
    if (c1 >= 0 && r1 < R) fwd[i * R + r1] = c1;
    for (int r = valid + lane; r < R; r += 32) fwd[i * R + r] = -1;
  }
}

// R25: insert (p << 32 | i) into node c's R-smallest set (CAS on the current maximum; the
// final set is the R smallest keys whatever the interleaving -- values only decrease).
// Keys carry the GLOBAL id of i (R25 orders ties by id, and stored positions are list-major).
__global__ void graph_reverse_kernel(const int32_t* __restrict__ fwd, int64_t n, int R,
                                     const int32_t* __restrict__ row_ids,
                                     unsigned long long* __restrict__ rev) {
  const int64_t tot = n * R;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < tot;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / R;
    const int p = (int)(t % R);
    const int32_t c = fwd[t];
    if (c < 0) continue;
    const unsigned long long key =
        ((unsigned long long)p << 32) | (unsigned long long)(uint32_t)row_ids[i];
    unsigned long long* slots = rev + (int64_t)c * R;
    while (true) {
      int m = 0;
      unsigned long long mv = __ldcg(slots);  // L2 reads: other SMs CAS these slots
      for (int s = 1; s < R; ++s) {
        const unsigned long long v = __ldcg(slots + s);
        if (v > mv) {
          mv = v;
          m = s;
        }
      }
      if (key >= mv) break;
      if (atomicCAS(&slots[m], mv, key) == mv) break;
    }
  }
}

// R26: one warp per node.
__global__ void __launch_bounds__(256) graph_merge_kernel(const int32_t* __restrict__ fwd,
                                                          const unsigned long long* __restrict__ rev,
                                                          int64_t n, int R,
                                                          const int32_t* __restrict__ pos_of,
                                                          int64_t row_offset,
                                                          int32_t* __restrict__ nbr) {
  __shared__ int32_t lst[8][GR_MAX_R];
  __shared__ unsigned long long srt[8][GR_MAX_R];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  int32_t* L = lst[warp];
  unsigned long long* S = srt[warp];
  const int64_t nw = (int64_t)gridDim.x * 8;
  for (int64_t c = blockIdx.x * 8 + warp; c < n; c += nw) {
    // sort the reverse keys ascending (empty = ~0 sorts last)
    const unsigned long long k0 = lane < R ? rev[c * R + lane] : ~0ull;
    const unsigned long long k1 = lane + 32 < R ? rev[c * R + lane + 32] : ~0ull;
    int r0 = 0, r1 = 0;
    for (int m = 0; m < R; ++m) {
      const unsigned long long km = __shfl_sync(0xffffffffu, m < 32 ? k0 : k1, m & 31);
      r0 += km < k0 || (km == k0 && m < lane);
      r1 += km < k1 || (km == k1 && m < lane + 32);
    }
    if (lane < R) S[r0] = k0;
    if (lane + 32 < R) S[r1] = k1;
    __syncwarp();
    int cnt = 0;
    auto present = [&](int32_t x) -> bool {
      const bool hit = (lane < cnt && L[lane] == x) || (lane + 32 < cnt && L[lane + 32] == x);
      return __ballot_sync(0xffffffffu, hit) != 0;
    };
    const int32_t* f = fwd + c * R;
    for (int t = 0; t < R / 2; ++t) {
      const int32_t x = f[t];
      if (x < 0) break;
      if (lane == 0) L[cnt] = x;
      ++cnt;
      __syncwarp();
    }
    for (int t = 0; t < R && cnt < R; ++t) {
      const unsigned long long kk = S[t];
      if (kk == ~0ull) break;
      const int32_t x = pos_of[(int64_t)(kk & 0xffffffffull) - row_offset];
      if (!present(x)) {
        if (lane == 0) L[cnt] = x;
        ++cnt;
      }
      __syncwarp();
    }
    for (int t = R / 2; t < R && cnt < R; ++t) {
      const int32_t x = f[t];
      if (x < 0) break;
      if (!present(x)) {
        if (lane == 0) L[cnt] = x;
        ++cnt;
      }
      __syncwarp();
    }
    for (int t = lane; t < R; t += 32) nbr[c * R + t] = t < cnt ? L[t] : -1;
    __syncwarp();
  }
}

// ------------------------------------------------------------------ search

struct SearchSmem {
  uint32_t hash[GR_HASH];
  __align__(16) float q[768];   // float4 slots, swizzled (q_slot_bf16 / q_slot_e4m3)
  unsigned long long key[2][GR_MAX_L];
  int32_t pos[2][GR_MAX_L];
  uint8_t flag[2][GR_MAX_L];
  int32_t npos[GR_MAX_NEW];               // rows to score this iteration
  unsigned long long nkey[GR_MAX_NEW];    // scored rows that can enter the list
  int32_t ipos[GR_MAX_NEW];
  int32_t chosen[8];
  int32_t n_new, n_ins, n_chosen;
  unsigned long long smax;                // best key scored in the step (maturity exit)
};

__device__ __forceinline__ int32_t read_ready(const int32_t* p) {
  if (p == nullptr) return 1;
  int32_t v;
  asm volatile("ld.relaxed.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// one bulk L2 prefetch of [p, p + bytes) (16-byte aligned, bytes a multiple of 16)
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// L2 eviction-priority policies (createpolicy) and loads that carry them
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint4 ldg_policy(const uint4* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ int32_t ldg_policy(const int32_t* p, uint64_t pol) {
  int32_t v;
  asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
}

__device__ __forceinline__ bool visit(uint32_t* hash, int32_t pos) {
  const uint32_t v = (uint32_t)pos + 1u;
  uint32_t h = ((uint32_t)pos * 2654435761u) >> (32 - GR_HASH_LOG);
  while (true) {
    const uint32_t old = atomicCAS(&hash[h], 0u, v);
    if (old == 0u) return true;
    if (old == v) return false;
    h = (h + 1) & (GR_HASH - 1);
  }
}

// The query sits in smem as float4 slots, swizzled so that the 8 lanes of one LDS.128 phase
// (consecutive chunks) hit 8 different 16-byte bank groups: bf16 chunk c (8 values) owns slots
// 2c, 2c+1 with its two halves swapped when bit 2 of c is set; e4m3 chunk c (16 values) owns
// slots 4c..4c+3 rotated by c >> 1.  (Unswizzled, the lanes' 32 / 64-byte strides gave 2- and
// 4-way conflicts: short-scoreboard stalls on the FMAs.)
__device__ __forceinline__ int q_slot_bf16(int c, int g) { return 2 * c + (g ^ ((c >> 2) & 1)); }
__device__ __forceinline__ int q_slot_e4m3(int c, int g) { return 4 * c + ((g + (c >> 1)) & 3); }

__device__ __forceinline__ float bf16x8_dot(const uint4 v, const float4* q4, int c) {
  const float4 qa = q4[q_slot_bf16(c, 0)];
  const float4 qb = q4[q_slot_bf16(c, 1)];
  const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v);
  const float2 f0 = __bfloat1622float2(b[0]), f1 = __bfloat1622float2(b[1]);
  const float2 f2 = __bfloat1622float2(b[2]), f3 = __bfloat1622float2(b[3]);
  float acc = f0.x * qa.x;
  acc = fmaf(f0.y, qa.y, acc);
  acc = fmaf(f1.x, qa.z, acc);
  acc = fmaf(f1.y, qa.w, acc);
  acc = fmaf(f2.x, qb.x, acc);
  acc = fmaf(f2.y, qb.y, acc);
  acc = fmaf(f3.x, qb.z, acc);
  acc = fmaf(f3.y, qb.w, acc);
  return acc;
}

// Score npos[0, cnt) into nkey (warp-cooperative, kRowsPerWarp rows in flight per warp;
// lane l holds 16-byte chunks l, l + 32, l + 64 of a row; the query is in smem).
// Rows whose key is not above `floor` (the list's L-th key once the list is full) cannot enter
// the list and are dropped here; the survivors go to (nkey, ipos)[0, n_ins).
template <int kSThreads, int kRowsPerWarp, bool kMature>
__device__ void score_rows(const GraphSearchArgs& a, SearchSmem& sm, int cnt, int nchunk,
                           unsigned long long floor) {
  constexpr int kSWarps = kSThreads / 32;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint4* X4 = reinterpret_cast<const uint4*>(a.X);
  // rows are read once per query (evict first); row ids are 4 bytes per 1.5 KB row, 84 MB at
  // C3, and fit the L2 when the row stream does not evict them (evict last)
  const uint64_t pol_stream = (a.prefetch & 4) ? policy_evict_first() : policy_evict_normal();
  const uint64_t pol_keep = (a.prefetch & 8) ? policy_evict_last() : policy_evict_normal();
  for (int j0 = warp * kRowsPerWarp; j0 < cnt; j0 += kSWarps * kRowsPerWarp) {
    uint4 v[kRowsPerWarp][3];
    int32_t p[kRowsPerWarp];
    uint32_t gid[kRowsPerWarp];
#pragma unroll
    for (int u = 0; u < kRowsPerWarp; ++u) {
      p[u] = j0 + u < cnt ? sm.npos[j0 + u] : -1;
      // the row's global id, loaded with its data (not after the dot product)
      gid[u] = (lane == 0 && p[u] >= 0)
                   ? (uint32_t)ldg_policy(a.row_ids + p[u], pol_keep) : 0u;
#pragma unroll
      for (int rd = 0; rd < 3; ++rd) {
        const int c = rd * 32 + lane;
        v[u][rd] = (p[u] >= 0 && c < nchunk)
                       ? ldg_policy(X4 + (int64_t)p[u] * nchunk + c, pol_stream)
                       : make_uint4(0, 0, 0, 0);
      }
    }
    // the query chunk is loaded from smem once per rd and reused by every row in flight
    // (rows outer would reload it per row: LDS latency exposed on the FMAs); per row the sum
    // order is unchanged (rd = 0, 1, 2)
    float acc[kRowsPerWarp];
#pragma unroll
    for (int u = 0; u < kRowsPerWarp; ++u) acc[u] = 0.f;
#pragma unroll
    for (int rd = 0; rd < 3; ++rd)
      if (rd * 32 + lane < nchunk) {
#pragma unroll
        for (int u = 0; u < kRowsPerWarp; ++u)
          acc[u] += bf16x8_dot(v[u][rd], reinterpret_cast<const float4*>(sm.q), rd * 32 + lane);
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int u = 0; u < kRowsPerWarp; ++u) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
#pragma unroll
    for (int u = 0; u < kRowsPerWarp; ++u) {
      if (lane == 0 && p[u] >= 0) {
        const unsigned long long key = make_key(acc[u], gid[u]);
        if (kMature) atomicMax(&sm.smax, key);
        if (key > floor) {
          const int t = atomicAdd(&sm.n_ins, 1);
          sm.nkey[t] = key;
          sm.ipos[t] = p[u];
          if (a.prefetch & 2) prefetch_l2(a.nbr + (int64_t)p[u] * a.R, (uint32_t)a.R * 4u);
        }
      }
    }
  }
}

// e4m3 byte at bits 31..24 of t -> fp32 bits of (value * 2^-120): the sign moves as is and
// the 7 exponent/mantissa bits land in the low exponent bits (eeee) and the top mantissa bits
// (mmm), i.e. the e4m3 exponent bias 7 becomes fp32's 127 (subnormals map to fp32 subnormals,
// exactly).  Three integer ops instead of the conversion-unit cvt path.
__device__ __forceinline__ float e4m3_top_to_f32(uint32_t t) {
  return __uint_as_float((t & 0x80000000u) | ((t >> 4) & 0x07F00000u));
}
constexpr int kF8QueryShift = 112;  // query values are pre-scaled by 2^112: products = x*q*2^-8

// 16 e4m3 values (one uint4) . 16 fp32 query values (pre-scaled by 2^kF8QueryShift)
__device__ __forceinline__ float e4m3x16_dot(const uint4 v, const float4* q4, int c) {
  // four independent 4-long FMA chains (one per 32-bit word), summed pairwise
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
  float acc[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float4 q = q4[q_slot_e4m3(c, i)];
    acc[i] = e4m3_top_to_f32(w[i] << 24) * q.x;
    acc[i] = fmaf(e4m3_top_to_f32(w[i] << 16), q.y, acc[i]);
    acc[i] = fmaf(e4m3_top_to_f32(w[i] << 8), q.z, acc[i]);
    acc[i] = fmaf(e4m3_top_to_f32(w[i]), q.w, acc[i]);
  }
  return (acc[0] + acc[1]) + (acc[2] + acc[3]);
}

constexpr int kF8RowsPerWarp = 4;  // 4 x 2 uint4 in flight per lane: 0 spills at 64 registers

// score_rows on the e4m3 copy (R34): a row is d8_pad bytes = nch 16-byte chunks, lane l holds
// chunks l and l + 32; twice the rows in flight of the bf16 path for the same registers.
template <int kSThreads, int kRowsPerWarp>
__device__ void score_rows_f8(const GraphSearchArgs& a, SearchSmem& sm, int cnt,
                              unsigned long long floor) {
  constexpr int kSWarps = kSThreads / 32;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int nch = a.d8_pad / 16;
  const uint4* X4 = reinterpret_cast<const uint4*>(a.X8);
  for (int j0 = warp * kRowsPerWarp; j0 < cnt; j0 += kSWarps * kRowsPerWarp) {
    uint4 v[kRowsPerWarp][2];
    int32_t p[kRowsPerWarp];
    uint32_t gid[kRowsPerWarp];
#pragma unroll
    for (int u = 0; u < kRowsPerWarp; ++u) {
      p[u] = j0 + u < cnt ? sm.npos[j0 + u] : -1;
      gid[u] = (lane == 0 && p[u] >= 0) ? (uint32_t)__ldg(a.row_ids + p[u]) : 0u;
#pragma unroll
      for (int rd = 0; rd < 2; ++rd) {
        const int c = rd * 32 + lane;
        v[u][rd] = (p[u] >= 0 && c < nch) ? __ldg(X4 + (int64_t)p[u] * nch + c)
                                          : make_uint4(0, 0, 0, 0);
      }
    }
    // each float4 of the query is loaded once and used by every row in flight (one FMA chain
    // per row; the rows give the ILP)
    float acc[kRowsPerWarp];
#pragma unroll
    for (int u = 0; u < kRowsPerWarp; ++u) acc[u] = 0.f;
    const float4* q4 = reinterpret_cast<const float4*>(sm.q);
#pragma unroll
    for (int rd = 0; rd < 2; ++rd)
      if (rd * 32 + lane < nch) {
        const int c = rd * 32 + lane;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float4 q = q4[q_slot_e4m3(c, i)];
#pragma unroll
          for (int u = 0; u < kRowsPerWarp; ++u) {
            const uint32_t w = i == 0 ? v[u][rd].x : i == 1 ? v[u][rd].y : i == 2 ? v[u][rd].z
                                                                              : v[u][rd].w;
            acc[u] = fmaf(e4m3_top_to_f32(w << 24), q.x, acc[u]);
            acc[u] = fmaf(e4m3_top_to_f32(w << 16), q.y, acc[u]);
            acc[u] = fmaf(e4m3_top_to_f32(w << 8), q.z, acc[u]);
            acc[u] = fmaf(e4m3_top_to_f32(w), q.w, acc[u]);
          }
        }
      }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int u = 0; u < kRowsPerWarp; ++u) acc[u] += __shfl_xor_sync(0xffffffffu, acc[u], o);
#pragma unroll
    for (int u = 0; u < kRowsPerWarp; ++u) {
      if (lane == 0 && p[u] >= 0) {
        const unsigned long long key = make_key(acc[u], gid[u]);
        if (key > floor) {
          const int t = atomicAdd(&sm.n_ins, 1);
          sm.nkey[t] = key;
          sm.ipos[t] = p[u];
          if (a.prefetch & 2) prefetch_l2(a.nbr + (int64_t)p[u] * a.R, (uint32_t)a.R * 4u);
        }
      }
    }
  }
}

// number of entries of the descending array a[0, n) that are > x
__device__ __forceinline__ int count_greater(const unsigned long long* a, int n,
                                             unsigned long long x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] > x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

template <int kSThreads, int kRowsPerWarp, bool kMature, bool kF8>
__global__ void __launch_bounds__(kSThreads, 1024 / kSThreads)
    graph_search_kernel(const GraphSearchArgs a, const GraphMatureArgs m) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  SearchSmem& sm = *reinterpret_cast<SearchSmem*>(smem_raw);
  const int q = blockIdx.x;
  const int lane = threadIdx.x % 32;
  const int nchunk = a.d_pad / 8;
#ifdef SA_TUNING_BUILD
  const bool dbg = a.dbg != nullptr && threadIdx.x == 0;
#else
  constexpr bool dbg = false;   // the product library never times phases
#endif
  unsigned long long dcy[4] = {0, 0, 0, 0};
  long long dt = 0;
  auto dmark = [&](int ph) {
    if (dbg) {
      const long long c = clock64();
      dcy[ph] += (unsigned long long)(c - dt);
      dt = c;
    }
  };
  if (dbg) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    a.dbg[(int64_t)q * 8] = g;
  }
  for (int i = threadIdx.x; i < GR_HASH; i += kSThreads) sm.hash[i] = 0u;
  if constexpr (kF8) {
    for (int i = threadIdx.x; i < a.d8_pad; i += kSThreads)
      sm.q[q_slot_e4m3(i >> 4, (i >> 2) & 3) * 4 + (i & 3)] =
          ldexpf(e4m3_top_to_f32((uint32_t)a.Q8[(int64_t)q * a.d8_pad + i] << 24),
                 120 + kF8QueryShift);
  } else {
    for (int i = threadIdx.x; i < a.d_pad; i += kSThreads)
      sm.q[q_slot_bf16(i >> 3, (i >> 2) & 1) * 4 + (i & 3)] =
          __bfloat162float(a.Q[(int64_t)q * a.d_pad + i]);
  }
  if (threadIdx.x == 0) {
    sm.n_new = 0;
    sm.n_ins = 0;
  }
  __syncthreads();
  // entries: the first stored row of each probed list (lists hold ascending global ids)
  for (int e = threadIdx.x; e < a.E; e += kSThreads) {
    const uint64_t pk = a.entry_keys[(int64_t)q * a.E + e];
    if (pk != 0ull) {
      const uint32_t l = key_id(pk);
      const int64_t lo = a.list_off[l], hi = a.list_off[l + 1];
      if (hi > lo && visit(sm.hash, (int32_t)lo)) sm.npos[atomicAdd(&sm.n_new, 1)] = (int32_t)lo;
    }
  }
  __syncthreads();
  int cur = 0;
  int n_new = sm.n_new;
  int cnt = 0;
  if constexpr (kF8) score_rows_f8<kSThreads, kF8RowsPerWarp>(a, sm, n_new, 0ull);
  else score_rows<kSThreads, kRowsPerWarp, false>(a, sm, n_new, nchunk, 0ull);
  __syncthreads();
  int expanded = 0;
  int scored = n_new;
  int visited = n_new;   // entries in the visited table
  double ema = 0.0;  // thread 0 (maturity exit)
  int steps = 0;     // iterations run (maturity exit)
  int iters = 0;
  if (dbg) dt = clock64();
  for (int it = 0;; ++it) {
    if (kMature) steps = it;
    iters = it;
    // ---- merge the surviving new rows into the sorted list (top-L); keys are distinct, so an
    // entry's new position = its rank in the old list + the number of new keys above it (v.v.)
    const int n_ins = sm.n_ins;
    if (n_ins > 0) {
      const int nxt = cur ^ 1;
      for (int i = threadIdx.x; i < cnt; i += kSThreads) {
        const unsigned long long x = sm.key[cur][i];
        int np = i;
        for (int j = 0; j < n_ins; ++j) np += sm.nkey[j] > x;
        if (np < a.L) {
          sm.key[nxt][np] = x;
          sm.pos[nxt][np] = sm.pos[cur][i];
          sm.flag[nxt][np] = sm.flag[cur][i];
        }
      }
      for (int j = threadIdx.x; j < n_ins; j += kSThreads) {
        const unsigned long long x = sm.nkey[j];
        int np = count_greater(sm.key[cur], cnt, x);
        for (int t = 0; t < n_ins; ++t) np += sm.nkey[t] > x;
        if (np < a.L) {
          sm.key[nxt][np] = x;
          sm.pos[nxt][np] = sm.ipos[j];
          sm.flag[nxt][np] = 0;
        }
      }
      cnt = min(a.L, cnt + n_ins);
      cur = nxt;
      __syncthreads();
    }
    dmark(0);
    // ---- maturity signal of step it (R28-R29): s_t = best key scored in the step, RQ_t over
    // the list's first / last entries after the merge, EMA in fp64 with the oracle's roundings
    bool stop = false;
    if constexpr (kMature) if (it > 0 && threadIdx.x == 0) {
      double r = 1.0;
      if (n_new > 0) {
        const double sb = key_score(sm.key[cur][0]), sw = key_score(sm.key[cur][cnt - 1]);
        if (sb != sw) r = __ddiv_rn(__dsub_rn(sb, (double)key_score(sm.smax)), __dsub_rn(sb, sw));
      }
      ema = it == 1 ? r
                    : __dadd_rn(__dmul_rn(m.alpha, r), __dmul_rn(__dsub_rn(1.0, m.alpha), ema));
      if (m.out_rq && it <= m.trace_cols) {
        m.out_rq[(int64_t)q * m.trace_cols + it - 1] = r;
        m.out_ema[(int64_t)q * m.trace_cols + it - 1] = ema;
      }
      stop = it % m.g == 0 && ema >= m.tau && read_ready(m.ready) != 0;
    }
    if (it >= a.T) break;
    // ---- pick the first w unexpanded entries (warp 0)
    if (threadIdx.x < 32) {
      int taken = 0;
      if constexpr (kMature) stop = __shfl_sync(0xffffffffu, stop, 0);
      for (int base = 0; base < cnt && taken < a.w && !stop; base += 32) {
        const int i = base + lane;
        const bool un = i < cnt && sm.flag[cur][i] == 0;
        unsigned m = __ballot_sync(0xffffffffu, un);
        __syncwarp();   // every lane's flag read precedes lane 0's writes below
        while (m && taken < a.w) {
          const int b = __ffs(m) - 1;
          m &= m - 1;
          if (lane == 0) {
            sm.chosen[taken] = sm.pos[cur][base + b];
            sm.flag[cur][base + b] = 1;
          }
          ++taken;
        }
      }
      if (lane == 0) {
        sm.n_chosen = taken;
        sm.n_new = 0;
        // every thread read n_ins at the top of this iteration; when it was nonzero the merge's
        // barrier orders those reads before this write, when zero there is nothing to reset
        if (n_ins != 0) sm.n_ins = 0;
        if constexpr (kMature) sm.smax = 0ull;
      }
    }
    __syncthreads();
    dmark(1);
    const int nc = sm.n_chosen;
    if (nc == 0) break;
    expanded += nc;
    // ---- forgettable visited set: when the table would pass 3/4 load, clear it and keep only
    // the list's rows.  The list evolves exactly as with the full visited set: a forgotten row
    // is not in the list, so it was scored below the list's L-th key (or dropped below it), the
    // L-th key only rises, and a re-scored copy is dropped by the floor test again -- only work
    // is repeated, never a list entry.
    if (visited + nc * a.R > GR_VISIT_CAP) {
      for (int i = threadIdx.x; i < GR_HASH; i += kSThreads) sm.hash[i] = 0u;
      __syncthreads();
      for (int i = threadIdx.x; i < cnt; i += kSThreads) visit(sm.hash, sm.pos[cur][i]);
      __syncthreads();
      visited = cnt;
    }
    // ---- neighbours not yet visited
    for (int t = threadIdx.x; t < nc * a.R; t += kSThreads) {
      const int32_t c = a.nbr[(int64_t)sm.chosen[t / a.R] * a.R + (t % a.R)];
      if (c >= 0 && visit(sm.hash, c)) {
        sm.npos[atomicAdd(&sm.n_new, 1)] = c;
        if (a.prefetch & 1) {
          if constexpr (kF8) prefetch_l2(a.X8 + (int64_t)c * a.d8_pad, (uint32_t)a.d8_pad);
          else prefetch_l2(a.X + (int64_t)c * a.d_pad, (uint32_t)a.d_pad * 2u);
        }
      }
    }
    __syncthreads();
    dmark(2);
    n_new = sm.n_new;
    scored += n_new;
    visited += n_new;
    if constexpr (kF8)
      score_rows_f8<kSThreads, kF8RowsPerWarp>(a, sm, n_new,
                                                 cnt == a.L ? sm.key[cur][a.L - 1] : 0ull);
    else
      score_rows<kSThreads, kRowsPerWarp, kMature>(a, sm, n_new, nchunk,
                                                   cnt == a.L ? sm.key[cur][a.L - 1] : 0ull);
    __syncthreads();
    dmark(3);
  }
  if (dbg) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    a.dbg[(int64_t)q * 8 + 1] = g;
    for (int i = 0; i < 4; ++i) a.dbg[(int64_t)q * 8 + 2 + i] = dcy[i];
    a.dbg[(int64_t)q * 8 + 6] = (unsigned long long)iters;
  }
  if constexpr (kF8) {
    // the whole list, re-keyed with stored positions, for the bf16 re-rank
    for (int i = threadIdx.x; i < a.L; i += kSThreads)
      a.out_keys[(int64_t)q * a.L + i] =
          i < cnt ? make_key(key_score(sm.key[cur][i]), (uint32_t)sm.pos[cur][i]) : 0ull;
  } else {
    for (int i = threadIdx.x; i < a.k; i += kSThreads) {
      const unsigned long long key = i < cnt ? sm.key[cur][i] : 0ull;
      a.out_ids[(int64_t)q * a.k + i] = key == 0ull ? -1 : (int64_t)key_id(key);
      a.out_scores[(int64_t)q * a.k + i] = key == 0ull ? -INFINITY : key_score(key);
    }
  }
  if (a.out_expanded && threadIdx.x == 0) {
    a.out_expanded[q] = expanded;
    a.out_expanded[a.nq + q] = scored;
  }
  if (kMature) {
    if (m.out_steps && threadIdx.x == 0) m.out_steps[q] = steps;
    if (m.out_rq)
      for (int t = steps + threadIdx.x; t < m.trace_cols; t += kSThreads) {
        m.out_rq[(int64_t)q * m.trace_cols + t] = __longlong_as_double(0x7ff8000000000000ll);
        m.out_ema[(int64_t)q * m.trace_cols + t] = __longlong_as_double(0x7ff8000000000000ll);
      }
  }
}

}  // namespace

cudaError_t launch_inverse_ids(const int32_t* row_ids, int64_t n, int64_t row_offset,
                               int32_t* pos_of, cudaStream_t s) {
  inverse_ids_kernel<<<grid_for(n, 256), 256, 0, s>>>(row_ids, n, row_offset, pos_of);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_knn_to_pos(const int64_t* ids, int64_t nb, int kk, int64_t p0,
                              const int32_t* pos_of, int64_t row_offset, int K, int32_t* knn,
                              cudaStream_t s) {
  knn_to_pos_kernel<<<grid_for(nb, 128), 128, 0, s>>>(ids, nb, kk, p0, pos_of, row_offset, K,
                                                      knn);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_graph_prune(const int32_t* knn, int64_t n, int K, int R, int32_t* fwd,
                               cudaStream_t s) {
  graph_prune_kernel<<<grid_for(n, 8), 256, 0, s>>>(knn, n, K, R, fwd);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_graph_reverse(const int32_t* fwd, int64_t n, int R, const int32_t* row_ids,
                                 uint64_t* rev, cudaStream_t s) {
  graph_reverse_kernel<<<grid_for(n * R, 256), 256, 0, s>>>(
      fwd, n, R, row_ids, reinterpret_cast<unsigned long long*>(rev));
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_graph_merge(const int32_t* fwd, const uint64_t* rev, int64_t n, int R,
                               const int32_t* pos_of, int64_t row_offset, int32_t* nbr,
                               cudaStream_t s) {
  graph_merge_kernel<<<grid_for(n, 8), 256, 0, s>>>(
      fwd, reinterpret_cast<const unsigned long long*>(rev), n, R, pos_of, row_offset, nbr);
  note_launch();
  return cudaGetLastError();
}

size_t graph_search_smem(int) { return sizeof(SearchSmem); }

template <int TH, int RW, bool M, bool F8>
cudaError_t launch_shape(const GraphSearchArgs& a, const GraphMatureArgs& m, int64_t nq,
                         cudaStream_t s) {
  const size_t smem = sizeof(SearchSmem);
  cudaError_t e =
      ensure_max_smem(reinterpret_cast<const void*>(graph_search_kernel<TH, RW, M, F8>), smem);
  if (e != cudaSuccess) return e;
  graph_search_kernel<TH, RW, M, F8><<<(unsigned)nq, TH, smem, s>>>(a, m);
  note_launch();
  return cudaGetLastError();
}

template <bool M, bool F8>
cudaError_t launch_shapes(const GraphSearchArgs& a, const GraphMatureArgs& m, int64_t nq,
                          cudaStream_t s) {
  if (nq <= 148) return launch_shape<1024, 3, M, F8>(a, m, nq, s);
  if (nq <= 296) return launch_shape<512, 3, M, F8>(a, m, nq, s);
  return launch_shape<256, 3, M, F8>(a, m, nq, s);
}

cudaError_t launch_graph_search(const GraphSearchArgs& a, const GraphMatureArgs* m, int64_t nq,
                                cudaStream_t s, bool fp8) {
  // Throughput shape: 256 threads x 3 rows in flight per warp at 4 CTAs/SM (64 registers,
  // ~45 KB smem), every query of a 512 batch resident at once.  Measured alternatives (C3,
  // L=160): 128 threads x 6 rows 0.84x, 128 x 8 (spills) 0.6x, 256 x 4 (spills) slower.
  // Latency shapes for small batches (agent steps): 1024 threads when at most one query per
  // SM (an iteration's ~100-200 new rows all in flight at once), 512 threads for two.
  // (C3, L=104: batch 1 0.32 ms, 64 0.40 ms, 148 0.43 ms vs 0.65 ms with the 256 shape.)
  if (fp8) return m ? cudaErrorInvalidValue : launch_shapes<false, true>(a, GraphMatureArgs{}, nq, s);
  return m ? launch_shapes<true, false>(a, *m, nq, s)
           : launch_shapes<false, false>(a, GraphMatureArgs{}, nq, s);
}

}  // namespace sa
