// ivf_small.cu -- IVF search of an agent-step batch in ONE cooperative launch (SURVEY.md §8(d)
// C5; DESIGN.md §4.2 "small batches").
//
// SearchAgent-X retrieves once per <search> tag (Alg. 1), a handful of
// queries at a time, and the engine stalls until the documents arrive: an agent step
// is latency-bound.  The batch path (probe kernel + select + inversion + list scan + merge)
// costs ~10 launches of fixed overhead for ~20 us of HBM work at batch 1.  Here the whole
// search -- R11's probe and the exact scan of the probed lists with the R5 ordering -- is
// one kernel of one CTA per SM.  Every byte it streams (centroids, then list rows and their
// ids) moves HBM -> smem by 1-D TMA bulk copies through a 3-stage ring of 32-row pieces
// (48 KB at d = 768) fed by a dedicated copy warp (full / empty mbarriers), so each SM keeps
// ~100-150 KB in flight while 16 warps score rows on the CUDA cores.
//   A  centroid keys: CTA b scores its 1/G slice of the bf16 centroids against every query
//      and keeps the keys (score, list id) in smem, plus its m best per query in global;
//   -- grid barrier
//   B  probe (exact top-nprobe keys, R11: ties -> lowest list id): every CTA reads the
//      published keys, takes T' = the nprobe-th largest of the CTAs' first m keys (<= the
//      nprobe-th largest key overall: it is the nprobe-th of a subset) and, when every CTA's
//      last published key is below T', ranks the published keys >= T' (all keys >= T' were
//      published); otherwise (slices correlated with the query) the CTAs append every key
//      >= T' and, after a second grid barrier, rank them (a 64-bit radix select when many);
//   C  scan: the probed lists are cut into 32-row pieces, CTA b takes an equal share (in
//      (query, list) order); a warp scores rows w and w + 16 of each piece against the query
//      held in registers and keeps a sorted top-k in registers (lane j = j-th best); the 16
//      warp lists are merged into one list per (CTA, query);
//   D  the last CTA to finish (a counter, no grid barrier) keeps the k best of the G per-CTA
//      lists of each query (R5 order) and writes the result (packed keys for a cross-rank
//      merge, or ids / scores padded -1 / -inf).
// Scores are fp32 sums of exact bf16 products on the CUDA cores (the batch path uses the
// tensor cores; the two agree up to fp32 rounding order, i.e. at near-ties, R36).
// List rows are read with an L2 evict-first policy (streamed once per step); the centroids
// with the default policy.
#include <cooperative_groups.h>
#include <cuda_bf16.h>

#include "ivf_small.cuh"
#include "keys.cuh"
#include "launch.cuh"
#include "ptx.cuh"

namespace sa {

namespace cg = cooperative_groups;

namespace {

constexpr int kCWarps = 16;                           // scoring warps
constexpr int kCThreads = 32 * kCWarps;
constexpr int kThreads = IVSM_THREADS;                // + the copy warp
constexpr int kWarps = kThreads / 32;
static_assert(kThreads == kCThreads + 32, "one copy warp");
constexpr int kPiece = 32;                            // rows per bulk copy
constexpr int kStages = 3;
constexpr int kMaxDPad = 768;
constexpr int kRowsBytes = kPiece * kMaxDPad * 2;     // 48 KB
constexpr int kIdBytes = 256;                         // a piece's ids (16-byte aligned range)
constexpr int kStageBytes = kRowsBytes + kIdBytes;
constexpr int kRingBytes = kStages * kStageBytes;
constexpr int kRingKeys = kRingBytes / 8;
constexpr int kMaxNp = IVSM_MAX_NQ * IVSM_MAX_NPROBE;
constexpr int kRankMax = 1024;   // fallback candidates ranked by counting; more -> radix select
constexpr int kFastCap = 512;    // published candidates per query on the fast path
constexpr int kSvCap = kCWarps * IVSM_MAX_K;          // survivors of a warp-list merge
static_assert((IVSM_MAX_NLIST + IVSM_MAX_NPROBE) <= kRingKeys, "probe candidates fit the ring");

struct PieceInfo {
  int64_t row0;
  int32_t rows, qi, o;   // stored rows [row0, +rows), query, output list
  int32_t pad;
};

struct __align__(16) SmallSmem {
  float4 qp[IVSM_MAX_NQ][3][2][32];           // the queries, bf16-rounded, widened to fp32,
                                              // lane-planar: elements [8 ch + 4 h, +4) of
                                              // chunk ch = lane + 32 u (conflict-free LDS.128)
  uint64_t full[kStages], empty[kStages];
  PieceInfo info[kStages];
  uint64_t lk[IVSM_MAX_NQ][IVSM_MAX_LOCAL];   // this CTA's centroid keys per query
  uint64_t wl[kCWarps][IVSM_MAX_K];           // warp lists at a flush
  uint64_t sv[kSvCap];                        // survivors of a warp-list merge
  uint64_t thr[IVSM_MAX_NQ];                  // probe thresholds T'
  int32_t probe[kMaxNp];                      // probe entries (query-major, by descending
                                              // key): the list's first stored row
  int32_t lend[kMaxNp];                       // each probe entry's list end
  int32_t seb[IVSM_MAX_STAGE], see[IVSM_MAX_STAGE];   // a maturity stage's entries
  int32_t pre[kMaxNp + 1];                    // exclusive prefix of pieces per probe entry
  uint32_t hist[256];
  uint64_t red[kWarps];
  int32_t ccnt[IVSM_MAX_NQ], unpub[IVSM_MAX_NQ];
  int32_t s_int[4];
};

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// 1-D bulk copy global -> this CTA's smem, completing `bytes` on the mbarrier.
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes,
                                         uint32_t bar, uint64_t policy, bool hint) {
  if (hint)
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "l"(policy)
        : "memory");
  else
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

__device__ __forceinline__ int32_t read_ready(const int32_t* p) {
  if (p == nullptr) return 1;
  int32_t v;
  asm volatile("ld.relaxed.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ int64_t globaltimer() {
  int64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Barrier of nth threads: the whole CTA, or the scoring warps alone (named barrier 1).
__device__ __forceinline__ void bsync(int nth) {
  if (nth == kThreads) __syncthreads();
  else asm volatile("bar.sync 1, %0;" ::"r"(nth) : "memory");
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t x = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += x;
  }
  return v;
}

__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t x = __shfl_xor_sync(0xffffffffu, v, o);
    v = x > v ? x : v;
  }
  return v;
}

// Max of one u64 per thread over the first nth threads (result to each of them).
__device__ __forceinline__ uint64_t block_max(uint64_t v, SmallSmem& sm, int nth) {
  v = warp_max_u64(v);
  bsync(nth);
  if ((threadIdx.x & 31) == 0) sm.red[threadIdx.x >> 5] = v;
  bsync(nth);
  uint64_t m = 0ull;
  for (int w = 0; w < nth / 32; ++w) m = sm.red[w] > m ? sm.red[w] : m;
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

// Descending bitonic sort of sv[0, P) in shared memory by nth threads (P a power of two).
__device__ void block_sort_desc(uint64_t* sv, int P, int nth) {
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      bsync(nth);
      for (int i = threadIdx.x; i < P; i += nth) {
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
  bsync(nth);
}

// The k best keys of L descending lists of k keys in smem (list j at lists[j * lstride],
// empty slots 0) -> out[0, k) descending (0-padded), by the first nth threads.  Every key of
// the top k is >= T = max_j lists[j][k-1] (k keys of one list are >= T), so only those
// survive to a sort.
__device__ void topk_of_lists(const uint64_t* lists, int L, int lstride, int k, uint64_t* sv,
                              int sv_cap, uint64_t* out, SmallSmem& sm, int nth) {
  uint64_t t = 0ull;
  for (int j = threadIdx.x; j < L; j += nth) {
    const uint64_t x = lists[j * lstride + k - 1];
    t = x > t ? x : t;
  }
  const uint64_t T = block_max(t, sm, nth);
  if (threadIdx.x == 0) sm.s_int[0] = 0;
  bsync(nth);
  for (int e = threadIdx.x; e < L * k; e += nth) {
    const uint64_t x = lists[(e / k) * lstride + e % k];
    if (x != 0ull && x >= T) {
      const int pos = atomicAdd(&sm.s_int[0], 1);
      if (pos < sv_cap) sv[pos] = x;
    }
  }
  bsync(nth);
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
    for (int i = m + threadIdx.x; i < P; i += nth) sv[i] = 0ull;
    block_sort_desc(sv, P, nth);
    for (int i = threadIdx.x; i < k; i += nth) out[i] = sv[i];
  }
  bsync(nth);
}

// The k best keys of L descending lists of k keys in smem (list j at lists[j * k], empty slots
// 0) -> out[0, k) descending (0-padded), by ONE warp: k rounds of "largest key below the
// previous one" (keys are distinct), each round skipping lists whose best key is already
// taken.  No CTA barrier, so the warps of a CTA merge different outputs concurrently.
__device__ void warp_topk_of_lists(const uint64_t* lists, int L, int k, uint64_t* out) {
  const int lane = threadIdx.x & 31;
  uint64_t prev = ~0ull;
  for (int r = 0; r < k; ++r) {
    uint64_t m = 0ull;
    for (int e = lane; e < L * k; e += 32) {
      const uint64_t x = lists[e];
      if (x < prev && x > m) m = x;
    }
    m = warp_max_u64(m);
    if (lane == 0) out[r] = m;
    prev = m;
    if (m == 0ull) {
      for (int r2 = r + 1 + lane; r2 < k; r2 += 32) out[r2] = 0ull;
      break;
    }
  }
  __syncwarp();
}

// The nprobe-th largest of the n distinct keys kb[0, n) (n >= nprobe), MSB-first radix
// select over the 64 key bits, by the whole CTA.
__device__ uint64_t radix_kth(const uint64_t* kb, int n, int nprobe, SmallSmem& sm) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t prefix = 0ull, mask = 0ull;
  int remaining = nprobe;
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += kThreads) sm.hist[i] = 0u;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += kThreads) {
      const uint64_t v = kb[i];
      if ((v & mask) == prefix) atomicAdd(&sm.hist[(v >> shift) & 255u], 1u);
    }
    __syncthreads();
    if (warp == 0) {
      // buckets from the top, 8 per lane: the first bucket where the count reaches
      // `remaining` holds the k-th key
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
    prefix |= (uint64_t)(uint32_t)sm.s_int[1] << shift;
    mask |= 255ull << shift;
    __syncthreads();
  }
  return prefix;
}

// ring keys the fast probe path needs: published [nq][G][mp], first-m [nq][G*m], candidates
__host__ __device__ inline int64_t fast_keys(int nq, int m, int G) {
  return (int64_t)nq * G * (m + IVSM_EXTRA) + (int64_t)nq * G * m + (int64_t)nq * kFastCap;
}

}  // namespace

bool ivf_small_fits(int nq, int nprobe, int nlist, int grid) {
  const int m = ivf_small_m(nprobe, grid);
  return nlist <= IVSM_MAX_NLIST && nlist <= (int64_t)IVSM_MAX_LOCAL * grid &&
         fast_keys(nq, m, grid) <= kRingKeys;
}

template <int NQ, bool MATURE>
__global__ void __launch_bounds__(kThreads, 1)
ivf_small_kernel(const IvfSmallArgs a, const SmallMatureArgs mo) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* ring = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
  uint64_t* ring64 = reinterpret_cast<uint64_t*>(ring);
  SmallSmem& sm = *reinterpret_cast<SmallSmem*>(ring + kRingBytes);
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x, b = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool copier = warp == kCWarps;
  const int nq = a.nq, k = a.k, nprobe = a.nprobe, d_pad = a.d_pad;
  const int nch = d_pad / 8;                    // 16-byte chunks per row
  const uint32_t row_bytes = (uint32_t)d_pad * 2;
  const int c0 = (int)((int64_t)b * a.nlist / G), c1 = (int)((int64_t)(b + 1) * a.nlist / G);
  const int nloc = c1 - c0;
  const int nA = (nloc + kPiece - 1) / kPiece;
  const uint32_t full0 = ptx::smem_u32(&sm.full[0]), empty0 = ptx::smem_u32(&sm.empty[0]);
  const uint32_t ring0 = ptx::smem_u32(ring);
  if (a.debug_ns && tid == 0) a.debug_ns[b * 8 + 0] = globaltimer();

  // the copy warp's lane 0 owns the ring: it initialises the barriers and starts the first
  // centroid copies at once (the scoring warps wait on them only after the CTA barrier below)
  if (copier && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(full0 + s * 8, 1);
      ptx::mbar_init(empty0 + s * 8, kCWarps);
    }
    ptx::fence_mbar_init();
    for (int i = 0; i < min(kStages, nA); ++i) {
      const uint32_t bytes = (uint32_t)min(kPiece, nloc - i * kPiece) * row_bytes;
      ptx::mbar_arrive_expect_tx(full0 + i * 8, bytes);
      bulk_g2s(ring0 + i * kStageBytes, a.C + (int64_t)(c0 + i * kPiece) * d_pad, bytes,
               full0 + i * 8, 0ull, false);
    }
  }
  // Pinned host queries: CTA 0 reads them over the host link (once) and stages them in device
  // memory; the other CTAs wait for its release flag and read them from L2.
  const bool host_q = a.Q_host != nullptr;
  if (host_q) {
    const int32_t expect = *a.seq + 1;   // *seq changes only at the end of the launch
    if (b == 0) {
      const int n = nq * a.d;
      if (a.q_f32) {
        const uint32_t* src = static_cast<const uint32_t*>(a.Q_host);
        uint32_t* dst = static_cast<uint32_t*>(const_cast<void*>(a.Q));
        for (int i = tid; i < n; i += kThreads) dst[i] = src[i];
      } else {
        const unsigned short* src = static_cast<const unsigned short*>(a.Q_host);
        unsigned short* dst = static_cast<unsigned short*>(const_cast<void*>(a.Q));
        for (int i = tid; i < n; i += kThreads) dst[i] = src[i];
      }
      __threadfence();
      __syncthreads();
      if (tid == 0) ptx::st_release_gpu(a.q_ready, expect);
    } else {
      if (tid == 0)
        while (ptx::ld_acquire_gpu(a.q_ready) != expect) __nanosleep(32);
      __syncthreads();
    }
  }
  // queries -> smem, RNE-rounded to bf16 (R3) then widened exactly; padding is zero
  for (int i = tid; i < NQ * kMaxDPad; i += kThreads) {   // every slot: zero past d
    const int qi = i / kMaxDPad, c = i % kMaxDPad;
    float v = 0.f;
    if (qi < nq && c < a.d) {
      const int64_t o = (int64_t)qi * a.d + c;
      if (a.q_f32) {
        const float* Qf = static_cast<const float*>(a.Q);
        v = __bfloat162float(__float2bfloat16_rn(host_q ? __ldcg(Qf + o) : Qf[o]));
      } else {
        const unsigned short* Qh = static_cast<const unsigned short*>(a.Q);
        v = __uint_as_float((uint32_t)(host_q ? __ldcg(Qh + o) : Qh[o]) << 16);
      }
    }
    const int ch = c >> 3, u = ch >> 5, ln = ch & 31, h = (c >> 2) & 1;
    reinterpret_cast<float*>(&sm.qp[qi][u][h][ln])[c & 3] = v;
  }
  if (b == 0) {   // ordered before every use by the grid barriers below
    for (int i = tid; i <= nq + (MATURE ? 2 : 0); i += kThreads) a.counters[i] = 0;
    if constexpr (MATURE) {
      for (int i = tid; i < nq * k; i += kThreads) mo.R[i] = 0ull;
      for (int qi = tid; qi < nq; qi += kThreads) {
        mo.ema[qi] = 0.0;
        mo.active[qi] = 1;
        mo.t_done[qi] = 0;
      }
      if (mo.trace_rq)
        for (int i = tid; i < nq * nprobe; i += kThreads) {
          mo.trace_rq[i] = __longlong_as_double(0x7ff8000000000000ll);
          mo.trace_ema[i] = __longlong_as_double(0x7ff8000000000000ll);
        }
    }
  }
  __syncthreads();

  // Ring position p (phase A: p = i; phase C: p = nA + j) uses stage p % kStages; its full
  // barrier completes phase p / kStages, its empty barrier (16 warp arrivals) likewise.
  // ---- A: this CTA's centroid keys
  if (copier) {
    if (lane == 0)
      for (int i = kStages; i < nA; ++i) {
        const int s = i % kStages;
        ptx::mbar_wait(empty0 + s * 8, (uint32_t)((i / kStages - 1) & 1));
        const uint32_t bytes = (uint32_t)min(kPiece, nloc - i * kPiece) * row_bytes;
        ptx::mbar_arrive_expect_tx(full0 + s * 8, bytes);
        bulk_g2s(ring0 + s * kStageBytes, a.C + (int64_t)(c0 + i * kPiece) * d_pad, bytes,
                 full0 + s * 8, 0ull, false);
      }
    __syncwarp();
  } else {
    for (int i = 0; i < nA; ++i) {
      const int s = i % kStages;
      ptx::mbar_wait(full0 + s * 8, (uint32_t)((i / kStages) & 1));
      const uint8_t* st = ring + s * kStageBytes;
      const int r0 = i * kPiece, rows = min(kPiece, nloc - r0);
      uint4 v[2][3];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint4* row = reinterpret_cast<const uint4*>(st + (warp + h * kCWarps) * row_bytes);
#pragma unroll
        for (int u = 0; u < 3; ++u) {
          const int ch = lane + 32 * u;
          v[h][u] = (warp + h * kCWarps < rows && ch < nch) ? row[ch] : make_uint4(0, 0, 0, 0);
        }
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(empty0 + s * 8);   // this warp is done with the stage
      // both rows against each query chunk: one pair of conflict-free LDS.128 per (chunk, query)
      float acc[2][NQ];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int qi = 0; qi < NQ; ++qi) acc[h][qi] = 0.f;
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        if (lane + 32 * u >= nch) break;
#pragma unroll
        for (int qi = 0; qi < NQ; ++qi) {
          const float4 qa = sm.qp[qi][u][0][lane];
          const float4 qb = sm.qp[qi][u][1][lane];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint4 w = v[h][u];
            float x = acc[h][qi];
            x = fmaf(__uint_as_float(w.x << 16), qa.x, x);
            x = fmaf(__uint_as_float(w.x & 0xFFFF0000u), qa.y, x);
            x = fmaf(__uint_as_float(w.y << 16), qa.z, x);
            x = fmaf(__uint_as_float(w.y & 0xFFFF0000u), qa.w, x);
            x = fmaf(__uint_as_float(w.z << 16), qb.x, x);
            x = fmaf(__uint_as_float(w.z & 0xFFFF0000u), qb.y, x);
            x = fmaf(__uint_as_float(w.w << 16), qb.z, x);
            x = fmaf(__uint_as_float(w.w & 0xFFFF0000u), qb.w, x);
            acc[h][qi] = x;
          }
        }
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int r = warp + h * kCWarps;
        if (r >= rows) break;
#pragma unroll
        for (int qi = 0; qi < NQ; ++qi) {
          float s2 = acc[h][qi];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) s2 += __shfl_xor_sync(0xffffffffu, s2, o);
          if (lane == 0 && qi < nq) sm.lk[qi][r0 + r] = make_key(s2, (uint32_t)(c0 + r0 + r));
        }
      }
      if (a.debug_ns && i == 0 && tid == 0) a.debug_ns[b * 8 + 6] = globaltimer();
    }
  }
  __syncthreads();
  // this CTA's mp = m + IVSM_EXTRA best keys per query, descending (0 where it holds fewer)
  const int m = ivf_small_m(nprobe, G);
  const int mp = m + IVSM_EXTRA;
  if (warp < nq) {
    uint64_t x[IVSM_MAX_LOCAL / 32];
#pragma unroll
    for (int j = 0; j < IVSM_MAX_LOCAL / 32; ++j) {
      const int c = lane + 32 * j;
      x[j] = c < nloc ? sm.lk[warp][c] : 0ull;
    }
    for (int r = 0; r < mp; ++r) {
      uint64_t mx = 0ull;
#pragma unroll
      for (int j = 0; j < IVSM_MAX_LOCAL / 32; ++j) mx = x[j] > mx ? x[j] : mx;
      mx = warp_max_u64(mx);
#pragma unroll
      for (int j = 0; j < IVSM_MAX_LOCAL / 32; ++j)
        if (x[j] == mx) x[j] = 0ull;     // keys are distinct: one owner (or mx == 0)
      if (lane == 0) a.top[((int64_t)warp * G + b) * mp + r] = mx;
    }
  }
  if (a.debug_ns && tid == 0) a.debug_ns[b * 8 + 1] = globaltimer();
  grid.sync();

  // ---- B: the probe sets (every CTA, every query)
  // probe entry e -> its list's stored rows [probe[e], lend[e]) (n_local < 2^31); the loads
  // overlap the ranking
  auto set_probe = [&](int e, uint32_t l) __attribute__((always_inline)) {
    sm.probe[e] = (int32_t)a.list_off[l];
    sm.lend[e] = (int32_t)a.list_off[l + 1];
  };
  {
    const int Gm = G * m, Gmp = G * mp;
    uint64_t* tk = ring64;                   // [nq][G][mp] published keys
    uint64_t* tm = tk + nq * Gmp;            // [nq][G * m] the CTAs' first m keys
    uint64_t* cs = tm + nq * Gm;             // [nq][kFastCap] published keys >= T'
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(a.top);
    for (int i0 = tid; i0 < nq * Gmp; i0 += 8 * kThreads) {   // 8 loads in flight per thread
      uint64_t x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * kThreads;
        x[u] = i < nq * Gmp ? __ldcg(src + i) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = i0 + u * kThreads;
        if (i >= nq * Gmp) break;
        tk[i] = x[u];
        const int qi = i / Gmp, r = i - qi * Gmp, bb = r / mp, jj = r - bb * mp;
        if (jj < m) tm[qi * Gm + bb * m + jj] = x[u];
      }
    }
    if (tid < nq) {
      sm.ccnt[tid] = 0;
      sm.unpub[tid] = 0;
    }
    __syncthreads();
    for (int p = tid; p < nq * Gm; p += kThreads) {
      const uint64_t x = tm[p];
      if (x == 0ull) continue;
      const uint64_t* L = tm + (p / Gm) * Gm;
      int rank = 0;
      for (int i = 0; i < Gm; ++i) rank += L[i] > x;
      if (rank == nprobe - 1) sm.thr[p / Gm] = x;   // keys distinct, >= nprobe nonzero ones
    }
    __syncthreads();
    for (int p = tid; p < nq * Gmp; p += kThreads) {
      const int qi = p / Gmp;
      const uint64_t x = tk[p];
      if (x != 0ull && x >= sm.thr[qi]) {
        if ((p - qi * Gmp) % mp == mp - 1) sm.unpub[qi] = 1;   // keys >= T' may be unpublished
        const int pos = atomicAdd(&sm.ccnt[qi], 1);
        if (pos < kFastCap) cs[qi * kFastCap + pos] = x;
      }
    }
    __syncthreads();
    bool fast = true;
    for (int qi = 0; qi < nq; ++qi) fast = fast && !sm.unpub[qi] && sm.ccnt[qi] <= kFastCap;
    if (fast) {   // grid-uniform: every CTA read the same published keys
      for (int p = tid; p < nq * kFastCap; p += kThreads) {
        const int qi = p / kFastCap, j = p - qi * kFastCap, n = sm.ccnt[qi];
        if (j >= n) continue;
        const uint64_t* C = cs + qi * kFastCap;
        const uint64_t x = C[j];
        int rank = 0;
        for (int i = 0; i < n; ++i) rank += C[i] > x;
        if (rank < nprobe) set_probe(qi * nprobe + rank, key_id(x));
      }
      __syncthreads();
    }
    if (a.debug_ns && tid == 0) a.debug_ns[b * 8 + 2] = globaltimer();
    if (!fast) {
      // every key >= T' of this CTA -> the query's candidates; rank them after a grid barrier
      for (int p = tid; p < nq * nloc; p += kThreads) {
        const int qi = p / nloc;
        const uint64_t x = sm.lk[qi][p - qi * nloc];
        if (x >= sm.thr[qi]) {
          const int pos = atomicAdd(&a.counters[qi], 1);
          a.pcand[(int64_t)qi * a.nlist + pos] = x;
        }
      }
      grid.sync();
      for (int qi = 0; qi < nq; ++qi) {
        uint64_t* kb = ring64;
        const int cq = __ldcg(a.counters + qi);
        for (int i = tid; i < cq; i += kThreads)
          kb[i] = __ldcg(reinterpret_cast<const unsigned long long*>(a.pcand) +
                         (int64_t)qi * a.nlist + i);
        __syncthreads();
        int n = cq;
        if (cq > kRankMax) {
          // many candidates: keep the keys >= the nprobe-th largest, then rank those
          const uint64_t kth = radix_kth(kb, cq, nprobe, sm);
          uint64_t* sel = kb + cq;
          if (tid == 0) sm.s_int[0] = 0;
          __syncthreads();
          for (int i = tid; i < cq; i += kThreads)
            if (kb[i] >= kth) sel[atomicAdd(&sm.s_int[0], 1)] = kb[i];
          __syncthreads();
          kb = sel;
          n = nprobe;
        }
        for (int j = tid; j < n; j += kThreads) {
          const uint64_t x = kb[j];
          int rank = 0;
          for (int i = 0; i < n; ++i) rank += kb[i] > x;
          if (rank < nprobe) set_probe(qi * nprobe + rank, key_id(x));
        }
        __syncthreads();
      }
    }
  }
  if (a.debug_ns && tid == 0) a.debug_ns[b * 8 + 3] = globaltimer();

  // ---- C: scan entries [0, E) -- stored rows [sm.probe[e], sm.lend[e]) of `ebeg`/`eend` --
  // in 32-row pieces, an equal share of pieces per CTA, continuing the ring at position pos.
  // Entry e belongs to query e / eq_div and to output list eo(e) = e / eo_div; each CTA
  // writes its top-k of every output list to cand[(b * nout + o) * k] (0-padded, zeros for
  // lists it did not touch).  Returns the next ring position.
  auto scan_entries = [&](const int32_t* ebeg, const int32_t* eend, int E, int eq_div,
                          int eo_div, int nout, uint64_t* cand, int pos, int gscan) -> int {
    {
      // exclusive prefix of piece counts over the scoring threads (E <= 2048: 4 per thread)
      int loc[4], s = 0;
      if (!copier) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int e = tid * 4 + i;
          const int c = e < E ? (eend[e] - ebeg[e] + kPiece - 1) / kPiece : 0;
          loc[i] = s;
          s += c;
        }
      }
      const uint32_t incl = warp_incl_scan((uint32_t)s);
      if (lane == 31) sm.red[warp] = incl;
      __syncthreads();
      if (!copier) {
        int base = 0;
        for (int w = 0; w < warp; ++w) base += (int)sm.red[w];
        base += (int)incl - s;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int e = tid * 4 + i;
          if (e < E) sm.pre[e] = base + loc[i];
        }
        if (tid == kCThreads - 1) sm.pre[E] = base + s;
      }
      for (int i = tid; i < nout * k; i += kThreads) cand[(int64_t)b * nout * k + i] = 0ull;
      ptx::fence_proxy_async_smem();   // the ring's generic-proxy use above precedes the copies
      __syncthreads();
    }
    const int total = sm.pre[E];
    // pieces of CTA b among the gscan scanning CTAs
    const int pb = (int)((int64_t)b * total / gscan), pe = (int)((int64_t)(b + 1) * total / gscan);
    const int nP = pe - pb;
    if (copier) {
      if (lane == 0) {
        const uint64_t pol = policy_evict_first();
        for (int j = 0; j < nP; ++j) {
          const int p = pb + j, ps = pos + j, s = ps % kStages;
          int lo = 0, hi = E - 1;   // the last entry e with pre[e] <= p (it has pieces)
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (sm.pre[mid] <= p) lo = mid;
            else hi = mid - 1;
          }
          const int32_t lend = eend[lo];
          PieceInfo pi;
          pi.row0 = ebeg[lo] + (int64_t)(p - sm.pre[lo]) * kPiece;
          pi.rows = (int32_t)(lend - pi.row0 < kPiece ? lend - pi.row0 : kPiece);
          pi.qi = lo / eq_div;
          pi.o = lo / eo_div;
          // the piece's ids: the 16-byte aligned range around them (row_ids is padded)
          const int64_t i0 = pi.row0 & ~int64_t(3), i1 = (pi.row0 + pi.rows + 3) & ~int64_t(3);
          if (ps >= kStages) ptx::mbar_wait(empty0 + s * 8, (uint32_t)((ps / kStages - 1) & 1));
          sm.info[s] = pi;
          const uint32_t rb = (uint32_t)pi.rows * row_bytes, ib = (uint32_t)(i1 - i0) * 4;
          ptx::mbar_arrive_expect_tx(full0 + s * 8, rb + ib);
          bulk_g2s(ring0 + s * kStageBytes, a.X + pi.row0 * d_pad, rb, full0 + s * 8, pol, true);
          bulk_g2s(ring0 + s * kStageBytes + kRowsBytes, a.row_ids + i0, ib, full0 + s * 8, pol,
                   true);
        }
      }
      __syncwarp();
    } else {
      // this warp's sorted top-k of the current output list: lane j holds the j-th best
      uint64_t L = 0ull, lthr = 0ull;
      int qcur = -1, ocur = -1;
      float qr[3][8];
      // the 16 warp lists -> this CTA's list of output o, merged by warp 0 alone (the first
      // barrier keeps the next flush from overwriting lists warp 0 may still be reading)
      uint64_t* wl = &sm.wl[0][0];   // [kCWarps][k], contiguous
      auto flush = [&](int o) __attribute__((always_inline)) {
        bsync(kCThreads);
        if (lane < k) wl[warp * k + lane] = L;
        bsync(kCThreads);
        if (warp == 0) warp_topk_of_lists(wl, kCWarps, k, cand + ((int64_t)b * nout + o) * k);
      };
      for (int j = 0; j < nP; ++j) {
        const int ps = pos + j, s = ps % kStages;
        ptx::mbar_wait(full0 + s * 8, (uint32_t)((ps / kStages) & 1));
        const PieceInfo pi = sm.info[s];
        if (pi.o != ocur) {   // uniform over the scoring warps (each takes every piece)
          if (ocur >= 0) flush(ocur);
          ocur = pi.o;
          L = 0ull;
          lthr = 0ull;
        }
        if (pi.qi != qcur) {
          qcur = pi.qi;
#pragma unroll
          for (int u = 0; u < 3; ++u) {   // zero past d_pad
            const float4 qa = sm.qp[qcur][u][0][lane], qb = sm.qp[qcur][u][1][lane];
            qr[u][0] = qa.x; qr[u][1] = qa.y; qr[u][2] = qa.z; qr[u][3] = qa.w;
            qr[u][4] = qb.x; qr[u][5] = qb.y; qr[u][6] = qb.z; qr[u][7] = qb.w;
          }
        }
        if (a.debug_ns && j == 0 && tid == 0) a.debug_ns[b * 8 + 7] = globaltimer();
        const uint8_t* st = ring + s * kStageBytes;
        const int32_t* ids = reinterpret_cast<const int32_t*>(st + kRowsBytes) + (pi.row0 & 3);
        uint4 v[2][3];
        int32_t id[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = warp + h * kCWarps;
          const uint4* row = reinterpret_cast<const uint4*>(st + r * row_bytes);
#pragma unroll
          for (int u = 0; u < 3; ++u) {
            const int ch = lane + 32 * u;
            v[h][u] = (r < pi.rows && ch < nch) ? row[ch] : make_uint4(0, 0, 0, 0);
          }
          id[h] = r < pi.rows ? ids[r] : 0;
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(empty0 + s * 8);   // this warp is done with the stage
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (warp + h * kCWarps >= pi.rows) break;
          float acc = 0.f;
#pragma unroll
          for (int u = 0; u < 3; ++u) {
            const uint4 w = v[h][u];   // zero past d_pad
            acc = fmaf(__uint_as_float(w.x << 16), qr[u][0], acc);
            acc = fmaf(__uint_as_float(w.x & 0xFFFF0000u), qr[u][1], acc);
            acc = fmaf(__uint_as_float(w.y << 16), qr[u][2], acc);
            acc = fmaf(__uint_as_float(w.y & 0xFFFF0000u), qr[u][3], acc);
            acc = fmaf(__uint_as_float(w.z << 16), qr[u][4], acc);
            acc = fmaf(__uint_as_float(w.z & 0xFFFF0000u), qr[u][5], acc);
            acc = fmaf(__uint_as_float(w.w << 16), qr[u][6], acc);
            acc = fmaf(__uint_as_float(w.w & 0xFFFF0000u), qr[u][7], acc);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
          const uint64_t key = make_key(acc, (uint32_t)id[h]);
          if (key > lthr) {   // warp-uniform: insert into the sorted register list
            uint64_t prev = __shfl_up_sync(0xffffffffu, L, 1);
            if (lane == 0) prev = ~0ull;
            const uint64_t nl = key > L ? (key > prev ? prev : key) : L;
            L = lane < k ? nl : 0ull;
            lthr = __shfl_sync(0xffffffffu, L, k - 1);
          }
        }
      }
      if (ocur >= 0) flush(ocur);
    }
    return pos + nP;
  };

  // The k best keys of each of the nl lists cand[(bb * nout + o0 + o) * k], bb < G, o < nl ->
  // dst + o * k, by the whole CTA (lists of as many outputs as fit the ring loaded in one
  // pass, one L2 round trip).  cand was written by other CTAs: read through L2.
  // `reserve` keys at the end of the ring are not touched (dst may live there).
  auto merge_outputs = [&](const uint64_t* cand, int nout, int o0, int nl, uint64_t* dst,
                           int reserve) {
    const int gk = G * k;
    const int fit = max(1, (kRingKeys - reserve) / gk);
    uint64_t* lists = ring64;
    for (int f0 = 0; f0 < nl; f0 += fit) {
      const int nf = min(fit, nl - f0);
      for (int i0 = tid; i0 < nf * gk; i0 += 8 * kThreads) {   // lists[of][bb][j], 8 in flight
        uint64_t x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + u * kThreads;
          const int of = i / gk, bb = (i - of * gk) / k, j = i - of * gk - bb * k;
          x[u] = i < nf * gk ? __ldcg(reinterpret_cast<const unsigned long long*>(cand) +
                                      ((int64_t)bb * nout + o0 + f0 + of) * k + j)
                             : 0ull;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (i0 + u * kThreads < nf * gk) lists[i0 + u * kThreads] = x[u];
      }
      __syncthreads();
      for (int of = warp; of < nf; of += kWarps)   // one output per warp
        warp_topk_of_lists(lists + of * gk, G, k, dst + (int64_t)(f0 + of) * k);
      __syncthreads();
    }
  };
  auto write_result = [&](int qi, int j, uint64_t key) {
    const int64_t o = (int64_t)qi * k + j;
    if (a.out_keys) {
      a.out_keys[o] = key;
    } else {
      a.out_ids[o] = key == 0ull ? -1 : (int64_t)key_id(key);
      a.out_scores[o] = key == 0ull ? -__int_as_float(0x7f800000) : key_score(key);
    }
  };

  if constexpr (!MATURE) {
    const int np = nq * nprobe;
    const int pos = scan_entries(sm.probe, sm.lend, np, nprobe, nprobe, nq, a.cand, nA, G);
    (void)pos;
    if (a.debug_ns && tid == 0) a.debug_ns[b * 8 + 4] = globaltimer();

    // ---- D: the last CTA to finish merges the G per-CTA lists of every query
    // (CTA barrier, then a gpu-scope acq_rel increment by one thread: releases this CTA's
    // lists, and the last CTA acquires everyone's)
    __syncthreads();
    if (tid == 0) sm.s_int[3] = ptx::atom_add_acq_rel_gpu(&a.counters[nq], 1);
    __syncthreads();
    if (sm.s_int[3] != G - 1) return;
    uint64_t* best = ring64 + kRingKeys - nq * k;   // past every merge's working set
    merge_outputs(a.cand, nq, 0, nq, best, nq * k);
    for (int i = tid; i < nq * k; i += kThreads) write_result(i / k, i % k, best[i]);
    if (a.done_host) __threadfence_system();   // results visible before the signal
    __syncthreads();
    if (a.done_host && tid == 0) {
      const int32_t v = *a.seq + 1;
      *a.seq = v;
      __threadfence_system();
      *reinterpret_cast<volatile int32_t*>(a.done_host) = v;
    }
    if (a.debug_ns && tid == 0) a.debug_ns[b * 8 + 5] = globaltimer();
  } else {
    // ---- maturity exit (§3.3; R14-R19): stage s scans lists
    // [s*g, (s+1)*g) of every active query; the last CTA to finish a stage merges each list's
    // per-CTA lists, inserts the lists into the running top-k R in probe-rank order, updates
    // RQ / EMA per list and takes the exit decision at the checkpoint, then releases the
    // next stage.  One launch; the engine-ready flag is read on the device.
    const int P = nprobe, g = mo.g;
    // CTAs 0..G-2 scan, CTA G-1 closes the stages.  Stage st's scan overlaps stage st-1's
    // closure: the entries of stage st are those of the queries still active after closure
    // st-2 (a superset of the true set -- a query that exits at closure st-1 just has its
    // stage-st lists ignored), and the per-CTA lists are double-buffered by stage parity.
    // The closer waits for every scanner's arrival at stage st, merges each list's per-CTA
    // lists, inserts the lists into the running top-k R in probe-rank order, updates RQ / EMA
    // per list, takes the exit decisions and releases the stage with the new active mask.
    const int Gs = G - 1;
    int32_t* arr = a.counters + nq;        // [2] scanners done with a stage, per parity
    int32_t* rel = a.counters + nq + 2;    // release word: closed stages | active mask << 16
    const int64_t cand_stage = (int64_t)G * nq * g * k;
    // tid 0: wait until stages [0, upto) are closed, or the search has ended (mask 0)
    auto wait_release = [&](int upto) -> uint32_t {
      int32_t v;
      while (true) {
        v = ptx::ld_acquire_gpu(rel);
        if ((v & 0xFFFF) >= upto || ((v & 0xFFFF) > 0 && ((uint32_t)v >> 16) == 0u)) break;
        __nanosleep(32);
      }
      return (uint32_t)v >> 16;
    };
    const uint32_t full_mask = (1u << nq) - 1u;
    if (b == G - 1) {
      // ---- the closer
      for (int i = tid; i < 2 * nq * g * k; i += kThreads)   // its own (empty) lists
        a.cand[(i / (nq * g * k)) * cand_stage + (int64_t)b * nq * g * k + i % (nq * g * k)] = 0ull;
      uint32_t cmask = full_mask;   // active after the previous closure
      for (int st = 0;; ++st) {
        const bool stamp = mo.stage_ns && st < 64 && tid == 0;
        if (tid == 0) {
          while (ptx::ld_acquire_gpu(arr + (st & 1)) < Gs) __nanosleep(32);
          if (stamp) mo.stage_ns[st * 4 + 2] = globaltimer();
        }
        __syncthreads();
        // the engine flag, read once per stage (its latency overlaps the merges)
        const int32_t ready = tid == 0 ? read_ready(mo.ready) : 0;
        const uint64_t* cand = a.cand + (st & 1) * cand_stage;
        // the stage's lists (exact top-k per list: its best key is element 0)
        uint64_t* lt = ring64 + kRingKeys - nq * g * k;
        merge_outputs(cand, nq * g, 0, nq * g, lt, nq * g * k);
        if (tid == 0) {
          sm.s_int[1] = ready;
          sm.s_int[2] = (int32_t)cmask;
        }
        __syncthreads();
        if (warp < nq && ((cmask >> warp) & 1u)) {
          const int qi = warp;
          uint64_t R = lane < k ? __ldcg(reinterpret_cast<const unsigned long long*>(mo.R) +
                                         (int64_t)qi * k + lane)
                                : 0ull;
          double ema = __ldcg(mo.ema + qi);
          // the g insertions in probe-rank order (shuffles only); lane j keeps step j's
          // (s_best, s_worst, s_t) keys, so the fp64 divisions below run side by side
          uint64_t kb = 0ull, kw = 0ull, ks = 0ull;
          const int ng = min(g, P - st * g);
          for (int j = 0; j < ng; ++j) {
            const uint64_t* lj = lt + (qi * g + j) * k;
            // R <- top-k(R u list): both descending, the list reversed across lanes makes the
            // 64 keys bitonic; one max/min step keeps the best 32 (bitonic), 5 more sort them
            const uint64_t lv = lane < k ? lj[lane] : 0ull;
            const uint64_t lrev = __shfl_sync(0xffffffffu, lv, 31 - lane);
            uint64_t x = R > lrev ? R : lrev;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              const uint64_t y = __shfl_xor_sync(0xffffffffu, x, o);
              x = (lane & o) ? (x < y ? x : y) : (x > y ? x : y);
            }
            R = lane < k ? x : 0ull;
            const uint64_t best = __shfl_sync(0xffffffffu, R, 0);
            const unsigned nz = __ballot_sync(0xffffffffu, R != 0ull);
            const uint64_t worst = nz ? __shfl_sync(0xffffffffu, R, 31 - __clz(nz)) : 0ull;
            if (lane == j) {
              kb = best;
              kw = worst;
              ks = lj[0];
            }
          }
          // signal (R15-R17) in fp64 from the fp32 scores, the oracle's two roundings
          double rq = 1.0;
          if (lane < ng && ks != 0ull && kb != 0ull) {
            const double sb = (double)key_score(kb), sw = (double)key_score(kw);
            const double s_t = (double)key_score(ks);
            if (sb != sw) rq = __ddiv_rn(__dsub_rn(sb, s_t), __dsub_rn(sb, sw));
          }
          for (int j = 0; j < ng; ++j) {   // the EMA recurrence, identical in every lane
            const double rj = __shfl_sync(0xffffffffu, rq, j);
            const int r = st * g + j;
            ema = r == 0 ? rj : __dadd_rn(__dmul_rn(mo.alpha, rj), __dmul_rn(1.0 - mo.alpha, ema));
            if (lane == j && mo.trace_rq) {
              mo.trace_rq[(int64_t)qi * P + r] = rj;
              mo.trace_ema[(int64_t)qi * P + r] = ema;
            }
          }
          if (lane < k) reinterpret_cast<unsigned long long*>(mo.R)[(int64_t)qi * k + lane] = R;
          if (lane == 0) {
            mo.ema[qi] = ema;
            // checkpoint after the stage (R18): t = lists scanned so far
            const int t = min((st + 1) * g, P);
            const bool exit_now = (t % g) == 0 && ema >= mo.tau && sm.s_int[1] != 0;
            if (exit_now || t >= P) {
              mo.t_done[qi] = t;
              atomicAnd(reinterpret_cast<unsigned*>(&sm.s_int[2]), ~(1u << qi));
            }
          }
        }
        __syncthreads();
        cmask = (uint32_t)sm.s_int[2];
        if (cmask == 0u) {   // the last queries finished: R -> the output
          for (int i = tid; i < nq * k; i += kThreads)
            write_result(i / k, i % k,
                         __ldcg(reinterpret_cast<const unsigned long long*>(mo.R) + i));
          for (int qi = tid; qi < nq; qi += kThreads)
            if (mo.out_t) mo.out_t[qi] = __ldcg(mo.t_done + qi);
        }
        __syncthreads();
        if (tid == 0) {
          arr[st & 1] = 0;
          if (stamp) mo.stage_ns[st * 4 + 3] = globaltimer();
          ptx::st_release_gpu(rel, (int32_t)((cmask << 16) | (uint32_t)(st + 1)));
        }
        if (cmask == 0u) break;
      }
    } else {
      // ---- the scanners
      int pos = nA;
      for (int st = 0;; ++st) {
        const bool stamp = mo.stage_ns && st < 64 && tid == 0 && b == 0;
        if (tid == 0) sm.s_int[2] = (int32_t)(st >= 2 ? wait_release(st - 1) : full_mask);
        __syncthreads();
        const uint32_t amask = (uint32_t)sm.s_int[2];
        __syncthreads();
        if (amask == 0u) break;
        if (stamp) mo.stage_ns[st * 4 + 0] = globaltimer();
        // this stage's entries: e = qi * g + j -> probe rank st * g + j of query qi
        for (int e = tid; e < nq * g; e += kThreads) {
          const int qi = e / g, r = st * g + e % g;
          const bool on = r < P && ((amask >> qi) & 1u);
          sm.seb[e] = on ? sm.probe[qi * P + r] : 0;
          sm.see[e] = on ? sm.lend[qi * P + r] : 0;
        }
        __syncthreads();
        pos = scan_entries(sm.seb, sm.see, nq * g, g, 1, nq * g, a.cand + (st & 1) * cand_stage,
                           pos, Gs);
        __syncthreads();
        if (stamp) mo.stage_ns[st * 4 + 1] = globaltimer();
        if (tid == 0) ptx::atom_add_acq_rel_gpu(arr + (st & 1), 1);   // releases the lists
      }
    }
  }
}

size_t ivf_small_smem_bytes() { return 128 + (size_t)kRingBytes + sizeof(SmallSmem); }

static cudaError_t launch_small(const IvfSmallArgs& a, const SmallMatureArgs& mo, bool mature,
                                int grid, cudaStream_t s) {
  if (a.nq < 1 || a.nq > IVSM_MAX_NQ || a.k < 1 || a.k > IVSM_MAX_K || a.nprobe < 1 ||
      a.nprobe > IVSM_MAX_NPROBE || a.nprobe > a.nlist || a.d_pad > kMaxDPad || a.d_pad % 64 ||
      grid < a.nq || !ivf_small_fits(a.nq, a.nprobe, a.nlist, grid) ||
      (int64_t)grid * a.k * 2 + (int64_t)a.nq * a.k > kRingKeys)
    return cudaErrorInvalidValue;
  if (mature && (mo.g < 1 || mo.g > IVSM_MAX_G || a.nq * mo.g > IVSM_MAX_STAGE || grid < 2 ||
                 (int64_t)grid * a.k * 2 + (int64_t)a.nq * mo.g * a.k > kRingKeys))
    return cudaErrorInvalidValue;
  const size_t smem = ivf_small_smem_bytes();
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
    e = cudaLaunchKernelEx(&cfg, kern, a, mo);
    note_launch();
    return e;
  };
  if (mature) {
    if (a.nq <= 1) return go(ivf_small_kernel<1, true>);
    if (a.nq <= 2) return go(ivf_small_kernel<2, true>);
    if (a.nq <= 4) return go(ivf_small_kernel<4, true>);
    return go(ivf_small_kernel<8, true>);
  }
  if (a.nq <= 1) return go(ivf_small_kernel<1, false>);
  if (a.nq <= 2) return go(ivf_small_kernel<2, false>);
  if (a.nq <= 4) return go(ivf_small_kernel<4, false>);
  return go(ivf_small_kernel<8, false>);
}

cudaError_t launch_ivf_small(const IvfSmallArgs& a, int grid, cudaStream_t s) {
  return launch_small(a, SmallMatureArgs{}, false, grid, s);
}

cudaError_t launch_ivf_small_mature(const IvfSmallArgs& a, const SmallMatureArgs& mo, int grid,
                                    cudaStream_t s) {
  return launch_small(a, mo, true, grid, s);
}

}  // namespace sa
