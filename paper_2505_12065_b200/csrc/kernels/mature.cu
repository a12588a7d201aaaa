// mature.cu -- non-stall maturity exit on IVF list order.
//
// PAPER.md §3.3: a normalised quality signal RQ_t of the newly discovered
// candidates, smoothed by an EMA (App. B.2), ends the search once it exceeds tau
// AND the LLM engine is ready; otherwise the search stops naturally.  Readings R14-R19
// (DESIGN.md §2): a step is one probed list in probe-rank order; s_t = the best score of
// the list; RQ_t = (s_best - s_t) / (s_best - s_worst) over the running top-k AFTER the
// list is inserted (1 when s_best == s_worst or the list is empty); EMA seeded with RQ_1,
// alpha = 2/(W+1); the exit test runs every g lists.
//
// The scan itself is ivf_scan_kernel run stage by stage (g lists per active query per
// stage) with the cross-list pruning bound off, so each (query, list) slot holds the exact
// top-k of its chunks and the list's best score.  These kernels are the per-stage glue:
// stage lists, the in-order merge + signal + exit decision, the loop condition, the output.
#include <cuda_runtime.h>

#include <cmath>

#include "keys.cuh"
#include "launch.cuh"
#include "mature.cuh"

namespace sa {

namespace {

constexpr int kUpdThreads = 256;
constexpr int kCandBlock = 1024;  // candidates examined per pass of the merge

__device__ __forceinline__ int32_t load_ready(const volatile int32_t* p) {
  if (p == nullptr) return 1;
  int32_t v;
  asm volatile("ld.relaxed.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void mature_init_kernel(MatureArgs a) {
  const int64_t n = (int64_t)a.nq * a.k;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    a.R[i] = 0ull;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.nq;
       i += (int64_t)gridDim.x * blockDim.x) {
    a.ema[i] = 0.0;
    a.active[i] = 1;
    a.t_done[i] = 0;
  }
  const int64_t nt = (int64_t)a.nq * a.nprobe_max;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nt;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (a.trace_rq) a.trace_rq[i] = __longlong_as_double(0x7ff8000000000000ll);
    if (a.trace_ema) a.trace_ema[i] = __longlong_as_double(0x7ff8000000000000ll);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.ctrl[0] = 0;
    a.ctrl[1] = a.nq;
    a.ctrl[2] = 0;
    a.ctrl[3] = 0;
  }
}

// Bitonic sort of buf[0, n2) descending (n2 a power of two), whole block.
__device__ void sort_desc(uint64_t* buf, int n2) {
  for (int sz = 2; sz <= n2; sz <<= 1)
    for (int st = sz >> 1; st > 0; st >>= 1) {
      for (int i = threadIdx.x; i < n2; i += blockDim.x) {
        const int j = i ^ st;
        if (j > i) {
          const bool desc = (i & sz) == 0;
          const uint64_t x = buf[i], y = buf[j];
          if (desc ? x < y : x > y) {
            buf[i] = y;
            buf[j] = x;
          }
        }
      }
      __syncthreads();
    }
}

// The last CTA of the update advances the stage and sets the WHILE condition.
__device__ void advance(const MatureArgs& a, cudaGraphConditionalHandle h) {
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&a.ctrl[3], 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (s_last && threadIdx.x == 0) {
    __threadfence();
    a.ctrl[3] = 0;
    const int s = a.ctrl[0] + 1;
    a.ctrl[0] = s;
    const bool more = atomicAdd(&a.ctrl[1], 0) > 0 && (int64_t)s * a.g < a.nprobe_max;
    cudaGraphSetConditional(h, more ? 1u : 0u);
  }
}

// One CTA per query: the stage's lists in probe-rank order.
__global__ void __launch_bounds__(kUpdThreads)
mature_update_kernel(MatureArgs a, cudaGraphConditionalHandle h) {
  extern __shared__ uint64_t buf[];  // [pow2 >= k + kCandBlock]
  __shared__ int s_cnt;
  __shared__ unsigned long long s_max;
  const int q = blockIdx.x;
  if (!a.active[q]) {
    advance(a, h);
    return;
  }
  const int s = a.ctrl[0];
  const int k = a.k;
  uint64_t* Rq = a.R + (size_t)q * k;
  for (int j = 0; j < a.g; ++j) {
    const int r = s * a.g + j;  // probe rank (0-based); step t = r + 1
    if (r >= a.nprobe_max) break;
    const int64_t e = (int64_t)q * a.g + j;
    const uint64_t* cand = a.part + (size_t)a.q_slot[e] * a.parts * k;
    const int64_t cnt = (a.q_slot[e + 1] - a.q_slot[e]) * (int64_t)a.parts * k;
    if (threadIdx.x == 0) s_max = 0ull;
    __syncthreads();
    // s_t: the list's best key (its partial lists hold each chunk's exact top-k)
    uint64_t m = 0ull;
    for (int64_t i = threadIdx.x; i < cnt; i += blockDim.x) m = max(m, cand[i]);
    if (m) atomicMax(&s_max, (unsigned long long)m);
    // R <- top-k(R u list): passes over blocks of candidates, keeping only keys above the
    // current k-th (once R is full), then a sort of R + survivors
    for (int64_t base = 0; base < cnt || base == 0; base += kCandBlock) {
      for (int i = threadIdx.x; i < k; i += blockDim.x) buf[i] = Rq[i];
      if (threadIdx.x == 0) s_cnt = 0;
      __syncthreads();
      const uint64_t floor_key = Rq[k - 1];  // 0 while R is not full
      const int64_t end = min(cnt, base + (int64_t)kCandBlock);
      for (int64_t i = base + threadIdx.x; i < end; i += blockDim.x) {
        const uint64_t c = cand[i];
        if (c > floor_key) buf[k + atomicAdd(&s_cnt, 1)] = c;
      }
      __syncthreads();
      const int tot = k + s_cnt;
      if (s_cnt > 0) {
        int n2 = 1;
        while (n2 < tot) n2 <<= 1;
        for (int i = tot + threadIdx.x; i < n2; i += blockDim.x) buf[i] = 0ull;
        __syncthreads();
        sort_desc(buf, n2);
        for (int i = threadIdx.x; i < k; i += blockDim.x) Rq[i] = buf[i];
      }
      __syncthreads();
      if (end >= cnt) break;
    }
    if (threadIdx.x == 0) {
      // signal (R15-R17), in fp64 from the fp32 scores
      double rq = 1.0;
      const uint64_t best = Rq[0];
      if (s_max != 0ull && best != 0ull) {
        int last = k - 1;
        while (Rq[last] == 0ull) --last;
        const double sb = (double)key_score(best), sw = (double)key_score(Rq[last]);
        const double st = (double)key_score((uint64_t)s_max);
        if (sb != sw) rq = __ddiv_rn(__dsub_rn(sb, st), __dsub_rn(sb, sw));
      }
      // no FMA contraction: the same two roundings as the oracle's a*x + (1-a)*prev
      const double ema =
          (r == 0) ? rq : __dadd_rn(__dmul_rn(a.alpha, rq), __dmul_rn(1.0 - a.alpha, a.ema[q]));
      a.ema[q] = ema;
      if (a.trace_rq) a.trace_rq[(size_t)q * a.nprobe_max + r] = rq;
      if (a.trace_ema) a.trace_ema[(size_t)q * a.nprobe_max + r] = ema;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    // checkpoint after the stage (R18): t = lists scanned so far
    const int t = min((s + 1) * a.g, a.nprobe_max);
    const bool checkpoint = (t % a.g) == 0;
    const bool exit_now = checkpoint && a.ema[q] >= a.tau && load_ready(a.ready) != 0;
    if (exit_now || t >= a.nprobe_max) {
      a.active[q] = 0;
      a.t_done[q] = t;
      atomicSub(&a.ctrl[1], 1);
    }
  }
  advance(a, h);
}

__global__ void mature_final_kernel(MatureArgs a, int64_t* out_ids, float* out_scores,
                                    int32_t* out_t) {
  const int64_t n = (int64_t)a.nq * a.k;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = a.R[i];
    out_ids[i] = key == 0ull ? -1 : (int64_t)key_id(key);
    out_scores[i] = key == 0ull ? -INFINITY : key_score(key);
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.nq;
       i += (int64_t)gridDim.x * blockDim.x)
    if (out_t) out_t[i] = a.t_done[i];
}

unsigned blocks_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  if (b < 1) b = 1;
  if (b > 1184) b = 1184;
  return (unsigned)b;
}

}  // namespace

cudaError_t launch_mature_init(const MatureArgs& a, cudaStream_t s) {
  const int64_t n = (int64_t)a.nq * (a.k > a.nprobe_max ? a.k : a.nprobe_max);
  mature_init_kernel<<<blocks_for(n), 256, 0, s>>>(a);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_mature_update(const MatureArgs& a, cudaGraphConditionalHandle h,
                                 cudaStream_t s) {
  int n2 = 1;
  while (n2 < a.k + kCandBlock) n2 <<= 1;
  const size_t smem = (size_t)n2 * sizeof(uint64_t);
  cudaError_t e = ensure_max_smem(reinterpret_cast<const void*>(mature_update_kernel), 64 * 1024);
  if (e != cudaSuccess) return e;
  mature_update_kernel<<<a.nq, kUpdThreads, smem, s>>>(a, h);
  note_launch();
  return cudaGetLastError();
}

cudaError_t launch_mature_final(const MatureArgs& a, int64_t* out_ids, float* out_scores,
                                int32_t* out_t, cudaStream_t s) {
  mature_final_kernel<<<blocks_for((int64_t)a.nq * a.k), 256, 0, s>>>(a, out_ids, out_scores,
                                                                       out_t);
  note_launch();
  return cudaGetLastError();
}

}  // namespace sa
