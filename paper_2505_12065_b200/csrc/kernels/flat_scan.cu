// flat_scan.cu -- fused exact inner-product scan + per-query running top-k (§8(a) a5).
//
// The retrieval step of SearchAgent-X is top-k search of query embeddings
// against the passage-embedding knowledge base (§2.1 "exact nearest
// neighbor (ENN) search"; vLLM_ENN "exhaustive search", App. B.3 P:394;
// k docs returned).  Here S = Q . X^T is computed tile by tile on
// the sm_100a tensor cores and reduced to a running top-k inside the kernel,
// so the score matrix never reaches HBM (BASELINE.json north_star).
//
// Mapping:
//   * MMA M side = 128 queries of one query block.  The block's bf16 rows live
//     in TMEM for the whole scan (A operand from TMEM, "TS" form): lane m =
//     query m, columns [A_COL, A_COL + d_pad/2) hold its 2-packed bf16.
//   * MMA N side = 64 corpus rows per tile, TMA-staged from HBM into a
//     FS_STAGES-deep smem ring (128-byte swizzle, one 64x64 box per K-step).
//   * fp32 accumulators: two 64-column TMEM buffers (cols 0 and 64) so the
//     epilogue drains tile t while the tensor core computes tile t+1.
//   * warp 0: TMA producer, warp 1: TMEM alloc + single-thread MMA issuer,
//     warps 2..5: epilogue, thread = query (TMEM lane quadrant = warp % 4).
//     Each epilogue thread keeps a size-k min-heap of packed keys; the
//     per-tile fast path is a 64-way max + one compare against the heap root.
//   * persistent grid: work item w = (query block qb, corpus slice s); slices
//     partition the corpus tiles; partial top-k lists go to part[q][s][k].
#include <cuda_bf16.h>

#include "flat_scan.cuh"
#include "keys.cuh"
#include "ptx.cuh"

namespace sa {

namespace {

constexpr int kBM = FS_BM;
constexpr int kBN = FS_BN;
constexpr int kBK = FS_BK;
constexpr int kStages = FS_STAGES;
constexpr int kStageBytes = kBN * kBK * 2;  // 8 KB
constexpr int kAccCols = kBN;               // fp32 columns per accumulator
constexpr int kACol = 2 * kAccCols;         // A (queries) starts after two accumulators
constexpr uint32_t kTmemCols = 512;

struct __align__(8) SmemTail {
  uint64_t full[kStages];
  uint64_t empty[kStages];
  uint64_t tmem_full[2];
  uint64_t tmem_empty[2];
  uint64_t a_full;
  uint32_t tmem_base;
};

__device__ __forceinline__ float heap_threshold(uint64_t root) {
  return root == 0ull ? -__int_as_float(0x7f800000) : key_score(root);
}

// Offer `key` to a size-k min-heap whose element i lives at h[i * kBM].
// Returns the new threshold score (score of the root).
__device__ __noinline__ float heap_offer(uint64_t* h, int k, uint64_t key) {
  if (key <= h[0]) return heap_threshold(h[0]);
  int i = 0;
  while (true) {
    int l = 2 * i + 1;
    if (l >= k) break;
    int r = l + 1;
    uint64_t hl = h[(size_t)l * kBM];
    int c = l;
    uint64_t hc = hl;
    if (r < k) {
      uint64_t hr = h[(size_t)r * kBM];
      if (hr < hl) { c = r; hc = hr; }
    }
    if (hc >= key) break;
    h[(size_t)i * kBM] = hc;
    i = c;
  }
  h[(size_t)i * kBM] = key;
  return heap_threshold(h[0]);
}

struct WorkItem {
  int qb, s;
  int64_t t0, t1;
};

__device__ __forceinline__ WorkItem work_item(int w, int S, int64_t T) {
  WorkItem wi;
  wi.qb = w / S;
  wi.s = w % S;
  wi.t0 = (int64_t)wi.s * T / S;
  wi.t1 = (int64_t)(wi.s + 1) * T / S;
  return wi;
}

}  // namespace

__global__ void __launch_bounds__(FS_THREADS, 1)
flat_scan_topk_kernel(const __grid_constant__ CUtensorMap tmap_x, const FlatScanArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* stage_base = smem;
  uint64_t* heap_s = reinterpret_cast<uint64_t*>(smem + kStages * kStageBytes);
  SmemTail* tail =
      reinterpret_cast<SmemTail*>(smem + kStages * kStageBytes + FS_KSMEM * kBM * sizeof(uint64_t));

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int S = a.S;
  const int n_work = a.QB * S;
  const int64_t T = (a.n_rows + kBN - 1) / kBN;
  const int num_kb = a.d_pad / kBK;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      ptx::mbar_init(ptx::smem_u32(&tail->full[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&tail->empty[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(ptx::smem_u32(&tail->tmem_full[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&tail->tmem_empty[i]), 4);
    }
    ptx::mbar_init(ptx::smem_u32(&tail->a_full), 4);
    ptx::fence_mbar_init();
    ptx::fence_proxy_async_smem();
  }
  if (warp == 0 && lane == 0) ptx::prefetch_tmap(&tmap_x);
  if (warp == 1) {
    ptx::tmem_alloc(ptx::smem_u32(&tail->tmem_base), kTmemCols);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tail->tmem_base;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
        WorkItem wi = work_item(w, S, T);
        for (int64_t t = wi.t0; t < wi.t1; ++t) {
          for (int kb = 0; kb < num_kb; ++kb) {
            ptx::mbar_wait(ptx::smem_u32(&tail->empty[stage]), phase ^ 1);
            const uint32_t fb = ptx::smem_u32(&tail->full[stage]);
            ptx::mbar_arrive_expect_tx(fb, kStageBytes);
            ptx::tma_load_2d(ptx::smem_u32(stage_base + stage * kStageBytes), &tmap_x, fb,
                             kb * kBK, (int32_t)(t * kBN));
            if (++stage == kStages) { stage = 0; phase ^= 1; }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===================== MMA issuer (one thread) =====================
    if (lane == 0) {
      const uint32_t idesc = ptx::umma_idesc_bf16(kBM, kBN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int cur_qb = -1;
      uint32_t a_phase = 0;
      for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
        WorkItem wi = work_item(w, S, T);
        if (wi.qb != cur_qb) {
          ptx::mbar_wait(ptx::smem_u32(&tail->a_full), a_phase);
          a_phase ^= 1;
          cur_qb = wi.qb;
          ptx::tc_fence_after();
        }
        for (int64_t t = wi.t0; t < wi.t1; ++t) {
          ptx::mbar_wait(ptx::smem_u32(&tail->tmem_empty[acc]), acc_phase ^ 1);
          ptx::tc_fence_after();
          const uint32_t d_tmem = tmem + acc * kAccCols;
          for (int kb = 0; kb < num_kb; ++kb) {
            ptx::mbar_wait(ptx::smem_u32(&tail->full[stage]), phase);
            ptx::tc_fence_after();
            const uint64_t bdesc = ptx::umma_desc_sw128(ptx::smem_u32(stage_base + stage * kStageBytes));
#pragma unroll
            for (int kk = 0; kk < kBK / 16; ++kk) {
              const uint32_t a_tmem = tmem + kACol + kb * (kBK / 2) + kk * 8;
              ptx::mma_bf16_ts(d_tmem, a_tmem, bdesc + (uint64_t)(kk * 2), idesc,
                               (kb | kk) != 0 ? 1u : 0u);
            }
            ptx::tc_commit(ptx::smem_u32(&tail->empty[stage]));
            if (++stage == kStages) { stage = 0; phase ^= 1; }
          }
          ptx::tc_commit(ptx::smem_u32(&tail->tmem_full[acc]));
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else {
    // ===================== epilogue: 4 warps, thread = query =====================
    const int quad = warp & 3;                 // TMEM lane quadrant this warp may access
    const int rib = quad * 32 + lane;          // row in query block
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    const int k = a.k;
    uint64_t* heap = (k <= FS_KSMEM) ? (heap_s + rib)
                                     : (a.heap_g + (size_t)blockIdx.x * k * kBM + rib);
    for (int i = 0; i < k; ++i) heap[(size_t)i * kBM] = 0ull;
    float thr = heap_threshold(0ull);
    int acc = 0;
    uint32_t acc_phase = 0;
    int cur_qb = -1;
    for (int w = blockIdx.x; w < n_work; w += gridDim.x) {
      WorkItem wi = work_item(w, S, T);
      const int64_t q = (int64_t)wi.qb * kBM + rib;
      if (wi.qb != cur_qb) {
        // Stage this query block into TMEM columns [kACol, kACol + d_pad/2).
        // All MMAs reading the previous block completed before the previous
        // item's last tmem_full commit, which this thread already consumed.
        const uint4* src = reinterpret_cast<const uint4*>(a.Q + (size_t)q * a.d_pad);
        for (int c = 0; c < num_kb; ++c) {
          uint32_t r[32];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            uint4 v = __ldg(src + c * 8 + i);
            r[4 * i + 0] = v.x; r[4 * i + 1] = v.y; r[4 * i + 2] = v.z; r[4 * i + 3] = v.w;
          }
          ptx::tmem_st32(tmem + lane_addr + kACol + c * 32, r);
        }
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&tail->a_full));
        cur_qb = wi.qb;
      }
      for (int64_t t = wi.t0; t < wi.t1; ++t) {
        ptx::mbar_wait(ptx::smem_u32(&tail->tmem_full[acc]), acc_phase);
        ptx::tc_fence_after();
        uint32_t r0[32], r1[32];
        ptx::tmem_ld32(tmem + lane_addr + acc * kAccCols, r0);
        ptx::tmem_ld32(tmem + lane_addr + acc * kAccCols + 32, r1);
        ptx::tmem_wait_ld();
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&tail->tmem_empty[acc]));
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }

        const int64_t row0 = t * kBN;
        if (a.mode == 1) {
          // debug: materialise the score tile (tests only)
          if (q < a.nq_pad) {
            float* dst = a.dbg + (size_t)q * a.n_rows;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              if (row0 + j < a.n_rows) dst[row0 + j] = __uint_as_float(r0[j]);
              if (row0 + 32 + j < a.n_rows) dst[row0 + 32 + j] = __uint_as_float(r1[j]);
            }
          }
          continue;
        }
        float m0 = __uint_as_float(r0[0]);
        float m1 = __uint_as_float(r1[0]);
#pragma unroll
        for (int j = 1; j < 32; ++j) {
          m0 = fmaxf(m0, __uint_as_float(r0[j]));
          m1 = fmaxf(m1, __uint_as_float(r1[j]));
        }
        if (fmaxf(m0, m1) >= thr) {
#pragma unroll
          for (int j = 0; j < 64; ++j) {
            const float s = __uint_as_float(j < 32 ? r0[j] : r1[j - 32]);
            if (s >= thr) {
              const int64_t row = row0 + j;
              if (row < a.n_rows) {
                const uint32_t id = a.id_base + (a.row_ids ? (uint32_t)a.row_ids[row] : (uint32_t)row);
                thr = heap_offer(heap, k, make_key(s, id));
              }
            }
          }
        }
      }
      if (a.mode == 0) {
        // flush this work item's partial list and reset the heap
        uint64_t* dst = a.part + ((size_t)q * S + wi.s) * k;
        for (int i = 0; i < k; ++i) {
          dst[i] = heap[(size_t)i * kBM];
          heap[(size_t)i * kBM] = 0ull;
        }
        thr = heap_threshold(0ull);
      }
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, kTmemCols);
  }
}

size_t flat_scan_smem_bytes() {
  return 1024 + (size_t)kStages * kStageBytes + (size_t)FS_KSMEM * kBM * sizeof(uint64_t) +
         sizeof(SmemTail);
}

cudaError_t launch_flat_scan(const CUtensorMap& tmap, const FlatScanArgs& a, int grid,
                             cudaStream_t stream) {
  static bool attr_set = false;
  const size_t smem = flat_scan_smem_bytes();
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(flat_scan_topk_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  flat_scan_topk_kernel<<<grid, FS_THREADS, smem, stream>>>(tmap, a);
  return cudaGetLastError();
}

}  // namespace sa
