// score_gemm.cu -- dense score dump S = Q . X^T on the sm_100a tensor cores (the IVF probe's
// centroid scores, SURVEY.md §8(a) a7, and the graph search's entry points).
//
// The probe scores every query against every centroid (PAPER.md's retrieval over the
// partitioned index, R11: the nprobe best lists by inner product), then an exact select
// (merge.cu) keeps the top-nprobe keys.  A probe is a small GEMM (C3: 512 x 16384 x 768,
// 12.9 GFLOP), so the flat scan's layout -- each unit stages its query block once into TMEM
// and scans a corpus slice -- pays that staging for only 3-4 tiles per unit.  Here both
// operands stream through one TMA ring, K-block by K-block, as in a plain GEMM:
//   * one CTA per SM, persistent over 128 x 128 output tiles (query block, centroid block);
//   * warp 8: TMA producer -- per K-block a 128 x 64 bf16 box of queries and one of centroids
//     (16 + 16 KB, SWIZZLE_128B) into a 5-stage ring (full / empty mbarriers);
//   * warp 9: TMEM allocation and the MMA issuer (tcgen05.mma kind::f16, SS form, M = N = 128,
//     K = 16 per instruction, fp32 accumulate) into two 128-column TMEM accumulators, so the
//     epilogue drains tile t while tile t+1 accumulates;
//   * warps 0..7: epilogue -- warp w reads TMEM lane quadrant w % 4 (32 queries) x 64 columns,
//     then writes them through a 4 KB XOR-swizzled smem tile so that every store instruction
//     writes one query's 32 consecutive scores (128 B).
// The per-row K order (K-blocks 0.., 16-wide steps) is the flat scan's, so the scores are the
// same fp32 sums of exact bf16 products.
#include <cuda_bf16.h>

#include "launch.cuh"
#include "ptx.cuh"
#include "score_gemm.cuh"

namespace sa {

namespace {

constexpr int kBM = 128;                 // queries per tile (MMA M)
constexpr int kBN = 128;                 // centroid rows per tile (MMA N)
constexpr int kBK = 64;                  // bf16 elements per K-block (one 128-byte swizzle row)
constexpr int kStages = 5;
constexpr int kBoxBytes = kBM * kBK * 2;  // 16 KB (both operands: 128 rows x 64)
constexpr int kStageBytes = 2 * kBoxBytes;
constexpr int kEpiWarps = 8;
constexpr int kThreads = 32 * (kEpiWarps + 2);
constexpr int kProducerWarp = kEpiWarps;
constexpr int kMmaWarp = kEpiWarps + 1;
constexpr uint32_t kTmemCols = 256;      // two fp32 accumulators of 128 columns
constexpr uint32_t kIdesc = ptx::umma_idesc_bf16(kBM, kBN);

struct __align__(8) Bars {
  uint64_t full[kStages];
  uint64_t empty[kStages];
  uint64_t tmem_full[2];
  uint64_t tmem_empty[2];
  uint32_t tmem_base;
};

constexpr size_t kSmemBytes = 1024 + (size_t)kStages * kStageBytes +
                              (size_t)kEpiWarps * 32 * 32 * sizeof(float) + sizeof(Bars);

__global__ void __launch_bounds__(kThreads, 1)
score_gemm_kernel(const __grid_constant__ CUtensorMap tmap_q,
                  const __grid_constant__ CUtensorMap tmap_x, const ScoreGemmArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* ring = smem;
  float* xpose = reinterpret_cast<float*>(smem + (size_t)kStages * kStageBytes);
  Bars* bars = reinterpret_cast<Bars*>(xpose + kEpiWarps * 32 * 32);
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0);
  const int lane = threadIdx.x % 32;
  const int QB = (int)((a.nq + kBM - 1) / kBM);
  const int NB = (int)((a.n_rows + kBN - 1) / kBN);
  const int n_tiles = QB * NB;
  const int num_kb = a.d_pad / kBK;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      ptx::mbar_init(ptx::smem_u32(&bars->full[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&bars->empty[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(ptx::smem_u32(&bars->tmem_full[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&bars->tmem_empty[i]), kEpiWarps);
    }
    ptx::fence_mbar_init();
    ptx::fence_proxy_async_smem();
  }
  if (warp == kProducerWarp && lane == 0) {
    ptx::prefetch_tmap(&tmap_q);
    ptx::prefetch_tmap(&tmap_x);
  }
  if (warp == kMmaWarp) {
    ptx::tmem_alloc(ptx::smem_u32(&bars->tmem_base), kTmemCols);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == kProducerWarp) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int w = blockIdx.x; w < n_tiles; w += gridDim.x) {
        // query block fastest: the CTAs running at once share centroid blocks in L2
        const int qb = w % QB, nb = w / QB;
        for (int kb = 0; kb < num_kb; ++kb) {
          ptx::mbar_wait(ptx::smem_u32(&bars->empty[stage]), phase ^ 1);
          const uint32_t fb = ptx::smem_u32(&bars->full[stage]);
          const uint32_t dst = ptx::smem_u32(ring + (size_t)stage * kStageBytes);
          ptx::mbar_arrive_expect_tx(fb, kStageBytes);
          ptx::tma_load_2d(dst, &tmap_q, fb, kb * kBK, qb * kBM);
          ptx::tma_load_2d(dst + kBoxBytes, &tmap_x, fb, kb * kBK, nb * kBN);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == kMmaWarp) {
    // ===================== MMA issuer (warp-convergent, elect.sync issues) =====================
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    const uint64_t desc0 = ptx::umma_desc_sw128(ptx::smem_u32(ring));
    for (int w = blockIdx.x; w < n_tiles; w += gridDim.x) {
      ptx::mbar_wait(ptx::smem_u32(&bars->tmem_empty[acc]), acc_phase ^ 1);
      ptx::tc_fence_after();
      const uint32_t d_tmem = tmem + (uint32_t)(acc * kBN);
      for (int kb = 0; kb < num_kb; ++kb) {
        ptx::mbar_wait(ptx::smem_u32(&bars->full[stage]), phase);
        ptx::tc_fence_after();
        const uint64_t adesc = desc0 + (uint64_t)(((size_t)stage * kStageBytes) >> 4);
        const uint64_t bdesc = adesc + (uint64_t)(kBoxBytes >> 4);
#pragma unroll
        for (int kk = 0; kk < kBK / 16; ++kk)
          ptx::mma_bf16_elect<1, false>(d_tmem, adesc + kk * 2, bdesc + kk * 2, kIdesc,
                                        (kb | kk) ? 1u : 0u);
        ptx::tc_commit_elect<1>(ptx::smem_u32(&bars->empty[stage]));
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
      ptx::tc_commit_elect<1>(ptx::smem_u32(&bars->tmem_full[acc]));
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    __syncwarp();
  } else {
    // ===================== epilogue: warp = (lane quadrant, column half) =====================
    const int quad = warp & 3;
    const int half = warp >> 2;
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    float* tb = xpose + warp * 1024;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int w = blockIdx.x; w < n_tiles; w += gridDim.x) {
      const int qb = w % QB, nb = w / QB;
      ptx::mbar_wait(ptx::smem_u32(&bars->tmem_full[acc]), acc_phase);
      ptx::tc_fence_after();
      uint32_t r0[32], r1[32];
      const uint32_t col = (uint32_t)(acc * kBN + half * 64);
      ptx::tmem_ld32(tmem + lane_addr + col, r0);
      ptx::tmem_ld32(tmem + lane_addr + col + 32, r1);
      ptx::tmem_wait_ld();
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&bars->tmem_empty[acc]));
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      const int64_t qbase = (int64_t)qb * kBM + quad * 32;   // lane l holds query qbase + l
      const int64_t c0 = (int64_t)nb * kBN + half * 64;
#pragma unroll
      for (int j = 0; j < 32; ++j) tb[lane * 32 + (j ^ lane)] = __uint_as_float(r0[j]);
      __syncwarp();
#pragma unroll 4
      for (int rr = 0; rr < 32; ++rr)
        if (qbase + rr < a.nq && c0 + lane < a.n_rows)
          a.out[(qbase + rr) * a.ldo + c0 + lane] = tb[rr * 32 + (lane ^ rr)];
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 32; ++j) tb[lane * 32 + (j ^ lane)] = __uint_as_float(r1[j]);
      __syncwarp();
#pragma unroll 4
      for (int rr = 0; rr < 32; ++rr)
        if (qbase + rr < a.nq && c0 + 32 + lane < a.n_rows)
          a.out[(qbase + rr) * a.ldo + c0 + 32 + lane] = tb[rr * 32 + (lane ^ rr)];
      __syncwarp();
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, kTmemCols);
  }
}

}  // namespace

bool score_gemm_applies(int d_pad) { return d_pad > 0 && d_pad % kBK == 0; }

cudaError_t launch_score_gemm(const CUtensorMap& tmap_q, const CUtensorMap& tmap_x,
                              const ScoreGemmArgs& a, int num_sms, cudaStream_t stream) {
  if (a.nq <= 0 || a.n_rows <= 0) return cudaSuccess;
  cudaError_t e = ensure_max_smem(reinterpret_cast<const void*>(score_gemm_kernel), kSmemBytes);
  if (e != cudaSuccess) return e;
  const int64_t tiles = ((a.nq + kBM - 1) / kBM) * ((a.n_rows + kBN - 1) / kBN);
  const int grid = (int)(tiles < num_sms ? tiles : num_sms);
  score_gemm_kernel<<<grid, kThreads, kSmemBytes, stream>>>(tmap_q, tmap_x, a);
  note_launch();
  return cudaGetLastError();
}

}  // namespace sa
