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
//   * MMA M side = queries.  Each CTA keeps its block of 128 bf16 query rows
//     resident for the whole scan: the first FS_KB_TMEM K-blocks in TMEM (A
//     operand from TMEM, "TS" form: lane m = query m, 2-packed bf16 columns),
//     any remaining K-blocks (d = 768: 4 of 12) in a 64 KB smem region read
//     with the SS form.  That keeps 256 TMEM columns free for two fp32
//     accumulator buffers at every d <= 768.
//   * MMA N side = 128 corpus rows per tile, TMA-staged from HBM into an smem
//     ring (128-byte swizzle, one box per 64-wide K step).
//   * CG = 2: a cluster of two CTAs is one cta_group::2 MMA of M = 256 (two
//     query blocks); each CTA stages half of the tile (64 rows) and the
//     leader issues the MMAs, so every SM receives half the corpus bytes per
//     FLOP of the CG = 1 layout (L2->SM traffic is the limiter).
//   * fp32 accumulators: two 128-column TMEM buffers, so the epilogue drains
//     tile t while the tensor core computes tile t+1.
//   * warps 0..7: epilogue -- thread = (query, column half),
//     each with a size-k min-heap of packed keys; per tile the fast path is
//     a 64-way max and one compare against the heap root; warp 8: TMA producer;
//     warp 9: TMEM alloc + MMA issuer (leader CTA); warp 10: bound warp.
//   * pruning bounds (exact: a candidate below a lower bound of the query's final
//     k-th score can never be returned; ties pass): q_hint = max of the published
//     heap roots, and the k-th largest of the heaps' BEST scores, computed by the
//     bound warp -- the heaps of a query cover disjoint rows, so k heaps' maxima are
//     k distinct candidates.  With ~100 heaps per query the latter tracks the k-th
//     best of every row scanned so far, so the per-tile slow path (a heap insert)
//     stays rare even while each heap is still filling.
//   * persistent grid: work item = (query group, corpus slice); partial
//     lists go to part[q][slice][half][k] and are merged by merge.cu.
//   (The IVF list scan, §8(a) a8, has its own kernel: ivf_scan.cu.)
#include <cuda_bf16.h>

#include "flat_scan.cuh"
#include "keys.cuh"
#include "launch.cuh"
#include "ptx.cuh"

namespace sa {

namespace {

constexpr int kBM = FS_BM;
constexpr int kBN = FS_BN;
constexpr int kBK = FS_BK;
constexpr int kEpiT = FS_EPI_THREADS;
constexpr uint32_t kTmemCols = 512;
constexpr int kASmemKb = FS_BM * FS_BK * 2;  // one 128-row x 64-col K-block of A in smem: 16 KB

constexpr int kKbPerStage = 2;
// tiles a unit may run ahead of units sharing its slice (C3: DRAM reads 51 -> 33 GB per batch
// vs 8; 2 gives 32.3 GB but no faster)
constexpr int kLockstepLag = 4;
constexpr int kLockstepSpinCap = 1 << 14;   // sleeps of one lockstep wait before pacing stops
constexpr int kBoundMaxK = 16;              // the bound warp serves k <= 16 (smem heaps)

template <int CG, bool F8 = false>
struct Cfg {
  static constexpr int kRowsPerCta = kBN / CG;              // corpus rows staged per CTA per tile
  static constexpr int kBoxBytes = kRowsPerCta * kBK * 2;  // one TMA box: rows x 64 bf16
  static constexpr int kStageBytes = kBoxBytes * kKbPerStage;
  static constexpr int kStages = CG == 1 ? 4 : 7;          // 128 / 112 KB of corpus in flight
  static constexpr uint32_t kIdesc =
      F8 ? ptx::umma_idesc_e4m3(kBM * CG, kBN) : ptx::umma_idesc_bf16(kBM * CG, kBN);
};

template <int CG>
struct __align__(8) SmemTail {
  uint64_t full[Cfg<CG>::kStages];
  uint64_t empty[Cfg<CG>::kStages];
  uint64_t tmem_full[2];
  uint64_t tmem_empty[2];
  uint64_t a_full;
  uint64_t a_tma;
  // bound warp -> epilogue: (query group << 32 | ordered k-th-of-maxima) per CTA query row
  uint64_t bound[FS_BM];
  int32_t bw_qkey;     // query group the epilogue is on (-1 none yet, -2 finished)
  int32_t tiles_done;  // tiles the epilogue (warp 0) has consumed
  uint32_t tmem_base;
};

__device__ __forceinline__ float heap_threshold(uint64_t root) {
  return root == 0ull ? -__int_as_float(0x7f800000) : key_score(root);
}

// Offer `key` to a size-k min-heap whose element i lives at h[i * kEpiT].
// Returns the new threshold score (score of the root).
__device__ __noinline__ float heap_offer(uint64_t* h, int k, uint64_t key) {
  if (key <= h[0]) return heap_threshold(h[0]);
  int i = 0;
  while (true) {
    int l = 2 * i + 1;
    if (l >= k) break;
    int r = l + 1;
    uint64_t hl = h[(size_t)l * kEpiT];
    int c = l;
    uint64_t hc = hl;
    if (r < k) {
      uint64_t hr = h[(size_t)r * kEpiT];
      if (hr < hl) { c = r; hc = hr; }
    }
    if (hc >= key) break;
    h[(size_t)i * kEpiT] = hc;
    i = c;
  }
  h[(size_t)i * kEpiT] = key;
  return heap_threshold(h[0]);
}

// One unit of work (query group, corpus slice); producer, MMA and epilogue decode it
// identically.  Pure arithmetic on the item index, so it is warp-uniform by construction.
struct WorkItem {
  int qkey;          // query group
  int s;             // corpus slice
  int32_t t0, t1;    // tile range
};

__device__ __forceinline__ WorkItem work_item(int w, const FlatScanArgs& a, int32_t T) {
  WorkItem wi;
  wi.qkey = w / a.S;
  wi.s = w % a.S;
  wi.t0 = (int32_t)((int64_t)wi.s * T / a.S);
  wi.t1 = (int32_t)((int64_t)(wi.s + 1) * T / a.S);
  return wi;
}

}  // namespace

template <int CG, bool F8, bool DUMP>
__global__ void __launch_bounds__(FS_THREADS, 1)
flat_scan_topk_kernel(const __grid_constant__ CUtensorMap tmap_x,
                      const __grid_constant__ CUtensorMap tmap_q, const FlatScanArgs a) {
  using C = Cfg<CG, F8>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* stage_base = smem;
  uint8_t* a_smem = smem + C::kStages * C::kStageBytes;  // [FS_KB_SMEM][128 rows][128 B], SW128
  uint64_t* heap_s = reinterpret_cast<uint64_t*>(a_smem + FS_KB_SMEM * kASmemKb);
  SmemTail<CG>* tail = reinterpret_cast<SmemTail<CG>*>(reinterpret_cast<uint8_t*>(heap_s) +
                                                       FS_KSMEM * kEpiT * sizeof(uint64_t));

  // Broadcast from lane 0 so the compiler knows role branches are warp-uniform (lets ptxas
  // keep the MMA operands in uniform registers instead of a per-MMA R2UR waterfall).
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0);
  // Role layout: warps 0..7 epilogue (warp % 4 = TMEM lane quadrant), warp 8 TMA producer,
  // warp 9 MMA issuer.  The warp scheduler prefers the highest warp id among eligible warps,
  // so the latency-critical single-thread producer/MMA loops win their sub-partition's issue
  // slot over the two epilogue warps that share it.
  constexpr int kProducerWarp = FS_EPI_WARPS;
  constexpr int kMmaWarp = FS_EPI_WARPS + 1;
  constexpr int kBoundWarp = FS_EPI_WARPS + 2;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = CG == 2 ? ptx::cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  const int unit = blockIdx.x / CG;        // CTA (CG=1) or CTA pair (CG=2)
  const int n_units = gridDim.x / CG;
  const int S = a.S;
  const int n_work = a.QP * S;
  const int32_t T = (int32_t)((a.n_rows + kBN - 1) / kBN);
  const int num_kb = a.d_pad / kBK;
  const int nacc = 2;
  const uint32_t a_col = (uint32_t)(nacc * kBN);          // A (TMEM part) after the accumulators
  const int kb_t = num_kb < FS_KB_TMEM ? num_kb : FS_KB_TMEM;  // K-blocks of A held in TMEM
  const int kb_s = num_kb - kb_t;                         // K-blocks of A held in smem

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::kStages; ++i) {
      ptx::mbar_init(ptx::smem_u32(&tail->full[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&tail->empty[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(ptx::smem_u32(&tail->tmem_full[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&tail->tmem_empty[i]), FS_EPI_WARPS * CG);
    }
    ptx::mbar_init(ptx::smem_u32(&tail->a_full), FS_EPI_WARPS * CG);
    ptx::mbar_init(ptx::smem_u32(&tail->a_tma), 1);
    tail->bw_qkey = -1;
    tail->tiles_done = 0;
    ptx::fence_mbar_init();
    ptx::fence_proxy_async_smem();
  }
  if (warp == kBoundWarp)
    for (int i = lane; i < FS_BM; i += 32) tail->bound[i] = 0ull;
  if (warp == kProducerWarp && lane == 0) {
    ptx::prefetch_tmap(&tmap_x);
    if (kb_s > 0) ptx::prefetch_tmap(&tmap_q);
  }
  if (warp == kMmaWarp) {
    if (CG == 2) {
      ptx::tmem_alloc_2sm(ptx::smem_u32(&tail->tmem_base), kTmemCols);
      ptx::tmem_relinquish_2sm();
    } else {
      ptx::tmem_alloc(ptx::smem_u32(&tail->tmem_base), kTmemCols);
      ptx::tmem_relinquish();
    }
  }
  ptx::tc_fence_before();
  if (CG == 2) ptx::cluster_sync(); else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tail->tmem_base;

  const int n_sl = (num_kb + kKbPerStage - 1) / kKbPerStage;  // ring stages per tile
  if (warp == kProducerWarp) {
    // ===================== TMA producer (both CTAs) =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t full0 = ptx::smem_u32(&tail->full[0]);
      // Soft lockstep (flat mode, one work item per unit, several query groups): the units
      // that scan the same corpus slice for different query groups publish their progress
      // and none runs more than kLockstepLag tiles ahead of another, so the slice is read
      // from HBM once and served from L2 to the other groups (37 slices x lag x 192 KB
      // stays well inside the 126 MB L2).  Only the pair leader's producer paces.
      // Pacing is only an L2 optimisation, and nothing guarantees the peer units are resident
      // (a plain cluster launch; other streams may hold SMs): a wait that lasts longer than
      // kLockstepSpinCap sleeps (>= ~4 ms, tiles take ~µs) turns pacing off for this unit,
      // so a unit never waits on a peer that has not been scheduled.
      bool lockstep = a.progress != nullptr && leader;
      const bool publish = lockstep;
      const int lag = a.lockstep_lag > 0 ? a.lockstep_lag : kLockstepLag;
      for (int w = unit; w < n_work; w += n_units) {
        const WorkItem wi = work_item(w, a, T);
        for (int32_t t = wi.t0; t < wi.t1; ++t) {
          if (publish) {
            const int32_t done = t - wi.t0;
            if ((done & 3) == 0) {
              ptx::st_release_gpu(a.progress + unit, done);   // published even if not pacing
              for (int g = 0; g < a.QP && lockstep; ++g) {
                const int p = g * S + wi.s;
                if (p == unit) continue;
                int spins = 0;
                while (ptx::ld_acquire_gpu(a.progress + p) < done - lag) {
                  if (++spins > kLockstepSpinCap) {
                    lockstep = false;
                    break;
                  }
                  __nanosleep(256);
                }
              }
            }
          }
          const int32_t row = t * kBN + (int32_t)rank * C::kRowsPerCta;
          for (int sl = 0; sl < n_sl; ++sl) {
            const int kb0 = sl * kKbPerStage;
            const int nkb = num_kb - kb0 < kKbPerStage ? num_kb - kb0 : kKbPerStage;
            ptx::mbar_wait(ptx::smem_u32(&tail->empty[stage]), phase ^ 1);
            const uint32_t dst = ptx::smem_u32(stage_base + stage * C::kStageBytes);
            const uint32_t fb = full0 + stage * 8;
            if (CG == 1) {
              ptx::mbar_arrive_expect_tx(fb, nkb * C::kBoxBytes);
              for (int j = 0; j < nkb; ++j)
                ptx::tma_load_2d(dst + j * C::kBoxBytes, &tmap_x, fb, (kb0 + j) * kBK, row);
            } else {
              if (leader) ptx::mbar_arrive_expect_tx(fb, 2 * nkb * C::kBoxBytes);
              const uint32_t fbl = ptx::mapa(fb, 0);
              for (int j = 0; j < nkb; ++j)
                ptx::tma_load_2d_2sm(dst + j * C::kBoxBytes, &tmap_x, fbl, (kb0 + j) * kBK, row);
            }
            if (++stage == C::kStages) { stage = 0; phase ^= 1; }
          }
        }
      }
      // Drain: wait until every stage has been released by its final MMA commit, so no
      // tcgen05.commit arrival can target this CTA's smem after it exits.
      for (int i = 0; i < C::kStages; ++i) {
        ptx::mbar_wait(ptx::smem_u32(&tail->empty[stage]), phase ^ 1);
        if (++stage == C::kStages) { stage = 0; phase ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp == kMmaWarp) {
    // ===================== MMA issuer (leader CTA; warp-convergent, elect.sync issues) ======
    if (leader) {
      const int n_work_u = __shfl_sync(0xffffffffu, n_work, 0);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int cur_qp = -1;
      uint32_t a_phase = 0;
      const uint64_t desc0 = ptx::umma_desc_sw128(ptx::smem_u32(stage_base));
      const uint64_t adesc0 = ptx::umma_desc_sw128(ptx::smem_u32(a_smem));
      const uint32_t full0 = ptx::smem_u32(&tail->full[0]);
      const uint32_t empty0 = ptx::smem_u32(&tail->empty[0]);
      for (int w = unit; w < n_work_u; w += n_units) {
        const WorkItem wi = work_item(w, a, T);
        if (wi.qkey != cur_qp) {
          ptx::mbar_wait(ptx::smem_u32(&tail->a_full), a_phase);
          a_phase ^= 1;
          cur_qp = wi.qkey;
          ptx::tc_fence_after();
        }
        for (int32_t t = wi.t0; t < wi.t1; ++t) {
          ptx::mbar_wait(ptx::smem_u32(&tail->tmem_empty[acc]), acc_phase ^ 1);
          ptx::tc_fence_after();
          const uint32_t d_tmem = tmem + (uint32_t)(acc * kBN);
          for (int sl = 0; sl < n_sl; ++sl) {
            ptx::mbar_wait(full0 + stage * 8, phase);
            ptx::tc_fence_after();
            const uint64_t sdesc = desc0 + (uint64_t)((stage * C::kStageBytes) >> 4);
#pragma unroll
            for (int j = 0; j < kKbPerStage; ++j) {
              const int kb = sl * kKbPerStage + j;
              if (kb < num_kb) {
                const uint64_t bdesc = sdesc + (uint64_t)((j * C::kBoxBytes) >> 4);
                if (kb < kb_t) {
                  const uint32_t a_tmem = tmem + a_col + (uint32_t)(kb * (kBK / 2));
#pragma unroll
                  for (int kk = 0; kk < kBK / 16; ++kk) {
                    if constexpr (F8)
                      ptx::mma_e4m3_elect<CG, true>(d_tmem, a_tmem + kk * 8, bdesc + kk * 2,
                                                    C::kIdesc, (kb | kk) ? 1u : 0u);
                    else
                      ptx::mma_bf16_elect<CG, true>(d_tmem, a_tmem + kk * 8, bdesc + kk * 2,
                                                    C::kIdesc, (kb | kk) ? 1u : 0u);
                  }
                } else {
                  const uint64_t adesc = adesc0 + (uint64_t)(((kb - kb_t) * kASmemKb) >> 4);
#pragma unroll
                  for (int kk = 0; kk < kBK / 16; ++kk) {
                    if constexpr (F8)
                      ptx::mma_e4m3_elect<CG, false>(d_tmem, adesc + kk * 2, bdesc + kk * 2,
                                                     C::kIdesc, 1u);
                    else
                      ptx::mma_bf16_elect<CG, false>(d_tmem, adesc + kk * 2, bdesc + kk * 2,
                                                     C::kIdesc, 1u);
                  }
                }
              }
            }
            ptx::tc_commit_elect<CG>(empty0 + stage * 8);
            if (++stage == C::kStages) { stage = 0; phase ^= 1; }
          }
          ptx::tc_commit_elect<CG>(ptx::smem_u32(&tail->tmem_full[acc]));
          if (++acc == nacc) { acc = 0; acc_phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == kBoundWarp) {
    // ===================== bound warp: k-th largest of the heaps' best scores ================
    // Lane i refreshes rows i, i+32, ... of the CTA's current query block: it reads the
    // query's q_max row (the best score of each of its heaps, published by the epilogue) and
    // keeps the k largest in a sorted register list; the k-th is a lower bound of the query's
    // final k-th score (k distinct rows).  Rounds run after the epilogue has processed 1, 2,
    // 4, 8, ... tiles of the current query block: the maxima move fast early and rarely
    // later, and each round reads every query's row from L2 (which the corpus stream needs).
    const int k = a.k;
    if (!DUMP && a.q_max != nullptr && k <= kBoundMaxK) {
      const int H = a.q_max_stride;
      int cur = -1, next_at = 0;
      while (true) {
        const int qkey = atomicAdd(&tail->bw_qkey, 0);   // shared flags: atomics (no data race)
        if (qkey == -2) break;
        const int done = atomicAdd(&tail->tiles_done, 0);
        if (qkey != cur) {
          cur = qkey;
          next_at = done + 1;
        }
        if (qkey >= 0 && done >= next_at) {
          next_at = done + (done > 1 ? done : 1);
#ifdef SA_TUNING_BUILD
          if (a.counters && lane == 0) atomicAdd(a.counters + 2, 1ull);
#endif
          for (int i = lane; i < FS_BM; i += 32) {
            const int64_t q = ((int64_t)qkey * CG + rank) * kBM + i;
            if (q >= a.nq) break;
            // descending top-k list in registers (static indices only), kth = its k-th entry
            uint32_t t[kBoundMaxK];
#pragma unroll
            for (int j = 0; j < kBoundMaxK; ++j) t[j] = 0u;
            uint32_t kth = 0u;
            // the row (stride a multiple of 4 words) in batches of 32 values: all 8 vector
            // loads of a batch are issued before any is used (one L2 round trip per batch)
            const uint4* row = reinterpret_cast<const uint4*>(a.q_max + q * H);
            for (int h0 = 0; h0 < H / 4; h0 += 8) {
              uint4 vb[8];
#pragma unroll
              for (int u = 0; u < 8; ++u)
                vb[u] = h0 + u < H / 4 ? ptx::ld_relaxed_gpu_v4(row + h0 + u)
                                       : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
              for (int u = 0; u < 32; ++u) {
                const uint4& w4 = vb[u >> 2];
                uint32_t v = (u & 3) == 0 ? w4.x : (u & 3) == 1 ? w4.y : (u & 3) == 2 ? w4.z : w4.w;
                if (v <= kth) continue;
#pragma unroll
                for (int j = 0; j < kBoundMaxK; ++j) {   // insert into the descending list
                  const uint32_t hi = v > t[j] ? v : t[j];
                  v = v > t[j] ? t[j] : v;
                  t[j] = hi;
                }
                // kth = t[k - 1] = the smallest of the first k entries (a min, not an index:
                // t stays in registers)
                kth = 0xFFFFFFFFu;
#pragma unroll
                for (int j = 0; j < kBoundMaxK; ++j)
                  kth = min(kth, t[j] | (j < k ? 0u : 0xFFFFFFFFu));
              }
            }
            if (kth != 0u)
              atomicExch(reinterpret_cast<unsigned long long*>(&tail->bound[i]),
                         ((unsigned long long)(uint32_t)qkey << 32) | kth);
            if (atomicAdd(&tail->bw_qkey, 0) != qkey) break;
          }
        }
        __nanosleep(500);
      }
    }
    __syncwarp();
  } else {
    // ===================== epilogue: 8 warps, thread = (query, column half) =====================
    const int ew = warp;                     // epilogue warp 0..7
    const int quad = warp & 3;               // TMEM lane quadrant this warp may access
    const int half = ew >> 2;                // accumulator columns [half*64, half*64+64)
    const int rib = quad * 32 + lane;        // query row within this CTA's block
    const int et = ew * 32 + lane;           // epilogue thread index 0..255
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    const int k = a.k;
    // Heaps live in smem for k <= FS_KSMEM (insertions are latency-critical: the epilogue
    // must finish a tile within one MMA tile time), for k <= FS_KSMEM_BIG when the whole A
    // operand sits in TMEM (the heaps then start at the unused smem A region, which directly
    // precedes heap_s: 64 + 32 KB = 48 x 256 keys), else in global scratch.
    static_assert(FS_KB_SMEM * kASmemKb + FS_KSMEM * kEpiT * 8 == FS_KSMEM_BIG * kEpiT * 8,
                  "smem A region + heap region must hold FS_KSMEM_BIG heaps");
    const bool heap_smem = k <= (kb_s == 0 ? FS_KSMEM_BIG : FS_KSMEM);
    uint64_t* heap = heap_smem ? ((kb_s == 0 ? reinterpret_cast<uint64_t*>(a_smem) : heap_s) + et)
                               : (a.heap_g + (size_t)blockIdx.x * k * kEpiT + et);
    if constexpr (!DUMP)
      for (int i = 0; i < k; ++i) heap[(size_t)i * kEpiT] = 0ull;
    float thr = heap_threshold(0ull);
#ifdef SA_TUNING_BUILD
    uint32_t c_pass = 0, c_ins = 0;
#define SA_FS_COUNT(x) ++x
#else
#define SA_FS_COUNT(x) (void)0
#endif
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t a_tma_phase = 0;
    const uint32_t a_full_leader = CG == 2 ? ptx::mapa(ptx::smem_u32(&tail->a_full), 0)
                                           : ptx::smem_u32(&tail->a_full);
    const uint32_t tmem_empty0 = CG == 2 ? ptx::mapa(ptx::smem_u32(&tail->tmem_empty[0]), 0)
                                         : ptx::smem_u32(&tail->tmem_empty[0]);
    // Stage query group `qkey`'s block into the A operand (TMEM K-blocks + smem K-blocks) and
    // arrive on a_full.  Callers guarantee every MMA that read the previous block has
    // completed (they consumed that block's last tmem_full).
    auto stage_a = [&](int qkey) __attribute__((always_inline)) {
      if (ew == 0 && lane == 0) atomicExch(&tail->bw_qkey, qkey);
      const int64_t q_row = ((int64_t)qkey * CG + rank) * kBM + rib;
      const bool q_ok = q_row < a.nq;
      const bool tma_thread = ew == 0 && lane == 0 && kb_s > 0;
      if (tma_thread) {
        // K-blocks [kb_t, num_kb) of this CTA's 128 query rows -> smem (SS operand)
        const uint32_t bar = ptx::smem_u32(&tail->a_tma);
        ptx::mbar_arrive_expect_tx(bar, (uint32_t)(kb_s * kASmemKb));
        const int32_t qrow0 = (int32_t)(((int64_t)qkey * CG + rank) * kBM);
        for (int j = 0; j < kb_s; ++j)
          ptx::tma_load_2d(ptx::smem_u32(a_smem + j * kASmemKb), &tmap_q, bar,
                           (kb_t + j) * kBK, qrow0);
      }
      // Rows of absent queries are left as they are: MMA output rows are independent and the
      // epilogue never reads the rows of invalid lanes, so a warp with no valid lane skips.
      if (half == 0 && __any_sync(0xffffffffu, q_ok)) {
        const uint4* src = reinterpret_cast<const uint4*>(a.Q + (size_t)q_row * a.d_pad);
        for (int c = 0; c < kb_t; ++c) {
          uint32_t r[32];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            uint4 v = q_ok ? __ldg(src + c * 8 + i) : make_uint4(0, 0, 0, 0);
            r[4 * i + 0] = v.x; r[4 * i + 1] = v.y; r[4 * i + 2] = v.z; r[4 * i + 3] = v.w;
          }
          ptx::tmem_st32(tmem + lane_addr + a_col + c * 32, r);
        }
        ptx::tmem_wait_st();
      }
      if (tma_thread) {
        ptx::mbar_wait(ptx::smem_u32(&tail->a_tma), a_tma_phase);
        a_tma_phase ^= 1;
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (CG == 2 && !leader) ptx::mbar_arrive_cluster(a_full_leader);
        else ptx::mbar_arrive(ptx::smem_u32(&tail->a_full));
      }
    };

    if (unit < n_work) stage_a(work_item(unit, a, T).qkey);
    for (int w = unit; w < n_work; w += n_units) {
      const WorkItem wi = work_item(w, a, T);
      const int wn = w + n_units;
      const bool has_next = wn < n_work;
      // the next item's query group (decoded lazily, at this item's last tile)
      const int64_t q = ((int64_t)wi.qkey * CG + rank) * kBM + rib;
      const bool valid = q < a.nq;
      if (wi.t1 <= wi.t0 && has_next) {
        const int nq_key = work_item(wn, a, T).qkey;
        if (nq_key != wi.qkey) stage_a(nq_key);
      }
      // Exact pruning bound shared by all heaps of a query (all corpus slices / column
      // halves): q_hint[q] = max over published heap roots.  Each root is the k-th best score
      // of a subset of q's candidates, so q's final k-th score is >= q_hint[q] and smaller
      // scores can never be returned (ties pass: s >= thr).  Roots are published as they rise
      // and the bound is re-read every 4 tiles, so every heap prunes with the best threshold
      // any heap of the query has reached.
      float hint = heap_threshold(0ull);
      uint32_t published = 0u;
      if (valid && a.q_hint) {
        const uint32_t h = __ldcg(a.q_hint + q);
        if (h != 0u) hint = float_from_ordered(h);
      }
      thr = fmaxf(thr, hint);
      uint32_t h_next = 0u;   // the bound, loaded one tile before it is used (L2 latency hidden)
      // this heap's best score so far (ordered), published to q_max for the bound warp
      uint32_t best_o = 0u;
      uint32_t* const my_max =
          a.q_max ? a.q_max + q * a.q_max_stride + wi.s * FS_LISTS_PER_ITEM + half : nullptr;
      for (int32_t t = wi.t0; t < wi.t1; ++t) {
        if (valid && ((t - wi.t0) & 3) == 3) {
          if (a.q_hint && h_next != 0u) hint = fmaxf(hint, float_from_ordered(h_next));
          const uint64_t b = atomicAdd(reinterpret_cast<unsigned long long*>(&tail->bound[rib]), 0ull);
          if ((uint32_t)(b >> 32) == (uint32_t)wi.qkey && (uint32_t)b != 0u)
            hint = fmaxf(hint, float_from_ordered((uint32_t)b));
          thr = fmaxf(thr, hint);
        }
        if (valid && a.q_hint && ((t - wi.t0) & 3) == 2) h_next = __ldcg(a.q_hint + q);
        ptx::mbar_wait(ptx::smem_u32(&tail->tmem_full[acc]), acc_phase);
        ptx::tc_fence_after();
        uint32_t r0[32], r1[32];
        const uint32_t col = (uint32_t)(acc * kBN + half * 64);
        if (a.experiment != 2) {
          ptx::tmem_ld32(tmem + lane_addr + col, r0);
          ptx::tmem_ld32(tmem + lane_addr + col + 32, r1);
          ptx::tmem_wait_ld();
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (CG == 2 && !leader) ptx::mbar_arrive_cluster(tmem_empty0 + acc * 8);
          else ptx::mbar_arrive(ptx::smem_u32(&tail->tmem_empty[acc]));
        }
        if (++acc == nacc) { acc = 0; acc_phase ^= 1; }
        if (ew == 0 && lane == 0) {
          atomicAdd(&tail->tiles_done, 1);
        }
        // The last accumulator of this item is in registers, so every MMA that read this
        // item's A operand has completed: stage the next item's queries now, before the
        // score processing, so the tensor core restarts as early as possible.
        if (t == wi.t1 - 1 && has_next) {
          const int nq_key = work_item(wn, a, T).qkey;
          if (nq_key != wi.qkey) stage_a(nq_key);
        }
        const int32_t row0 = t * kBN + half * 64;
        if constexpr (DUMP) {
          // Score dump (IVF probe, graph entry points, tests): the warp's 32 queries x 64
          // columns go through a 4 KB smem tile per 32 columns (XOR-swizzled, conflict-free)
          // so every store instruction writes one query's 32 consecutive scores (128 B)
          // instead of 32 scattered words.  The lanes hold consecutive queries.  heap_s is
          // free in this mode (no heaps).
          if (a.experiment == 0 && __any_sync(0xffffffffu, valid)) {
            float* tb = reinterpret_cast<float*>(heap_s) + ew * 1024;
            const int64_t qbase = q - lane;
#pragma unroll
            for (int j = 0; j < 32; ++j) tb[lane * 32 + (j ^ lane)] = __uint_as_float(r0[j]);
            __syncwarp();
#pragma unroll 4
            for (int rr = 0; rr < 32; ++rr)
              if (qbase + rr < a.nq && row0 + lane < a.n_rows)
                a.dbg[(qbase + rr) * a.n_rows + row0 + lane] = tb[rr * 32 + (lane ^ rr)];
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 32; ++j) tb[lane * 32 + (j ^ lane)] = __uint_as_float(r1[j]);
            __syncwarp();
#pragma unroll 4
            for (int rr = 0; rr < 32; ++rr)
              if (qbase + rr < a.nq && row0 + 32 + lane < a.n_rows)
                a.dbg[(qbase + rr) * a.n_rows + row0 + 32 + lane] = tb[rr * 32 + (lane ^ rr)];
            __syncwarp();
          }
          continue;
        }
        if (!valid || (a.experiment != 0 && a.experiment != 3)) continue;

        // maxima of the 4 groups of 16 columns, then of the tile: a passing tile visits only
        // the groups whose maximum passes (usually one), not all 64 columns
        float gm[4];
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const uint32_t* r = g < 2 ? r0 : r1;
          const int b = (g & 1) * 16;
          float x = fmaxf(__uint_as_float(r[b]), __uint_as_float(r[b + 1]));
#pragma unroll
          for (int j = 2; j < 16; j += 2)
            x = fmaxf(x, fmaxf(__uint_as_float(r[b + j]), __uint_as_float(r[b + j + 1])));
          gm[g] = x;
        }
        const float mt = fmaxf(fmaxf(gm[0], gm[1]), fmaxf(gm[2], gm[3]));
        if (a.experiment == 3) {   // timing experiment: the 64-way max only, no insertion
          if (mt == 1234.5f) a.part[0] = 0ull;
          continue;
        }
        if (mt >= thr) {
          SA_FS_COUNT(c_pass);
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            if (gm[g] < thr) continue;
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) {
              const int j = g * 16 + jj;
              const float s = __uint_as_float(j < 32 ? r0[j] : r1[j - 32]);
              if (s >= thr) {
                const int32_t row = row0 + j;
                if (row < a.n_rows) {
                  const uint32_t id =
                      a.id_base + (a.row_ids ? (uint32_t)a.row_ids[row] : (uint32_t)row);
                  const uint64_t key = make_key(s, id);
                  SA_FS_COUNT(c_ins);
                  thr = fmaxf(heap_offer(heap, k, key), hint);
                  const uint32_t o = (uint32_t)(key >> 32);
                  if (my_max && o > best_o) {
                    best_o = o;
                    ptx::st_relaxed_gpu_u32(my_max, o);
                  }
                }
              }
            }
          }
          if (a.q_hint) {
            const uint64_t root = heap[0];
            const uint32_t o = (uint32_t)(root >> 32);
            if (root != 0ull && o > published) {
              atomicMax(a.q_hint + q, o);
              published = o;
            }
          }
        }
      }
      if constexpr (!DUMP) {
        // flush this work item's partial list and reset the heap
        if (valid) {
          uint64_t* dst = a.part + (((size_t)q * S + wi.s) * FS_LISTS_PER_ITEM + half) * k;
          for (int i = 0; i < k; ++i) dst[i] = heap[(size_t)i * kEpiT];
          const uint64_t root = heap[0];
          if (a.q_hint && root != 0ull) atomicMax(a.q_hint + q, (uint32_t)(root >> 32));
        }
        for (int i = 0; i < k; ++i) heap[(size_t)i * kEpiT] = 0ull;
        thr = heap_threshold(0ull);
      }
    }
    if (ew == 0 && lane == 0) atomicExch(&tail->bw_qkey, -2);
#ifdef SA_TUNING_BUILD
    if (a.counters) {
      atomicAdd(a.counters + 0, (unsigned long long)c_pass);
      atomicAdd(a.counters + 1, (unsigned long long)c_ins);
    }
#endif
  }

  ptx::tc_fence_before();
  if (CG == 2) ptx::cluster_sync(); else __syncthreads();
  if (warp == kMmaWarp) {
    ptx::tc_fence_after();
    if (CG == 2) ptx::tmem_dealloc_2sm(tmem, kTmemCols);
    else ptx::tmem_dealloc(tmem, kTmemCols);
  }
}

size_t flat_scan_smem_bytes(int cta_group) {
  const size_t fixed = (size_t)FS_KB_SMEM * kASmemKb + (size_t)FS_KSMEM * kEpiT * sizeof(uint64_t);
  if (cta_group == 2)
    return 1024 + (size_t)Cfg<2>::kStages * Cfg<2>::kStageBytes + fixed + sizeof(SmemTail<2>);
  return 1024 + (size_t)Cfg<1>::kStages * Cfg<1>::kStageBytes + fixed + sizeof(SmemTail<1>);
}

cudaError_t launch_flat_scan(const CUtensorMap& tmap, const CUtensorMap& tmap_q, const FlatScanArgs& a, int cta_group,
                             int grid, cudaStream_t stream) {
  const size_t smem = flat_scan_smem_bytes(cta_group);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(FS_THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)cta_group;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = ensure_max_smem(reinterpret_cast<const void*>(kern), smem);
    if (e != cudaSuccess) return e;
    e = cudaLaunchKernelEx(&cfg, kern, tmap, tmap_q, a);
    note_launch();
    return e;
  };
  // instantiations: (CG, F8, DUMP); the score dump (FS_MODE_DEBUG) has its own, heap-free one
  if (a.mode == FS_MODE_DEBUG) {
    if (a.fp8) return cudaErrorInvalidValue;
    return cta_group == 2 ? go(flat_scan_topk_kernel<2, false, true>)
                          : go(flat_scan_topk_kernel<1, false, true>);
  }
  if (a.fp8) {
    return cta_group == 2 ? go(flat_scan_topk_kernel<2, true, false>)
                          : go(flat_scan_topk_kernel<1, true, false>);
  }
  return cta_group == 2 ? go(flat_scan_topk_kernel<2, false, false>)
                        : go(flat_scan_topk_kernel<1, false, false>);
}

}  // namespace sa
