// ivf_scan.cu -- list-major IVF scan with fused partial top-k (
// DESIGN.md §4.2).
//
// A work item is (inverted list l, block of <= 32 queries that probe l, row chunk of l).
// The list rows are the MMA's M side: 128-row tiles stream HBM -> smem through a TMA ring
// (128B swizzle) and are the A operand; the item's probing queries are the N side (B
// operand, N = 16 or 32), gathered from the staged query batch into a double-buffered smem
// block by dedicated gather warps one item ahead, so neither the tensor core nor the epilogue
// waits for a query gather.  Scores land in TMEM as [128 list rows x N queries] fp32.
//
// Epilogue: 8 warps; warp w reads TMEM lane quadrant w % 4 (32 list rows) and columns
// [16 * (w / 4), +16) (16 probers).  Per tile and column a warp compares its 32 scores with
// the prober's threshold, ballots the survivors and hands them one by one (shuffle) to the
// lane that owns that column's heap -- a size-k min-heap per (warp, prober).  At the end of
// the item every heap is written to the prober's output slot (4 partial lists per (query,
// probe, chunk): one per lane quadrant) and merged by merge.cu.  The pruning threshold of a
// prober is max(its heap root, q_hint[q]) -- q_hint is the max of the published roots of all
// heaps of the query, a lower bound of its final k-th score (exact: ties pass, s >= thr).
//
// Roles: warps 0..7 epilogue, warp 8 TMA producer (claims items from a global counter one
// item ahead and publishes them decoded, so no consumer touches item metadata in global
// memory), warp 9 MMA issuer (warp-convergent, elect.sync), warps 10..13 prober gather (the
// item's query rows into the double-buffered B operand, released by an MMA commit).
#include <cuda_bf16.h>

#include "ivf_scan.cuh"
#include "keys.cuh"
#include "launch.cuh"
#include "ptx.cuh"

namespace sa {

namespace {

constexpr int kBM = IVS_BM;
constexpr int kBK = 64;
constexpr int kNQ = IVS_NQ;
constexpr int kEpiWarps = 8;
constexpr int kGatherWarps = 4;
constexpr int kProducerWarp = kEpiWarps;
constexpr int kMmaWarp = kEpiWarps + 1;
constexpr int kGather0 = kEpiWarps + 2;               // first prober-gather warp
constexpr int kThreads = 32 * (kGather0 + kGatherWarps);
constexpr int kKbPerStage = 2;
constexpr int kBoxBytes = kBM * kBK * 2;              // one 128-row x 64-col box: 16 KB
constexpr int kStageBytes = kBoxBytes * kKbPerStage;  // 32 KB
constexpr int kStages = 3;
constexpr int kMaxKb = 12;                            // d_pad <= 768
constexpr int kBKbBytes = kNQ * kBK * 2;              // one K-block of a prober block: 4 KB
constexpr int kBBytes = kMaxKb * kBKbBytes;           // 48 KB per prober block buffer
constexpr int kNAcc = 4;
constexpr uint32_t kTmemCols = kNAcc * kNQ;           // 128
constexpr int kTailRows = 32;
constexpr int kItemQ = 4;

struct __align__(8) Tail {
  uint64_t full[kStages];
  uint64_t empty[kStages];
  uint64_t acc_full[kNAcc];
  uint64_t acc_empty[kNAcc];
  uint64_t b_full[2];
  uint64_t b_empty[2];
  uint64_t iq_full[kItemQ];
  uint64_t iq_empty[kItemQ];
  int32_t iq[kItemQ][6];   // decoded items: w (-1 = no more work), e0, chunk, cnt, r0, r1
  uint32_t tmem_base;
};

struct Item {
  int32_t e0, chunk, cnt;  // probers lq_ent[e0, e0 + cnt), chunk index
  int32_t r0, r1;          // stored rows [r0, r1)
  int32_t ntiles;
};

__device__ __forceinline__ Item decode_raw(int4 it, const IvfScanArgs& a) {
  const int32_t lo = (int32_t)a.list_off[it.x], hi = (int32_t)a.list_off[it.x + 1];
  Item r;
  r.e0 = it.y;
  r.chunk = it.z;
  r.cnt = it.w;
  r.r0 = lo + it.z * a.chunk_rows;
  r.r1 = hi < r.r0 + a.chunk_rows ? hi : r.r0 + a.chunk_rows;
  r.ntiles = (r.r1 - r.r0 + kBM - 1) / kBM;
  return r;
}

// Stage geometry of a tile with `left` stored rows (<= kBM used): a full tile stages two
// 128-row K-blocks (16 KB each) per ring slot; a chunk tail of nbox 32-row boxes packs its
// K-blocks at nbox * 4 KB spacing, 8 / 4 / 2 of them per slot for nbox = 1 / 2 / 3, so a short
// list costs few ring round trips.  The MMA still reads 128 rows from each K-block's base:
// rows past the tail are other K-blocks' (or other slots') bytes, masked by r1 in the epilogue.
struct TileGeom {
  int kbb;   // bytes of one K-block in the slot (1 KB aligned: the SW128 atom)
  int kps;   // K-blocks per slot
  int nbox;  // 32-row boxes per K-block (4 = one full 128-row box)
};
__device__ __forceinline__ TileGeom tile_geom(int32_t left) {
  TileGeom g;
  if (left >= kBM) {
    g.nbox = 4;
    g.kbb = kBoxBytes;
    g.kps = kKbPerStage;
  } else {
    g.nbox = (left + kTailRows - 1) / kTailRows;
    g.kbb = g.nbox * kTailRows * kBK * 2;
    g.kps = g.nbox == 1 ? 8 : g.nbox == 2 ? 4 : 2;
  }
  return g;
}

__device__ __forceinline__ float threshold_of(uint64_t root) {
  return root == 0ull ? -__int_as_float(0x7f800000) : key_score(root);
}

// Offer `key` to a size-k min-heap whose element i lives at h[i * IVS_HEAPS]; returns the
// score of the new root (-inf while the heap is not full).
__device__ __noinline__ float heap_push(uint64_t* h, int k, uint64_t key) {
  if (key <= h[0]) return threshold_of(h[0]);
  int i = 0;
  while (true) {
    const int l = 2 * i + 1;
    if (l >= k) break;
    const int r = l + 1;
    const uint64_t hl = h[(size_t)l * IVS_HEAPS];
    int c = l;
    uint64_t hc = hl;
    if (r < k) {
      const uint64_t hr = h[(size_t)r * IVS_HEAPS];
      if (hr < hl) { c = r; hc = hr; }
    }
    if (hc >= key) break;
    h[(size_t)i * IVS_HEAPS] = hc;
    i = c;
  }
  h[(size_t)i * IVS_HEAPS] = key;
  return threshold_of(h[0]);
}

}  // namespace

template <bool F8>
__global__ void __launch_bounds__(kThreads, 1)
ivf_scan_kernel(const __grid_constant__ CUtensorMap tmap_x,
                const __grid_constant__ CUtensorMap tmap_tail, const IvfScanArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* ring = smem;
  uint8_t* bbuf = ring + kStages * kStageBytes;  // [2][kMaxKb][32 rows][128 B], SW128
  uint64_t* heap_s = reinterpret_cast<uint64_t*>(bbuf + 2 * kBBytes);
  Tail* tail = reinterpret_cast<Tail*>(reinterpret_cast<uint8_t*>(heap_s) +
                                       IVS_KSMEM * IVS_HEAPS * sizeof(uint64_t));

  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x / 32), 0);
  const int lane = threadIdx.x % 32;
  const int n_work = *a.n_items;
  const int num_kb = a.d_pad / kBK;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      ptx::mbar_init(ptx::smem_u32(&tail->full[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&tail->empty[i]), 1);
    }
    for (int i = 0; i < kNAcc; ++i) {
      ptx::mbar_init(ptx::smem_u32(&tail->acc_full[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&tail->acc_empty[i]), kEpiWarps);
    }
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(ptx::smem_u32(&tail->b_full[i]), kGatherWarps);
      ptx::mbar_init(ptx::smem_u32(&tail->b_empty[i]), 1);
    }
    for (int i = 0; i < kItemQ; ++i) {
      ptx::mbar_init(ptx::smem_u32(&tail->iq_full[i]), 1);
      ptx::mbar_init(ptx::smem_u32(&tail->iq_empty[i]), 1 + kEpiWarps + kGatherWarps);
    }
    ptx::fence_mbar_init();
    ptx::fence_proxy_async_smem();
  }
  if (warp == kProducerWarp && lane == 0) {
    ptx::prefetch_tmap(&tmap_x);
    ptx::prefetch_tmap(&tmap_tail);
  }
  if (warp == kMmaWarp) {
    ptx::tmem_alloc(ptx::smem_u32(&tail->tmem_base), kTmemCols);
    ptx::tmem_relinquish();
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = tail->tmem_base;

  // consumer side of the item queue: item #i of this CTA (-1 = no more work)
  // consumer side of the item queue: item #i of this CTA (w = -1: no more work).  The fields
  // are ordered by the mbarriers; they are accessed with atomics only so that racecheck,
  // which does not model mbarrier ordering, sees no plain conflicting accesses.
  auto take_item = [&](int i, Item& it) __attribute__((always_inline)) -> int {
    const int slot = i % kItemQ;
    ptx::mbar_wait(ptx::smem_u32(&tail->iq_full[slot]), (uint32_t)((i / kItemQ) & 1));
    int v = 0;
    if (lane < 6) v = atomicAdd(&tail->iq[slot][lane], 0);
    __syncwarp();
    if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&tail->iq_empty[slot]));
    const int w = __shfl_sync(0xffffffffu, v, 0);
    it.e0 = __shfl_sync(0xffffffffu, v, 1);
    it.chunk = __shfl_sync(0xffffffffu, v, 2);
    it.cnt = __shfl_sync(0xffffffffu, v, 3);
    it.r0 = __shfl_sync(0xffffffffu, v, 4);
    it.r1 = __shfl_sync(0xffffffffu, v, 5);
    it.ntiles = (it.r1 - it.r0 + kBM - 1) / kBM;
    return w;
  };

  if (warp == kProducerWarp) {
    // ===================== item fetch + TMA producer =====================
    if (lane == 0) {
      // Items are claimed from the global counter one item ahead and decoded (items[], then
      // list_off[]) while the current item's first slot is in flight, so neither the atomic
      // nor the dependent loads stall the ring at an item boundary.
      int fetched = 0;
      auto push = [&](int w, const Item& it) {
        const int slot = fetched % kItemQ;
        ptx::mbar_wait(ptx::smem_u32(&tail->iq_empty[slot]),
                       (uint32_t)(((fetched / kItemQ) & 1) ^ 1));
        atomicExch(&tail->iq[slot][0], w);
        atomicExch(&tail->iq[slot][1], it.e0);
        atomicExch(&tail->iq[slot][2], it.chunk);
        atomicExch(&tail->iq[slot][3], it.cnt);
        atomicExch(&tail->iq[slot][4], it.r0);
        atomicExch(&tail->iq[slot][5], it.r1);
        ptx::mbar_arrive(ptx::smem_u32(&tail->iq_full[slot]));
        ++fetched;
      };
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t full0 = ptx::smem_u32(&tail->full[0]);
      int claimed = atomicAdd(a.item_counter, 1);
      int cur = claimed < n_work ? claimed : -1;
      Item it{};
      if (cur >= 0) it = decode_raw(a.items[cur], a);
      push(cur, it);
      claimed = cur >= 0 ? atomicAdd(a.item_counter, 1) : n_work;   // in flight
      while (cur >= 0) {
        const int nxt = claimed < n_work ? claimed : -1;
        const int4 raw = nxt >= 0 ? a.items[nxt] : make_int4(0, 0, 0, 0);   // in flight
        Item itn{};
        bool pushed = false;
        for (int32_t t = 0; t < it.ntiles; ++t) {
          const int32_t row = it.r0 + t * kBM;
          const int32_t left = it.r1 - row;
          const TileGeom g = tile_geom(left);
          for (int kb0 = 0; kb0 < num_kb; kb0 += g.kps) {
            const int nkb = num_kb - kb0 < g.kps ? num_kb - kb0 : g.kps;
            ptx::mbar_wait(ptx::smem_u32(&tail->empty[stage]), phase ^ 1);
            const uint32_t dst = ptx::smem_u32(ring + stage * kStageBytes);
            const uint32_t fb = full0 + stage * 8;
            ptx::mbar_arrive_expect_tx(fb, nkb * g.kbb);
            if (g.nbox == 4) {
              for (int j = 0; j < nkb; ++j)
                ptx::tma_load_2d(dst + j * g.kbb, &tmap_x, fb, (kb0 + j) * kBK, row);
            } else {
              // chunk tail: 32-row boxes only (a full box would drag in the next list's rows)
              for (int j = 0; j < nkb; ++j)
                for (int bx = 0; bx < g.nbox; ++bx)
                  ptx::tma_load_2d(dst + j * g.kbb + bx * kTailRows * kBK * 2, &tmap_tail, fb,
                                   (kb0 + j) * kBK, row + bx * kTailRows);
            }
            if (++stage == kStages) { stage = 0; phase ^= 1; }
            if (!pushed) {   // the next item, decoded behind this slot's copies
              pushed = true;
              if (nxt >= 0) itn = decode_raw(raw, a);
              push(nxt, itn);
              claimed = nxt >= 0 ? atomicAdd(a.item_counter, 1) : n_work;
            }
          }
        }
        cur = nxt;
        it = itn;
      }
      // drain: every stage released by its final MMA commit before the CTA may exit
      for (int i = 0; i < kStages; ++i) {
        ptx::mbar_wait(ptx::smem_u32(&tail->empty[stage]), phase ^ 1);
        if (++stage == kStages) { stage = 0; phase ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp == kMmaWarp) {
    // ===================== MMA issuer (warp-convergent; elect.sync issues) =====================
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    const uint64_t adesc0 = ptx::umma_desc_sw128(ptx::smem_u32(ring));
    const uint64_t bdesc0 = ptx::umma_desc_sw128(ptx::smem_u32(bbuf));
    const uint32_t full0 = ptx::smem_u32(&tail->full[0]);
    const uint32_t empty0 = ptx::smem_u32(&tail->empty[0]);
    for (int i = 0;; ++i) {
      Item it;
      const int w = take_item(i, it);
      if (w < 0) break;
      const uint32_t idesc = F8 ? ptx::umma_idesc_e4m3(kBM, it.cnt <= 16 ? 16 : 32)
                                : ptx::umma_idesc_bf16(kBM, it.cnt <= 16 ? 16 : 32);
      const int buf = i & 1;
      ptx::mbar_wait(ptx::smem_u32(&tail->b_full[buf]), (uint32_t)((i >> 1) & 1));
      ptx::tc_fence_after();
      const uint64_t bdesc_buf = bdesc0 + (uint64_t)((buf * kBBytes) >> 4);
      for (int32_t t = 0; t < it.ntiles; ++t) {
        ptx::mbar_wait(ptx::smem_u32(&tail->acc_empty[acc]), acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem + (uint32_t)(acc * kNQ);
        const TileGeom g = tile_geom(it.r1 - (it.r0 + t * kBM));
        for (int kb0 = 0; kb0 < num_kb; kb0 += g.kps) {
          ptx::mbar_wait(full0 + stage * 8, phase);
          ptx::tc_fence_after();
          const uint64_t sdesc = adesc0 + (uint64_t)((stage * kStageBytes) >> 4);
          for (int j = 0; j < g.kps; ++j) {
            const int kb = kb0 + j;
            if (kb < num_kb) {
              const uint64_t ad = sdesc + (uint64_t)((j * g.kbb) >> 4);
              const uint64_t bd = bdesc_buf + (uint64_t)((kb * kBKbBytes) >> 4);
#pragma unroll
              for (int kk = 0; kk < kBK / 16; ++kk) {
                if constexpr (F8)
                  ptx::mma_e4m3_elect<1, false>(d_tmem, ad + kk * 2, bd + kk * 2, idesc,
                                                (kb | kk) ? 1u : 0u);
                else
                  ptx::mma_bf16_elect<1, false>(d_tmem, ad + kk * 2, bd + kk * 2, idesc,
                                                (kb | kk) ? 1u : 0u);
              }
            }
          }
          ptx::tc_commit_elect<1>(empty0 + stage * 8);
          if (++stage == kStages) { stage = 0; phase ^= 1; }
        }
        ptx::tc_commit_elect<1>(ptx::smem_u32(&tail->acc_full[acc]));
        if (++acc == kNAcc) { acc = 0; acc_phase ^= 1; }
      }
      ptx::tc_commit_elect<1>(ptx::smem_u32(&tail->b_empty[buf]));   // prober buffer free
    }
    __syncwarp();
  } else if (warp >= kGather0) {
    // ===================== prober gather: 4 warps =====================
    // Item i's probers -> prober buffer i & 1 (128B-swizzled K-major rows: 16-byte chunk c of
    // row r of a K-block at c ^ (r & 7)) once the MMAs of item i - 2 released it, then
    // b_full.  Dedicated warps, so the epilogue never waits on these dependent loads.
    const uint4* Q4 = reinterpret_cast<const uint4*>(a.Q);
    const int row_chunks = num_kb * 8;  // 16-byte chunks per query row
    const int gt = (warp - kGather0) * 32 + lane;
    constexpr int kGT = 32 * kGatherWarps;
    for (int i = 0;; ++i) {
      Item it;
      if (take_item(i, it) < 0) break;
      const int buf = i & 1;
      ptx::mbar_wait(ptx::smem_u32(&tail->b_empty[buf]), (uint32_t)(((i >> 1) & 1) ^ 1));
      const int total = it.cnt * row_chunks;
      uint8_t* base = bbuf + buf * kBBytes;
      for (int c0 = gt; c0 < total; c0 += 8 * kGT) {
        uint4 v[8];
        int dst[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int c = c0 + u * kGT;
          dst[u] = -1;
          if (c < total) {
            const int r = c / row_chunks, rem = c - r * row_chunks;
            const int kb = rem >> 3, ch = rem & 7;
            const int q = __ldg(&a.lq_ent[it.e0 + r].x);
            v[u] = __ldg(Q4 + (size_t)q * row_chunks + rem);
            dst[u] = kb * kBKbBytes + (r >> 3) * 1024 + (r & 7) * 128 + ((ch ^ (r & 7)) << 4);
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (dst[u] >= 0) *reinterpret_cast<uint4*>(base + dst[u]) = v[u];
      }
      ptx::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&tail->b_full[buf]));
    }
  } else {
    // ===================== epilogue: 8 warps =====================
    const int ew = warp;
    const int quad = ew & 3;   // TMEM lane quadrant: list rows [32 * quad, +32) of a tile
    const int half = ew >> 2;  // prober columns [16 * half, +16)
    const int et = ew * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    const int k = a.k;
    const bool use_hint = a.q_hint != nullptr;  // shared pruning bound (off: exact per-item top-k)
    const int col = half * 16 + lane;  // prober owned by this lane (lanes 0..15)
    uint64_t* heap = (k <= IVS_KSMEM)
                         ? heap_s + (ew * 16 + (lane & 15))
                         : a.heap_g + (size_t)blockIdx.x * k * IVS_HEAPS + (ew * 16 + (lane & 15));
    if (lane < 16)
      for (int i = 0; i < k; ++i) heap[(size_t)i * IVS_HEAPS] = 0ull;
    int acc = 0;
    uint32_t acc_phase = 0;
    // per-item metadata is loaded one item ahead (prober entry) or at the item's start (output
    // slot, used at its end) so that no dependent global load sits on the critical path
    Item it, itn;
    int w = take_item(0, it);
    int2 e_cur = make_int2(0, 0);
    if (w >= 0 && lane < 16 && col < it.cnt) e_cur = a.lq_ent[it.e0 + col];
    for (int i = 0; w >= 0; ++i) {
      const int wn = take_item(i + 1, itn);
      int2 e_nxt = make_int2(0, 0);
      if (wn >= 0 && lane < 16 && col < itn.cnt) e_nxt = a.lq_ent[itn.e0 + col];   // in flight
      const bool own = lane < 16 && col < it.cnt;
      int64_t q = 0;
      int pj = 0;
      float hint = threshold_of(0ull);
      int64_t slot0 = 0;
      if (own) {
        q = e_cur.x;
        pj = e_cur.y;
        slot0 = a.q_slot[(size_t)q * a.nprobe + pj];   // in flight until the flush
        const uint32_t h = use_hint ? __ldcg(a.q_hint + q) : 0u;
        if (h != 0u) hint = float_from_ordered(h);
      }
      float thr = hint;
      uint32_t published = 0u;
      const int ncol = it.cnt - half * 16;  // columns of this warp (uniform)
      for (int32_t t = 0; t < it.ntiles; ++t) {
        const int32_t row = it.r0 + t * kBM + quad * 32 + lane;
        const bool rvalid = row < it.r1;
        // this lane's row id, loaded before the wait (used only if a score passes)
        const uint32_t id = !rvalid ? 0u : a.row_ids ? (uint32_t)__ldg(a.row_ids + row) : (uint32_t)row;
        ptx::mbar_wait(ptx::smem_u32(&tail->acc_full[acc]), acc_phase);
        ptx::tc_fence_after();
        uint32_t r[16];
        if (ncol > 0) {
          ptx::tmem_ld16(tmem + lane_addr + (uint32_t)(acc * kNQ + half * 16), r);
          ptx::tmem_wait_ld();
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(ptx::smem_u32(&tail->acc_empty[acc]));
        if (++acc == kNAcc) { acc = 0; acc_phase ^= 1; }
        if (ncol <= 0) continue;
        if (use_hint && own && (t & 3) == 3) {
          const uint32_t h = __ldcg(a.q_hint + q);
          if (h != 0u) {
            hint = fmaxf(hint, float_from_ordered(h));
            thr = fmaxf(thr, hint);
          }
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (j >= ncol) break;
          const float th = __shfl_sync(0xffffffffu, thr, j);
          const float s = __uint_as_float(r[j]);
          const bool pass = rvalid && s >= th;
          uint32_t m = __ballot_sync(0xffffffffu, pass);
          if (m) {
            const uint64_t key = pass ? make_key(s, id) : 0ull;
            while (m) {
              const int src = __ffs(m) - 1;
              m &= m - 1;
              const uint64_t kk = __shfl_sync(0xffffffffu, key, src);
              if (lane == j) thr = fmaxf(heap_push(heap, k, kk), hint);
            }
            if (lane == j) {
              const uint64_t root = heap[0];
              const uint32_t o = (uint32_t)(root >> 32);
              if (use_hint && root != 0ull && o > published) {
                atomicMax(a.q_hint + q, o);
                published = o;
              }
            }
          }
        }
      }
      // flush this item's partial lists (one per lane quadrant) and reset the heaps
      if (own) {
        const size_t slot = (size_t)(slot0 + it.chunk);
        uint64_t* dst = a.part + (slot * IVS_PARTS + quad) * k;
        for (int i2 = 0; i2 < k; ++i2) {
          dst[i2] = heap[(size_t)i2 * IVS_HEAPS];
          heap[(size_t)i2 * IVS_HEAPS] = 0ull;
        }
      }
      w = wn;
      it = itn;
      e_cur = e_nxt;
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, kTmemCols);
  }
}

size_t ivf_scan_smem_bytes() {
  return 1024 + (size_t)kStages * kStageBytes + 2 * (size_t)kBBytes +
         (size_t)IVS_KSMEM * IVS_HEAPS * sizeof(uint64_t) + sizeof(Tail);
}

cudaError_t launch_ivf_scan(const CUtensorMap& tmap_x, const CUtensorMap& tmap_tail,
                            const IvfScanArgs& a, int grid, cudaStream_t stream) {
  const size_t smem = ivf_scan_smem_bytes();
  auto go = [&](auto kern) -> cudaError_t {
    cudaError_t e = ensure_max_smem(reinterpret_cast<const void*>(kern), smem);
    if (e != cudaSuccess) return e;
    kern<<<grid, kThreads, smem, stream>>>(tmap_x, tmap_tail, a);
    note_launch();
    return cudaGetLastError();
  };
  return a.fp8 ? go(ivf_scan_kernel<true>) : go(ivf_scan_kernel<false>);
}

}  // namespace sa
