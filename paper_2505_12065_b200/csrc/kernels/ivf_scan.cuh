// ivf_scan.cuh -- launcher interface of the list-major IVF scan kernel.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace sa {

constexpr int IVS_BM = 128;    // list rows per tile (MMA M = TMEM lanes)
constexpr int IVS_NQ = 32;     // probing queries per work item (MMA N in {16, 32})
constexpr int IVS_PARTS = 4;   // partial lists per (prober, item): one per TMEM lane quadrant
constexpr int IVS_KSMEM = 16;  // heaps in smem for k <= 16, else in global scratch
constexpr int IVS_HEAPS = 128; // (epilogue warp, column) heaps per CTA

struct IvfScanArgs {
  const __nv_bfloat16* Q;  // staged queries [nq, d_pad] bf16
  int32_t d_pad;           // multiple of 64, <= 768
  int32_t k;               // 1..256
  const int32_t* row_ids;  // stored row -> global id (nullptr: the stored position)
  uint64_t* part;          // out: [slot][IVS_PARTS][k] packed keys (unordered, 0 = empty)
  uint64_t* heap_g;        // scratch [grid][k][IVS_HEAPS] when k > IVS_KSMEM
  const int4* items;       // [*n_items] {list, first prober in lq_ent, chunk, prober count <= 32}
  const int32_t* n_items;  // device scalar
  const int64_t* list_off; // [nlist + 1] stored-row range of each list
  const int2* lq_ent;      // (query, probe rank) pairs grouped by list
  const int64_t* q_slot;   // [nq * nprobe] first output slot of (query, probe rank)
  int32_t nprobe;
  int32_t chunk_rows;      // rows per work item (multiple of IVS_BM)
  uint32_t* q_hint;        // [nq] ordered-fp32 lower bound of each query's k-th score (zeroed);
                           // nullptr: no shared bound (every partial list is its exact top-k)
  int32_t* item_counter;   // zeroed global counter: dynamic item scheduling
  int32_t fp8;             // 1: e4m3 rows and queries (kind::f8f6f4) passed as 16-bit pairs:
                           // Q [nq, d_pad pairs], tensor maps over the e4m3 copy; row_ids may
                           // then be nullptr (keys carry stored positions for the re-rank)
};

size_t ivf_scan_smem_bytes();
// tmap_x: stored corpus, 128-row x 64-col boxes; tmap_tail: the same with 32-row boxes.
cudaError_t launch_ivf_scan(const CUtensorMap& tmap_x, const CUtensorMap& tmap_tail,
                            const IvfScanArgs& a, int grid, cudaStream_t stream);

}  // namespace sa
