// flat_scan.cuh -- launcher interface of the fused scan + top-k kernel.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace sa {

constexpr int FS_BM = 128;       // query rows per CTA (TMEM lanes)
constexpr int FS_BN = 128;       // corpus rows per tile (MMA N, accumulator columns)
constexpr int FS_BK = 64;        // bf16 per 128-byte swizzle row (one TMA box column extent)
constexpr int FS_EPI_WARPS = 8;  // two warps per TMEM lane quadrant, 64 columns each
constexpr int FS_THREADS = 96 + 32 * FS_EPI_WARPS;  // 8 epilogue warps, TMA, MMA, bound warp
constexpr int FS_EPI_THREADS = 32 * FS_EPI_WARPS;
constexpr int FS_MAX_DPAD = 768; // queries: up to 8 K-blocks in TMEM + 4 in smem
constexpr int FS_KB_TMEM = 8;    // K-blocks of the A operand held in TMEM (256 columns)
constexpr int FS_KB_SMEM = 4;    // K-blocks of the A operand held in smem (64 KB)
constexpr int FS_KSMEM = 16;     // running heaps in smem for k <= 16, else in global scratch
constexpr int FS_KSMEM_BIG = 48; // ... or k <= 48 when the A operand fits TMEM (d_pad <= 512):
                                 // the heaps then also take the unused 64 KB A region
constexpr int FS_TAIL_ROWS = 32;  // box rows of the index's tail tensor map (IVF list tails,
                                  // ivf_scan.cu)
constexpr int FS_LISTS_PER_ITEM = 2;  // partial lists per (query, work item): one per column half

// largest k whose running heaps stay in shared memory for this d_pad
inline int fs_heap_smem_cap(int32_t d_pad) {
  return d_pad <= FS_KB_TMEM * FS_BK ? FS_KSMEM_BIG : FS_KSMEM;
}

enum FlatScanMode : int32_t {
  FS_MODE_TOPK = 0,   // work item = (query group, corpus slice), running top-k
  FS_MODE_DEBUG = 1,  // raw score dump (IVF probe, graph entry points, tests)
};

struct FlatScanArgs {
  const __nv_bfloat16* Q;  // staged queries [>= nq rows, d_pad] bf16, zero padded columns
  int64_t nq;              // real query rows (rows >= nq are never read)
  int64_t nq_pad;          // multiple of FS_BM * cta_group (flat modes)
  int32_t d_pad;           // multiple of 64, <= FS_MAX_DPAD
  int64_t n_rows;          // corpus rows (the tensor map covers exactly these)
  int32_t QP;              // flat: query groups = nq_pad / (FS_BM * cta_group)
  int32_t S;               // flat: corpus slices per query group
  int32_t k;               // 1..256
  const int32_t* row_ids;  // optional row -> id map (nullptr: id = row)
  uint32_t id_base;        // added to the id stored in each key
  uint64_t* part;          // out: [nq_pad][S][FS_LISTS_PER_ITEM][k] packed keys (unordered)
  uint64_t* heap_g;        // scratch [grid][k][FS_EPI_THREADS] when k > FS_KSMEM
  float* dbg;              // debug: [nq_pad][n_rows] raw scores
  int32_t mode;            // FlatScanMode
  uint32_t* q_hint;        // optional [nq] ordered-fp32 lower bound of each query's k-th score
                           // (zero-initialised by the caller; 0 = none)
  uint32_t* q_max;         // optional [nq][q_max_stride] ordered-fp32 best score of each heap
                           // of a query (heap index = slice * FS_LISTS_PER_ITEM + half; zeroed
                           // by the caller): the bound warp's k-th-of-maxima bound (flat_scan.cu)
  int32_t q_max_stride;    // >= S * FS_LISTS_PER_ITEM, a multiple of 4 (unused entries stay 0)
  int32_t* progress;       // optional [units] tile progress for soft lockstep (zeroed; one
                           // work item per unit and QP > 1)
  int32_t experiment;      // timing experiments only (tuning builds, SA_EXPERIMENT): 1 = skip score
                           // processing, 2 = also skip the TMEM loads, 3 = the 64-way max
                           // only (no insertion).  0 in production.
  int32_t lockstep_lag;    // tiles a unit may run ahead of the units sharing its slice (0 = 4)
  unsigned long long* counters;  // tuning builds only (SA_FS_COUNT): [0] passing (thread, tile)
                           // pairs, [1] heap insertions, [2] bound-warp rounds
  int32_t fp8;             // 1: Q and the corpus are e4m3 bytes (kind::f8f6f4 MMAs), passed
                           // as 16-bit pairs -- d_pad counts PAIRS of e4m3 values (bytes / 2),
                           // so TMA boxes, swizzle, descriptors and TMEM columns are the bf16
                           // ones byte for byte.
};

// cta_group = 1: one CTA per query block of 128 (M=128, box 128 rows).
// cta_group = 2: CTA pairs (cluster of 2) share each corpus tile, M=256 (box 64 rows per CTA).
size_t flat_scan_smem_bytes(int cta_group);
// tmap: corpus rows (box 128 rows for cta_group 1, 64 for 2); tmap_q: the staged queries
// (box 128 rows, rows = nq), used for the K-blocks of the A operand that live in smem.
cudaError_t launch_flat_scan(const CUtensorMap& tmap, const CUtensorMap& tmap_q,
                             const FlatScanArgs& a, int cta_group, int grid, cudaStream_t stream);

}  // namespace sa
