// flat_scan.cuh -- launcher interface of the fused scan + top-k kernel.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

namespace sa {

constexpr int FS_BM = 128;      // queries per CTA (TMEM lanes)
constexpr int FS_BN = 64;       // corpus rows per accumulator tile
constexpr int FS_BK = 64;       // bf16 per 128-byte swizzle row (one TMA box column extent)
constexpr int FS_STAGES = 18;   // TMA ring depth (8 KB per stage)
constexpr int FS_KSMEM = 32;    // heaps live in smem for k <= 32, else in global scratch
constexpr int FS_THREADS = 192; // warp 0 TMA, warp 1 MMA, warps 2..5 epilogue
constexpr int FS_MAX_DPAD = 768;// A operand in TMEM: 128 + d_pad/2 <= 512 columns

struct FlatScanArgs {
  const __nv_bfloat16* Q;  // staged queries [nq_pad, d_pad] bf16, zero padded
  int64_t nq_pad;          // multiple of FS_BM
  int32_t d_pad;           // multiple of 64, <= FS_MAX_DPAD
  int64_t n_rows;          // corpus rows scanned (tensor map covers exactly these)
  int32_t QB;              // query blocks = nq_pad / FS_BM
  int32_t S;               // corpus slices per query block
  int32_t k;               // 1..256
  const int32_t* row_ids;  // optional row -> id map (nullptr: id = row)
  uint32_t id_base;        // added to the id stored in each key
  uint64_t* part;          // out: [nq_pad][S][k] packed keys (unordered within a list)
  uint64_t* heap_g;        // scratch [grid][k][FS_BM] when k > FS_KSMEM
  float* dbg;              // mode 1: [nq_pad][n_rows] raw scores
  int32_t mode;            // 0 = top-k, 1 = debug score dump
};

size_t flat_scan_smem_bytes();
cudaError_t launch_flat_scan(const CUtensorMap& tmap, const FlatScanArgs& a, int grid,
                             cudaStream_t stream);

}  // namespace sa
