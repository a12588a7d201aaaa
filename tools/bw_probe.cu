// bw_probe.cu -- TMA streaming bandwidth from L2-resident and HBM-resident buffers,
// with 64-row x 128-byte SW128 boxes (the flat-scan corpus tile shape).
#include <cstdio>
#include <cstdint>
#include <cudaTypedefs.h>
#include "../paper_2505_12065_b200/csrc/kernels/ptx.cuh"
using namespace sa::ptx;

constexpr int STAGES = 16;
__global__ void __launch_bounds__(64, 1) stream(const __grid_constant__ CUtensorMap m, int64_t rows, int box_rows,
                                                int cols_blocks, int reps) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t full[STAGES];
  const int stage_bytes = box_rows * 128;
  if (threadIdx.x == 0) { for (int i = 0; i < STAGES; ++i) mbar_init(smem_u32(&full[i]), 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t tiles = rows / box_rows;
    int64_t per = tiles / gridDim.x;
    int64_t t0 = blockIdx.x * per;
    uint32_t phase[STAGES] = {0};
    int64_t n = 0;
    for (int r = 0; r < reps; ++r)
      for (int64_t t = t0; t < t0 + per; ++t)
        for (int kb = 0; kb < cols_blocks; ++kb) {
          int s = n % STAGES;
          if (n >= STAGES) { mbar_wait(smem_u32(&full[s]), phase[s]); phase[s] ^= 1; }
          mbar_arrive_expect_tx(smem_u32(&full[s]), stage_bytes);
          tma_load_2d(smem_u32(smem + s * stage_bytes), &m, smem_u32(&full[s]), kb * 64, (int)(t * box_rows));
          ++n;
        }
    for (int64_t j = n - STAGES; j < n; ++j) { if (j < 0) continue; int s = j % STAGES; mbar_wait(smem_u32(&full[s]), phase[s]); phase[s] ^= 1; }
  }
}

int main() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  const int cols = 768;
  for (int64_t rows : {(int64_t)40000, (int64_t)4000000}) {     // 61 MB (L2) and 6.1 GB (HBM)
    void* buf; cudaMalloc(&buf, rows * cols * 2); cudaMemset(buf, 0, rows * cols * 2);
    for (int box_rows : {64, 128, 256}) {
      CUtensorMap m;
      cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
      cuuint64_t str[1] = {(cuuint64_t)cols * 2};
      cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
      cuuint32_t es[2] = {1, 1};
      enc(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      int smem = STAGES * box_rows * 128 + 1024;
      cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      int reps = rows < 100000 ? 50 : 2;
      for (int grid : {148}) {
        stream<<<grid, 64, smem>>>(m, rows, box_rows, cols / 64, 1);
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        stream<<<grid, 64, smem>>>(m, rows, box_rows, cols / 64, reps);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        int64_t tiles = rows / box_rows; int64_t per = tiles / grid;
        double bytes = (double)per * grid * box_rows * cols * 2 * reps;
        printf("rows=%lld box_rows=%d grid=%d: %.1f GB/s  (err=%s)\n", (long long)rows, box_rows, grid,
               bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
      }
    }
    cudaFree(buf);
  }
  return 0;
}
