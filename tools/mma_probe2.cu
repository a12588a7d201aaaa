// mma_probe2.cu -- cycles per tcgen05.mma with a minimal, unrolled issue loop.
#include <cstdio>
#include <cstdint>
#include "../paper_2505_12065_b200/csrc/kernels/ptx.cuh"
using namespace sa::ptx;

template <int N, bool ATMEM>
__global__ void probe(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_mbar_init(); }
  if (warp == 0) { tmem_alloc(smem_u32(&tbase), 512); tmem_relinquish(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  uint32_t tmem = tbase;
  constexpr uint32_t idesc = umma_idesc_bf16(128, N);
  uint64_t bdesc = umma_desc_sw128(smem_u32(smem));
  uint64_t adesc = umma_desc_sw128(smem_u32(smem + 65536));
  if (warp == 0 && lane == 0) {
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; i += 16) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (ATMEM) mma_bf16_ts(tmem, tmem + 384 + (j & 3) * 8, bdesc + (j & 3) * 2, idesc, 1u);
        else mma_bf16_ss(tmem, adesc + (j & 3) * 2, bdesc + (j & 3) * 2, idesc, 1u);
      }
    }
    tc_commit(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int N, bool ATMEM>
void run(int grid, unsigned long long* d) {
  int iters = 8192;
  auto k = probe<N, ATMEM>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  k<<<grid, 128, 160 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
  unsigned long long h[148]; cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0; for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("N=%3d A=%s grid=%3d  %.1f cyc/mma (floor %d)\n", N, ATMEM ? "tmem" : "smem", grid,
         (double)mx / iters, N / 2);
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 148 * 8);
  for (int grid : {1, 148}) {
    run<64, true>(grid, d); run<128, true>(grid, d); run<256, false>(grid, d);
    run<64, false>(grid, d); run<128, false>(grid, d);
  }
  return 0;
}
