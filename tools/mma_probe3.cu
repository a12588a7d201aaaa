// mma_probe3.cu -- cycles per cta_group::2 tcgen05.mma (M=256, N=128), TS vs SS, per CTA pair.
#include <cstdio>
#include <cstdint>
#include "../paper_2505_12065_b200/csrc/kernels/ptx.cuh"
using namespace sa::ptx;

template <bool ATMEM, int N>
__global__ void __cluster_dims__(2, 1, 1) probe(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  uint32_t rank = cluster_ctarank();
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_mbar_init(); }
  if (warp == 0) { tmem_alloc_2sm(smem_u32(&tbase), 512); tmem_relinquish_2sm(); }
  tc_fence_before(); cluster_sync(); tc_fence_after();
  uint32_t tmem = tbase;
  constexpr uint32_t idesc = umma_idesc_bf16(256, N);
  uint64_t bdesc = umma_desc_sw128(smem_u32(smem));
  uint64_t adesc = umma_desc_sw128(smem_u32(smem + 65536));
  if (warp == 0 && rank == 0) {
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; i += 16) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if (ATMEM) mma_bf16_elect<2, true>(tmem, tmem + 256 + (j & 3) * 8, bdesc + (j & 3) * 2, idesc, 1u);
        else mma_bf16_elect<2, false>(tmem, adesc + (j & 3) * 2, bdesc + (j & 3) * 2, idesc, 1u);
      }
    }
    tc_commit_elect<2>(smem_u32(&bar));
    mbar_wait(smem_u32(&bar), 0);
    unsigned long long t1 = clock64();
    if (lane == 0) out[blockIdx.x / 2] = t1 - t0;
  }
  if (warp == 0 && rank == 1) mbar_wait(smem_u32(&bar), 0);
  tc_fence_before(); cluster_sync();
  if (warp == 0) { tc_fence_after(); tmem_dealloc_2sm(tmem, 512); }
}

template <bool ATMEM, int N>
void run(int pairs, unsigned long long* d) {
  int iters = 8192;
  auto k = probe<ATMEM, N>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  k<<<pairs * 2, 128, 160 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); exit(1); }
  unsigned long long h[74]; cudaMemcpy(h, d, pairs * 8, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0; for (int i = 0; i < pairs; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("2CTA M=256 N=%d A=%s pairs=%d: %.1f cyc/mma (floor %d)\n", N, ATMEM ? "tmem" : "smem", pairs,
         (double)mx / iters, 256 * N / 512);
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 74 * 8);
  for (int pairs : {1, 74}) {
    run<true, 128>(pairs, d); run<false, 128>(pairs, d); run<true, 256>(pairs, d); run<false, 256>(pairs, d); run<true, 64>(pairs, d);
  }
  return 0;
}
