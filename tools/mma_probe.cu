// mma_probe.cu -- microbenchmark: cycles per tcgen05.mma (kind::f16, M=128) as a function of
// N, A source (TMEM/SMEM), number of independent accumulator chains, and issue style.
// Not part of the library; used to choose the flat-scan tile shape.
#include <cstdio>
#include <cstdint>
#include "../paper_2505_12065_b200/csrc/kernels/ptx.cuh"
using namespace sa::ptx;

__global__ void probe(int N, int a_tmem_mode, int chains, int iters, int uniform_issue,
                      unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) { mbar_init(smem_u32(&bar), 1); fence_mbar_init(); }
  if (warp == 0) { tmem_alloc(smem_u32(&tbase), 512); tmem_relinquish(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  uint32_t tmem = tbase;
  uint32_t idesc = umma_idesc_bf16(128, N);
  uint64_t bdesc = umma_desc_sw128(smem_u32(smem));
  uint64_t adesc = umma_desc_sw128(smem_u32(smem + 65536));
  if (warp == 0) {
    unsigned long long t0 = clock64();
    if (uniform_issue) {
      for (int i = 0; i < iters; ++i) {
        int c = i % chains;
        uint32_t d = tmem + c * N;
        uint32_t acc = (i >= chains) ? 1u : 0u;
        uint32_t e;
        asm volatile("{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\nselp.u32 %0, 1, 0, p;\n}" : "=r"(e));
        if (e) {
          if (a_tmem_mode) mma_bf16_ts(d, tmem + 384 + (i & 3) * 8, bdesc + (i & 3) * 2, idesc, acc);
          else mma_bf16_ss(d, adesc + (i & 3) * 2, bdesc + (i & 3) * 2, idesc, acc);
        }
        __syncwarp();
      }
      if (lane == 0) tc_commit(smem_u32(&bar));
      __syncwarp();
    } else if (lane == 0) {
      for (int i = 0; i < iters; ++i) {
        int c = i % chains;
        uint32_t d = tmem + c * N;
        uint32_t acc = (i >= chains) ? 1u : 0u;
        if (a_tmem_mode) mma_bf16_ts(d, tmem + 384 + (i & 3) * 8, bdesc + (i & 3) * 2, idesc, acc);
        else mma_bf16_ss(d, adesc + (i & 3) * 2, bdesc + (i & 3) * 2, idesc, acc);
      }
      tc_commit(smem_u32(&bar));
    }
    __syncwarp();
    mbar_wait(smem_u32(&bar), 0);
    unsigned long long t1 = clock64();
    if (lane == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  int iters = 4096;
  printf("N  A    chains uniform  cyc/mma  (ideal floor N/2)\n");
  for (int uniform = 0; uniform < 2; ++uniform)
  for (int amode = 1; amode >= 0; --amode)
  for (int N : {64, 128, 256})
  for (int chains : {1, 2, 4}) {
    if (amode == 1 && chains * N > 384) continue;
    if (amode == 0 && chains * N > 512) continue;
    probe<<<148, 128, 160 * 1024>>>(N, amode, chains, iters, uniform, d);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
    unsigned long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0; for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    printf("%3d %s %d %d  %.1f  (%d)\n", N, amode ? "tmem" : "smem", chains, uniform,
           (double)mx / iters, N / 2);
  }
  return 0;
}
