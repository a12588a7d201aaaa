// bulk_probe.cu -- HBM -> smem streaming rate of 1-D TMA bulk copies (cp.async.bulk) on one
// B200, as a function of the copy size, ring depth and the number of copies per stage.
// Each of 148 CTAs (one per SM) streams its contiguous 1/148 of a 4 GiB buffer through a
// ring of S stages; one thread issues, all threads wait and touch one word per 512 B (so
// the consumer is never the bottleneck).  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -O3 -o tools/bulk_probe tools/bulk_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nW_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

__device__ __forceinline__ void bulk_hint(uint32_t dst, const void* src, uint32_t bytes,
                                          uint32_t bar) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}

__global__ void stream_kernel(const uint8_t* buf, size_t per_cta, int piece, int S, int split,
                              unsigned long long* sink, int hint = 0, size_t stride = 0) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bars[16];
  const size_t base = (size_t)blockIdx.x * (stride ? stride : per_cta);
  const int n = (int)(per_cta / piece);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(smem_u32(&bars[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int i) {
    const int s = i % S;
    mbar_expect(smem_u32(&bars[s]), piece);
    const int sub = piece / split;
    for (int c = 0; c < split; ++c)
      if (hint) bulk_hint(smem_u32(sm + (size_t)s * piece + c * sub), buf + base + (size_t)i * piece + c * sub,
           sub, smem_u32(&bars[s]));
      else bulk(smem_u32(sm + (size_t)s * piece + c * sub), buf + base + (size_t)i * piece + c * sub,
           sub, smem_u32(&bars[s]));
  };
  if (threadIdx.x == 0)
    for (int i = 0; i < S && i < n; ++i) issue(i);
  unsigned long long acc = 0;
  for (int i = 0; i < n; ++i) {
    const int s = i % S;
    mbar_wait(smem_u32(&bars[s]), (i / S) & 1);
    for (int o = threadIdx.x * 512; o < piece; o += blockDim.x * 512)
      acc += *reinterpret_cast<const uint32_t*>(sm + (size_t)s * piece + o);
    __syncthreads();
    if (threadIdx.x == 0 && i + S < n) issue(i + S);
  }
  if (acc == 0x123456789ull) sink[0] = acc;
}

// agent-step-like consumer: 16 warps, each copies rows w and w + 16 (1536 B) of the 32-row
// piece to registers, the stage is released, then a 768-term fp32 dot + warp reduction.
__global__ void agent_kernel(const uint8_t* buf, int npieces, size_t stride, int compute,
                             unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bars[4];
  const int S = 3, piece = 49152;
  const size_t base = (size_t)blockIdx.x * stride;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) mbar_init(smem_u32(&bars[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int i) {
    const int s = i % S;
    mbar_expect(smem_u32(&bars[s]), piece);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(sm + (size_t)s * piece)),
        "l"(buf + base + (size_t)i * piece), "r"(piece), "r"(smem_u32(&bars[s])), "l"(pol)
        : "memory");
  };
  if (threadIdx.x == 0)
    for (int i = 0; i < S && i < npieces; ++i) issue(i);
  float tot = 0.f;
  for (int i = 0; i < npieces; ++i) {
    const int s = i % S;
    mbar_wait(smem_u32(&bars[s]), (i / S) & 1);
    uint4 v[2][3];
    for (int h = 0; h < 2; ++h)
      for (int u = 0; u < 3; ++u)
        v[h][u] = reinterpret_cast<const uint4*>(sm + (size_t)s * piece + (warp + 16 * h) * 1536)[lane + 32 * u];
    __syncthreads();
    if (threadIdx.x == 0 && i + S < npieces) issue(i + S);
    if (compute)
      for (int h = 0; h < 2; ++h) {
        float acc = 0.f;
        for (int u = 0; u < 3; ++u) {
          const uint4 w = v[h][u];
          acc = fmaf(__uint_as_float(w.x << 16), 0.5f, acc);
          acc = fmaf(__uint_as_float(w.x & 0xFFFF0000u), 0.25f, acc);
          acc = fmaf(__uint_as_float(w.y << 16), 0.5f, acc);
          acc = fmaf(__uint_as_float(w.y & 0xFFFF0000u), 0.25f, acc);
          acc = fmaf(__uint_as_float(w.z << 16), 0.5f, acc);
          acc = fmaf(__uint_as_float(w.z & 0xFFFF0000u), 0.25f, acc);
          acc = fmaf(__uint_as_float(w.w << 16), 0.5f, acc);
          acc = fmaf(__uint_as_float(w.w & 0xFFFF0000u), 0.25f, acc);
        }
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        tot += acc;
      }
    else
      tot += __uint_as_float(v[0][0].x ^ v[1][2].w);
  }
  if (tot == 1.2345f) sink[0] = 1;
}

int main() {
  const size_t total = 4ull << 30;
  uint8_t* buf;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int pieces[] = {8192, 16384, 32768, 49152};
  const int stages[] = {2, 3, 4, 6, 8, 12};
  const int splits[] = {1, 4};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int piece : pieces)
    for (int S : stages)
      for (int split : splits) {
        if ((size_t)piece * S > 196 * 1024) continue;
        const size_t per_cta = (total / sms) / piece * piece;
        stream_kernel<<<sms, 128, piece * S>>>(buf, per_cta, piece, S, split, sink);
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r)
          stream_kernel<<<sms, 128, piece * S>>>(buf, per_cta, piece, S, split, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double gbs = 5.0 * per_cta * sms / (ms * 1e-3) / 1e9;
        printf("piece %6d B  stages %2d  split %d  in-flight/SM %4d KB : %7.0f GB/s  (%s)\n", piece,
               S, split, piece * S / 1024, gbs, cudaGetErrorString(cudaGetLastError()));
      }
  // short streams (an agent step: ~13 pieces of 48 KB per SM), misaligned starts, hint on/off
  for (int hint = 0; hint < 2; ++hint)
    for (int npieces : {1, 2, 4, 13, 26}) {
      const int piece = 49152, S = 3;
      const size_t per_cta = (size_t)npieces * piece;
      const size_t stride = 27ull * 1024 * 1024 + 512;   // scattered, 512-B aligned starts
      stream_kernel<<<sms, 128, piece * S>>>(buf, per_cta, piece, S, 1, sink, hint, stride);
      cudaEventRecord(e0);
      for (int r = 0; r < 50; ++r)
        stream_kernel<<<sms, 128, piece * S>>>(buf, per_cta, piece, S, 1, sink, hint, stride);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("short: %2d pieces x 48 KB per SM, hint %d: %6.1f us per launch, %6.0f GB/s\n",
             npieces, hint, ms * 1e3 / 50, 50.0 * per_cta * sms / (ms * 1e-3) / 1e9);
    }
  cudaFuncSetAttribute(agent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int compute = 0; compute < 2; ++compute)
    for (int npieces : {4, 13, 26, 104}) {
      const size_t stride = 27ull * 1024 * 1024 + 512;
      agent_kernel<<<sms, 512, 3 * 49152>>>(buf, npieces, stride, compute, sink);
      cudaEventRecord(e0);
      for (int r = 0; r < 50; ++r) agent_kernel<<<sms, 512, 3 * 49152>>>(buf, npieces, stride, compute, sink);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("agent-like 512 thr: %3d pieces, compute %d: %6.1f us per launch, %6.0f GB/s (%s)\n",
             npieces, compute, ms * 1e3 / 50, 50.0 * npieces * 49152.0 * sms / (ms * 1e-3) / 1e9,
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
