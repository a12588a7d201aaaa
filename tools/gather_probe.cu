// gather_probe.cu -- HBM bandwidth of RANDOM row gathers on one B200: the access pattern of
// the graph beam search (graph.cu: whole 1536-byte bf16 rows, or 768-byte e4m3 rows, at
// uniformly random positions of a 32 GB corpus).  The sequential copy figure in
// MEASURED_PEAKS.json is the roofline the bench reports against; this probe measures what a
// random-row stream can reach, as a function of the rows in flight per SM.
//
//   reg:  each warp loads R rows at a time into registers (lane l: 16-byte chunks l, l+32, ..),
//         B threads per CTA, as many CTAs as fit (the graph kernel's form, without its phases)
//   bulk: one lane per warp issues cp.async.bulk of whole rows into a per-warp smem ring of
//         S slots (mbarrier per slot), the warp touches each row when it lands
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_probe tools/gather_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

template <int R>
__global__ void gather_reg(const uint4* __restrict__ X, int64_t n_rows, int nch, int iters,
                           uint32_t seed, unsigned long long* sink) {
  const int lane = threadIdx.x & 31;
  const uint64_t gw = (uint64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    uint4 v[R][3];
#pragma unroll
    for (int u = 0; u < R; ++u) {
      const int64_t row = (int64_t)(mix64(((gw * iters + it) * R + u) ^ ((uint64_t)seed << 40)) %
                                    (uint64_t)n_rows);
#pragma unroll
      for (int rd = 0; rd < 3; ++rd) {
        const int c = rd * 32 + lane;
        v[u][rd] = c < nch ? __ldg(X + row * nch + c) : make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < R; ++u)
#pragma unroll
      for (int rd = 0; rd < 3; ++rd) acc ^= v[u][rd].x ^ v[u][rd].y ^ v[u][rd].z ^ v[u][rd].w;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// one warp per ring; S slots of `bytes` each; the warp streams `iters` random rows
__global__ void gather_bulk(const uint8_t* __restrict__ X, int64_t n_rows, uint32_t bytes, int S,
                            int iters, uint32_t seed, unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t sm[];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31, nw = blockDim.x / 32;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm) + warp * 32;
  uint8_t* ring = sm + nw * 32 * 8 + (size_t)warp * S * bytes;
  const uint64_t gw = (uint64_t)blockIdx.x * nw + warp;
  if (lane == 0)
    for (int s = 0; s < S; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar + s)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  auto issue = [&](int it) {
    const int s = it % S;
    const int64_t row =
        (int64_t)(mix64((gw * iters + it) ^ ((uint64_t)seed << 40)) % (uint64_t)n_rows);
    const uint32_t b = smem_u32(bar + s);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
            "r"(smem_u32(ring + (size_t)s * bytes)),
        "l"(X + row * bytes), "r"(bytes), "r"(b)
        : "memory");
  };
  if (lane == 0)
    for (int it = 0; it < S && it < iters; ++it) issue(it);
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    const int s = it % S;
    const uint32_t par = (uint32_t)((it / S) & 1);
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(
            smem_u32(bar + s)),
        "r"(par)
        : "memory");
    const uint4* r4 = reinterpret_cast<const uint4*>(ring + (size_t)s * bytes);
    for (int c = lane; c < (int)(bytes / 16); c += 32) acc ^= r4[c].x ^ r4[c].w;
    __syncwarp();
    if (lane == 0 && it + S < iters) issue(it + S);
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

int main() {
  const int64_t row_bytes_bf16 = 1536;
  const int64_t n_rows = 21015324;
  const size_t total = (size_t)n_rows * row_bytes_bf16;
  uint8_t* X;
  if (cudaMalloc(&X, total) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(X, 1, total);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int sms = 148;
  auto run_reg = [&](auto kern, int R, int threads, int ctas_per_sm, int64_t rb) {
    const int nch = (int)(rb / 16);
    const int64_t nr = (int64_t)(total / rb);
    const int grid = sms * ctas_per_sm;
    const int warps = grid * threads / 32;
    const int iters = (int)((8ll << 30) / ((int64_t)warps * R * rb));  // ~8 GB per launch
    kern<<<grid, threads>>>(reinterpret_cast<const uint4*>(X), nr, nch, iters, 1u, sink);
    cudaEventRecord(e0);
    for (int r = 0; r < 3; ++r)
      kern<<<grid, threads>>>(reinterpret_cast<const uint4*>(X), nr, nch, iters, 2u + r, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = 3.0 * warps * (double)iters * R * rb;
    printf("reg  row %5lld B  R %d  threads %4d x %d CTAs/SM  in-flight/SM %4lld KB : %6.0f GB/s (%s)\n",
           (long long)rb, R, threads, ctas_per_sm,
           (long long)(threads / 32 * ctas_per_sm * R * rb / 1024), bytes / (ms * 1e6),
           cudaGetErrorString(cudaGetLastError()));
  };
  for (int64_t rb : {row_bytes_bf16, (int64_t)768}) {
    run_reg(gather_reg<1>, 1, 256, 4, rb);
    run_reg(gather_reg<2>, 2, 256, 4, rb);
    run_reg(gather_reg<3>, 3, 256, 4, rb);
    run_reg(gather_reg<4>, 4, 256, 4, rb);
    run_reg(gather_reg<3>, 3, 256, 8, rb);
    run_reg(gather_reg<6>, 6, 256, 4, rb);
    run_reg(gather_reg<8>, 8, 128, 8, rb);
  }
  for (int64_t rb : {row_bytes_bf16, (int64_t)768, (int64_t)3072}) {
    for (int S : {2, 4, 8, 16}) {
      for (int threads : {256, 512, 1024}) {
        const size_t smem = (size_t)(threads / 32) * (32 * 8 + S * rb);
        if (smem > 220 * 1024) continue;
        cudaFuncSetAttribute(gather_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const int64_t nr = (int64_t)(total / rb);
        const int grid = sms;
        const int warps = grid * threads / 32;
        const int iters = (int)((8ll << 30) / ((int64_t)warps * rb));
        gather_bulk<<<grid, threads, smem>>>(X, nr, (uint32_t)rb, S, iters, 1u, sink);
        cudaEventRecord(e0);
        for (int r = 0; r < 3; ++r)
          gather_bulk<<<grid, threads, smem>>>(X, nr, (uint32_t)rb, S, iters, 2u + r, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double bytes = 3.0 * warps * (double)iters * rb;
        printf("bulk row %5lld B  S %2d  threads %4d  in-flight/SM %4lld KB : %6.0f GB/s (%s)\n",
               (long long)rb, S, threads, (long long)(threads / 32 * S * rb / 1024),
               bytes / (ms * 1e6), cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
