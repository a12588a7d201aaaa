// condgraph_probe.cu -- does compute-sanitizer synccheck understand mbarriers in kernels that
// run inside a WHILE conditional graph node?  (sa_search_mature's stage loop reports "Barrier
// error: Missing init" there while the same kernel launched directly is clean.)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/condgraph_probe tools/condgraph_probe.cu
//   compute-sanitizer --tool synccheck /tmp/condgraph_probe [direct|graph]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>

__global__ void mbar_kernel(int* out) {
  __shared__ __align__(8) unsigned long long bar;
  __shared__ int val;
  const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 32) {
    val = 7 + blockIdx.x;
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(b) : "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile(
        "{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
        "@!P1 bra W;\n}\n" ::"r"(b)
        : "memory");
    if (threadIdx.x == 0) out[blockIdx.x] = val;
  }
}

__global__ void count_kernel(int* ctr, cudaGraphConditionalHandle h) {
  if (threadIdx.x == 0 && blockIdx.x == 0) cudaGraphSetConditional(h, ++*ctr < 3 ? 1u : 0u);
}

int main(int argc, char** argv) {
  const bool graph = argc > 1 && std::strcmp(argv[1], "graph") == 0;
  int *out, *ctr;
  cudaMalloc(&out, 8 * sizeof(int));
  cudaMalloc(&ctr, sizeof(int));
  cudaMemset(ctr, 0, sizeof(int));
  cudaStream_t s;
  cudaStreamCreate(&s);
  if (!graph) {
    for (int i = 0; i < 3; ++i) mbar_kernel<<<8, 64, 0, s>>>(out);
  } else {
    cudaGraph_t g;
    cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle h;
    cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t cn;
    cudaGraphAddNode(&cn, g, nullptr, 0, &cp);
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    mbar_kernel<<<8, 64, 0, s>>>(out);
    count_kernel<<<1, 32, 0, s>>>(ctr, h);
    cudaGraph_t g2;
    cudaStreamEndCapture(s, &g2);
    cudaGraphExec_t ex;
    cudaGraphInstantiate(&ex, g, 0);
    cudaGraphLaunch(ex, s);
  }
  cudaError_t e = cudaStreamSynchronize(s);
  int h[8];
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  int c = 0;
  cudaMemcpy(&c, ctr, sizeof(int), cudaMemcpyDeviceToHost);
  std::printf("%s: %s, out[0..7] = %d..%d, loop iterations %d\n", graph ? "graph" : "direct",
              cudaGetErrorString(e), h[0], h[7], graph ? c : 3);
  return e == cudaSuccess ? 0 : 1;
}
