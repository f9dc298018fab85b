// launch_probe.cu -- dev probe: the cost of a kernel boundary in a captured
// graph, with and without programmatic dependent launch (PDL): a chain of K
// near-empty kernels (grid = SMs, 128 threads; each waits for its
// predecessor, then lets its successor launch) replayed as one graph.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/launch_probe tools/launch_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void step(int* buf, int k) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0) buf[blockIdx.x] += k;
}

static float run(int K, bool pdl, int blocks, int threads, size_t smem) {
  int* buf;
  cudaMalloc(&buf, 4096 * 4);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaFuncSetAttribute(step, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaGraph_t g;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int k = 0; k < K; ++k) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = (pdl && k > 0) ? 1 : 0;
    cudaLaunchKernelEx(&cfg, step, buf, k);
  }
  cudaStreamEndCapture(st, &g);
  cudaGraphExec_t ge;
  cudaGraphInstantiate(&ge, g, 0);
  for (int i = 0; i < 20; ++i) cudaGraphLaunch(ge, st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, st);
  for (int i = 0; i < 200; ++i) cudaGraphLaunch(ge, st);
  cudaEventRecord(e1, st);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1000.f / 200 / K;
}

int main() {
  for (size_t smem : {(size_t)0, (size_t)200 * 1024})
    for (int pdl = 0; pdl < 2; ++pdl)
      for (int blocks : {148, 592})
        printf("smem %3zu KB  pdl %d  blocks %3d: %.2f us per kernel (chain of 24)\n", smem / 1024, pdl, blocks,
               run(24, pdl, blocks, 128, smem));
  return 0;
}
