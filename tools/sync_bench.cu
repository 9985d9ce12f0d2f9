// Micro-benchmark: cost of cooperative grid.sync() vs dependent kernel nodes in a CUDA
// graph (with and without programmatic dependent launch), on the B200.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void syncs(int n, int* x) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < n; ++i) { if (threadIdx.x == 0 && blockIdx.x == 0) x[0] += 1; g.sync(); }
}
__global__ void tiny(int* x) { if (threadIdx.x == 0 && blockIdx.x == 0) x[0] += 1; }
__global__ void tiny_pdl(int* x) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0 && blockIdx.x == 0) x[0] += 1;
  asm volatile("griddepcontrol.launch_dependents;");
}
__global__ void custom_bar(int n, unsigned* cnt, volatile unsigned* gen, int* x) {
  // sense-reversal barrier: one arrival per CTA
  for (int i = 0; i < n; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned g0 = *gen;
      __threadfence();
      if (atomicAdd(cnt, 1) == gridDim.x - 1) { *cnt = 0; __threadfence(); *gen = g0 + 1; }
      else { while (*gen == g0) { } }
      __threadfence();
    }
    __syncthreads();
  }
}
int main() {
  int* x; cudaMalloc(&x, 64); unsigned* c; cudaMalloc(&c, 64); cudaMemset(c, 0, 64);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int N = 200;
  int cfg[][2] = {{1, 1024}, {1, 512}, {1, 256}, {2, 1024}, {4, 256}, {8, 256}};
  for (auto& cf : cfg) {
    int grid = cf[0] * nsm, tpb = cf[1], n = N;
    void* args[] = {&n, &x};
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(a, s);
      cudaLaunchCooperativeKernel((void*)syncs, grid, tpb, args, 0, s);
      cudaEventRecord(b, s); cudaEventSynchronize(b);
    }
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("grid.sync  %4d CTAs x %4d thr: %.3f us/sync\n", grid, tpb, ms * 1e3 / N);
    void* args2[] = {&n, &c, &c + 0, &x};
    unsigned* gen = c + 16;
    void* args3[] = {&n, &c, &gen, &x};
    for (int w = 0; w < 2; ++w) {
      cudaEventRecord(a, s);
      cudaLaunchCooperativeKernel((void*)custom_bar, grid, tpb, args3, 0, s);
      cudaEventRecord(b, s); cudaEventSynchronize(b);
    }
    cudaEventElapsedTime(&ms, a, b);
    printf("custom bar %4d CTAs x %4d thr: %.3f us/sync  (err %s)\n", grid, tpb, ms * 1e3 / N, cudaGetErrorString(cudaGetLastError()));
  }
  for (int grid : {1, 148, 592, 1184}) {
    for (int pdl = 0; pdl < 2; ++pdl) {
      cudaGraph_t g; cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
      for (int i = 0; i < N; ++i) {
        if (!pdl) tiny<<<grid, 256, 0, s>>>(x);
        else {
          cudaLaunchConfig_t lc = {}; lc.gridDim = grid; lc.blockDim = 256; lc.stream = s;
          cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = 1; lc.attrs = at; lc.numAttrs = 1;
          cudaLaunchKernelEx(&lc, tiny_pdl, x);
        }
      }
      cudaStreamEndCapture(s, &g); cudaGraphInstantiate(&ge, g, 0);
      for (int w = 0; w < 2; ++w) {
        cudaEventRecord(a, s); cudaGraphLaunch(ge, s); cudaEventRecord(b, s); cudaEventSynchronize(b);
      }
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("graph node grid=%4d pdl=%d: %.3f us/kernel (err %s)\n", grid, pdl, ms * 1e3 / N, cudaGetErrorString(cudaGetLastError()));
    }
  }
  for (int grid : {148, 1184}) {
    cudaEventRecord(a, s);
    for (int i = 0; i < N; ++i) tiny<<<grid, 256, 0, s>>>(x);
    cudaEventRecord(b, s); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("stream launch grid=%4d: %.3f us/kernel\n", grid, ms * 1e3 / N);
  }
  return 0;
}
