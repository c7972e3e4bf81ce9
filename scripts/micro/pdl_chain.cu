// Floor of a PDL-chained kernel sequence: A (256 CTAs x 192 thr) -> B (32 CTAs x 256 thr) -> A ...
// each kernel: launch_dependents, griddepcontrol.wait, one store.  Also A -> A chains and plain
// (no PDL) launches, inside a CUDA graph, timed with events.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void kA(int* p, int x) {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) p[blockIdx.x] = x;
}
__global__ void kB(int* p, int x) {
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) p[1024 + blockIdx.x] = x + p[blockIdx.x];
}
static void launch(void (*k)(int*, int), dim3 g, dim3 b, int* p, int x, cudaStream_t s, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = g; cfg.blockDim = b; cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k, p, x);
}
int main() {
  int* p; cudaMalloc(&p, 1 << 20);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  for (int mode = 0; mode < 4; ++mode) {      // 0: A-B pdl, 1: A-B plain, 2: A-A pdl, 3: A-A plain
    const bool pdl = mode == 0 || mode == 2, pair = mode < 2;
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int l = 0; l < 28; ++l) {
      launch(kA, dim3(256), dim3(192), p, l, s, pdl && l > 0);
      if (pair) launch(kB, dim3(32), dim3(256), p, l, s, pdl);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    for (int i = 0; i < 20; ++i) cudaGraphLaunch(ge, s);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, s);
    for (int i = 0; i < 200; ++i) cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const char* nm[] = {"A->B PDL", "A->B plain", "A->A PDL", "A->A plain"};
    printf("%-12s %.2f us per layer (28 layers per graph)\n", nm[mode], ms * 1e3 / 200 / 28);
  }
  return 0;
}
