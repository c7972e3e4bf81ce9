// Legacy tensor path on sm_100a: throughput and latency of mma.sync.m16n8k16 bf16 -> fp32
// (the step kernel's QK / PV instruction).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hmma_rate hmma_rate.cu
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ void mma16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
template <int CH>
__global__ void k(float* out, long long* cyc, int iters, uint32_t seed) {
  float acc[CH][4] = {};
  uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) mma16816(acc[c], a0, a1, a2, a3, b0, b1);
  }
  long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int CH>
void run(int warps, const char* what) {
  float* out; long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  k<CH><<<148, warps * 32>>>(out, cyc, 16, 1);
  k<CH><<<148, warps * 32>>>(out, cyc, iters, 1);
  cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double mma_per_smsp = (double)iters * CH * warps / 4.0;
  printf("%-28s warps/SM %2d chains %d: %.2f cycles per HMMA per SMSP, %.1f cycles per HMMA per warp\n", what, warps, CH,
         h[0] / mma_per_smsp, (double)h[0] / (iters * CH));
  cudaFree(out); cudaFree(cyc);
}
int main() {
  run<1>(1, "latency (1 dependent chain)");
  run<8>(1, "1 warp, 8 chains");
  run<8>(4, "4 warps, 8 chains");
  run<8>(8, "8 warps, 8 chains");
  run<8>(16, "16 warps, 8 chains");
  run<4>(32, "32 warps, 4 chains");
  return 0;
}
