#include <cstdio>
__global__ void k(unsigned long long* out) {
  unsigned long long prev, t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prev));
  unsigned long long mind = ~0ull; int changes = 0; long long c0 = clock64();
  for (int i = 0; i < 200000; ++i) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t != prev) { if (t - prev < mind) mind = t - prev; changes++; prev = t; }
  }
  long long c1 = clock64();
  out[0] = mind; out[1] = changes; out[2] = c1 - c0; out[3] = t;
}
int main() { unsigned long long* d; cudaMalloc(&d, 64); k<<<1,1>>>(d); unsigned long long h[4]; cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
  printf("min tick %llu ns, changes %llu over %llu cycles (%.1f us at 1.965 GHz), mod1024 %llu\n", h[0], h[1], h[2], h[2]/1965.0, h[3] % 1024); }
