// Unit check of the tcgen05 (UMMA) operand conventions the step kernel relies on, on the store
// layout of kv_internal.cuh (8-row groups, 128-byte column blocks, chunk ^ (row & 7)):
//   S[128 tok][16]  = K[128 tok][128 d] . q[16][128 d]^T      A K-major SW128, B K-major SW128
//   O[128 d][32]    = V[128 tok][128 d]^T . P[32][128 tok]^T  A MN-major SW128, B K-major SW128
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_check umma_check.cu && ./umma_check
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint32_t tile_off(int row, int c) {   // D = 128
  return ((uint32_t)(row >> 3) << 11) + ((uint32_t)(c >> 3) << 10) + ((uint32_t)(row & 7) << 7) +
         ((uint32_t)((c & 7) ^ (row & 7)) << 4);
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// SM100 shared-memory matrix descriptor: start >> 4 [0,14), LBO >> 4 [16,30), SBO >> 4 [32,46),
// version 1 [46,48), base offset 0, layout type [61,64) (SWIZZLE_128B = 2)
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
// instruction descriptor: f32 accumulate, bf16 A/B, majors, N >> 3 at [17,23), M >> 4 at [24,29)
__host__ __device__ constexpr uint32_t idesc(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t tmem, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
               " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
               ::"r"(tmem), "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(mbar) : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t n) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(n)); }
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t par) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(a), "r"(par) : "memory");
  } while (!ok);
}

__global__ void k(const __nv_bfloat16* K, const __nv_bfloat16* q, const __nv_bfloat16* V, const __nv_bfloat16* P,
                  float* S_out, float* O_out, int mn_lbo, int mn_sbo) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* sK = sm;                 // 32 KB
  unsigned char* sV = sm + 32768;         // 32 KB
  unsigned char* sq = sm + 65536;         // 16 rows: 4 KB
  unsigned char* sP = sm + 69632;         // 32 rows: 8 KB
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 77824);
  uint32_t* tbase = reinterpret_cast<uint32_t*>(sm + 77840);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 128 * 16; i += 128) {              // 16-byte chunks
    const int r = i / 16, c = i % 16;
    *reinterpret_cast<uint4*>(sK + tile_off(r, c)) = *reinterpret_cast<const uint4*>(K + r * 128 + c * 8);
    *reinterpret_cast<uint4*>(sV + tile_off(r, c)) = *reinterpret_cast<const uint4*>(V + r * 128 + c * 8);
  }
  for (int i = tid; i < 16 * 16; i += 128) {
    const int r = i / 16, c = i % 16;
    *reinterpret_cast<uint4*>(sq + tile_off(r, c)) = *reinterpret_cast<const uint4*>(q + r * 128 + c * 8);
  }
  for (int i = tid; i < 32 * 16; i += 128) {
    const int r = i / 16, c = i % 16;
    *reinterpret_cast<uint4*>(sP + tile_off(r, c)) = *reinterpret_cast<const uint4*>(P + r * 128 + c * 8);
  }
  if (tid == 0) { mbar_init(smem_u32(bar), 1); mbar_init(smem_u32(bar + 1), 1); }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;\n" ::"r"(smem_u32(tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tm = *tbase;
  if (tid == 0) {
    const uint32_t idS = idesc(128, 16, 0, 0);
    for (int kk = 0; kk < 8; ++kk) {                      // K = d in steps of 16 (32 B)
      const uint32_t off = (kk >> 2) * 1024 + (kk & 3) * 32;
      mma(tm, sdesc(smem_u32(sK) + off, 16, 2048), sdesc(smem_u32(sq) + off, 16, 2048), idS, kk > 0);
    }
    commit(smem_u32(bar));
    const uint32_t idO = idesc(128, 32, 1, 0);
    for (int kk = 0; kk < 8; ++kk) {                      // K = tokens in steps of 16 (two 8-row groups)
      mma(tm + 32, sdesc(smem_u32(sV) + kk * 4096, mn_lbo, mn_sbo),
          sdesc(smem_u32(sP) + (kk >> 2) * 1024 + (kk & 3) * 32, 16, 2048), idO, kk > 0);
    }
    commit(smem_u32(bar + 1));
  }
  mbar_wait(smem_u32(bar), 0);
  mbar_wait(smem_u32(bar + 1), 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  uint32_t r[32];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(tm + ((uint32_t)(32 * w) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
  for (int j = 0; j < 16; ++j) S_out[(32 * w + lane) * 16 + j] = __uint_as_float(r[j]);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                 "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                 "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
               : "r"(tm + 32 + ((uint32_t)(32 * w) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
  for (int j = 0; j < 32; ++j) O_out[(32 * w + lane) * 32 + j] = __uint_as_float(r[j]);
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;\n" ::"r"(tm));
}

int main(int argc, char** argv) {
  srand(3);
  auto rnd = [] { return (float)(rand() % 2001 - 1000) / 500.0f; };
  std::vector<__nv_bfloat16> K(128 * 128), V(128 * 128), q(16 * 128), P(32 * 128);
  std::vector<float> Kf(K.size()), Vf(V.size()), qf(q.size()), Pf(P.size());
  for (size_t i = 0; i < K.size(); ++i) { K[i] = __float2bfloat16(rnd()); Kf[i] = __bfloat162float(K[i]); }
  for (size_t i = 0; i < V.size(); ++i) { V[i] = __float2bfloat16(rnd()); Vf[i] = __bfloat162float(V[i]); }
  for (size_t i = 0; i < q.size(); ++i) { q[i] = __float2bfloat16(rnd()); qf[i] = __bfloat162float(q[i]); }
  for (size_t i = 0; i < P.size(); ++i) { P[i] = __float2bfloat16(rnd()); Pf[i] = __bfloat162float(P[i]); }
  __nv_bfloat16 *dK, *dV, *dq, *dP;
  float *dS, *dO;
  cudaMalloc(&dK, K.size() * 2); cudaMalloc(&dV, V.size() * 2); cudaMalloc(&dq, q.size() * 2); cudaMalloc(&dP, P.size() * 2);
  cudaMalloc(&dS, 128 * 16 * 4); cudaMalloc(&dO, 128 * 32 * 4);
  cudaMemcpy(dK, K.data(), K.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dV, V.data(), V.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dq, q.data(), q.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dP, P.data(), P.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  const int cand[][2] = {{1024, 2048}, {2048, 1024}};
  for (auto& cd : cand) {
    cudaMemset(dS, 0, 128 * 16 * 4);
    cudaMemset(dO, 0, 128 * 32 * 4);
    k<<<1, 128, 80 * 1024>>>(dK, dq, dV, dP, dS, dO, cd[0], cd[1]);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<float> S(128 * 16), O(128 * 32);
    cudaMemcpy(S.data(), dS, S.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
    double es = 0, eo = 0;
    for (int t = 0; t < 128; ++t)
      for (int h = 0; h < 16; ++h) {
        double ref = 0;
        for (int d = 0; d < 128; ++d) ref += (double)Kf[t * 128 + d] * qf[h * 128 + d];
        es = fmax(es, fabs(ref - S[t * 16 + h]));
      }
    for (int d = 0; d < 128; ++d)
      for (int n = 0; n < 32; ++n) {
        double ref = 0;
        for (int t = 0; t < 128; ++t) ref += (double)Vf[t * 128 + d] * Pf[n * 128 + t];
        eo = fmax(eo, fabs(ref - O[d * 32 + n]));
      }
    printf("MN-major LBO=%d SBO=%d: max|S err| = %.3g, max|O err| = %.3g\n", cd[0], cd[1], es, eo);
  }
  return 0;
}
