// GPU twin of synth.py: integer counter hash -> bf16 bit patterns (see synth.py docstring).
// Every fp32 operation is a single IEEE round-to-nearest op (__fmul_rn/__fadd_rn, no FMA),
// so the bytes equal the numpy generator's.
#include "../../include/kv_synth.h"
#include <cuda_runtime.h>
#include <cstdint>

namespace {
constexpr uint64_t GOLD = 0x9E3779B97F4A7C15ull, M1 = 0xBF58476D1CE4E5B9ull, M2 = 0x94D049BB133111EBull;
constexpr int TID_K = 0, TID_V = 1, TID_Q = 2, TID_SAL = 3, TID_DIR = 4;
__device__ __constant__ float SIG_K = 0.8660254f, SIG_V = 0.8660254f, SIG_Q = 0.8660254f, C_Q = 1.0f,
                              W_MAG = 0.25f, TWO_M15 = 3.0517578125e-05f;

__device__ __forceinline__ uint64_t sm64(uint64_t x) {
  uint64_t z = x + GOLD;
  z = (z ^ (z >> 30)) * M1;
  z = (z ^ (z >> 27)) * M2;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t row_key(uint64_t seed, int64_t tid, int64_t a, int64_t b, int64_t c, int64_t d) {
  uint64_t h = sm64(seed);
  h = sm64(h ^ (uint64_t)tid);
  h = sm64(h ^ (uint64_t)a);
  h = sm64(h ^ (uint64_t)b);
  h = sm64(h ^ (uint64_t)c);
  h = sm64(h ^ (uint64_t)d);
  return h;
}
__device__ __forceinline__ float gauss(uint64_t u) {
  const int64_t s = (int64_t)(u & 0xFFFF) + (int64_t)((u >> 16) & 0xFFFF) + (int64_t)((u >> 32) & 0xFFFF) +
                    (int64_t)(u >> 48);
  return __fmul_rn((float)(s - 131070), TWO_M15);
}
__device__ __forceinline__ uint16_t bf16_rne(float x) {
  uint32_t u = __float_as_uint(x);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
__device__ __forceinline__ float salience(uint64_t seed, int b, int pos, int P, int ks, float sig_a) {
  float a = __fmul_rn(gauss(sm64(row_key(seed, TID_SAL, b, pos, 0, 0))), sig_a);
  if (pos >= P && pos < P + ks) a = __fadd_rn(a, __fmul_rn(4.0f, sig_a));
  return a;
}
__device__ __forceinline__ float direction(uint64_t seed, int l, int g, int dim) {
  const uint64_t u = sm64(row_key(seed, TID_DIR, l, g, 0, 0) + (uint64_t)dim);
  return (u >> 63) ? -W_MAG : W_MAG;
}

__global__ void k_gen_kv(uint64_t seed, int which, int L, int B, int Hkv, int d, int pos0, int npos, int P,
                         int ks, float sig_a, uint16_t* out, int l0) {
  const size_t total = (size_t)L * B * Hkv * npos * d;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    size_t r = e;
    const int dim = (int)(r % d); r /= d;
    const int p = (int)(r % npos); r /= npos;
    const int h = (int)(r % Hkv); r /= Hkv;
    const int b = (int)(r % B); r /= B;
    const int l = l0 + (int)r;                  // layers [l0, l0 + L)
    const int pos = pos0 + p;
    const uint64_t key = row_key(seed, which == 0 ? TID_K : TID_V, l, b, h, pos);
    const float x = gauss(sm64(key + (uint64_t)dim));
    float val;
    if (which == 1) val = __fmul_rn(x, SIG_V);
    else val = __fadd_rn(__fmul_rn(x, SIG_K), __fmul_rn(salience(seed, b, pos, P, ks, sig_a), direction(seed, l, h, dim)));
    out[e] = bf16_rne(val);
  }
}

__global__ void k_gen_q(uint64_t seed, int t0, int T, int L, int B, int Hq, int Hkv, int d, uint16_t* out) {
  const int G = Hq / Hkv;
  const size_t total = (size_t)T * L * B * Hq * d;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (size_t)gridDim.x * blockDim.x) {
    size_t r = e;
    const int dim = (int)(r % d); r /= d;
    const int h = (int)(r % Hq); r /= Hq;
    const int b = (int)(r % B); r /= B;
    const int l = (int)(r % L); r /= L;
    const int t = t0 + (int)r;
    const float x = gauss(sm64(row_key(seed, TID_Q, t, l, b, h) + (uint64_t)dim));
    out[e] = bf16_rne(__fadd_rn(__fmul_rn(x, SIG_Q), __fmul_rn(C_Q, direction(seed, l, h / G, dim))));
  }
}
int grid_for(size_t total) {
  size_t g = (total + 255) / 256;
  return (int)(g > 148 * 64 ? 148 * 64 : (g ? g : 1));
}
}  // namespace

extern "C" int kv_synth_kv(uint64_t seed, int which, int L, int B, int Hkv, int d, int pos0, int npos,
                           int prompt_len, int sink_size, float sig_a, void* out, void* stream) {
  const size_t total = (size_t)L * B * Hkv * npos * d;
  if (total == 0) return 0;
  k_gen_kv<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(seed, which, L, B, Hkv, d, pos0, npos, prompt_len,
                                                            sink_size, sig_a, (uint16_t*)out, 0);
  return (int)cudaGetLastError();
}
extern "C" int kv_synth_kv_layer(uint64_t seed, int which, int layer, int B, int Hkv, int d, int pos0, int npos,
                                 int prompt_len, int sink_size, float sig_a, void* out, void* stream) {
  const size_t total = (size_t)B * Hkv * npos * d;
  if (total == 0) return 0;
  k_gen_kv<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(seed, which, 1, B, Hkv, d, pos0, npos, prompt_len,
                                                            sink_size, sig_a, (uint16_t*)out, layer);
  return (int)cudaGetLastError();
}
extern "C" int kv_synth_q(uint64_t seed, int t0, int T, int L, int B, int Hq, int Hkv, int d, void* out,
                          void* stream) {
  const size_t total = (size_t)T * L * B * Hq * d;
  if (total == 0) return 0;
  k_gen_q<<<grid_for(total), 256, 0, (cudaStream_t)stream>>>(seed, t0, T, L, B, Hq, Hkv, d, (uint16_t*)out);
  return (int)cudaGetLastError();
}
extern "C" int kv_synth_row(uint64_t seed, int which, int L, int B, int Hkv, int d, int pos, int prompt_len,
                            int sink_size, float sig_a, void* out, void* stream) {
  return kv_synth_kv(seed, which, L, B, Hkv, d, pos, 1, prompt_len, sink_size, sig_a, out, stream);
}
