/*
 * kv_synth.h -- seeded synthetic-input generator (GPU twin of
 * paper_2605_09490_b200/synth/synth.py).  Test/bench plumbing, not the method:
 * it writes bf16 K/V/q bit patterns into device buffers.  Byte-identical to the
 * CPU generator for the same (seed, indices).  Returns 0 or a cudaError_t value.
 */
#ifndef KV_SYNTH_H_
#define KV_SYNTH_H_
#include <stdint.h>
#if defined(__GNUC__)
#define KV_SYNTH_API __attribute__((visibility("default")))
#else
#define KV_SYNTH_API
#endif

#ifdef __cplusplus
extern "C" {
#endif
/* out: device bf16 [L][B][Hkv][npos][d] of K (which=0) or V (which=1), positions pos0.. */
KV_SYNTH_API int kv_synth_kv(uint64_t seed, int which, int L, int B, int Hkv, int d, int pos0, int npos,
                int prompt_len, int sink_size, float sig_a, void* out, void* stream);
/* out: device bf16 [B][Hkv][npos][d]: layer `layer` of kv_synth_kv's tensor (same bytes), so a large
 * prefix can be generated and loaded one layer at a time */
KV_SYNTH_API int kv_synth_kv_layer(uint64_t seed, int which, int layer, int B, int Hkv, int d, int pos0, int npos,
                      int prompt_len, int sink_size, float sig_a, void* out, void* stream);
/* out: device bf16 [T][L][B][Hq][d] of queries for steps t0..t0+T-1 */
KV_SYNTH_API int kv_synth_q(uint64_t seed, int t0, int T, int L, int B, int Hq, int Hkv, int d, void* out, void* stream);
/* out: device bf16 [L][B][Hkv][d] K (which=0) / V (which=1) rows of one position (per-step append) */
KV_SYNTH_API int kv_synth_row(uint64_t seed, int which, int L, int B, int Hkv, int d, int pos,
                 int prompt_len, int sink_size, float sig_a, void* out, void* stream);
#ifdef __cplusplus
}
#endif
#endif
