// Internal device-side view of a kv_tier ctx (shared by the kernels of libkvtier.so).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

namespace kvt {

constexpr int T0 = 0, T1 = 1, T2 = 2, T3 = 3;
constexpr int NTRACE = 24;        // debug trace slots per CTA (KVTIER_TRACE=1)
constexpr int CNT_STRIDE = 8;     // cnt[buf][b][8]: |T0| |T1| |T2| |T3| |visible at event| pad..
constexpr int ZRING = 4;          // max logits/ML ring slots (score kernels lag the decode chain);
                                  // DevView::zring <= ZRING are used (zring_of in ctx.cu)
constexpr int ZBATCH = 1;         // launches whose score updates one score kernel applies (layer order;
                                  // measured: batching 4 made the kernel too big to share SMs with the chain)

// kv_tier_scorer: VATP (1) and combined (3) weight increments by ||v||; redundancy (2) and
// combined (3) rank by I - rho (DESIGN AMB-30/31)
__host__ __device__ constexpr bool scorer_uses_vnorm(int s) { return s == 1 || s == 3; }
__host__ __device__ constexpr bool scorer_uses_red(int s) { return s == 2 || s == 3 || s == 5; }
// windowed (4) and R-KV (5): classify ranks the max-pooled score of the last w steps (AMB-32)
__host__ __device__ constexpr bool scorer_uses_window(int s) { return s == 4 || s == 5; }
constexpr int RKV_ALPHA = 8;        // observation steps
constexpr int RKV_HALF_POOL = 3;    // max-pool kernel 7

// Mutable device state (graph-static kernels read it instead of taking args).
struct DevState {
  int n;            // current sequence length: positions [0, n)
  int t;            // decode step
  int cur;          // ping-pong buffer holding the live stores / lists
  int n_event;      // n at the last committed manage event
  int err;          // sticky error bits: 1 = non-finite probability/score, 2 = tier store overflow (shard),
                    // 4 = a device-side wait hit its 2 s watchdog
  int scur;         // row-store buffer (always 0: the stores are single-buffered, migrate works in place)
  int pad0, pad1;
  unsigned long long d2h_rows;   // rows written to the pinned host stores
  int nn;           // 1: this rank holds the step's new token (always 1 unless sequence-sharded)
};

struct DevView {
  int B, L, Hq, Hkv, G, D, Nmax;
  int cap0, cap1, cap2;
  int P, ks, kw;
  int hbm_bp, evict_bp, t2_bp, evict_mode;
  int policy, budget;   // kv_tier_policy (tier policy of a5), kept tokens (H2O / RANDOM)
  int scorer;           // kv_tier_scorer (a4 increment: attention, or attention x ||v|| for VATP)
  float* vnorm;         // VATP / combined: [L][B][Hkv][Nmax] fp32 L2 norm of each token's V row (else null)
  float* red;           // redundancy / combined: [B][Hkv][Nmax] fp32 R_part = sum_l cos(k_i, k_{i-1})
  uint16_t* lastk;      // redundancy / combined: [L][B][Hkv][D] bf16 key of the last appended token
  float* snap;          // windowed / R-KV: [B][Hkv][Nmax] S_part at the start of the observation window
  float* pool;          // windowed / R-KV: classify scratch [B][Nmax] compacted scores + [B][Nmax] int indices
  int interval;         // Delta (kv_tier_config::manage_interval; binding for windowed scorers)
  int* zlayer;          // [ZRING] layer of the launch that filled each logit slot
  int zring;            // logit ring slots in use (2..ZRING): the ring stays inside the L2 carve-out
  unsigned policy_seed;
  int stream_mode;      // staging_tokens == 0
  int host_t1;          // N1: T1 attended on the host (kv_tier_set_host_t1); kernels skip T1
  int out_fp32;
  int split;            // CTAs per (b, g) cluster
  int variant;          // decode-attention kernel variant (warps x pipeline stages)
  int seq_w, seq_r;     // sequence sharding: positions in 64-blocks, block k owned by rank k % seq_w
  int hN;               // rows per group of the pinned host stores (N_max, or a shard's own positions)
  int score_grid;       // CTAs of the score-flush kernel (runs beside the attention chain)
  unsigned long long* trace;   // debug: per-CTA %globaltimer checkpoints (null = off)
  float* zbuf;          // [ZRING][B*Hkv][zrows][8] logits (log2 domain) of recent launches
  float* ml;            // [ZRING][B*Hkv][16] per-head (max, 1/sum) of recent launches
  int zrows;            // virtual rows per unit (N_max + padding)
  float* part;          // [B*Hkv][split][part_stride] per-CTA partials (m[8], l[8], o[G][D])
  int part_stride;
  // whole-step kernel (step.cu): step_k CTAs in all; step_s > 1: a cluster of step_s CTAs per kv
  // head (row slices), else step_m kv heads per CTA.  step_k = 0: the step runs per layer.
  int step_k, step_s, step_m;
  int split_req;        // kv_tier_config::split (0 = auto): also fixes the step kernel's CTAs per kv head
  int step_nw;          // consumer warps per CTA: 8 (one CTA per SM) or 4 (two CTAs per SM)
  int step_um;          // 1: the tcgen05 consumer (4 softmax warps + the MMA-issuing warp, one CTA per SM)
  int step_um_ok;       // kv_tier_config::step_kernel == 2
  int* step_done;       // [L][B] CTAs of request b that finished layer l (zeroed by k_begin_step)
  void* hot_base;       // L2 access-policy window over the small hot buffers
  size_t hot_bytes;
  float hot_hit;        // hitRatio of the window: persisting carve-out / window bytes (<= 1)
  int4* moves;          // [B][mcap] {src tier, src row, dst tier | dst row << 2, position}
  int* mcount;          // [B] moves of the last plan (<= mcap)
  int mcap;             // moves per request (>= N: an event never overflows)
  int mchunk;           // mtemp holds B * mcap * mchunk rows: mchunk pairs at the worst-case move count
  unsigned* gbar;       // grid barrier counter of k_migrate_rows (zeroed by k_plan)
  int c0_load;          // prefix positions loaded into T0 (the rest start in T1, AMB-26)
  int* scratch;         // [B][Nmax] plan scratch (hole rows)
  __nv_bfloat16* mtemp; // [B * mcap * mchunk][2][D] rows in flight during a migrate chunk
  __nv_bfloat16* k0[2]; __nv_bfloat16* v0[2];        // T0 store  [L][B][Hkv][cap0][D]
  __nv_bfloat16* k1[2]; __nv_bfloat16* v1[2];        // T1 staging [L][B][Hkv][cap1][D] (stream: [2][B][Hkv][cap1][D] in k1[0]/v1[0])
  int8_t* c2k[2]; int8_t* c2v[2];                      // T2 codes  [L][B][Hkv][cap2][D]
  float* s2k[2]; float* s2v[2];                        // T2 scales [L][B][Hkv][cap2]
  int* idx[2][3];                                      // [buf][tier] -> [B][cap_tier] ascending positions
  int* idxvis[2];                                      // [buf] -> [B][Nmax] ascending visible positions at event
  uint8_t* tier[2];                                    // [buf] -> [B][Nmax]
  int* rowof[2];                                       // [buf] -> [B][Nmax] row within the tier store
  int* cnt[2];                                         // [buf] -> [B][CNT_STRIDE]
  float* S;                                            // S_part [B][Hkv][Nmax]
  float* fS;                                           // scratch [B][Nmax]
  DevState* st;
  __nv_bfloat16* hk1; __nv_bfloat16* hv1;            // pinned host T1 [L][B][Hkv][hN][D] (mapped; host_row)
  int8_t* hc2k; int8_t* hc2v; float* hs2k; float* hs2v;   // pinned host T2 (mapped, may be null)
};

#ifndef KVT_INLINE_OFFLOAD
#define KVT_INLINE_OFFLOAD 0   // A/B builds only (-DKVT_INLINE_OFFLOAD=1): offload inside the migrate kernel
#endif

__device__ __forceinline__ unsigned long long gtimer() {   // %globaltimer (ns): watchdogs, debug traces
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// RANDOM tier policy: rank key of (request, position) = high 32 bits of
// splitmix64(splitmix64(seed << 32 | req) ^ pos) (the oracle implements the same generator).
__host__ __device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ unsigned random_key32(unsigned seed, int req, int pos) {
  return (unsigned)(splitmix64(splitmix64(((unsigned long long)seed << 32) | (unsigned)req) ^ (unsigned)pos) >> 32);
}
// (n_new, n_hbm, n_t2) of a manage event under the tier policy (kv_tier.h kv_tier_policy)
__host__ __device__ __forceinline__ void policy_counts(int policy, int budget, int hbm_bp, int evict_bp, int t2_bp,
                                                       int evict_mode, long long n_prot, long long nl, long long n3,
                                                       long long* n_new, long long* n_hbm, long long* n_t2) {
  if (policy == 1) {                 // STREAMING: only the protected sinks + window stay
    *n_new = nl; *n_hbm = 0; *n_t2 = 0;
    return;
  }
  if (policy == 2 || policy == 3) {  // H2O / RANDOM: protected + the top budget - |P| live tokens
    long long keep = budget - n_prot;
    keep = keep < 0 ? 0 : (keep > nl ? nl : keep);
    *n_new = nl - keep; *n_hbm = keep; *n_t2 = 0;
    return;
  }
  long long nn;                      // HIERARCHY: Alg. 1 floors in basis points (AMB-8/9/11)
  if (evict_mode == 0) {
    nn = ((long long)evict_bp * (nl + n3)) / 10000 - n3;
    if (nn < 0) nn = 0;
  } else {
    nn = ((long long)evict_bp * nl) / 10000;
  }
  const long long surv = nl - nn;
  *n_new = nn;
  *n_hbm = ((long long)hbm_bp * surv) / 10000;
  *n_t2 = ((long long)t2_bp * (surv - *n_hbm)) / 10000;
}

// ring slot of launch index i = zfirst + j: batches start ZBATCH-aligned and zring % ZBATCH == 0
// (ZBATCH = 1), so a batch never wraps and the slot is i itself (no division in the score passes)
__device__ __forceinline__ int zslot_of(const DevView&, int i) { return i; }
static_assert(ZBATCH == 1, "zring_of must keep zring % ZBATCH == 0 if ZBATCH grows");

// a4 weight of token (layer, unit, pos): 1 (Eq. 1) or its V-row norm (VATP)
__device__ __forceinline__ float score_weight(const DevView& v, int layer, int unit, int pos) {
  return scorer_uses_vnorm(v.scorer) ? v.vnorm[((size_t)layer * v.B * v.Hkv + unit) * v.Nmax + pos] : 1.f;
}

// Sequence sharding: block-cyclic ownership of SEQ_BLOCK-position blocks.
// A rank's tier stores and index lists hold only its own positions; the tier array and the
// scores cover every position (tiers are identical on every rank).
constexpr int SEQ_BLOCK = 64;
__host__ __device__ __forceinline__ bool seq_own(int seq_w, int seq_r, int pos) {
  return seq_w <= 1 || (pos / SEQ_BLOCK) % seq_w == seq_r;
}
// owned positions below n
__host__ __device__ __forceinline__ int seq_owned_below(int seq_w, int seq_r, int n) {
  if (seq_w <= 1) return n;
  const int full = n / SEQ_BLOCK, rem = n % SEQ_BLOCK;
  int c = (full / seq_w) * SEQ_BLOCK + (full % seq_w > seq_r ? SEQ_BLOCK : 0);
  if (full % seq_w == seq_r) c += rem;
  return c;
}
// position of the j-th owned position (ascending)
__host__ __device__ __forceinline__ int seq_pos_of(int seq_w, int seq_r, int j) {
  if (seq_w <= 1) return j;
  return ((j / SEQ_BLOCK) * seq_w + seq_r) * SEQ_BLOCK + j % SEQ_BLOCK;
}

// Row of position pos of group grp in the pinned host T1/T2 stores ([L][B][H_kv][hN] rows): a
// sequence shard keeps only its own positions there too (row = owned index).
__host__ __device__ __forceinline__ size_t host_row(const DevView& v, size_t grp, int pos) {
  return grp * (size_t)v.hN + (size_t)(v.seq_w > 1 ? seq_owned_below(v.seq_w, v.seq_r, pos) : pos);
}

__device__ __forceinline__ size_t grp_of(const DevView& v, int l, int b, int g) {
  return ((size_t)l * v.B + b) * v.Hkv + g;
}

// bf16 K/V rows in the T0 store and the T1 staging are stored pre-swizzled in the 128-byte
// swizzle atom of the tensor cores: every group of 8 rows holds its 128-byte column blocks one
// after the other (d = 64: one block, plain rows; d = 128: [8 rows x cols 0..63 | 8 rows x cols
// 64..127], 2 KB), and inside a block the 16-byte chunk c of row j sits at chunk c ^ (j & 7).  A
// linear bulk copy of whole 8-row groups into shared memory therefore lands in the layout both
// ldmatrix (bank-conflict-free) and a K-major / MN-major SWIZZLE_128B UMMA descriptor read.
// swz_off(j, e, D): element e of row j relative to j * D.
__host__ __device__ __forceinline__ int swz_off(int j, int e, int D) {
  const int c = (e >> 3) & 7, r = j & 7;
  return D == 128 ? ((e >> 6) << 9) + (r << 6) - (r << 7) + ((c ^ r) << 3) + (e & 7)
                  : (((c ^ r) << 3) | (e & 7));
}
// byte offset of 16-byte chunk c (0 .. D/8-1) of row `row` inside a shared-memory tile of rows
// (the same layout, tile starting at an 8-row boundary)
template <int D>
__device__ __forceinline__ uint32_t tile_off(int row, int c) {
  if constexpr (D == 128)
    return ((uint32_t)(row >> 3) << 11) + ((uint32_t)(c >> 3) << 10) + ((uint32_t)(row & 7) << 7) +
           ((uint32_t)((c & 7) ^ (row & 7)) << 4);
  else
    return ((uint32_t)row << 7) + ((uint32_t)(c ^ (row & 7)) << 4);
}
constexpr int STORE_SLACK_ROWS = 128;   // rows of slack after each bf16 store buffer

__device__ __forceinline__ float bf16_bits_to_f(uint16_t h) { return __uint_as_float(((uint32_t)h) << 16); }

// Redundancy (AMB-30), one full warp: c = cos(k_new, k_prev) of layer `layer`, unit (b, g), with
// k_prev the unit's previous key (lastk, zero before the first row); R_part[unit][pos] += c
// (layers append in ascending order, so the fp32 sum runs over l ascending); then k_new
// becomes the previous key.  krow: the new key's bf16 row (global memory).
__device__ __forceinline__ void redund_append(const DevView& v, int layer, int unit, int pos, const uint16_t* krow) {
  const int lane = threadIdx.x & 31;
  uint16_t* prev = v.lastk + ((size_t)layer * v.B * v.Hkv + unit) * v.D;
  float dot = 0.f, na = 0.f, nb = 0.f;
  for (int e = lane; e < v.D; e += 32) {
    const float a = bf16_bits_to_f(krow[e]), p = bf16_bits_to_f(prev[e]);
    dot = fmaf(a, p, dot);
    na = fmaf(a, a, na);
    nb = fmaf(p, p, nb);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    dot += __shfl_xor_sync(0xffffffffu, dot, off);
    na += __shfl_xor_sync(0xffffffffu, na, off);
    nb += __shfl_xor_sync(0xffffffffu, nb, off);
  }
  __syncwarp();
  for (int e = lane; e < v.D; e += 32) prev[e] = krow[e];
  if (lane == 0) {
    const float c = (na > 0.f && nb > 0.f) ? __fdiv_rn(dot, __fsqrt_rn(__fmul_rn(na, nb))) : 0.f;
    float* r = v.red + (size_t)unit * v.Nmax + pos;
    *r = __fadd_rn(*r, c);
  }
}

// fp32 -> bf16 round-to-nearest-even on the bit pattern (finite inputs)
__device__ __forceinline__ uint16_t f_to_bf16_bits(float x) {
  uint32_t u = __float_as_uint(x);
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}

}  // namespace kvt

// Launchers (defined in the .cu files, called by ctx.cu)
namespace kvt {
cudaError_t launch_begin_step(const DevView& v, cudaStream_t s);
cudaError_t launch_append(const DevView& v, int layer, const void* k, const void* vv, cudaStream_t s);
cudaError_t launch_load_prefix(const DevView& v, int layer, const void* k, const void* vv, int n0, cudaStream_t s);
cudaError_t launch_init_meta(const DevView& v, int n0, cudaStream_t s);
cudaError_t launch_decode_attn(const DevView& v, int layer, const void* q, const void* knew, const void* vnew,
                               void* o, int zpar, int pdl, cudaStream_t s, float* lse = nullptr);
cudaError_t launch_set_ml(const DevView& v, int zslot, const float* lse, cudaStream_t s);
cudaError_t launch_vnorm_prefix(const DevView& v, int layer, const void* vv, int n0, cudaStream_t s);
cudaError_t launch_t1_score_add(const DevView& v, const float* inc, cudaStream_t s);
cudaError_t launch_redund_prefix(const DevView& v, int layer, const void* k, int n0, cudaStream_t s);
cudaError_t launch_lse_combine(const float* op, const float* lp, int world, int rows, int d, float* oo, float* lo,
                               cudaStream_t s, float* ml = nullptr, int G = 1, size_t rs_o = 0, size_t rs_l = 0,
                               int pdl = 0);
// rs_o / rs_l: floats between consecutive ranks' o / (m, l) parts (0 = packed: rows * d, rows * 2)
cudaError_t launch_score_flush(const DevView& v, int zfirst, int nz, cudaStream_t s);
cudaError_t launch_score_update(const DevView& v, int layer, const float* probs, cudaStream_t s);
cudaError_t launch_end_step(const DevView& v, cudaStream_t s);
cudaError_t launch_classify(const DevView& v, const float* Sx, int parts, cudaStream_t s,
                            const float* snapx = nullptr);
cudaError_t launch_plan(const DevView& v, cudaStream_t s);
cudaError_t launch_migrate_rows(const DevView& v, cudaStream_t s);
cudaError_t launch_offload_rows(const DevView& v, cudaStream_t s);
cudaError_t launch_commit(const DevView& v, cudaStream_t s);
cudaError_t launch_prefetch(const DevView& v, int layer, cudaStream_t s);
size_t attn_smem_bytes(const DevView& v);
size_t merge_smem_bytes(const DevView& v);
cudaError_t attn_configure(const DevView& v);
size_t step_smem_bytes(const DevView& v);
cudaError_t step_configure(const DevView& v, int* clusters);
cudaError_t launch_decode_step(const DevView& v, const void* q, const void* knew, const void* vnew, void* o, int score,
                               cudaStream_t s);
}  // namespace kvt
