// Host side of libkvtier.so: config validation, memory carving, host-side state
// machine of Alg. 1, stream/event ordering, and the C ABI entry points.
#include "../../include/kv_tier.h"
#include "kv_internal.cuh"

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <dlfcn.h>
#include <nccl.h>      // types only: the functions are resolved at run time (no link-time NCCL)

using namespace kvt;

// NCCL, resolved from the libnccl.so.2 already in the process (torch's), else dlopen'ed: the
// library loads and runs without NCCL unless a ctx is created with an nccl_unique_id.
namespace {
struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};
const NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
    a.group_start = reinterpret_cast<decltype(a.group_start)>(dlsym(h, "ncclGroupStart"));
    a.group_end = reinterpret_cast<decltype(a.group_end)>(dlsym(h, "ncclGroupEnd"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.all_gather && a.group_start && a.group_end && a.error_string;
    return a;
  }();
  return api;
}
}  // namespace

struct kv_tier_ctx {
  kv_tier_config cfg;
  kv_tier_sizes sz;
  DevView v;
  // host mirror of the uniform-per-request state (all requests share n and P)
  int n = 0, t = 0, cur = 0, n0 = -1;
  int c[4] = {0, 0, 0, 0};            // |T0| |T1| |T2| |T3|
  int pend[4] = {0, 0, 0, 0};         // counts computed by the last classify
  int n_event = 0, nvis_event = 0;
  bool classified = false, step_open = false, loaded = false;
  std::vector<int> loaded_layers;
  void* host_t1 = nullptr;            // cudaHostAlloc base (K then V)
  void* host_t2 = nullptr;            // codes K, codes V, scales K, scales V
  cudaEvent_t ev_step_begin = nullptr, ev_migrated = nullptr, ev_offload_done = nullptr;
  cudaEvent_t ev_slot_free[2] = {nullptr, nullptr};
  std::vector<cudaEvent_t> ev_prefetched;
  std::vector<int> prefetched_step;
  std::vector<int> appended_step;          // step in which layer l's new row was written
  bool offload_pending = false;
  bool capturing = false;
  struct {                                 // host state saved by kv_tier_capture_begin
    int n, t, c0;
    bool classified;
    std::vector<int> pstep, astep;
  } cap;
  // per-layer ABI: may decode_attention chain to the previous library launch with programmatic
  // dependent launch?  Only when that launch was this step's decode_attention / append on the
  // same stream (begin_step, score flushes and migrate change state the kernel's prologue reads).
  bool pdl_ok = false;
  void* pdl_stream = nullptr;
  int zslot_next = 0;                      // logits/ML ring slot of the next fused decode_attention (0 at step start)
  int zpend_first = 0, zpend_n = 0;        // launches whose score update is not yet issued
  bool slot_busy[ZRING] = {};              // a score kernel may still read the slot
  bool scores_pending = false;             // score kernels not yet joined back into the main stream
  cudaStream_t score_stream = nullptr;     // a4 score updates run here, off the attention chain
  cudaStream_t offload_stream = nullptr;   // differential staging: rows entering T1/T2 -> pinned host
  cudaEvent_t ev_merged[ZRING] = {}, ev_scored[ZRING] = {}, ev_score_tail = nullptr;
  bool slot_recorded[2] = {false, false};   // ev_slot_free[x] recorded within the open step
  int lse_pending = -1;                    // score slot of a decode_attention_lse awaiting the global (M, L)
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  unsigned long long* trace = nullptr;     // debug timeline buffer (KVTIER_TRACE=1)
  // N1 host-T1 mode (kv_tier_set_host_t1)
  int mig_epoch = 0, h1_epoch = -1;        // migrates issued / epoch of the host copy of the T1 lists
  std::vector<int> h1_idx, h1_cnt;         // [B][cap1] T1 positions (store order), [B] |T1|
  std::vector<float> h1_z;                 // [B][H_q][cap1] logits of the last host_t1_attention
  int h1_layer = -1;                       // layer whose logits h1_z holds (-1: none pending)
  float* h1_inc[2] = {nullptr, nullptr};   // pinned mapped score increments, double-buffered
  // kv_tier_host_t1_layer: pinned q / partial / lse staging and device partials
  uint16_t* h1_q = nullptr;
  float* h1_o = nullptr;                   // [B][H_q][d] host partial o, then [B][H_q][2] lse, then lse_global
  float* d1_parts = nullptr;               // device: o parts [2][B][H_q][d], lse parts [2][B][H_q][2], lse [B][H_q][2]
  cudaEvent_t ev_q = nullptr;
  cudaEvent_t ev_inc[2] = {nullptr, nullptr};
  bool inc_used[2] = {false, false};
  // sequence sharding with a library-owned communicator (kv_tier_init with an nccl_unique_id):
  // every layer's (o, m, l) all-gather + LSE combine + score rescale run inside kv_tier_step /
  // the step graph; events all-gather S_part inside kv_tier_classify
  ncclComm_t comm = nullptr;
  float* x_recv = nullptr;                 // [W] slots of x_slot floats: [B][H_q][d] o part, then [B][H_q][2] (m, l)
  size_t x_slot = 0;                       // floats per rank slot (rounded up to 16 B)
  float* x_lse = nullptr;                  // [L][B][H_q][2] global (M, L) per layer
  float* x_scores = nullptr;               // [W][B][H_kv][N_max] all-gathered S_part (events)
  float* x_snaps = nullptr;                // [W][B][H_kv][N_max] all-gathered S_part snapshots (windowed scorers)
  std::string err;
};

static inline float __uint_as_float_host(uint32_t u) {
  float f;
  memcpy(&f, &u, 4);
  return f;
}

namespace {

thread_local std::string g_err;

kv_tier_status fail(kv_tier_ctx* ctx, kv_tier_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  if (ctx) ctx->err = buf;
  g_err = buf;
  return st;
}

kv_tier_status cuda_check(kv_tier_ctx* ctx, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return KV_TIER_OK;
  return fail(ctx, KV_TIER_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }
int round16(long long x) { return (int)((x + 15) / 16 * 16); }

// CTAs per unit: one wave of at most 2 decode CTAs per SM (rounding up would start a second,
// partial wave: measured at 14B, 3 -> 2 CTAs per unit took 382 -> 401 steps/s)
int split_of(const kv_tier_config& c) {
  if (c.split > 0) return c.split;
  const int units = c.num_requests * c.num_kv_heads;
  return std::max(1, std::min(8, (2 * 148) / units));
}

int auto_split(const kv_tier_config& c) { return split_of(c); }

// Logit ring slots: as many as fit a 60 MB share of the L2 persisting carve-out (2..ZRING).  A
// ring larger than that thrashes L2 against the KV stream; long layers need fewer slots (the
// score kernel lags the chain by about a layer).  Measured (profiles/r01/zring_r01.md): 32B
// B=16 2 slots 146 vs 4 slots 128 steps/s; 14B 3 slots 431, 4 slots 416, 2 slots 369; 7B 4
// slots 3005 vs 2 slots 2499.
int zring_of(const kv_tier_config& c) {
  const size_t slot = (size_t)c.num_requests * c.num_kv_heads * (c.max_tokens + 64) * 8 * 4;
  int k = ZRING;
  while (k > 2 && (size_t)k * slot > ((size_t)60 << 20)) --k;
  return k;
}

kv_tier_status validate(const kv_tier_config* c) {
  if (!c) return fail(nullptr, KV_TIER_E_INVAL, "null config");
  if (c->num_requests < 1 || c->num_requests > 1024) return fail(nullptr, KV_TIER_E_INVAL, "num_requests out of range");
  if (c->num_layers < 1) return fail(nullptr, KV_TIER_E_INVAL, "num_layers < 1");
  if (c->num_kv_heads < 1 || c->num_q_heads % c->num_kv_heads != 0)
    return fail(nullptr, KV_TIER_E_INVAL, "num_q_heads must be a multiple of num_kv_heads");
  if (c->num_q_heads / c->num_kv_heads > 8) return fail(nullptr, KV_TIER_E_INVAL, "GQA group > 8 not supported");
  if (c->head_dim != 64 && c->head_dim != 128) return fail(nullptr, KV_TIER_E_INVAL, "head_dim must be 64 or 128");
  if (c->max_tokens < 2) return fail(nullptr, KV_TIER_E_INVAL, "max_tokens < 2");
  if (c->prompt_len < 0 || c->sink_size < 0 || c->window_size < 1)
    return fail(nullptr, KV_TIER_E_INVAL, "window_size must be >= 1 (AMB-20) and P, k_s >= 0");
  if (c->hbm_ratio_bp > 10000 || c->evict_ratio_bp > 10000 || c->t2_fraction_bp > 10000)
    return fail(nullptr, KV_TIER_E_INVAL, "ratios are basis points in [0, 10000]");
  if (c->evict_mode != 0 && c->evict_mode != 1) return fail(nullptr, KV_TIER_E_INVAL, "bad evict_mode");
  if (c->staging_tokens != 0 && c->staging_tokens != KV_TIER_STAGING_ALL)
    return fail(nullptr, KV_TIER_E_INVAL, "staging_tokens must be 0 (stream) or KV_TIER_STAGING_ALL (differential)");
  if (c->shard != KV_TIER_SHARD_REQUEST && c->shard != KV_TIER_SHARD_KVHEAD && c->shard != KV_TIER_SHARD_SEQUENCE)
    return fail(nullptr, KV_TIER_E_INVAL, "shard must be REQUEST, KVHEAD or SEQUENCE");
  if (c->world < 1 || c->rank < 0 || c->rank >= c->world) return fail(nullptr, KV_TIER_E_INVAL, "need 0 <= rank < world");
  if (c->split < 0 || c->split > 64) return fail(nullptr, KV_TIER_E_INVAL, "split must be in [0, 64]");
  if (c->variant < 0 || c->variant > 5) return fail(nullptr, KV_TIER_E_INVAL, "variant must be in [0, 5]");
  if (c->step_kernel < 0 || c->step_kernel > 3)
    return fail(nullptr, KV_TIER_E_INVAL, "step_kernel must be 0 (auto), 1 (mma.sync), 2 (tcgen05) or 3 (per-layer kernels)");
  if (c->policy < KV_TIER_POLICY_HIERARCHY || c->policy > KV_TIER_POLICY_RANDOM)
    return fail(nullptr, KV_TIER_E_INVAL, "policy must be a kv_tier_policy");
  if (c->scorer < KV_TIER_SCORER_ATTENTION || c->scorer > KV_TIER_SCORER_RKV)
    return fail(nullptr, KV_TIER_E_INVAL, "scorer must be a kv_tier_scorer");

  if (scorer_uses_window(c->scorer) && c->manage_interval < 1)
    return fail(nullptr, KV_TIER_E_INVAL, "windowed scorers need manage_interval >= 1 (the observation window follows it)");

  if ((c->policy == KV_TIER_POLICY_H2O || c->policy == KV_TIER_POLICY_RANDOM) && c->budget < 1)
    return fail(nullptr, KV_TIER_E_INVAL, "H2O / RANDOM need budget >= 1 kept tokens per request");
  return KV_TIER_OK;
}

// Capacities (rows per (l, b, g)).  T0 holds the steady state, not the whole chain: after an
// event P u the top n_hbm survivors, plus the Delta tokens appended before the next event
// (AMB-25), n_hbm <= beta * (N - |P|) (Alg. 1); a longer prefix starts partly in T1
// (AMB-26).  T1 (staging / stream ring) and T2 hold the offloaded share.  Every store is single-
// buffered: migrate moves rows in place (chunked through mtemp).
int delta_slack(const kv_tier_config& c) { return std::max(16, c.manage_interval) + 16; }
void capacities(const kv_tier_config& c, int* cap0, int* cap1, int* cap2) {
  const long long N = c.max_tokens;
  const long long prot = std::min<long long>(N, (long long)c.prompt_len + c.sink_size + c.window_size);
  // a sequence shard stores only its own positions: every store is bounded by that count
  const long long own = c.shard == KV_TIER_SHARD_SEQUENCE
                            ? seq_owned_below(c.world, c.rank, (int)N) + SEQ_BLOCK : N;
  const long long Nc = std::min<long long>(N, own);
  long long keep;                                            // live tokens an event may keep in T0
  if (c.policy == KV_TIER_POLICY_STREAMING) keep = 0;
  else if (c.policy == KV_TIER_POLICY_H2O || c.policy == KV_TIER_POLICY_RANDOM) keep = c.budget;
  else keep = ((long long)c.hbm_ratio_bp * (N - prot) + 9999) / 10000;
  long long c0 = std::min<long long>(Nc, prot + keep + delta_slack(c));
  const long long load0 = std::max<long long>(0, c0 - delta_slack(c));     // prefix rows loaded into T0
  const long long off = ((long long)(10000 - c.hbm_ratio_bp) * N + 9999) / 10000 + 2;
  long long c1 = std::min<long long>(Nc, std::max<long long>(off, Nc - load0));
  long long c2 = c.t2_fraction_bp ? std::min<long long>(Nc, (off * c.t2_fraction_bp + 9999) / 10000 + 2) : 0;
  if (c.shard == KV_TIER_SHARD_SEQUENCE && c.world > 1) {
    // a shard's T1/T2 share tracks the global fraction (block-cyclic ownership): 1.25x its fair
    // share + one block; a classify that would exceed it sets the device capacity flag (E_CAPACITY)
    c1 = std::min<long long>(c1, (off * 5 + 4 * c.world - 1) / (4 * c.world) + SEQ_BLOCK);
    if (c2) c2 = std::min<long long>(c2, (c2 * 5 + 4 * c.world - 1) / (4 * c.world) + SEQ_BLOCK);
  }
  *cap0 = round16(c0);
  *cap1 = round16(c1);
  *cap2 = round16(c2);
}

struct Layout {
  size_t off_k0[2], off_v0[2], off_k1[2], off_v1[2], off_c2k[2], off_c2v[2], off_s2k[2], off_s2v[2];
  size_t off_idx[2][3], off_vis[2], off_tier[2], off_row[2], off_cnt[2], off_S, off_fS, off_st, off_z, off_ml;
  size_t off_part, off_uctr, off_moves, off_mcount, off_scratch, off_mtemp, total, hot_begin, off_vnorm, off_zlayer;
  size_t off_red, off_lastk, off_snap, off_pool, off_sdone;
  size_t b_t0, b_t1, b_t2, b_scores, b_meta;
};

int split_of(const kv_tier_config& c);
int zring_of(const kv_tier_config& c);

// Whole-step kernel (step.cu): s CTAs per kv head (a cluster, s <= 16) or m kv heads per CTA;
// 8 consumer warps per CTA (one CTA per SM) or 4 (two per SM).  Every CTA of a request must be
// resident at once (they wait on each other layer by layer), so a shape qualifies only if all
// B*H_kv/m clusters fit the GPU together.  Among those, the one engaging the most SMs wins, then
// the one-CTA-per-SM shape.  Sets v.step_k (total CTAs, 0 = no
// shape fits), v.step_s, v.step_m, v.step_nw.
void step_plan(DevView& v, int nsm) {
  int best = 0, bs = 0, bm = 0, bnw = 0, bum = 0, brank = 0;
  // candidates in preference order on ties: the tcgen05 consumer, 8 mma.sync warps, 4 warps
  const int um_ok = (v.D == 128 && v.cap2 == 0) ? v.step_um_ok : 0;   // the tcgen05 consumer applies
  for (int cand = 0; cand < 3; ++cand) {
    const int um = cand == 0 ? um_ok : 0, nw = cand == 2 ? 4 : 8;
    if (cand == 0 && !um_ok) continue;
    const int per_sm = nw == 8 ? 1 : 2, rank = 3 - cand;
    for (int m = 8; m >= 1; m >>= 1) {
      if (v.Hkv % m) continue;
      if (um && m != 1) continue;                    // the tcgen05 consumer: one kv head per cluster
      for (int s = um ? 2 : 1; s <= (m == 1 ? 16 : 1); ++s) {
        if (v.split_req > 0 && (s != v.split_req || m != 1)) continue;   // the config's split, if given
        const int clusters_needed = v.B * v.Hkv / m, total = clusters_needed * s;
        if (total > per_sm * nsm) continue;
        v.step_k = total; v.step_s = s; v.step_m = m; v.step_nw = um ? 4 : nw; v.step_um = um;
        if (step_smem_bytes(v) > (nw == 8 ? 227 * 1024 : 113 * 1024)) continue;
        int clusters = 0;
        if (step_configure(v, &clusters) != cudaSuccess) { cudaGetLastError(); continue; }
        if (clusters < clusters_needed) continue;
        // SMs engaged; ties: the tcgen05 consumer, then one CTA per SM (measured at 7B: 8 warps x
        // 128 CTAs 3593 steps/s, 4 warps x 256 CTAs 3353)
        const int sms = total / per_sm, best_sms = best ? best / (bnw == 8 || bum ? 1 : 2) : 0;
        if (sms > best_sms || (sms == best_sms && rank > brank)) {
          best = total; bs = s; bm = m; bnw = um ? 4 : nw; bum = um; brank = rank;
        }
      }
    }
  }
  v.step_k = best; v.step_s = bs; v.step_m = bm; v.step_nw = bnw; v.step_um = bum;
  if (best) { int c = 0; step_configure(v, &c); }   // leave the chosen shape's attributes set
}

// Rows per group of the pinned host stores: every position, or a sequence shard's own ones.
int host_rows_of(const kv_tier_config& c) {
  return c.shard == KV_TIER_SHARD_SEQUENCE && c.world > 1 ? seq_owned_below(c.world, c.rank, c.max_tokens) + SEQ_BLOCK
                                                         : c.max_tokens;
}


// Rows a migrate may move per request: every position at most once, so an event never overflows.
size_t mcap_of(const kv_tier_config& c) {
  const size_t n = c.shard == KV_TIER_SHARD_SEQUENCE ? (size_t)seq_owned_below(c.world, c.rank, c.max_tokens) + SEQ_BLOCK
                                                    : (size_t)c.max_tokens;
  return (n + 15) / 16 * 16;
}
// (layer, kv head) pairs per migrate chunk: mtemp (B * mcap rows of 4d bytes per pair) stays
// within 64 MB.  KVTIER_MCHUNK (test hook) forces smaller chunks; results never depend on it.
int mchunk_of(const kv_tier_config& c) {
  const size_t per = (size_t)c.num_requests * mcap_of(c) * 4 * c.head_dim;
  int k = (int)std::max<size_t>(1, ((size_t)64 << 20) / per);
  k = std::min(k, c.num_layers * c.num_kv_heads);
  if (const char* ov = getenv("KVTIER_MCHUNK")) k = std::max(1, std::min(k, atoi(ov)));
  return k;
}

Layout make_layout(const kv_tier_config& c, int cap0, int cap1, int cap2) {
  Layout L{};
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o += align256(bytes); return r; };
  const size_t LBH = (size_t)c.num_layers * c.num_requests * c.num_kv_heads;
  const size_t BH = (size_t)c.num_requests * c.num_kv_heads;
  const size_t D = c.head_dim, B = c.num_requests, N = c.max_tokens;
  const bool stream = c.staging_tokens == 0;
  size_t s0 = o;
  const size_t SL = STORE_SLACK_ROWS;
  L.off_k0[0] = L.off_k0[1] = take((LBH * cap0 + SL) * D * 2);     // single-buffered row stores
  L.off_v0[0] = L.off_v0[1] = take((LBH * cap0 + SL) * D * 2);
  L.b_t0 = o - s0; s0 = o;
  const size_t g1 = stream ? 2 * BH : LBH;                      // stream mode: a 2-layer ring
  L.off_k1[0] = L.off_k1[1] = take((g1 * cap1 + SL) * D * 2);
  L.off_v1[0] = L.off_v1[1] = take((g1 * cap1 + SL) * D * 2);
  L.b_t1 = o - s0; s0 = o;
  L.off_c2k[0] = L.off_c2k[1] = take(LBH * cap2 * D);
  L.off_c2v[0] = L.off_c2v[1] = take(LBH * cap2 * D);
  L.off_s2k[0] = L.off_s2k[1] = take(LBH * cap2 * 4);
  L.off_s2v[0] = L.off_s2v[1] = take(LBH * cap2 * 4);
  L.b_t2 = o - s0; s0 = o;
  // migrate staging (cold): the move list and one chunk of (layer, kv head) pairs in flight
  const size_t mcap = mcap_of(c);
  L.off_moves = take(B * mcap * 16);
  L.off_mcount = take(B * 4);
  L.off_scratch = take(B * N * 4);
  L.off_mtemp = take(B * mcap * (size_t)mchunk_of(c) * 2 * D * 2);
  // hot, small: kept resident in L2 (access-policy window from off_S to the end)
  L.off_S = take(BH * N * 4);
  L.off_z = take(zring_of(c) * BH * (N + 64) * 8 * 4);   // logits of recent launches (score update)
  L.off_ml = take(ZRING * BH * 16 * 4);
  const size_t nslots = BH * (split_of(c) + 1);                          // per-CTA partials + new token
  L.off_part = take(nslots * (16 + 8 * D) * 4);
  L.off_sdone = take((size_t)c.num_layers * B * 4);                     // step kernel layer counters
  L.off_uctr = take(256);                                                 // migrate grid barrier
  L.off_zlayer = take(ZRING * 4);
  L.off_vnorm = take(scorer_uses_vnorm(c.scorer) ? LBH * N * 4 : 0);     // VATP / combined: V-row norms
  L.off_red = take(scorer_uses_red(c.scorer) ? BH * N * 4 : 0);          // redundancy partials R_part
  L.off_lastk = take(scorer_uses_red(c.scorer) ? LBH * D * 2 : 0);       // previous key per (layer, kv head)
  L.off_snap = take(scorer_uses_window(c.scorer) ? BH * N * 4 : 0);      // windowed: S_part snapshot
  L.off_pool = take(scorer_uses_window(c.scorer) ? 2 * B * N * 4 : 0);   // windowed: compacted scores + indices
  L.b_scores = o - s0; s0 = o;
  for (int i = 0; i < 2; ++i) {
    L.off_idx[i][0] = take(B * cap0 * 4);
    L.off_idx[i][1] = take(B * std::max(cap1, 1) * 4);
    L.off_idx[i][2] = take(B * std::max(cap2, 1) * 4);
    L.off_vis[i] = take(B * N * 4);
    L.off_tier[i] = take(B * N);
    L.off_row[i] = take(B * N * 4);
    L.off_cnt[i] = take(B * CNT_STRIDE * 4);
  }
  L.off_fS = take(B * N * 4);
  L.off_st = take(sizeof(DevState));
  L.hot_begin = L.off_S;
  L.b_meta = o - s0;
  L.total = o;
  return L;
}

int n_protected(const kv_tier_config& c, int n) {
  const int a = std::min(c.prompt_len + c.sink_size, n);
  const int w0 = std::max(0, n - c.window_size);
  return a + (n - std::max(w0, a));
}

}  // namespace

extern "C" {

const char* kv_tier_version(void) { return "kvtier-b200 0.2 (sm_100a: bulk-copy ring + mma.sync split decode, PDL merge chain)"; }

const char* kv_tier_last_error(const kv_tier_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_err.c_str();
}

kv_tier_status kv_tier_query_sizes(const kv_tier_config* cfg, kv_tier_sizes* out) {
  kv_tier_status st = validate(cfg);
  if (st != KV_TIER_OK) return st;
  if (!out) return fail(nullptr, KV_TIER_E_INVAL, "null sizes");
  int cap0, cap1, cap2;
  capacities(*cfg, &cap0, &cap1, &cap2);
  Layout L = make_layout(*cfg, cap0, cap1, cap2);
  memset(out, 0, sizeof(*out));
  out->device_arena = L.total;
  out->t0_store = L.b_t0;
  out->t1_staging = L.b_t1;
  out->t2_store = L.b_t2;
  out->scores = L.b_scores;
  out->meta = L.b_meta;
  const size_t rows = (size_t)cfg->num_layers * cfg->num_requests * cfg->num_kv_heads * host_rows_of(*cfg);
  out->host_t1 = rows * cfg->head_dim * 2 * 2;     // T1 (and a prefix longer than T0's load share) lives here
  out->host_t2 = cfg->t2_fraction_bp ? rows * (cfg->head_dim + 4) * 2 : 0;
  out->cap_t0 = cap0;
  out->cap_t1 = cap1;
  out->cap_t2 = cap2;
  return KV_TIER_OK;
}

kv_tier_status kv_tier_init(const kv_tier_config* cfg, const kv_tier_buffers* buf, const void* nccl_unique_id,
                            kv_tier_ctx** out) {
  kv_tier_status st = validate(cfg);
  if (st != KV_TIER_OK) return st;
  if (!buf || !buf->device_arena || !out) return fail(nullptr, KV_TIER_E_INVAL, "null buffers/out");
  if (nccl_unique_id && cfg->shard != KV_TIER_SHARD_SEQUENCE)
    return fail(nullptr, KV_TIER_E_INVAL, "an nccl_unique_id is only used by sequence sharding (the other splits have no collective on the step)");
  if (nccl_unique_id && !cfg->out_fp32)
    return fail(nullptr, KV_TIER_E_INVAL, "sequence sharding with a communicator combines o in fp32: out_fp32 must be 1");
  if (scorer_uses_window(cfg->scorer) && cfg->shard == KV_TIER_SHARD_SEQUENCE && cfg->world > 1 && !nccl_unique_id)
    return fail(nullptr, KV_TIER_E_INVAL, "windowed scorers on sequence shards need the library's communicator "
                "(their classify all-gathers every shard's S_part and snapshot)");
  if (nccl_unique_id && !nccl_api().ok)
    return fail(nullptr, KV_TIER_E_NCCL, "libnccl.so.2 not found in the process or on the loader path");
  if (((uintptr_t)buf->device_arena) & 255) return fail(nullptr, KV_TIER_E_INVAL, "device_arena must be 256-B aligned");
  cudaError_t e = cudaSetDevice(cfg->device);
  if (e != cudaSuccess) return fail(nullptr, KV_TIER_E_CUDA, "cudaSetDevice: %s", cudaGetErrorString(e));
  kv_tier_ctx* ctx = new kv_tier_ctx();
  ctx->cfg = *cfg;
  kv_tier_query_sizes(cfg, &ctx->sz);
  int cap0 = ctx->sz.cap_t0, cap1 = ctx->sz.cap_t1, cap2 = ctx->sz.cap_t2;
  Layout L = make_layout(*cfg, cap0, cap1, cap2);
  char* A = reinterpret_cast<char*>(buf->device_arena);
  DevView& v = ctx->v;
  memset(&v, 0, sizeof(v));
  v.B = cfg->num_requests; v.L = cfg->num_layers; v.Hq = cfg->num_q_heads; v.Hkv = cfg->num_kv_heads;
  v.G = v.Hq / v.Hkv; v.D = cfg->head_dim; v.Nmax = cfg->max_tokens;
  v.cap0 = cap0; v.cap1 = cap1; v.cap2 = cap2;
  v.P = cfg->prompt_len; v.ks = cfg->sink_size; v.kw = cfg->window_size;
  v.hbm_bp = (int)cfg->hbm_ratio_bp; v.evict_bp = (int)cfg->evict_ratio_bp; v.t2_bp = (int)cfg->t2_fraction_bp;
  v.evict_mode = cfg->evict_mode;
  v.policy = cfg->policy;
  v.budget = cfg->budget;
  v.policy_seed = cfg->policy_seed;
  v.stream_mode = cfg->staging_tokens == 0;
  v.out_fp32 = cfg->out_fp32;
  v.split = auto_split(*cfg);
  v.split_req = cfg->split;
  v.variant = cfg->variant;
  v.step_um_ok = cfg->step_kernel == 2 ? 1 : 0;
  v.seq_w = cfg->shard == KV_TIER_SHARD_SEQUENCE ? cfg->world : 1;
  v.seq_r = cfg->shard == KV_TIER_SHARD_SEQUENCE ? cfg->rank : 0;
  v.score_grid = 148;                       // score-flush CTAs beside the per-layer chain (measured best)
  for (int i = 0; i < 2; ++i) {
    v.k0[i] = reinterpret_cast<__nv_bfloat16*>(A + L.off_k0[i]);
    v.v0[i] = reinterpret_cast<__nv_bfloat16*>(A + L.off_v0[i]);
    v.k1[i] = reinterpret_cast<__nv_bfloat16*>(A + L.off_k1[i]);
    v.v1[i] = reinterpret_cast<__nv_bfloat16*>(A + L.off_v1[i]);
    v.c2k[i] = reinterpret_cast<int8_t*>(A + L.off_c2k[i]);
    v.c2v[i] = reinterpret_cast<int8_t*>(A + L.off_c2v[i]);
    v.s2k[i] = reinterpret_cast<float*>(A + L.off_s2k[i]);
    v.s2v[i] = reinterpret_cast<float*>(A + L.off_s2v[i]);
    for (int T = 0; T < 3; ++T) v.idx[i][T] = reinterpret_cast<int*>(A + L.off_idx[i][T]);
    v.idxvis[i] = reinterpret_cast<int*>(A + L.off_vis[i]);
    v.tier[i] = reinterpret_cast<uint8_t*>(A + L.off_tier[i]);
    v.rowof[i] = reinterpret_cast<int*>(A + L.off_row[i]);
    v.cnt[i] = reinterpret_cast<int*>(A + L.off_cnt[i]);
  }
  v.S = reinterpret_cast<float*>(A + L.off_S);
  v.zbuf = reinterpret_cast<float*>(A + L.off_z);
  v.ml = reinterpret_cast<float*>(A + L.off_ml);
  v.zrows = cfg->max_tokens + 64;
  v.zring = zring_of(*cfg);
  v.part = reinterpret_cast<float*>(A + L.off_part);
  v.part_stride = 16 + 8 * v.D;
  v.step_k = v.step_s = v.step_m = v.step_nw = 0;
  v.step_done = reinterpret_cast<int*>(A + L.off_sdone);
  v.zlayer = reinterpret_cast<int*>(A + L.off_zlayer);
  v.scorer = cfg->scorer;
  v.vnorm = scorer_uses_vnorm(cfg->scorer) ? reinterpret_cast<float*>(A + L.off_vnorm) : nullptr;
  v.red = scorer_uses_red(cfg->scorer) ? reinterpret_cast<float*>(A + L.off_red) : nullptr;
  v.lastk = scorer_uses_red(cfg->scorer) ? reinterpret_cast<uint16_t*>(A + L.off_lastk) : nullptr;
  v.snap = scorer_uses_window(cfg->scorer) ? reinterpret_cast<float*>(A + L.off_snap) : nullptr;
  v.pool = scorer_uses_window(cfg->scorer) ? reinterpret_cast<float*>(A + L.off_pool) : nullptr;
  v.interval = cfg->manage_interval;
  v.hot_base = A + L.hot_begin;
  v.hot_bytes = L.total - L.hot_begin;
  v.moves = reinterpret_cast<int4*>(A + L.off_moves);
  v.mcount = reinterpret_cast<int*>(A + L.off_mcount);
  v.mcap = (int)mcap_of(*cfg);
  v.mchunk = mchunk_of(*cfg);
  v.c0_load = std::max(0, cap0 - delta_slack(*cfg));
  v.scratch = reinterpret_cast<int*>(A + L.off_scratch);
  v.mtemp = reinterpret_cast<__nv_bfloat16*>(A + L.off_mtemp);
  v.gbar = reinterpret_cast<unsigned*>(A + L.off_uctr);
  v.fS = reinterpret_cast<float*>(A + L.off_fS);
  v.st = reinterpret_cast<DevState*>(A + L.off_st);
  // pinned, mapped host stores (NUMA placement follows the calling thread's node)
  v.hN = host_rows_of(*cfg);
  const size_t rows = (size_t)v.L * v.B * v.Hkv * v.hN;
  if (ctx->sz.host_t1) {
    e = cudaHostAlloc(&ctx->host_t1, ctx->sz.host_t1, cudaHostAllocMapped | cudaHostAllocPortable);
    if (e != cudaSuccess) { delete ctx; return fail(nullptr, KV_TIER_E_OOM, "cudaHostAlloc(T1 %zu B): %s", (size_t)0, cudaGetErrorString(e)); }
    void* dptr = nullptr;
    cudaHostGetDevicePointer(&dptr, ctx->host_t1, 0);
    v.hk1 = reinterpret_cast<__nv_bfloat16*>(dptr);
    v.hv1 = v.hk1 + rows * v.D;
  }
  if (ctx->sz.host_t2) {
    e = cudaHostAlloc(&ctx->host_t2, ctx->sz.host_t2, cudaHostAllocMapped | cudaHostAllocPortable);
    if (e != cudaSuccess) { if (ctx->host_t1) cudaFreeHost(ctx->host_t1); delete ctx; return fail(nullptr, KV_TIER_E_OOM, "cudaHostAlloc(T2): %s", cudaGetErrorString(e)); }
    void* dptr = nullptr;
    cudaHostGetDevicePointer(&dptr, ctx->host_t2, 0);
    char* h = reinterpret_cast<char*>(dptr);
    v.hc2k = reinterpret_cast<int8_t*>(h);
    v.hc2v = reinterpret_cast<int8_t*>(h + rows * v.D);
    v.hs2k = reinterpret_cast<float*>(h + 2 * rows * v.D);
    v.hs2v = reinterpret_cast<float*>(h + 2 * rows * v.D + rows * 4);
  }
#if KVT_TRACE
  {                                         // debug builds: per-(layer, CTA) timeline buffer
    const size_t tb = (size_t)v.L * std::max(v.split * v.B * v.Hkv, 2 * 148) * NTRACE * sizeof(unsigned long long);
    if (cudaMalloc(&ctx->trace, tb) == cudaSuccess) { cudaMemset(ctx->trace, 0, tb); v.trace = ctx->trace; }
  }
#endif
  const size_t smem_need = std::max(attn_smem_bytes(v), merge_smem_bytes(v));
  if (smem_need > 227 * 1024) {
    const size_t need = smem_need;
    if (ctx->host_t1) cudaFreeHost(ctx->host_t1);
    if (ctx->host_t2) cudaFreeHost(ctx->host_t2);
    delete ctx;
    return fail(nullptr, KV_TIER_E_INVAL, "decode kernel needs %zu B shared memory (> 227 KB): raise split or pick a smaller variant", need);
  }
  e = cudaMemset(buf->device_arena, 0, ctx->sz.device_arena);   // stale rows read as masked padding stay finite
  if (e == cudaSuccess) {
    // scores, logits, partials and index lists stay L2-resident while K/V streams past them
    int maxp = 0;
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, cfg->device);
    size_t want = std::min<size_t>(v.hot_bytes, (size_t)maxp);
    size_t cur_lim = 0;
    cudaDeviceGetLimit(&cur_lim, cudaLimitPersistingL2CacheSize);
    if (want > cur_lim) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
    int maxw = 0;
    cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, cfg->device);
    v.hot_bytes = std::min<size_t>(v.hot_bytes, (size_t)maxw);
    // the persisting share of the window must fit the carve-out, or the hot lines evict each other
    size_t lim = 0;
    cudaDeviceGetLimit(&lim, cudaLimitPersistingL2CacheSize);
    v.hot_hit = v.hot_bytes > 0 ? (float)std::min(1.0, (double)lim / (double)v.hot_bytes) : 0.f;
    cudaGetLastError();                  // persistence is an optimisation: ignore if unsupported
  }
  if (e == cudaSuccess) e = attn_configure(v);
  if (e == cudaSuccess && !v.stream_mode && v.seq_w <= 1 && cfg->step_kernel != 3) {
    // kv_tier_step / the step graph: all layers in one launch, one thread-block cluster per request
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, cfg->device);
    step_plan(v, nsm);
  }
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_step_begin, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_migrated, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_offload_done, cudaEventDisableTiming);
  for (int i = 0; i < 2 && e == cudaSuccess; ++i) e = cudaEventCreateWithFlags(&ctx->ev_slot_free[i], cudaEventDisableTiming);
  for (int i = 0; i < ZRING && e == cudaSuccess; ++i) {
    e = cudaEventCreateWithFlags(&ctx->ev_merged[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_scored[i], cudaEventDisableTiming);
  }
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_score_tail, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->score_stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->offload_stream, cudaStreamNonBlocking);
  ctx->ev_prefetched.assign(v.L, nullptr);
  for (int l = 0; l < v.L && e == cudaSuccess; ++l) e = cudaEventCreateWithFlags(&ctx->ev_prefetched[l], cudaEventDisableTiming);
  if (e != cudaSuccess) {
    kv_tier_status s2 = fail(nullptr, KV_TIER_E_CUDA, "init: %s", cudaGetErrorString(e));
    kv_tier_destroy(ctx);
    return s2;
  }
  ctx->loaded_layers.assign(v.L, 0);
  ctx->prefetched_step.assign(v.L, -1);
  ctx->appended_step.assign(v.L, -1);
  if (nccl_unique_id) {
    // sequence sharding: a library-owned communicator and its exchange buffers (the layer
    // partials of one rank; every rank's; the global (M, L) per layer; all ranks' S_part)
    ncclUniqueId id;
    memcpy(&id, nccl_unique_id, sizeof(id));
    const ncclResult_t r = nccl_api().comm_init_rank(&ctx->comm, cfg->world, id, cfg->rank);
    if (r != ncclSuccess) {
      ctx->comm = nullptr;
      kv_tier_destroy(ctx);
      return fail(nullptr, KV_TIER_E_NCCL, "ncclCommInitRank: %s", nccl_api().error_string(r));
    }
    const size_t rows = (size_t)v.B * v.Hq, W = (size_t)cfg->world;
    ctx->x_slot = (rows * (v.D + 2) + 3) & ~(size_t)3;
    e = cudaMalloc(&ctx->x_recv, W * ctx->x_slot * 4);
    if (e == cudaSuccess) e = cudaMalloc(&ctx->x_lse, (size_t)v.L * rows * 2 * 4);
    if (e == cudaSuccess) e = cudaMalloc(&ctx->x_scores, W * v.B * v.Hkv * (size_t)v.Nmax * 4);
    if (e == cudaSuccess && v.snap) e = cudaMalloc(&ctx->x_snaps, W * v.B * v.Hkv * (size_t)v.Nmax * 4);
    if (e != cudaSuccess) {
      kv_tier_destroy(ctx);
      return fail(nullptr, KV_TIER_E_OOM, "sequence-shard exchange buffers: %s", cudaGetErrorString(e));
    }
  }
  *out = ctx;
  return KV_TIER_OK;
}

kv_tier_status kv_tier_nccl_unique_id(void* out, size_t bytes) {
  if (!out || bytes < sizeof(ncclUniqueId))
    return fail(nullptr, KV_TIER_E_INVAL, "need %zu bytes for the NCCL unique id", sizeof(ncclUniqueId));
  if (!nccl_api().ok) return fail(nullptr, KV_TIER_E_NCCL, "libnccl.so.2 not found in the process or on the loader path");
  ncclUniqueId id;
  const ncclResult_t r = nccl_api().get_unique_id(&id);
  if (r != ncclSuccess) return fail(nullptr, KV_TIER_E_NCCL, "ncclGetUniqueId: %s", nccl_api().error_string(r));
  memcpy(out, &id, sizeof(id));
  return KV_TIER_OK;
}

kv_tier_status kv_tier_destroy(kv_tier_ctx* ctx) {
  if (!ctx) return KV_TIER_OK;
  cudaDeviceSynchronize();
  if (ctx->host_t1) cudaFreeHost(ctx->host_t1);
  if (ctx->host_t2) cudaFreeHost(ctx->host_t2);
  if (ctx->ev_step_begin) cudaEventDestroy(ctx->ev_step_begin);
  if (ctx->ev_migrated) cudaEventDestroy(ctx->ev_migrated);
  if (ctx->ev_offload_done) cudaEventDestroy(ctx->ev_offload_done);
  for (auto& ev : ctx->ev_slot_free) if (ev) cudaEventDestroy(ev);
  for (auto& ev : ctx->ev_prefetched) if (ev) cudaEventDestroy(ev);
  if (ctx->graph_exec) cudaGraphExecDestroy(ctx->graph_exec);
  if (ctx->graph) cudaGraphDestroy(ctx->graph);
  if (ctx->trace) cudaFree(ctx->trace);
  for (int i = 0; i < ZRING; ++i) {
    if (ctx->ev_merged[i]) cudaEventDestroy(ctx->ev_merged[i]);
    if (ctx->ev_scored[i]) cudaEventDestroy(ctx->ev_scored[i]);
  }
  if (ctx->ev_score_tail) cudaEventDestroy(ctx->ev_score_tail);
  if (ctx->score_stream) cudaStreamDestroy(ctx->score_stream);
  if (ctx->offload_stream) cudaStreamDestroy(ctx->offload_stream);
  for (int i = 0; i < 2; ++i) {
    if (ctx->h1_inc[i]) cudaFreeHost(ctx->h1_inc[i]);
    if (ctx->ev_inc[i]) cudaEventDestroy(ctx->ev_inc[i]);
  }
  if (ctx->h1_q) cudaFreeHost(ctx->h1_q);
  if (ctx->h1_o) cudaFreeHost(ctx->h1_o);
  if (ctx->d1_parts) cudaFree(ctx->d1_parts);
  if (ctx->ev_q) cudaEventDestroy(ctx->ev_q);
  if (ctx->comm) nccl_api().comm_destroy(ctx->comm);
  for (float* p : {ctx->x_recv, ctx->x_lse, ctx->x_scores, ctx->x_snaps})
    if (p) cudaFree(p);
  delete ctx;
  return KV_TIER_OK;
}

kv_tier_status kv_tier_load_prefix(kv_tier_ctx* ctx, int32_t layer, const void* k, const void* v, int32_t n0,
                                   void* stream) {
  if (!ctx) return fail(nullptr, KV_TIER_E_INVAL, "null ctx");
  if (layer < 0 || layer >= ctx->v.L) return fail(ctx, KV_TIER_E_INVAL, "layer out of range");
  if (!k || !v) return fail(ctx, KV_TIER_E_INVAL, "null k/v");
  if (ctx->t > 0 || ctx->step_open) return fail(ctx, KV_TIER_E_STATE, "load_prefix after decoding started");
  if (scorer_uses_red(ctx->v.scorer) &&
      layer != (int)std::count(ctx->loaded_layers.begin(), ctx->loaded_layers.end(), 1))
    return fail(ctx, KV_TIER_E_STATE, "redundancy scorers: load prefix layers once each, in ascending order (AMB-30)");
  {
    const int own0 = n0 < 0 ? 0 : seq_owned_below(ctx->v.seq_w, ctx->v.seq_r, n0);
    const int over = std::max(0, own0 - ctx->v.c0_load);       // prefix rows that start in T1 (AMB-26)
    if (n0 < 0 || n0 + 1 > ctx->v.Nmax || over > ctx->v.cap1 || (over > 0 && ctx->sz.host_t1 == 0))
      return fail(ctx, KV_TIER_E_CAPACITY, "prefix of %d tokens exceeds T0 + T1 capacity %d + %d / N_max %d", n0,
                  ctx->v.c0_load, ctx->v.cap1, ctx->v.Nmax);
  }
  if (ctx->n0 >= 0 && ctx->n0 != n0) return fail(ctx, KV_TIER_E_INVAL, "n0 differs between layers");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (ctx->n0 < 0) {
    kv_tier_status st = cuda_check(ctx, launch_init_meta(ctx->v, n0, s), "init_meta");
    if (st) return st;
    ctx->n0 = n0;
    ctx->n = n0;
    const int own0 = seq_owned_below(ctx->v.seq_w, ctx->v.seq_r, n0);
    ctx->c[0] = std::min(own0, ctx->v.c0_load);
    ctx->c[1] = own0 - ctx->c[0];
    ctx->c[2] = ctx->c[3] = 0;
    ctx->n_event = n0;
    ctx->nvis_event = ctx->c[0];
  }
  if (n0 > 0) {
    kv_tier_status st = cuda_check(ctx, launch_load_prefix(ctx->v, layer, k, v, n0, s), "load_prefix");
    if (!st && scorer_uses_vnorm(ctx->v.scorer))
      st = cuda_check(ctx, launch_vnorm_prefix(ctx->v, layer, v, n0, s), "load_prefix (V norms)");
    if (!st && scorer_uses_red(ctx->v.scorer))
      st = cuda_check(ctx, launch_redund_prefix(ctx->v, layer, k, n0, s), "load_prefix (key redundancy)");
    if (st) return st;
  }
  ctx->loaded_layers[layer] = 1;
  ctx->loaded = std::all_of(ctx->loaded_layers.begin(), ctx->loaded_layers.end(), [](int x) { return x != 0; });
  return KV_TIER_OK;
}

kv_tier_status kv_tier_begin_step(kv_tier_ctx* ctx, void* stream) {
  if (!ctx) return fail(nullptr, KV_TIER_E_INVAL, "null ctx");
  if (!ctx->loaded) return fail(ctx, KV_TIER_E_STATE, "load_prefix not called for every layer");
  if (ctx->step_open) return fail(ctx, KV_TIER_E_STATE, "begin_step twice without end_step");
  if (ctx->n + 1 > ctx->v.Nmax) return fail(ctx, KV_TIER_E_CAPACITY, "N_max=%d reached", ctx->v.Nmax);
  if (ctx->c[0] + 1 > ctx->v.cap0)
    return fail(ctx, KV_TIER_E_CAPACITY, "T0 store full (%d rows): call classify/migrate every Delta steps", ctx->v.cap0);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  kv_tier_status st = cuda_check(ctx, launch_begin_step(ctx->v, s), "begin_step");
  if (st) return st;
  st = cuda_check(ctx, cudaEventRecord(ctx->ev_step_begin, s), "event");
  if (st) return st;
  ctx->c[0] += seq_own(ctx->v.seq_w, ctx->v.seq_r, ctx->n) ? 1 : 0;
  ctx->n += 1;
  ctx->step_open = true;
  ctx->pdl_ok = false;
  ctx->classified = false;
  ctx->slot_recorded[0] = ctx->slot_recorded[1] = false;
  ctx->zslot_next = 0;
  ctx->zpend_n = 0;
  return KV_TIER_OK;
}

kv_tier_status kv_tier_append(kv_tier_ctx* ctx, int32_t layer, const void* k_new, const void* v_new, void* stream) {
  if (!ctx) return fail(nullptr, KV_TIER_E_INVAL, "null ctx");
  if (!ctx->step_open) return fail(ctx, KV_TIER_E_STATE, "append outside begin_step/end_step");
  if (layer < 0 || layer >= ctx->v.L) return fail(ctx, KV_TIER_E_INVAL, "layer out of range");
  if (!k_new || !v_new) return fail(ctx, KV_TIER_E_INVAL, "null k/v");
  kv_tier_status st = cuda_check(ctx, launch_append(ctx->v, layer, k_new, v_new, reinterpret_cast<cudaStream_t>(stream)), "append");
  if (!st) ctx->appended_step[layer] = ctx->t;
  // the append writes only the new row, which a following decode reads after its dependency wait
  ctx->pdl_ok = !st && ctx->pdl_stream == stream && ctx->pdl_ok;
  return st;
}

kv_tier_status kv_tier_prefetch(kv_tier_ctx* ctx, int32_t layer, void* side) {
  if (!ctx) return fail(nullptr, KV_TIER_E_INVAL, "null ctx");
  if (layer < 0 || layer >= ctx->v.L) return fail(ctx, KV_TIER_E_INVAL, "layer out of range");
  if (!ctx->v.stream_mode) return KV_TIER_OK;     // differential: staging already holds T1
  if (!ctx->step_open) return fail(ctx, KV_TIER_E_STATE, "prefetch outside a step");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(side);
  // ev_step_begin orders this after all earlier main-stream work (incl. the previous
  // step's attention on both ring slots); slot reuse within the step waits on the
  // attention that last read the slot.
  cudaError_t e = cudaStreamWaitEvent(s, ctx->ev_step_begin, 0);
  if (e == cudaSuccess && ctx->slot_recorded[layer & 1]) e = cudaStreamWaitEvent(s, ctx->ev_slot_free[layer & 1], 0);
  if (e == cudaSuccess && ctx->offload_pending && !ctx->capturing) e = cudaStreamWaitEvent(s, ctx->ev_offload_done, 0);
  if (e == cudaSuccess) e = launch_prefetch(ctx->v, layer, s);
  if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_prefetched[layer], s);
  if (e == cudaSuccess) ctx->prefetched_step[layer] = ctx->t;
  return cuda_check(ctx, e, "prefetch");
}

// a4 on the score stream: S_part += sum_h exp2(z - M)/L for the pending launches (layer order),
// once the last of them has merged.  Slots are batched ZBATCH-aligned from slot 0 each step.
static cudaError_t issue_scores(kv_tier_ctx* ctx, cudaStream_t s) {
  const int z0 = ctx->zpend_first, nz = ctx->zpend_n;
  (void)s;
  cudaError_t e = cudaSuccess;
  for (int j = 0; j < nz && e == cudaSuccess; ++j)    // launches may sit on different streams
    e = cudaStreamWaitEvent(ctx->score_stream, ctx->ev_merged[(z0 + j) % ctx->v.zring], 0);
  if (e == cudaSuccess) e = launch_score_flush(ctx->v, z0, nz, ctx->score_stream);
  if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_scored[z0], ctx->score_stream);
  if (e == cudaSuccess) {
    for (int j = 0; j < nz; ++j) ctx->slot_busy[(z0 + j) % ctx->v.zring] = true;
    ctx->scores_pending = true;
    ctx->zpend_n = 0;
  }
  return e;
}

static kv_tier_status decode_attention_impl(kv_tier_ctx* ctx, int32_t layer, const void* q, const void* k_new,
                                            const void* v_new, void* o, int32_t fuse_score_update, void* stream,
                                            int pdl, float* lse = nullptr) {
  if (!ctx) return fail(nullptr, KV_TIER_E_INVAL, "null ctx");
  if (ctx->v.seq_w > 1 && !lse)
    return fail(ctx, KV_TIER_E_STATE, "sequence shard: use kv_tier_decode_attention_lse (partial softmax statistics)");
  if (ctx->lse_pending >= 0)
    return fail(ctx, KV_TIER_E_STATE, "the previous decode_attention_lse still waits for kv_tier_score_update_lse");
  if (lse && ((uintptr_t)lse & 7)) return fail(ctx, KV_TIER_E_INVAL, "lse must be 8-B aligned");
  if (layer < 0 || layer >= ctx->v.L) return fail(ctx, KV_TIER_E_INVAL, "layer out of range");
  if (!q || !o) return fail(ctx, KV_TIER_E_INVAL, "null q/o");
  if ((k_new == nullptr) != (v_new == nullptr)) return fail(ctx, KV_TIER_E_INVAL, "k_new and v_new go together");
  if (((uintptr_t)q & 15) || ((uintptr_t)o & 15)) return fail(ctx, KV_TIER_E_INVAL, "q/o must be 16-B aligned");
  if (!ctx->step_open) return fail(ctx, KV_TIER_E_STATE, "decode_attention outside begin_step/end_step");
  if (!k_new && ctx->appended_step[layer] != ctx->t)
    return fail(ctx, KV_TIER_E_STATE, "layer %d: no new-token row (pass k_new/v_new or call kv_tier_append)", layer);
  if (ctx->v.host_t1 && !lse)
    return fail(ctx, KV_TIER_E_STATE, "host-T1 mode: the GPU result is partial, use kv_tier_decode_attention_lse");
  if (ctx->v.stream_mode && !ctx->v.host_t1 && ctx->prefetched_step[layer] != ctx->t)
    return fail(ctx, KV_TIER_E_STATE, "stream mode: kv_tier_prefetch(layer %d) must precede decode_attention in every step", layer);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSuccess;
  if (ctx->v.stream_mode) e = cudaStreamWaitEvent(s, ctx->ev_prefetched[layer], 0);
  const int zpar = fuse_score_update ? ctx->zslot_next : -1;
  // the ring slot's previous score kernel must be done before its logits are overwritten
  if (e == cudaSuccess && zpar >= 0 && ctx->slot_busy[zpar])
    e = cudaStreamWaitEvent(s, ctx->ev_scored[zpar - zpar % ZBATCH], 0);
  if (e == cudaSuccess) e = launch_decode_attn(ctx->v, layer, q, k_new, v_new, o, zpar, pdl, s, lse);
  if (e == cudaSuccess && zpar >= 0 && lse) {   // the update waits for the global (M, L)
    ctx->lse_pending = zpar;
    ctx->zslot_next = (zpar + 1) % ctx->v.zring;
    if (k_new) ctx->appended_step[layer] = ctx->t;
    return cuda_check(ctx, e, "decode_attention_lse");
  }
  if (e == cudaSuccess && zpar >= 0) e = cudaEventRecord(ctx->ev_merged[zpar], s);
  if (e == cudaSuccess && zpar >= 0) {
    if (ctx->zpend_n == 0) ctx->zpend_first = zpar;
    ctx->zpend_n += 1;
    ctx->zslot_next = (zpar + 1) % ctx->v.zring;
    if (ctx->zpend_n == ZBATCH) e = issue_scores(ctx, s);
  }
  if (e == cudaSuccess && ctx->v.stream_mode) {
    e = cudaEventRecord(ctx->ev_slot_free[layer & 1], s);
    ctx->slot_recorded[layer & 1] = true;
  }
  if (e == cudaSuccess && k_new) ctx->appended_step[layer] = ctx->t;
  return cuda_check(ctx, e, "decode_attention");
}

kv_tier_status kv_tier_decode_attention(kv_tier_ctx* ctx, int32_t layer, const void* q, const void* k_new,
                                        const void* v_new, void* o, int32_t fuse_score_update, void* stream) {
  // consecutive layers chain with programmatic dependent launch (the prologue streams this layer's
  // K/V while the previous kernel -- the previous layer's merge, or caller kernels in between --
  // finishes; q and the new token are read after griddepcontrol.wait)
  const int pdl = ctx && ctx->pdl_ok && ctx->pdl_stream == stream && !ctx->v.stream_mode ? 1 : 0;
  kv_tier_status st = decode_attention_impl(ctx, layer, q, k_new, v_new, o, fuse_score_update, stream, pdl);
  if (ctx) {
    ctx->pdl_ok = st == KV_TIER_OK;
    ctx->pdl_stream = stream;
  }
  return st;
}

kv_tier_status kv_tier_decode_attention_lse(kv_tier_ctx* ctx, int32_t layer, const void* q, const void* k_new,
                                            const void* v_new, void* o, float* lse, int32_t fuse_score_update,
                                            void* stream) {
  if (!lse) return fail(ctx, KV_TIER_E_INVAL, "null lse");
  return decode_attention_impl(ctx, layer, q, k_new, v_new, o, fuse_score_update, stream, 0, lse);
}

kv_tier_status kv_tier_lse_combine(const float* o_parts, const float* lse_parts, int32_t world, int32_t rows,
                                   int32_t d, float* o_out, float* lse_out, void* stream) {
  if (!o_parts || !lse_parts || !o_out || !lse_out || world < 1 || rows < 0 || d < 4 || d % 4)
    return fail(nullptr, KV_TIER_E_INVAL, "lse_combine: null pointer or bad shape (world >= 1, d %% 4 == 0)");
  if ((((uintptr_t)o_parts) | ((uintptr_t)o_out)) & 15 || (((uintptr_t)lse_parts) | ((uintptr_t)lse_out)) & 7)
    return fail(nullptr, KV_TIER_E_INVAL, "lse_combine: o must be 16-B and lse 8-B aligned");
  if (rows == 0) return KV_TIER_OK;
  return cuda_check(nullptr, launch_lse_combine(o_parts, lse_parts, world, rows, d, o_out, lse_out,
                                                reinterpret_cast<cudaStream_t>(stream)), "lse_combine");
}

// ml_set: the slot's (M, 1/L) were already written (seq_step's combine kernel writes them)
static kv_tier_status score_update_lse_impl(kv_tier_ctx* ctx, const float* lse_global, void* stream, bool ml_set) {
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const int z = ctx->lse_pending;
  cudaError_t e = ml_set ? cudaSuccess : launch_set_ml(ctx->v, z, lse_global, s);
  if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_merged[z], s);
  if (e == cudaSuccess) {
    if (ctx->zpend_n == 0) ctx->zpend_first = z;
    ctx->zpend_n += 1;
    if (ctx->zpend_n == ZBATCH) e = issue_scores(ctx, s);
  }
  if (e == cudaSuccess) ctx->lse_pending = -1;
  return cuda_check(ctx, e, "score_update_lse");
}
kv_tier_status kv_tier_score_update_lse(kv_tier_ctx* ctx, const float* lse_global, void* stream) {
  if (!ctx) return fail(nullptr, KV_TIER_E_INVAL, "null ctx");
  if (!lse_global || ((uintptr_t)lse_global & 7)) return fail(ctx, KV_TIER_E_INVAL, "lse_global must be an 8-B aligned device pointer");
  if (ctx->lse_pending < 0) return fail(ctx, KV_TIER_E_STATE, "no decode_attention_lse awaits its score update");
  return score_update_lse_impl(ctx, lse_global, stream, false);
}

kv_tier_status kv_tier_visible_count(const kv_tier_ctx* ctx, int32_t* n_vis) {
  if (!ctx || !n_vis) return fail(nullptr, KV_TIER_E_INVAL, "null arg");
  *n_vis = ctx->nvis_event + seq_owned_below(ctx->v.seq_w, ctx->v.seq_r, ctx->n) -
           seq_owned_below(ctx->v.seq_w, ctx->v.seq_r, ctx->n_event);
  return KV_TIER_OK;
}

kv_tier_status kv_tier_layout(const kv_tier_ctx* ctx, int32_t* counts4, int32_t* shape4) {
  if (!ctx) return fail(nullptr, KV_TIER_E_INVAL, "null ctx");
  if (counts4) {
    for (int i = 0; i < 3; ++i) counts4[i] = ctx->c[i];
    counts4[3] = seq_owned_below(ctx->v.seq_w, ctx->v.seq_r, ctx->n) - ctx->c[0] - ctx->c[1] - ctx->c[2];
  }
  if (shape4) {
    shape4[0] = ctx->v.step_k;
    shape4[1] = ctx->v.step_s;
    shape4[2] = ctx->v.step_m;
    shape4[3] = ctx->v.step_um ? 5 : ctx->v.step_nw;
  }
  return KV_TIER_OK;
}

kv_tier_status kv_tier_score_update(kv_tier_ctx* ctx, int32_t layer, const float* probs, void* stream) {
  if (!ctx) return fail(nullptr, KV_TIER_E_INVAL, "null ctx");
  if (!probs) return fail(ctx, KV_TIER_E_INVAL, "null probs");
  if (ctx->v.seq_w > 1) return fail(ctx, KV_TIER_E_STATE, "standalone score update is not defined for sequence shards");
  if (layer < 0 || layer >= ctx->v.L) return fail(ctx, KV_TIER_E_INVAL, "layer out of range");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSuccess;
  if (e == cudaSuccess) e = launch_score_update(ctx->v, layer, probs, s);
  return cuda_check(ctx, e, "score_update");
}

kv_tier_status kv_tier_end_step(kv_tier_ctx* ctx, void* stream) {
  if (!ctx) return fail(nullptr, KV_TIER_E_INVAL, "null ctx");
  if (!ctx->step_open) return fail(ctx, KV_TIER_E_STATE, "end_step without begin_step");
  if (ctx->lse_pending >= 0) return fail(ctx, KV_TIER_E_STATE, "end_step before kv_tier_score_update_lse");
  cudaError_t e = cudaSuccess;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (e == cudaSuccess && ctx->zpend_n > 0) e = issue_scores(ctx, s);
  if (e == cudaSuccess && ctx->scores_pending) {     // join the score stream: S_part is complete for this step
    e = cudaEventRecord(ctx->ev_score_tail, ctx->score_stream);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ctx->ev_score_tail, 0);
  }
  if (e == cudaSuccess) e = launch_end_step(ctx->v, s);
  kv_tier_status st = cuda_check(ctx, e, "end_step");
  if (st) return st;
  ctx->scores_pending = false;
  for (auto& b : ctx->slot_busy) b = false;
  ctx->zslot_next = 0;
  ctx->zpend_n = 0;
  ctx->step_open = false;
  ctx->pdl_ok = false;
  ctx->t += 1;
  return KV_TIER_OK;
}

static kv_tier_status classify_impl(kv_tier_ctx* ctx, const float* Sx, int parts, void* stream,
                                    const float* snapx = nullptr);

kv_tier_status kv_tier_classify(kv_tier_ctx* ctx, void* stream) {
  if (!ctx) return fail(nullptr, KV_TIER_E_INVAL, "null ctx");
  if (ctx->comm) {
    // sequence shards: every rank classifies the sum of all ranks' S_part (one owner per
    // position, so the sum is exact), all-gathered here over the library's communicator
    const DevView& v = ctx->v;
    const size_t cnt = (size_t)v.B * v.Hkv * v.Nmax;
    const NcclApi& nc = nccl_api();
    ncclResult_t r = nc.group_start();
    if (r == ncclSuccess)
      r = nc.all_gather(v.S, ctx->x_scores, cnt, ncclFloat32, ctx->comm, reinterpret_cast<cudaStream_t>(stream));
    if (r == ncclSuccess && v.snap)            // windowed scorers: every shard's snapshot too (AMB-32)
      r = nc.all_gather(v.snap, ctx->x_snaps, cnt, ncclFloat32, ctx->comm, reinterpret_cast<cudaStream_t>(stream));
    const ncclResult_t r2 = nc.group_end();
    if (r == ncclSuccess) r = r2;
    if (r != ncclSuccess) return fail(ctx, KV_TIER_E_NCCL, "all-gather of S_part: %s", nc.error_string(r));
    return classify_impl(ctx, ctx->x_scores, ctx->cfg.world, stream, v.snap ? ctx->x_snaps : nullptr);
  }
  if ((ctx->cfg.shard == KV_TIER_SHARD_KVHEAD || ctx->cfg.shard == KV_TIER_SHARD_SEQUENCE) && ctx->cfg.world > 1)
    return fail(ctx, KV_TIER_E_STATE, "KV-head sharding: classify needs every shard's scores (kv_tier_classify_gathered)");
  return classify_impl(ctx, nullptr, 1, stream);
}

kv_tier_status kv_tier_classify_gathered(kv_tier_ctx* ctx, const float* S_all, int32_t parts, void* stream) {
  if (!ctx) return fail(nullptr, KV_TIER_E_INVAL, "null ctx");
  if (!S_all || parts < 1) return fail(ctx, KV_TIER_E_INVAL, "S_all must be a device pointer and parts >= 1");
  if (((uintptr_t)S_all) & 3) return fail(ctx, KV_TIER_E_INVAL, "S_all must be 4-B aligned");
  if (scorer_uses_red(ctx->v.scorer) && ctx->v.seq_w <= 1)   // KV-head shards: R_part is per shard
    return fail(ctx, KV_TIER_E_STATE, "redundancy scorers classify from the ctx's own R_part (kv_tier_classify)");
  if (scorer_uses_window(ctx->v.scorer))
    return fail(ctx, KV_TIER_E_STATE, "windowed scorers classify from the ctx's own S_part snapshot (kv_tier_classify)");
  return classify_impl(ctx, S_all, parts, stream);
}

kv_tier_status kv_tier_scores_device(kv_tier_ctx* ctx, void** ptr, size_t* bytes) {
  if (!ctx || !ptr || !bytes) return fail(ctx, KV_TIER_E_INVAL, "null arg");
  *ptr = ctx->v.S;
  *bytes = (size_t)ctx->v.B * ctx->v.Hkv * ctx->v.Nmax * sizeof(float);
  return KV_TIER_OK;
}

static kv_tier_status classify_impl(kv_tier_ctx* ctx, const float* Sx, int parts, void* stream, const float* snapx) {
  if (!ctx->loaded) return fail(ctx, KV_TIER_E_STATE, "no prefix loaded");
  if (ctx->step_open) return fail(ctx, KV_TIER_E_STATE, "classify inside a step (call after the last layer's score update)");
  const kv_tier_config& c = ctx->cfg;
  const long long n = ctx->n, np = n_protected(c, ctx->n), n3 = ctx->c[3];
  const long long nl = n - np - n3;
  long long n_new, n_hbm, n_t2;
  policy_counts(c.policy, c.budget, (int)c.hbm_ratio_bp, (int)c.evict_ratio_bp, (int)c.t2_fraction_bp, c.evict_mode,
                np, nl, n3, &n_new, &n_hbm, &n_t2);
  const long long surv = nl - n_new;
  const int p0 = (int)(np + n_hbm), p1 = (int)(surv - n_hbm - n_t2), p2 = (int)n_t2, p3 = (int)(n3 + n_new);
  if (ctx->v.seq_w <= 1 && (p0 > ctx->v.cap0 || p1 > ctx->v.cap1 || p2 > ctx->v.cap2))   // shards: own counts <= caps
    return fail(ctx, KV_TIER_E_CAPACITY, "tier counts %d/%d/%d exceed capacities %d/%d/%d", p0, p1, p2,
                ctx->v.cap0, ctx->v.cap1, ctx->v.cap2);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSuccess;
  if (ctx->offload_pending) e = cudaStreamWaitEvent(s, ctx->ev_offload_done, 0);
  if (e == cudaSuccess) e = launch_classify(ctx->v, Sx, parts, s, snapx);
  kv_tier_status st = cuda_check(ctx, e, "classify");
  if (st) return st;
  ctx->pend[0] = p0; ctx->pend[1] = p1; ctx->pend[2] = p2; ctx->pend[3] = p3;
  ctx->classified = true;
  return KV_TIER_OK;
}

kv_tier_status kv_tier_migrate(kv_tier_ctx* ctx, void* main_stream, void* side) {
  if (!ctx) return fail(nullptr, KV_TIER_E_INVAL, "null ctx");
  if (!ctx->classified) return fail(ctx, KV_TIER_E_STATE, "migrate without a preceding classify");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(main_stream);
  (void)side;          // differential staging offloads on the ctx's own stream, stream mode in the migrate kernel
  ctx->mig_epoch += 1;                       // host-T1 mode re-reads the T1 lists
  // plan the new row layout, then move only the rows that change, in place: one cooperative
  // launch over chunks of (layer, kv head) pairs (gather + offload of rows entering T1/T2 ->
  // grid barrier -> scatter)
  cudaError_t e = launch_plan(ctx->v, s);
  const int npairs = ctx->v.L * ctx->v.Hkv;
  (void)npairs;
  if (e == cudaSuccess) e = launch_migrate_rows(ctx->v, s);
  if (e == cudaSuccess) e = launch_commit(ctx->v, s);
  if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_migrated, s);
  if (ctx->v.stream_mode || KVT_INLINE_OFFLOAD) {   // rows entering T1/T2 already written by the migrate kernel
    if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_offload_done, s);
  } else {                                   // copy them out beside the next steps (P:643's overlap)
    if (e == cudaSuccess) e = cudaStreamWaitEvent(ctx->offload_stream, ctx->ev_migrated, 0);
    if (e == cudaSuccess) e = launch_offload_rows(ctx->v, ctx->offload_stream);
    if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_offload_done, ctx->offload_stream);
  }
  kv_tier_status st = cuda_check(ctx, e, "migrate");
  if (st) return st;
  ctx->offload_pending = true;
  for (int i = 0; i < 4; ++i) ctx->c[i] = ctx->pend[i];
  ctx->cur ^= 1;
  ctx->n_event = ctx->n;
  ctx->nvis_event = ctx->n - ctx->c[3];
  if (ctx->v.seq_w > 1) {                  // a shard's own counts are decided on the device
    int cn[CNT_STRIDE];
    e = cudaStreamSynchronize(s);
    if (e == cudaSuccess) e = cudaMemcpy(cn, ctx->v.cnt[ctx->cur], sizeof(cn), cudaMemcpyDeviceToHost);
    st = cuda_check(ctx, e, "migrate (sequence shard counts)");
    if (st) return st;
    for (int i = 0; i < 3; ++i) ctx->c[i] = cn[i];
    ctx->c[3] = seq_owned_below(ctx->v.seq_w, ctx->v.seq_r, ctx->n) - cn[4];
    ctx->nvis_event = cn[4];
  }
  ctx->classified = false;
  return KV_TIER_OK;
}

// One decode step of a sequence shard with the library's communicator: per
// layer, this rank's partial softmax (o normalised by its own sum, (m, l) in the log2 domain) ->
// ncclAllGather of every rank's partial -> LSE combine in rank order (deterministic, Eq. 3 over
// the union of the shards) -> the score update rescaled by the global (M, L) (Eq. 1).  Every
// call is stream-ordered, so the whole step captures into one CUDA graph.
static kv_tier_status seq_step(kv_tier_ctx* ctx, const void* q, const void* k_new, const void* v_new, void* o,
                               int32_t fuse_score_update, void* stream, void* side) {
  if (!q || !k_new || !v_new || !o) return fail(ctx, KV_TIER_E_INVAL, "null step buffer");
  if (!fuse_score_update) return fail(ctx, KV_TIER_E_INVAL, "sequence shards fuse the score update (the combine rescales it)");
  const DevView& v = ctx->v;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  const size_t rows = (size_t)v.B * v.Hq, W = (size_t)ctx->cfg.world;
  const size_t qs = rows * v.D, ks = (size_t)v.B * v.Hkv * v.D;
  const char* qb = reinterpret_cast<const char*>(q);
  const char* kb = reinterpret_cast<const char*>(k_new);
  const char* vb = reinterpret_cast<const char*>(v_new);
  float* ob = reinterpret_cast<float*>(o);
  // in-place all-gather: this rank's partial is written straight into its own slot of the receive
  // buffer, one packed (o, m, l) slot per rank -> one ncclAllGather per layer, no send copy
  const size_t slot = ctx->x_slot;
  float* o_send = ctx->x_recv + (size_t)ctx->cfg.rank * slot;
  float* l_send = o_send + rows * v.D;
  kv_tier_status st = kv_tier_begin_step(ctx, stream);
  if (v.stream_mode)
    for (int l = 0; l < std::min(2, v.L) && !st; ++l) st = kv_tier_prefetch(ctx, l, side);
  for (int l = 0; l < v.L && !st; ++l) {
    // PDL: the decode's prologue (barriers, first K/V tiles) overlaps the previous layer's combine;
    // q and the new rows are read after griddepcontrol.wait
    st = decode_attention_impl(ctx, l, qb + l * qs * 2, kb + l * ks * 2, vb + l * ks * 2, o_send, 1, stream,
                               l > 0 && !v.stream_mode ? 1 : 0, l_send);
    if (st) break;
    // (also at world 1, where it is a copy: the one-GPU tests then run the multi-rank code path)
    const NcclApi& nc = nccl_api();
    const ncclResult_t r = nc.all_gather(o_send, ctx->x_recv, slot, ncclFloat32, ctx->comm, s);
    if (r != ncclSuccess) return fail(ctx, KV_TIER_E_NCCL, "layer %d all-gather: %s", l, nc.error_string(r));
    float* lse_l = ctx->x_lse + (size_t)l * rows * 2;
    // the combine also writes the pending score slot's (M, 1/L): no separate set_ml launch
    float* mlz = v.ml + (size_t)ctx->lse_pending * v.B * v.Hkv * 16;
    st = cuda_check(ctx, launch_lse_combine(ctx->x_recv, ctx->x_recv + rows * v.D, (int)W, (int)rows, v.D,
                                            ob + (size_t)l * qs, lse_l, s, mlz, v.G, slot, slot,
                                            v.stream_mode ? 0 : 1), "lse_combine");
    if (!st) st = score_update_lse_impl(ctx, lse_l, stream, true);
    if (!st && v.stream_mode && l + 2 < v.L) st = kv_tier_prefetch(ctx, l + 2, side);
  }
  if (st) return st;
  return kv_tier_end_step(ctx, stream);
}

kv_tier_status kv_tier_step(kv_tier_ctx* ctx, const void* q, const void* k_new, const void* v_new, void* o,
                            int32_t fuse_score_update, void* stream, void* side) {
  if (!ctx) return fail(nullptr, KV_TIER_E_INVAL, "null ctx");
  if (ctx->comm) return seq_step(ctx, q, k_new, v_new, o, fuse_score_update, stream, side);
  if (ctx->v.seq_w > 1) return fail(ctx, KV_TIER_E_STATE, "sequence shards without a communicator combine every layer: drive decode_attention_lse per layer");
  if (!q || !k_new || !v_new || !o) return fail(ctx, KV_TIER_E_INVAL, "null step buffer");
  const DevView& v = ctx->v;
  const size_t qs = (size_t)v.B * v.Hq * v.D, ks = (size_t)v.B * v.Hkv * v.D;
  const size_t os = qs * (v.out_fp32 ? 4 : 2);
  const char* qb = reinterpret_cast<const char*>(q);
  const char* kb = reinterpret_cast<const char*>(k_new);
  const char* vb = reinterpret_cast<const char*>(v_new);
  char* ob = reinterpret_cast<char*>(o);
  kv_tier_status st = kv_tier_begin_step(ctx, stream);
  if (st) return st;
  if (v.step_k > 0 && !v.host_t1) {
    // every layer in one launch: a1 + a3 + a4 with the per-request layer dependency inside
    st = cuda_check(ctx, launch_decode_step(v, q, k_new, v_new, o, fuse_score_update, reinterpret_cast<cudaStream_t>(stream)),
                    "decode_step");
    if (st) return st;
    for (int l = 0; l < v.L; ++l) ctx->appended_step[l] = ctx->t;
    return kv_tier_end_step(ctx, stream);
  }
  if (v.stream_mode)
    for (int l = 0; l < std::min(2, v.L) && !st; ++l) st = kv_tier_prefetch(ctx, l, side);
  // a1 fused into the attention kernel; consecutive layers chained with programmatic
  // dependent launch (each kernel's prologue overlaps the previous layer's tail)
  for (int l = 0; l < v.L && !st; ++l) {
    st = decode_attention_impl(ctx, l, qb + l * qs * 2, kb + l * ks * 2, vb + l * ks * 2, ob + l * os,
                               fuse_score_update, stream, l > 0 && !v.stream_mode);
    if (!st && v.stream_mode && l + 2 < v.L) st = kv_tier_prefetch(ctx, l + 2, side);
  }
  if (st) return st;
  return kv_tier_end_step(ctx, stream);
}

// External capture of a whole decoder step (the caller's CUDA graph holds this ctx's step calls
// between its own kernels): the host state machine runs once during the capture and is restored
// afterwards; kv_tier_graph_advance then advances it once per replay (kernels read the step and
// tier counters from device memory, so one graph serves every step).
kv_tier_status kv_tier_capture_begin(kv_tier_ctx* ctx) {
  if (!ctx) return fail(nullptr, KV_TIER_E_INVAL, "null ctx");
  if (ctx->step_open) return fail(ctx, KV_TIER_E_STATE, "capture inside a step");
  if (!ctx->loaded) return fail(ctx, KV_TIER_E_STATE, "no prefix loaded");
  if (ctx->capturing) return fail(ctx, KV_TIER_E_STATE, "capture already open");
  ctx->cap.n = ctx->n;
  ctx->cap.t = ctx->t;
  ctx->cap.c0 = ctx->c[0];
  ctx->cap.classified = ctx->classified;
  ctx->cap.pstep = ctx->prefetched_step;
  ctx->cap.astep = ctx->appended_step;
  ctx->capturing = true;
  ctx->pdl_ok = false;
  return KV_TIER_OK;
}
kv_tier_status kv_tier_capture_end(kv_tier_ctx* ctx) {
  if (!ctx) return fail(nullptr, KV_TIER_E_INVAL, "null ctx");
  if (!ctx->capturing) return fail(ctx, KV_TIER_E_STATE, "no capture open");
  ctx->capturing = false;
  ctx->pdl_ok = false;
  ctx->n = ctx->cap.n; ctx->t = ctx->cap.t; ctx->c[0] = ctx->cap.c0; ctx->classified = ctx->cap.classified;
  ctx->step_open = false;
  ctx->prefetched_step = ctx->cap.pstep;
  ctx->appended_step = ctx->cap.astep;
  ctx->zslot_next = 0;
  ctx->zpend_n = 0;
  for (auto& b : ctx->slot_busy) b = false;
  ctx->scores_pending = false;
  return KV_TIER_OK;
}
kv_tier_status kv_tier_graph_advance(kv_tier_ctx* ctx) {
  if (!ctx) return fail(nullptr, KV_TIER_E_INVAL, "null ctx");
  if (ctx->step_open || ctx->capturing) return fail(ctx, KV_TIER_E_STATE, "advance inside a step or a capture");
  if (ctx->n + 1 > ctx->v.Nmax) return fail(ctx, KV_TIER_E_CAPACITY, "N_max=%d reached", ctx->v.Nmax);
  if (ctx->c[0] + 1 > ctx->v.cap0) return fail(ctx, KV_TIER_E_CAPACITY, "T0 store full (%d rows)", ctx->v.cap0);
  ctx->c[0] += seq_own(ctx->v.seq_w, ctx->v.seq_r, ctx->n) ? 1 : 0;
  ctx->n += 1;
  ctx->t += 1;
  ctx->classified = false;
  return KV_TIER_OK;
}

kv_tier_status kv_tier_step_graph_capture(kv_tier_ctx* ctx, const void* q, const void* k_new, const void* v_new,
                                          void* o, int32_t fuse_score_update, void* stream, void* side) {
  if (!ctx) return fail(nullptr, KV_TIER_E_INVAL, "null ctx");
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  if (s == nullptr) return fail(ctx, KV_TIER_E_INVAL, "capture needs a non-default stream");
  kv_tier_status st = kv_tier_capture_begin(ctx);
  if (st) return st;
  if (ctx->graph_exec) { cudaGraphExecDestroy(ctx->graph_exec); ctx->graph_exec = nullptr; }
  if (ctx->graph) { cudaGraphDestroy(ctx->graph); ctx->graph = nullptr; }
  cudaError_t e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
  if (e != cudaSuccess) { kv_tier_capture_end(ctx); return cuda_check(ctx, e, "begin capture"); }
  st = kv_tier_step(ctx, q, k_new, v_new, o, fuse_score_update, stream, side);
  cudaGraph_t g = nullptr;
  e = cudaStreamEndCapture(s, &g);
  kv_tier_capture_end(ctx);
  if (st) { if (g) cudaGraphDestroy(g); return st; }
  if (e != cudaSuccess) return cuda_check(ctx, e, "end capture");
  e = cudaGraphInstantiate(&ctx->graph_exec, g, 0);
  if (e != cudaSuccess) { cudaGraphDestroy(g); return cuda_check(ctx, e, "graph instantiate"); }
  ctx->graph = g;
  return KV_TIER_OK;
}
kv_tier_status kv_tier_step_graph_launch(kv_tier_ctx* ctx, void* stream) {
  if (!ctx) return fail(nullptr, KV_TIER_E_INVAL, "null ctx");
  if (!ctx->graph_exec) return fail(ctx, KV_TIER_E_STATE, "no step graph captured");
  if (ctx->step_open) return fail(ctx, KV_TIER_E_STATE, "graph launch inside a step");
  if (ctx->n + 1 > ctx->v.Nmax) return fail(ctx, KV_TIER_E_CAPACITY, "N_max=%d reached", ctx->v.Nmax);
  if (ctx->c[0] + 1 > ctx->v.cap0) return fail(ctx, KV_TIER_E_CAPACITY, "T0 store full (%d rows)", ctx->v.cap0);
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  cudaError_t e = cudaSuccess;
  if (ctx->offload_pending && ctx->v.stream_mode) e = cudaStreamWaitEvent(s, ctx->ev_offload_done, 0);
  if (e == cudaSuccess) e = cudaGraphLaunch(ctx->graph_exec, s);
  kv_tier_status st = cuda_check(ctx, e, "graph launch");
  if (st) return st;
  ctx->c[0] += seq_own(ctx->v.seq_w, ctx->v.seq_r, ctx->n) ? 1 : 0;
  ctx->n += 1;
  ctx->t += 1;
  ctx->classified = false;
  return KV_TIER_OK;
}

kv_tier_status kv_tier_sync(kv_tier_ctx* ctx) {
  if (!ctx) return fail(nullptr, KV_TIER_E_INVAL, "null ctx");
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return fail(ctx, KV_TIER_E_CUDA, "async CUDA error: %s", cudaGetErrorString(e));
  DevState h;
  e = cudaMemcpy(&h, ctx->v.st, sizeof(h), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return fail(ctx, KV_TIER_E_CUDA, "state read: %s", cudaGetErrorString(e));
  if (h.err & 2) return fail(ctx, KV_TIER_E_CAPACITY, "a tier store of this sequence shard overflowed at classify (its share of T1/T2 exceeded 1.25x the fair share)");
  if (h.err & 4) return fail(ctx, KV_TIER_E_CUDA, "a device-side wait timed out (2 s watchdog: a co-scheduled CTA never arrived)");
  if (h.err) return fail(ctx, KV_TIER_E_NUMERIC, "non-finite probability or score detected on device");
  if (h.n != ctx->n || h.cur != ctx->cur)
    return fail(ctx, KV_TIER_E_STATE, "device/host state diverged (n %d/%d cur %d/%d)", h.n, ctx->n, h.cur, ctx->cur);
  return KV_TIER_OK;
}

kv_tier_status kv_tier_census(kv_tier_ctx* ctx, int32_t* counts, int64_t* d2h_rows) {
  kv_tier_status st = kv_tier_sync(ctx);
  if (st) return st;
  if (counts) {
    std::vector<int> cn((size_t)ctx->v.B * CNT_STRIDE);
    cudaError_t e = cudaMemcpy(cn.data(), ctx->v.cnt[ctx->cur], cn.size() * 4, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_check(ctx, e, "census");
    for (int b = 0; b < ctx->v.B; ++b) {
      // counts over [0, n): T3 is n - |visible| (positions appended since the event are T0)
      for (int i = 0; i < 3; ++i) counts[b * 4 + i] = cn[b * CNT_STRIDE + i];
      counts[b * 4 + 3] = seq_owned_below(ctx->v.seq_w, ctx->v.seq_r, ctx->n) - cn[b * CNT_STRIDE + 0] -
                          cn[b * CNT_STRIDE + 1] - cn[b * CNT_STRIDE + 2];
    }
  }
  if (d2h_rows) {
    DevState h;
    cudaMemcpy(&h, ctx->v.st, sizeof(h), cudaMemcpyDeviceToHost);
    *d2h_rows = (int64_t)h.d2h_rows;
  }
  return KV_TIER_OK;
}

kv_tier_status kv_tier_position(const kv_tier_ctx* ctx, int32_t* n, int32_t* t) {
  if (!ctx) return fail(nullptr, KV_TIER_E_INVAL, "null ctx");
  if (n) *n = ctx->n;
  if (t) *t = ctx->t;
  return KV_TIER_OK;
}

// Per-request tier counts |T0| |T1| |T2| of the live buffer (uniform across requests except
// under sequence sharding, where a shard's own counts depend on the request's tiers).
static kv_tier_status req_counts(kv_tier_ctx* ctx, std::vector<int>& cb) {
  kv_tier_status st = kv_tier_sync(ctx);
  if (st) return st;
  std::vector<int> cn((size_t)ctx->v.B * CNT_STRIDE);
  cudaError_t e = cudaMemcpy(cn.data(), ctx->v.cnt[ctx->cur], cn.size() * 4, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_check(ctx, e, "export counts");
  cb.assign((size_t)ctx->v.B * 3, 0);
  for (int b = 0; b < ctx->v.B; ++b)
    for (int T = 0; T < 3; ++T) cb[(size_t)b * 3 + T] = cn[(size_t)b * CNT_STRIDE + T];
  return KV_TIER_OK;
}

// Bytes of one request's export `what` given its counts c[3].
static size_t export_bytes_req(const kv_tier_ctx* ctx, int32_t what, const int* c) {
  const size_t H = ctx->v.Hkv, D = ctx->v.D, n = ctx->n;
  switch (what) {
    case KV_TIER_X_SCORES: case KV_TIER_X_REDUNDANCY: case KV_TIER_X_SNAPSHOT: return H * n * 4;
    case KV_TIER_X_TIERS: return n;
    case KV_TIER_X_IDX_T0: return (size_t)c[0] * 4;
    case KV_TIER_X_IDX_T1: return (size_t)c[1] * 4;
    case KV_TIER_X_IDX_T2: return (size_t)c[2] * 4;
    case KV_TIER_X_T0_ROWS: return H * c[0] * 2 * D * 2;
    case KV_TIER_X_T1_ROWS: case KV_TIER_X_STAGING: return H * c[1] * 2 * D * 2;
    case KV_TIER_X_T2_CODES: return H * c[2] * 2 * D;
    case KV_TIER_X_T2_SCALES: return H * c[2] * 2 * 4;
    default: return (size_t)-1;
  }
}

kv_tier_status kv_tier_export_size(kv_tier_ctx* ctx, int32_t what, size_t* bytes) {
  if (!ctx || !bytes) return fail(nullptr, KV_TIER_E_INVAL, "null arg");
  if (ctx->step_open) return fail(ctx, KV_TIER_E_STATE, "export inside a step");
  std::vector<int> cb;
  kv_tier_status st = req_counts(ctx, cb);
  if (st) return st;
  size_t tot = 0;
  for (int b = 0; b < ctx->v.B; ++b) {
    const size_t x = export_bytes_req(ctx, what, &cb[(size_t)b * 3]);
    if (x == (size_t)-1) return fail(ctx, KV_TIER_E_INVAL, "unknown export %d", what);
    tot += x;
  }
  *bytes = tot;
  return KV_TIER_OK;
}

kv_tier_status kv_tier_export(kv_tier_ctx* ctx, int32_t what, int32_t layer, void* host_dst, size_t bytes) {
  size_t need = 0;
  kv_tier_status st = kv_tier_export_size(ctx, what, &need);
  if (st) return st;
  if (!host_dst || bytes != need) return fail(ctx, KV_TIER_E_INVAL, "export %d needs %zu bytes, got %zu", what, need, bytes);
  if (layer < 0 || layer >= ctx->v.L) return fail(ctx, KV_TIER_E_INVAL, "layer out of range");
  std::vector<int> cb;
  st = req_counts(ctx, cb);                 // (synchronised)
  if (st) return st;
  const DevView& v = ctx->v;
  const int cur = ctx->cur;
  DevState hs;
  cudaError_t e = cudaMemcpy(&hs, v.st, sizeof(hs), cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_check(ctx, e, "export state");
  const int sb = hs.scur;              // row-store buffer
  const size_t B = v.B, H = v.Hkv, D = v.D, N = v.Nmax, n = ctx->n;
  char* out = reinterpret_cast<char*>(host_dst);
  auto d2h = [&](void* dst, const void* src, size_t nbytes) {
    return cudaMemcpy(dst, src, nbytes, cudaMemcpyDeviceToHost);
  };
  const int caps[3] = {v.cap0, v.cap1, v.cap2};
  // store-order index list of tier T for request b and the permutation to ascending positions
  auto order = [&](int T, size_t b, std::vector<int>& pos, std::vector<int>& perm) {
    const int cnt = cb[b * 3 + T];
    pos.assign((size_t)std::max(cnt, 1), 0);
    cudaError_t ee = d2h(pos.data(), v.idx[cur][T] + b * caps[T], (size_t)cnt * 4);
    perm.resize(cnt);
    for (int j = 0; j < cnt; ++j) perm[j] = j;
    std::sort(perm.begin(), perm.end(), [&](int x, int y) { return pos[x] < pos[y]; });
    return ee;
  };
  std::vector<int> pos, perm;
  size_t off = 0;                      // this request's byte offset in host_dst
  for (size_t b = 0; b < B && e == cudaSuccess; ++b) {
    const int* c = &cb[b * 3];
    char* ob = out + off;
    off += export_bytes_req(ctx, what, c);
    if (what == KV_TIER_X_SCORES) {
      for (size_t g = 0; g < H && e == cudaSuccess; ++g) e = d2h(ob + g * n * 4, v.S + (b * H + g) * N, n * 4);
    } else if (what == KV_TIER_X_REDUNDANCY) {
      if (!v.red) memset(ob, 0, H * n * 4);
      for (size_t g = 0; g < H && v.red && e == cudaSuccess; ++g) e = d2h(ob + g * n * 4, v.red + (b * H + g) * N, n * 4);
    } else if (what == KV_TIER_X_SNAPSHOT) {
      if (!v.snap) memset(ob, 0, H * n * 4);
      for (size_t g = 0; g < H && v.snap && e == cudaSuccess; ++g) e = d2h(ob + g * n * 4, v.snap + (b * H + g) * N, n * 4);
    } else if (what == KV_TIER_X_TIERS) {
      e = d2h(ob, v.tier[cur] + b * N, n);
    } else if (what >= KV_TIER_X_IDX_T0 && what <= KV_TIER_X_IDX_T2) {
      const int T = what - KV_TIER_X_IDX_T0;
      e = order(T, b, pos, perm);
      int* o32 = reinterpret_cast<int*>(ob);
      for (int j = 0; j < c[T]; ++j) o32[j] = pos[perm[j]];
    } else if (what == KV_TIER_X_T0_ROWS || what == KV_TIER_X_STAGING) {
      const bool t0 = what == KV_TIER_X_T0_ROWS;
      if (!t0 && v.stream_mode) return fail(ctx, KV_TIER_E_STATE, "no persistent staging in stream mode");
      const int T = t0 ? 0 : 1;
      const int cnt = c[T];
      const int cap = caps[T];
      const __nv_bfloat16* Ks = t0 ? v.k0[sb] : v.k1[sb];
      const __nv_bfloat16* Vs = t0 ? v.v0[sb] : v.v1[sb];
      std::vector<uint16_t> tk((size_t)((cnt + 7) & ~7) * D), tv((size_t)((cnt + 7) & ~7) * D);   // whole 8-row groups
      e = order(T, b, pos, perm);
      for (size_t g = 0; g < H && e == cudaSuccess; ++g) {
        const size_t grp = ((size_t)layer * B + b) * H + g;
        e = d2h(tk.data(), Ks + grp * cap * D, tk.size() * 2);
        if (e == cudaSuccess) e = d2h(tv.data(), Vs + grp * cap * D, tv.size() * 2);
        uint16_t* o16 = reinterpret_cast<uint16_t*>(ob) + (g * cnt) * 2 * D;
        for (int jj = 0; jj < cnt; ++jj) {
          const int j = perm[jj];
          for (size_t el = 0; el < D; ++el) {     // undo the store swizzle
            o16[(size_t)jj * 2 * D + el] = tk[(size_t)j * D + swz_off(j, (int)el, (int)D)];
            o16[(size_t)jj * 2 * D + D + el] = tv[(size_t)j * D + swz_off(j, (int)el, (int)D)];
          }
        }
      }
    } else if (what == KV_TIER_X_T1_ROWS) {
      const int cnt = c[1];
      const size_t rows = (size_t)v.L * B * H * v.hN;
      const uint16_t* hk = reinterpret_cast<const uint16_t*>(ctx->host_t1);
      const uint16_t* hv = hk ? hk + rows * D : nullptr;
      if (cnt > 0 && !hk) return fail(ctx, KV_TIER_E_STATE, "no host T1 store");
      e = order(1, b, pos, perm);
      for (size_t g = 0; g < H && e == cudaSuccess; ++g) {
        const size_t grp = ((size_t)layer * B + b) * H + g;
        uint16_t* o16 = reinterpret_cast<uint16_t*>(ob) + (g * cnt) * 2 * D;
        for (int jj = 0; jj < cnt; ++jj) {
          const int p = pos[perm[jj]];
          memcpy(o16 + (size_t)jj * 2 * D, hk + host_row(v, grp, p) * D, D * 2);
          memcpy(o16 + (size_t)jj * 2 * D + D, hv + host_row(v, grp, p) * D, D * 2);
        }
      }
    } else if (what == KV_TIER_X_T2_CODES || what == KV_TIER_X_T2_SCALES) {
      const int cnt = c[2];
      const bool codes = what == KV_TIER_X_T2_CODES;
      std::vector<int8_t> ck((size_t)cnt * D + 1), cv((size_t)cnt * D + 1);
      std::vector<float> sk((size_t)cnt + 1), sv((size_t)cnt + 1);
      e = order(2, b, pos, perm);
      for (size_t g = 0; g < H && e == cudaSuccess; ++g) {
        const size_t grp = ((size_t)layer * B + b) * H + g;
        if (codes) {
          e = d2h(ck.data(), v.c2k[sb] + grp * v.cap2 * D, (size_t)cnt * D);
          if (e == cudaSuccess) e = d2h(cv.data(), v.c2v[sb] + grp * v.cap2 * D, (size_t)cnt * D);
          int8_t* o8 = reinterpret_cast<int8_t*>(ob) + (g * cnt) * 2 * D;
          for (int jj = 0; jj < cnt; ++jj) {
            memcpy(o8 + (size_t)jj * 2 * D, ck.data() + (size_t)perm[jj] * D, D);
            memcpy(o8 + (size_t)jj * 2 * D + D, cv.data() + (size_t)perm[jj] * D, D);
          }
        } else {
          e = d2h(sk.data(), v.s2k[sb] + grp * v.cap2, (size_t)cnt * 4);
          if (e == cudaSuccess) e = d2h(sv.data(), v.s2v[sb] + grp * v.cap2, (size_t)cnt * 4);
          float* of = reinterpret_cast<float*>(ob) + (g * cnt) * 2;
          for (int jj = 0; jj < cnt; ++jj) { of[2 * jj] = sk[perm[jj]]; of[2 * jj + 1] = sv[perm[jj]]; }
        }
      }
    }
  }
  return cuda_check(ctx, e, "export");
}

kv_tier_status kv_tier_debug_trace_len(const kv_tier_ctx* ctx, size_t* n) {
  if (!ctx || !n) return fail(nullptr, KV_TIER_E_INVAL, "null arg");
  *n = (size_t)ctx->v.L * (std::max(ctx->v.split * ctx->v.B * ctx->v.Hkv, 2 * 148)) * NTRACE;
  return KV_TIER_OK;
}

kv_tier_status kv_tier_debug_trace(kv_tier_ctx* ctx, uint64_t* host_dst, size_t n) {
  if (!ctx || !host_dst) return fail(ctx, KV_TIER_E_INVAL, "null arg");
  const size_t need = (size_t)ctx->v.L * (std::max(ctx->v.split * ctx->v.B * ctx->v.Hkv, 2 * 148)) * NTRACE;
  if (!ctx->trace) return fail(ctx, KV_TIER_E_STATE, "tracing off (set KVTIER_TRACE=1 before kv_tier_init)");
  if (n != need) return fail(ctx, KV_TIER_E_INVAL, "trace needs %zu entries", need);
  cudaError_t e = cudaDeviceSynchronize();
  if (e == cudaSuccess) e = cudaMemcpy(host_dst, ctx->trace, need * 8, cudaMemcpyDeviceToHost);
  return cuda_check(ctx, e, "trace");
}

// ------------------------------------------------------------------ N1: host-side T1 attention
// SURVEY §8f N1 (ScoutAttention-style): T1 is attended where it lives.  Per layer
// q goes down and (o, m, l) plus the T1 score increments come up -- O(B·H_q·d + B·H_kv·|T1|)
// floats instead of |T1| rows.  The host loops are the same softmax as the decode kernel's
// (log2 domain, fp32), split by tier and recombined by kv_tier_lse_combine (Eq. 3).
// 2^x for x <= 0 on the host, vectorisable (no libm call): x = n + f, |f| <= 1/2, 2^f by its
// degree-7 Taylor polynomial in f·ln2 (relative error < 1e-8, below fp32 rounding), times 2^n
// built in the exponent bits.  Inputs below -126 return 2^-126 (negligible against l >= 1).
static inline float h1_exp2(float x) {
  x = std::max(x, -126.f);
  const float n = __builtin_rintf(x);
  const float t = (x - n) * 0.69314718056f;
  float p = 1.f / 5040.f;
  p = p * t + 1.f / 720.f;
  p = p * t + 1.f / 120.f;
  p = p * t + 1.f / 24.f;
  p = p * t + 1.f / 6.f;
  p = p * t + 0.5f;
  p = p * t + 1.f;
  p = p * t + 1.f;
  return p * __uint_as_float_host((uint32_t)((int)n + 127) << 23);
}

// One (request, kv head) of the host T1 partial, G a compile-time group size.  Pass 1: each K
// row converted once; the G dot products run interleaved in G vector accumulators (independent
// FMA chains, no per-head latency chain), z[h][j] = fp32(q_h·k_j)·sl2, m_h = max.  Pass 2, R = 16
// rows at a time: p = 2^(z - m) vectorised over rows (h1_exp2, no libm call), then o_h += p_r v_r
// with each V row converted once.  Inlined into h1_unit's target clones (AVX-512 / AVX2 / base).
extern "C++" {
template <int G>
static inline __attribute__((always_inline)) void h1_body(int n1, int D, float sl2, const uint16_t* q,
    const uint16_t* hk, const uint16_t* hv, const int* idx, size_t row0, int seq_w, int seq_r, float* z,
    size_t zst, float* o, float* lse) {
  constexpr int R = 16, V = 16;
  alignas(64) float qf[G][128], acc[G][128], row[128], pb[G][R];
  float m[G], l[G];
  for (int h = 0; h < G; ++h) {
    for (int e = 0; e < D; ++e) {
      qf[h][e] = __uint_as_float_host((uint32_t)q[(size_t)h * D + e] << 16);
      acc[h][e] = 0.f;
    }
    m[h] = -INFINITY;
    l[h] = 0.f;
  }
  auto rowp = [&](int pos) {
    return row0 + (size_t)(seq_w > 1 ? seq_owned_below(seq_w, seq_r, pos) : pos);
  };
  constexpr int PF = 4;                    // software prefetch distance (rows are scattered)
  for (int j = 0; j < n1; ++j) {           // pass 1: z and m
    const uint16_t* kr = hk + rowp(idx[j]) * D;
    if (j + PF < n1) {
      const char* nx = reinterpret_cast<const char*>(hk + rowp(idx[j + PF]) * D);
      for (int c = 0; c < D * 2; c += 64) __builtin_prefetch(nx + c, 0, 0);
    }
#pragma omp simd
    for (int e = 0; e < D; ++e) row[e] = __uint_as_float_host((uint32_t)kr[e] << 16);
    alignas(64) float va[G][V];
    for (int h = 0; h < G; ++h)
#pragma omp simd
      for (int k = 0; k < V; ++k) va[h][k] = 0.f;
    for (int e0 = 0; e0 < D; e0 += V)
      for (int h = 0; h < G; ++h)
#pragma omp simd
        for (int k = 0; k < V; ++k) va[h][k] += qf[h][e0 + k] * row[e0 + k];
    for (int h = 0; h < G; ++h) {
      float sdot = 0.f;
#pragma omp simd reduction(+ : sdot)
      for (int k = 0; k < V; ++k) sdot += va[h][k];
      const float zr = sdot * sl2;
      z[(size_t)h * zst + j] = zr;
      m[h] = std::max(m[h], zr);
    }
  }
  for (int j0 = 0; j0 < n1; j0 += R) {     // pass 2: p vectorised over R rows, then o
    const int nb = std::min(R, n1 - j0);
    for (int h = 0; h < G; ++h) {
      const float* zh = z + (size_t)h * zst + j0;
      float ls = 0.f;
#pragma omp simd reduction(+ : ls)
      for (int r = 0; r < R; ++r) {
        const float p = r < nb ? h1_exp2(zh[r < nb ? r : 0] - m[h]) : 0.f;
        pb[h][r] = p;
        ls += p;
      }
      l[h] += ls;
    }
    for (int r = 0; r < nb; ++r) {
      const uint16_t* vr = hv + rowp(idx[j0 + r]) * D;
      if (j0 + r + PF < n1) {
        const char* nx = reinterpret_cast<const char*>(hv + rowp(idx[j0 + r + PF]) * D);
        for (int c = 0; c < D * 2; c += 64) __builtin_prefetch(nx + c, 0, 0);
      }
#pragma omp simd
      for (int e = 0; e < D; ++e) row[e] = __uint_as_float_host((uint32_t)vr[e] << 16);
      for (int h = 0; h < G; ++h) {
        const float p = pb[h][r];
#pragma omp simd
        for (int e = 0; e < D; ++e) acc[h][e] += p * row[e];
      }
    }
  }
  for (int h = 0; h < G; ++h) {
    const float inv = l[h] > 0.f ? 1.f / l[h] : 0.f;
    for (int e = 0; e < D; ++e) o[(size_t)h * D + e] = acc[h][e] * inv;
    lse[(size_t)h * 2] = m[h];
    lse[(size_t)h * 2 + 1] = l[h];
  }
}
}  // extern "C++"

// Measured on the 7B shape (G = 7, 16 host threads, same-box A/B, scripts/exp_h1_only.py):
// libm exp2f per element 61 steps/s, vectorised exp2 65, + software prefetch of the scattered
// rows 8 ahead 72 (24 ahead: 56; 4 ahead: 75-96 on a box whose baseline also drifted 72 -> 99).
// The loop is bound by host memory latency on scattered 256-B rows, not by FMAs.
__attribute__((target_clones("avx512f", "avx2", "default")))
static void h1_unit(int n1, int G, int D, float sl2, const uint16_t* q, const uint16_t* hk, const uint16_t* hv,
                    const int* idx, size_t row0, int seq_w, int seq_r, float* z, size_t zst, float* o, float* lse) {
  switch (G) {
#define H1_CASE(g) case g: h1_body<g>(n1, D, sl2, q, hk, hv, idx, row0, seq_w, seq_r, z, zst, o, lse); break;
    H1_CASE(1) H1_CASE(2) H1_CASE(3) H1_CASE(4) H1_CASE(5) H1_CASE(6) H1_CASE(7) H1_CASE(8)
#undef H1_CASE
    default: break;
  }
}

// Eq. 1 increments of one (request, kv head)'s T1 tokens: inc[j] = sum_h 2^(z_hj - M_h) / L_h.
__attribute__((target_clones("avx512f", "avx2", "default")))
static void h1_scores(int n1, int G, const float* z, size_t zst, const float* lse_g, float* inc) {
  for (int j = 0; j < n1; ++j) inc[j] = 0.f;
  for (int h = 0; h < G; ++h) {
    const float M = lse_g[(size_t)h * 2], L = lse_g[(size_t)h * 2 + 1];
    const float invL = L > 0.f ? 1.f / L : 0.f;
    const float* zh = z + (size_t)h * zst;
#pragma omp simd
    for (int j = 0; j < n1; ++j) inc[j] += h1_exp2(zh[j] - M) * invL;
  }
}

kv_tier_status kv_tier_set_host_t1(kv_tier_ctx* ctx, int32_t on) {
  if (!ctx) return fail(nullptr, KV_TIER_E_INVAL, "null ctx");
  if (ctx->step_open) return fail(ctx, KV_TIER_E_STATE, "set_host_t1 inside a step");
  if (on && ctx->v.scorer != KV_TIER_SCORER_ATTENTION) return fail(ctx, KV_TIER_E_STATE, "host-T1 mode supports the attention scorer");
  if (on && ctx->v.seq_w > 1) return fail(ctx, KV_TIER_E_STATE, "host-T1 mode: not with sequence sharding");
  const size_t ninc = (size_t)ctx->v.B * ctx->v.Hkv * std::max(ctx->v.cap1, 1);
  for (int i = 0; on && i < 2; ++i) {
    if (!ctx->h1_inc[i]) {
      cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&ctx->h1_inc[i]), ninc * 4, cudaHostAllocMapped | cudaHostAllocPortable);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_inc[i], cudaEventDisableTiming);
      if (e != cudaSuccess) return cuda_check(ctx, e, "set_host_t1 (staging)");
    }
  }
  if (on && !ctx->h1_q) {
    const size_t rows = (size_t)ctx->v.B * ctx->v.Hq, D = ctx->v.D;
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&ctx->h1_q), rows * D * 2, cudaHostAllocPortable);
    if (e == cudaSuccess) e = cudaHostAlloc(reinterpret_cast<void**>(&ctx->h1_o), rows * (D + 4) * 4, cudaHostAllocPortable);
    if (e == cudaSuccess) e = cudaMalloc(reinterpret_cast<void**>(&ctx->d1_parts), rows * (2 * D + 6) * 4);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_q, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_check(ctx, e, "set_host_t1 (layer staging)");
  }
  ctx->v.host_t1 = on ? 1 : 0;
  ctx->h1_epoch = -1;
  ctx->h1_layer = -1;
  return KV_TIER_OK;
}

kv_tier_status kv_tier_host_t1_attention(kv_tier_ctx* ctx, int32_t layer, const void* q_host, float* o_part,
                                         float* lse_part) {
  if (!ctx) return fail(nullptr, KV_TIER_E_INVAL, "null ctx");
  if (!ctx->v.host_t1) return fail(ctx, KV_TIER_E_STATE, "host-T1 mode is off (kv_tier_set_host_t1)");
  if (!ctx->step_open) return fail(ctx, KV_TIER_E_STATE, "host_t1_attention outside begin_step/end_step");
  if (layer < 0 || layer >= ctx->v.L) return fail(ctx, KV_TIER_E_INVAL, "layer out of range");
  if (!q_host || !o_part || !lse_part) return fail(ctx, KV_TIER_E_INVAL, "null q/o/lse");
  const DevView& v = ctx->v;
  const int B = v.B, Hq = v.Hq, Hkv = v.Hkv, G = v.G, D = v.D, cap1 = std::max(v.cap1, 1);
  if (ctx->h1_epoch != ctx->mig_epoch) {     // first call after a migrate: read the T1 lists
    std::vector<int> cn((size_t)B * CNT_STRIDE);
    ctx->h1_idx.assign((size_t)B * cap1, 0);
    ctx->h1_cnt.assign(B, 0);
    cudaError_t e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemcpy(cn.data(), v.cnt[ctx->cur], cn.size() * 4, cudaMemcpyDeviceToHost);
    if (e == cudaSuccess && v.cap1 > 0)
      e = cudaMemcpy(ctx->h1_idx.data(), v.idx[ctx->cur][1], (size_t)B * v.cap1 * 4, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return cuda_check(ctx, e, "host_t1_attention (T1 lists)");
    for (int b = 0; b < B; ++b) ctx->h1_cnt[b] = cn[(size_t)b * CNT_STRIDE + 1];
    ctx->h1_z.assign((size_t)B * Hq * cap1, 0.f);
    ctx->h1_epoch = ctx->mig_epoch;
  }
  const size_t rows = (size_t)v.L * B * Hkv * v.hN;
  const uint16_t* hk = reinterpret_cast<const uint16_t*>(ctx->host_t1);
  if (!hk && std::any_of(ctx->h1_cnt.begin(), ctx->h1_cnt.end(), [](int c) { return c > 0; }))
    return fail(ctx, KV_TIER_E_STATE, "T1 tokens without a host T1 store");   // (beta = 100 % keeps T1 empty)
  const uint16_t* hv = hk ? hk + rows * D : nullptr;
  const uint16_t* q = reinterpret_cast<const uint16_t*>(q_host);
  const float sl2 = (float)(1.4426950408889634 / std::sqrt((double)D));
  const size_t zst = (size_t)cap1;
#pragma omp parallel for schedule(dynamic, 1)
  for (int bg = 0; bg < B * Hkv; ++bg) {       // one (request, kv head): each T1 row read once for its G heads
    const int b = bg / Hkv, g = bg % Hkv;
    const size_t grp = ((size_t)layer * B + b) * Hkv + g;
    const size_t bh0 = (size_t)b * Hq + (size_t)g * G;
    h1_unit(ctx->h1_cnt[b], G, D, sl2, q + bh0 * D, hk, hv, ctx->h1_idx.data() + (size_t)b * cap1,
            grp * (size_t)v.hN, v.seq_w, v.seq_r, ctx->h1_z.data() + bh0 * zst, zst, o_part + bh0 * D,
            lse_part + bh0 * 2);
  }
  ctx->h1_layer = layer;
  return KV_TIER_OK;
}

kv_tier_status kv_tier_host_t1_score_update(kv_tier_ctx* ctx, int32_t layer, const float* lse_global_host,
                                            void* stream) {
  if (!ctx) return fail(nullptr, KV_TIER_E_INVAL, "null ctx");
  if (!lse_global_host) return fail(ctx, KV_TIER_E_INVAL, "null lse_global");
  if (!ctx->v.host_t1 || ctx->h1_layer != layer)
    return fail(ctx, KV_TIER_E_STATE, "host_t1_score_update(layer %d) must follow host_t1_attention of that layer", layer);
  const DevView& v = ctx->v;
  const int B = v.B, Hq = v.Hq, Hkv = v.Hkv, G = v.G, cap1 = std::max(v.cap1, 1);
  const int buf = layer & 1;
  cudaError_t e = cudaSuccess;
  if (ctx->inc_used[buf]) e = cudaEventSynchronize(ctx->ev_inc[buf]);   // its previous scatter is done
  if (e != cudaSuccess) return cuda_check(ctx, e, "host_t1_score_update (staging)");
  float* inc = ctx->h1_inc[buf];
#pragma omp parallel for schedule(static)
  for (int bg = 0; bg < B * Hkv; ++bg) {   // Eq. 1: sum over the group's q heads of 2^(z - M) / L
    const int b = bg / Hkv, g = bg % Hkv;
    const size_t bh0 = (size_t)b * Hq + (size_t)g * G;
    h1_scores(ctx->h1_cnt[b], G, ctx->h1_z.data() + bh0 * cap1, (size_t)cap1, lse_global_host + bh0 * 2,
              inc + (size_t)bg * cap1);
  }
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  float* dinc = nullptr;
  e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&dinc), inc, 0);
  if (e == cudaSuccess) e = launch_t1_score_add(v, dinc, s);
  if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_inc[buf], s);
  if (e == cudaSuccess) ctx->inc_used[buf] = true;
  ctx->h1_layer = -1;
  return cuda_check(ctx, e, "host_t1_score_update");
}

// One whole host-T1 layer (the sequence of kv_tier.h's N1 block) in a single call: q down,
// GPU partial, host partial, combine, both score updates.  Two host waits per layer (q on the
// host; the combined (M, L) on the host).
kv_tier_status kv_tier_host_t1_layer(kv_tier_ctx* ctx, int32_t layer, const void* q, const void* k_new,
                                     const void* v_new, float* o, void* stream) {
  if (!ctx) return fail(nullptr, KV_TIER_E_INVAL, "null ctx");
  if (!ctx->v.host_t1 || !ctx->h1_q) return fail(ctx, KV_TIER_E_STATE, "host-T1 mode is off (kv_tier_set_host_t1)");
  if (!ctx->v.out_fp32) return fail(ctx, KV_TIER_E_STATE, "kv_tier_host_t1_layer needs out_fp32 = 1");
  if (!q || !o || ((uintptr_t)o & 15)) return fail(ctx, KV_TIER_E_INVAL, "q / o (16-B aligned fp32) required");
  const DevView& v = ctx->v;
  const size_t rows = (size_t)v.B * v.Hq, D = v.D;
  cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
  float* po = ctx->d1_parts;                 // [2][rows][D]
  float* pl = po + 2 * rows * D;             // [2][rows][2]
  float* lg = pl + 4 * rows;                 // [rows][2]
  float* ho = ctx->h1_o;                     // host o [rows][D], lse [rows][2], lse_global [rows][2]
  float* hl = ho + rows * D;
  float* hg = hl + 2 * rows;
  cudaError_t e = cudaMemcpyAsync(ctx->h1_q, q, rows * D * 2, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_q, s);
  if (e != cudaSuccess) return cuda_check(ctx, e, "host_t1_layer (q down)");
  kv_tier_status st = decode_attention_impl(ctx, layer, q, k_new, v_new, po, 1, stream, 0, pl);
  if (st) return st;
  e = cudaEventSynchronize(ctx->ev_q);
  if (e != cudaSuccess) return cuda_check(ctx, e, "host_t1_layer (q wait)");
  st = kv_tier_host_t1_attention(ctx, layer, ctx->h1_q, ho, hl);
  if (st) return st;
  e = cudaMemcpyAsync(po + rows * D, ho, rows * D * 4, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(pl + 2 * rows, hl, rows * 2 * 4, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = launch_lse_combine(po, pl, 2, (int)rows, (int)D, o, lg, s);
  if (e != cudaSuccess) return cuda_check(ctx, e, "host_t1_layer (combine)");
  st = kv_tier_score_update_lse(ctx, lg, stream);
  if (st) return st;
  e = cudaMemcpyAsync(hg, lg, rows * 2 * 4, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_q, s);
  if (e == cudaSuccess) e = cudaEventSynchronize(ctx->ev_q);
  if (e != cudaSuccess) return cuda_check(ctx, e, "host_t1_layer (lse up)");
  return kv_tier_host_t1_score_update(ctx, layer, hg, stream);
}

kv_tier_status kv_tier_import_scores(kv_tier_ctx* ctx, const float* host_S, size_t bytes) {
  if (!ctx || !host_S) return fail(ctx, KV_TIER_E_INVAL, "null arg");
  const size_t B = ctx->v.B, H = ctx->v.Hkv, N = ctx->v.Nmax, n = ctx->n;
  if (bytes != B * H * n * 4) return fail(ctx, KV_TIER_E_INVAL, "import_scores needs %zu bytes", B * H * n * 4);
  if (ctx->step_open) return fail(ctx, KV_TIER_E_STATE, "import inside a step");
  cudaError_t e = cudaDeviceSynchronize();
  for (size_t bg = 0; bg < B * H && e == cudaSuccess; ++bg)
    e = cudaMemcpy(ctx->v.S + bg * N, host_S + bg * n, n * 4, cudaMemcpyHostToDevice);
  return cuda_check(ctx, e, "import_scores");
}

}  // extern "C"
