/*
 * kv_tier.h -- C ABI of the B200 (sm_100a) tiered-KV decode hot path of
 * arXiv 2605.09490, "Semantics-aware four-tier KV memory hierarchy".
 *
 * Citations: P:n = PAPER.md line n (section / equation / algorithm named),
 * AMB-k = the reading of an ambiguous passage adopted in DESIGN.md.
 *
 * The per-decode-step path (Alg. 1):
 *   kv_tier_begin_step            new position n joins T0 (window)
 *   kv_tier_append      (layer)   its K/V row of layer l -> T0 store           (a1)
 *   kv_tier_prefetch    (layer)   T1 rows -> HBM staging (stream mode)         (a2)
 *   kv_tier_decode_attention (l)  GQA attention over T0+T1+T2 (Eq. 3, Prop. 1) (a3)
 *                                 + fused cumulative score update (Eq. 1)      (a4)
 *   kv_tier_end_step              t += 1
 *   kv_tier_classify              every Delta steps: tiers T0..T3              (a5)
 *   kv_tier_migrate               apply tier transitions to the stores         (a6)
 *
 * Conventions (all functions):
 *   - Return kv_tier_status: 0 = OK, < 0 = error.  No aborts, no exceptions.
 *     Argument errors are detected synchronously (E_INVAL / E_STATE / E_CAPACITY).
 *     Asynchronous CUDA errors and the device-side numeric flag (non-finite
 *     probability or score, AMB-2) surface at the next call that synchronises
 *     (kv_tier_sync / census / export) as E_CUDA / E_NUMERIC.
 *     kv_tier_last_error() returns a message for the last failure.
 *   - Every device call is asynchronous and stream-ordered on the stream passed
 *     (a cudaStream_t, passed as void*; NULL = legacy default stream).
 *   - Pointers marked "device" must be device-accessible, 16-byte aligned,
 *     contiguous, and are owned by the caller; the library never frees them.
 *   - bf16 = IEEE bfloat16 bit patterns (uint16).  Positions are 0-based (AMB-6).
 *   - One ctx per (process, device); a ctx is not thread-safe.
 */
#ifndef KV_TIER_H_
#define KV_TIER_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define KV_TIER_API __attribute__((visibility("default")))
#else
#define KV_TIER_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  KV_TIER_OK = 0,
  KV_TIER_E_INVAL = -1,     /* bad argument / shape mismatch, empty visible set */
  KV_TIER_E_CUDA = -2,      /* CUDA runtime error (possibly from an earlier async launch) */
  KV_TIER_E_NCCL = -3,      /* NCCL missing, communicator creation or a collective failed */
  KV_TIER_E_STATE = -4,     /* call out of order (e.g. migrate without classify) */
  KV_TIER_E_CAPACITY = -5,  /* a tier store would overflow its capacity */
  KV_TIER_E_OOM = -6,       /* host pinned allocation failed */
  KV_TIER_E_NUMERIC = -7    /* non-finite probability or score seen on device (AMB-2) */
} kv_tier_status;

/* Eviction budget semantics (AMB-9). TOTAL: |T3| = floor(r * |U_all|) over the run;
 * PER_EVENT: literal Alg. 1, n_evict = floor(r * |U|) at every event. */
typedef enum { KV_TIER_EVICT_TOTAL = 0, KV_TIER_EVICT_PER_EVENT = 1 } kv_tier_evict_mode;

/* Multi-GPU partitioning.  Without an nccl_unique_id the library runs no collective
 * and the caller (paper_2605_09490_b200/dist.py, torch.distributed over NCCL) moves the bytes;
 * with one (sequence sharding only) the library owns the communicator (see SEQUENCE below).
 *   REQUEST  each rank owns B requests; no collective anywhere on the path.
 *   KVHEAD   each rank owns H_kv / world kv heads (num_q_heads / num_kv_heads in the config
 *            are the rank's LOCAL counts; its global kv heads are rank*H_kv .. +H_kv-1).
 *            The step is local.  Tiers are per token across all heads (AMB-3, Alg. 1),
 *            so at an event every rank all-gathers S_part (kv_tier_scores_device) and calls
 *            kv_tier_classify_gathered: identical S -> identical tiers on every rank, summed
 *            in ascending global head order exactly as unsharded (bit-exact).
 *   SEQUENCE positions are owned block-cyclically: block k = positions [64k, 64k+64) belongs
 *            to rank k % world.  A rank's tier stores, index lists and
 *            census hold its own positions only; the tier array and S_part cover every
 *            position.  load_prefix takes the FULL prefix and keeps the rank's rows; the new
 *            token of a step is stored by its owner only.  Per layer the rank calls
 *            kv_tier_decode_attention_lse (o normalised by its own partial sum, plus its
 *            (max, sum) per head), the caller combines the ranks' partials (o = sum_r w_r o_r
 *            / sum_r w_r, w_r = 2^(m_r - M) l_r, M = max_r m_r: the LSE merge of Eq. 3 split
 *            by position) and hands the global (M, L) back through kv_tier_score_update_lse,
 *            which completes the fused score update with the exact global probabilities.
 *            At an event: all-gather S_part, kv_tier_classify_gathered (sum over ranks is
 *            exact: every position has one owner), migrate.  Without a communicator
 *            kv_tier_step / the step graph and kv_tier_score_update are E_STATE (the exchange
 *            sits between the layers).
 *            WITH a communicator (kv_tier_init given an nccl_unique_id from
 *            kv_tier_nccl_unique_id, one per job, every rank passing the same bytes): kv_tier_step
 *            and the step graph run the whole step on the library's NCCL communicator -- per
 *            layer decode_attention_lse (the rank's (o, m, l) written straight into its own slot
 *            of a packed receive buffer) -> ONE in-place ncclAllGather of the slots -> the LSE
 *            combine (rank order, deterministic) into o -> kv_tier_score_update_lse -- captured
 *            as one CUDA graph; kv_tier_classify all-gathers S_part itself.  out_fp32 must be 1. */
typedef enum { KV_TIER_SHARD_REQUEST = 0, KV_TIER_SHARD_KVHEAD = 1, KV_TIER_SHARD_SEQUENCE = 2 } kv_tier_shard;

/* Tier policy of a5 (the paper's pure-eviction baselines, §4.1, on
 * the same classify/migrate/decode path).  P = the protected set (prompt, sinks, window).
 *   HIERARCHY  the paper's four tiers (Alg. 1): beta / r / f2 as configured.
 *   STREAMING  StreamingLLM-style: every live non-protected token -> T3 (keep sinks + window).
 *   H2O        heavy hitters: keep P + the top max(0, budget - |P|) live tokens by cumulative
 *              score (ties: the newer token), the rest -> T3; no T1/T2.
 *   RANDOM     as H2O but ranked by a seeded hash of (policy_seed, request, position)
 *              (splitmix64, high 32 bits) instead of the score: uniform random removal.
 * budget (H2O/RANDOM) counts kept tokens per request, protected ones included. */
typedef enum { KV_TIER_POLICY_HIERARCHY = 0, KV_TIER_POLICY_STREAMING = 1, KV_TIER_POLICY_H2O = 2,
               KV_TIER_POLICY_RANDOM = 3 } kv_tier_policy;

/* Token scorer of a4 ("better scoring methods are plugins").
 *   ATTENTION  Eq. 1: S_i += sum_h p_{l,h,i}.
 *   VATP       value-aware attention: S_i += fp32(sum_h p_{l,h,i}) * ||v_{l,g,i}||_2, the
 *              fp32 L2 norm of the token's bf16 V row of layer l, kv head g, fixed when the row
 *              is loaded / appended.
 *   REDUNDANCY "attn - redundancy" (R-KV): S as ATTENTION; classify ranks by
 *              I_i - rho_i, I_i = fp32(S_i / S_max over the live set), rho_i the mean over layers
 *              and kv heads of c_i = cos(k_i, k_{i-1}) of the original key rows (DESIGN AMB-30/31).
 *              c is formed when a row is loaded / appended (the ctx keeps the previous key of
 *              every layer and kv head), so prefix layers must be loaded in ascending order.
 *   COMBINED   "attn x val - redundancy": S as VATP, ranked as REDUNDANCY.
 *   WINDOW     windowed attention (R-KV's "last alpha = 8 observation tokens"; App. E
 *              P:976): S as ATTENTION; classify ranks by W_i = fp32(sum_g S_part[g][i]) -
 *              fp32(sum_g S_snap[g][i]), max-pooled (kernel 7, stride 1) over the non-T3
 *              positions in ascending order.  S_snap is a copy of S_part the library takes at
 *              kv_tier_begin_step of step t when (t + w - 1) % Delta == 0, w = min(8, Delta)
 *              (cfg.manage_interval is then binding: call classify at steps t % Delta == 0 for
 *              the window to be the last w steps; DESIGN AMB-32).
 *   RKV        R-KV's Z = lambda I - (1 - lambda) R (App. E), lambda = 0.07:
 *              I_i = fp32(Wpool_i / max of Wpool over the live set) (0 if that max is 0),
 *              R_i = rho_i as REDUNDANCY; Z = fp32(0.07f * I) - fp32(0.93f * rho) (AMB-33).
 *   REDUNDANCY / COMBINED / RKV: every sequence shard appends every new key to its previous-key
 *   state and R_part covers all positions on every shard (identical copies), so sequence shards
 *   classify from their own R_part (also through kv_tier_classify_gathered); under KV-head
 *   sharding R_part is per shard and kv_tier_classify_gathered returns E_STATE.  WINDOW / RKV: no
 *   classify_gathered (E_STATE); on sequence shards only with the library's communicator
 *   (kv_tier_init E_INVAL without an nccl_unique_id): its kv_tier_classify all-gathers every
 *   shard's S_part and snapshot and pools over the global cache order of the tier array. */
typedef enum { KV_TIER_SCORER_ATTENTION = 0, KV_TIER_SCORER_VATP = 1, KV_TIER_SCORER_REDUNDANCY = 2,
               KV_TIER_SCORER_COMBINED = 3, KV_TIER_SCORER_WINDOW = 4, KV_TIER_SCORER_RKV = 5 } kv_tier_scorer;

#define KV_TIER_STAGING_ALL 0xFFFFFFFFu   /* differential mode: staging holds all of T1 (§3.4) */

typedef struct {
  int32_t  num_requests;     /* B  (this rank's requests)                            */
  int32_t  num_layers;       /* L                                                     */
  int32_t  num_q_heads;      /* H_q                                                   */
  int32_t  num_kv_heads;     /* H_kv; q head h reads kv head h / (H_q/H_kv) (AMB-4)   */
  int32_t  head_dim;         /* d in {64, 128}                                        */
  int32_t  max_tokens;       /* N_max per request: positions [0, N_max)               */
  int32_t  prompt_len;       /* P (protected)                                  */
  int32_t  sink_size;        /* k_s = 4                              */
  int32_t  window_size;      /* k_w = 128                             */
  int32_t  manage_interval;  /* Delta = 64; informative, the caller schedules */
  uint32_t hbm_ratio_bp;     /* beta in basis points (AMB-8)                   */
  uint32_t evict_ratio_bp;   /* r in basis points                              */
  uint32_t t2_fraction_bp;   /* f2: share of offloaded survivors placed in T2 (AMB-11) */
  int32_t  evict_mode;       /* kv_tier_evict_mode                                    */
  uint32_t staging_tokens;   /* KV_TIER_STAGING_ALL = differential (paper §3.4);
                                0 = stream mode: T1 rows re-fetched from pinned host
                                memory every step (strict DDR residency, AMB-13)      */
  int32_t  device;           /* CUDA device ordinal                                   */
  int32_t  rank, world, shard;
  int32_t  out_fp32;         /* 1: o is fp32 [B][H_q][d]; 0: bf16                      */
  int32_t  split;            /* CTAs per (request, kv head), <= 64; 0 = auto.  The
                                whole-step kernel (kv_tier_step) takes it as its cluster
                                size when <= 16 and the shape fits, else runs per layer */
  int32_t  variant;          /* decode kernel (consumer warps, stages): 0 (4,3) 1 (4,4)
                                2 (8,2) 3 (8,3) 4 (4,2) 5 (4,6)                        */
  int32_t  policy;           /* kv_tier_policy (0 = the paper's hierarchy)             */
  int32_t  budget;           /* kept tokens per request (H2O / RANDOM)                 */
  uint32_t policy_seed;      /* RANDOM                                                 */
  int32_t  scorer;           /* kv_tier_scorer (0 = Eq. 1 attention score)             */
  int32_t  step_kernel;      /* whole-step kernel consumer: 0 = auto (= 1, measured faster on
                                every shape tried), 1 = mma.sync (legacy tensor
                                path, 16-row slices per warp), 2 = tcgen05 / TMEM (d = 128,
                                no T2 rows, a cluster per kv head; else the step runs the
                                mma.sync consumer), 3 = none: kv_tier_step / the step graph
                                run the per-layer kernels (k_decode_attn + merge, chained
                                with PDL) as sequence shards always do                     */
} kv_tier_config;

typedef struct kv_tier_ctx kv_tier_ctx;

typedef struct {
  size_t device_arena;       /* bytes of device memory the caller must provide         */
  size_t t0_store, t1_staging, t2_store, scores, meta;   /* breakdown (informative)    */
  size_t host_t1, host_t2;   /* pinned host bytes the library allocates                */
  int32_t cap_t0, cap_t1, cap_t2;                        /* rows per (l, b, g)          */
} kv_tier_sizes;

typedef struct {
  void* device_arena;        /* device, >= sizes.device_arena bytes, 256-B aligned     */
} kv_tier_buffers;

/* Validate cfg and report the memory it needs.  Capacities (rows per layer, request and
 * kv head): T0 = N_max (the prefill prefix starts all-T0); T1 staging and the T2
 * store = the offloaded share ceil((1-beta) N_max) (+ f2 share for T2).  Stores are
 * double-buffered: migrate rebuilds the next buffer from the current one. */
KV_TIER_API kv_tier_status kv_tier_query_sizes(const kv_tier_config* cfg, kv_tier_sizes* out);

/* Create a ctx over caller-owned device memory; pins host T1/T2 stores
 * (cudaHostAlloc, mapped).  nccl_unique_id: NULL, or (sequence sharding only, out_fp32 = 1) the
 * 128 bytes of an ncclUniqueId every rank of the job passes: the ctx then owns an NCCL
 * communicator of cfg->world ranks (collective: every rank must call kv_tier_init) plus its
 * exchange buffers (cudaMalloc: 4 B x ((W + 1) B H_q (d + 2) + L B H_q 2 + W B H_kv N_max)),
 * freed by kv_tier_destroy.  E_NCCL if NCCL is unavailable or the communicator fails;
 * E_INVAL for an id with another shard mode. */
KV_TIER_API kv_tier_status kv_tier_init(const kv_tier_config* cfg, const kv_tier_buffers* buf,
                            const void* nccl_unique_id, kv_tier_ctx** out);

/* A fresh ncclUniqueId (rank 0 calls it and sends the bytes to the other ranks).  out: host,
 * >= 128 bytes.  NCCL is resolved at run time from the process (torch's libnccl.so.2) or the
 * loader path; E_NCCL if absent. */
KV_TIER_API kv_tier_status kv_tier_nccl_unique_id(void* out, size_t bytes);
KV_TIER_API kv_tier_status kv_tier_destroy(kv_tier_ctx* ctx);

/* Initial chain (prefill result, Alg. 1): positions [0, n0) of layer `layer`
 * all enter T0 with score 0.  k, v: device bf16 [B][H_kv][n0][d].  Must be called
 * for every layer with the same n0 before the first begin_step. */
KV_TIER_API kv_tier_status kv_tier_load_prefix(kv_tier_ctx* ctx, int32_t layer, const void* k, const void* v,
                                   int32_t n0, void* stream);

/* Start decode step t: position n (the new token, Alg. 1) joins T0 and the
 * window (protected).  E_CAPACITY if T0 or N_max would overflow. */
KV_TIER_API kv_tier_status kv_tier_begin_step(kv_tier_ctx* ctx, void* stream);

/* a1: write the new token's K/V of layer `layer`.  k_new, v_new: device bf16 [B][H_kv][d]. */
KV_TIER_API kv_tier_status kv_tier_append(kv_tier_ctx* ctx, int32_t layer, const void* k_new, const void* v_new,
                              void* stream);

/* a2 (stream mode only; no-op in differential mode): gather layer `layer`'s T1 rows
 * from pinned host memory into a 2-slot HBM staging ring on `side` (zero-copy
 * reads over the host link), layer-ahead.  decode_attention(layer) waits on it. */
KV_TIER_API kv_tier_status kv_tier_prefetch(kv_tier_ctx* ctx, int32_t layer, void* side);

/* a1 + a3 + a4: o[b][h] = sum_{i visible} softmax_i(q[b][h].k_i / sqrt d) v_i with
 * visible = T0 u T1 u T2 (T3 masked, Eq. 3; T2 rows dequantised, AMB-12), and,
 * if fuse_score_update, S_part[b][g][i] += sum_{h in g} p_{b,h,i} from the exact, globally
 * normalised probabilities (Eq. 1, AMB-1/14/15).
 * q: device bf16 [B][H_q][d]; o: device [B][H_q][d] fp32 (out_fp32) or bf16.
 * k_new, v_new: device bf16 [B][H_kv][d] rows of the new token for this layer, appended
 * to T0 inside the kernel (a1 fused); pass NULL for both if kv_tier_append already wrote
 * them this step.  E_STATE if neither happened. */
KV_TIER_API kv_tier_status kv_tier_decode_attention(kv_tier_ctx* ctx, int32_t layer, const void* q,
                                                    const void* k_new, const void* v_new, void* o,
                                                    int32_t fuse_score_update, void* stream);

/* a3 with the partial softmax statistics (sequence sharding; any mode): as
 * kv_tier_decode_attention, but o is normalised by this ctx's own partial sum and lse
 * (device fp32 [B][H_q][2]) receives (m, l) per head: m = max_i z_i in the log2 domain
 * (z = q.k / sqrt(d) * log2(e)) and l = sum_i 2^(z_i - m) over this ctx's visible tokens.
 * With fuse_score_update the score update of this launch waits for
 * kv_tier_score_update_lse (E_STATE if another decode/end_step comes first). */
KV_TIER_API kv_tier_status kv_tier_decode_attention_lse(kv_tier_ctx* ctx, int32_t layer, const void* q,
                                                        const void* k_new, const void* v_new, void* o, float* lse,
                                                        int32_t fuse_score_update, void* stream);

/* Rank combine of sequence-shard partials (the LSE merge of Eq. 3 split by position; no ctx):
 * o_parts device fp32 [world][rows][d] (each rank's o normalised by its own partial sum),
 * lse_parts [world][rows][2] (m in the log2 domain, l); writes o_out [rows][d] and
 * lse_out [rows][2] = (M, L) with M = max_r m_r, w_r = 2^(m_r - M) l_r (0 for m_r = -inf),
 * L = sum_r w_r and o = sum_r w_r o_r / L (0 if L = 0), summed in rank order (deterministic).
 * rows = B * H_q.  d % 4 == 0 and 16-B aligned pointers, else E_INVAL. */
KV_TIER_API kv_tier_status kv_tier_lse_combine(const float* o_parts, const float* lse_parts, int32_t world,
                                               int32_t rows, int32_t d, float* o_out, float* lse_out, void* stream);

/* Completes the pending fused score update of the last kv_tier_decode_attention_lse with the
 * GLOBAL per-head (M, L) (device fp32 [B][H_q][2], same encoding; the combination of every
 * rank's lse): S_part += sum_h 2^(z - M) / L over this ctx's tokens.  lse_global must stay
 * valid until the update has run on `stream`. */
KV_TIER_API kv_tier_status kv_tier_score_update_lse(kv_tier_ctx* ctx, const float* lse_global, void* stream);

/* ---- N1: host-side T1 partial attention (ScoutAttention-style prior art P:120,
 * P:215; strict DDR residency of T1).  With host-T1 mode on, kv_tier_decode_attention_lse
 * attends T0 ∪ T2 ∪ {new token} only (T1 skipped; no kv_tier_prefetch needed in stream mode)
 * and the host cores attend T1 in the pinned host store, so per layer only q goes down and
 * (o, m, l) plus the T1 score increments come up, instead of |T1| rows.  One layer:
 *   decode_attention_lse(o_gpu, lse_gpu) ; host_t1_attention(q_host -> o_host, lse_host) ;
 *   lse_combine([o_gpu, o_host], [lse_gpu, lse_host]) -> o, lse ;
 *   score_update_lse(lse) ; host_t1_score_update(lse copied to the host).
 * Attention scorer, request / KV-head sharding, split kernel with the merge kernel only;
 * kv_tier_decode_attention, kv_tier_step and graph capture return E_STATE in this mode. */
KV_TIER_API kv_tier_status kv_tier_set_host_t1(kv_tier_ctx* ctx, int32_t on);   /* outside a step */
/* Host T1 partial of `layer` in the open step.  q_host: bf16 [B][H_q][d] host memory (the step's
 * query); writes o_part fp32 [B][H_q][d] = sum_j 2^(z_j - m) v_j / l and lse_part fp32 [B][H_q][2]
 * = (m, l) over the request's T1 tokens j, z_j = fp32(q·k_j)·log2(e)/sqrt(d) (the decode kernel's
 * encoding; m = -inf, l = 0, o = 0 when |T1| = 0).  OpenMP over (b, h); the first call after a
 * migrate synchronises the device once to read the new T1 lists.  Keeps z for the score update. */
KV_TIER_API kv_tier_status kv_tier_host_t1_attention(kv_tier_ctx* ctx, int32_t layer, const void* q_host,
                                                     float* o_part, float* lse_part);
/* Eq. 1 for the T1 tokens of the layer last passed to kv_tier_host_t1_attention (E_STATE
 * otherwise): lse_global_host fp32 [B][H_q][2] host copy of the combined (M, L);
 * S_part[b][g][i] += fp32(sum_{h in g} 2^(z_hi - M_h) / L_h), formed on the host and scattered
 * by a kernel on `stream` from double-buffered mapped pinned memory (the call waits for the
 * scatter two layers back before reusing its buffer). */
KV_TIER_API kv_tier_status kv_tier_host_t1_score_update(kv_tier_ctx* ctx, int32_t layer, const float* lse_global_host,
                                                        void* stream);
/* The whole N1 sequence of one layer in one call (out_fp32 = 1): q device bf16 [B][H_q][d],
 * k_new / v_new as kv_tier_decode_attention, o device fp32 [B][H_q][d] = exact attention over
 * every visible token.  Uses ctx-owned pinned / device staging; blocks the calling thread twice
 * (q on the host, combined (M, L) on the host). */
KV_TIER_API kv_tier_status kv_tier_host_t1_layer(kv_tier_ctx* ctx, int32_t layer, const void* q, const void* k_new,
                                                 const void* v_new, float* o, void* stream);

/* a4 standalone (external probabilities, e.g. from another attention kernel):
 * probs: device fp32 [B][H_q][n_vis] over the visible tokens in ascending position
 * order; S_part[b][g][i] += fp32(sum_{h in g} probs[b][h][j(i)]).  n_vis is
 * returned by kv_tier_visible_count. */
KV_TIER_API kv_tier_status kv_tier_score_update(kv_tier_ctx* ctx, int32_t layer, const float* probs, void* stream);
KV_TIER_API kv_tier_status kv_tier_visible_count(const kv_tier_ctx* ctx, int32_t* n_vis);

/* Tier counts of the current step's layout, per request [|T0|, |T1|, |T2|, |T3|] over positions
 * [0, n) (the same for every request unless sequence-sharded: then this rank's request 0).  Host
 * mirror, no device synchronisation (unlike kv_tier_census).  Also reports the step kernel's
 * work split: shape[0] = CTAs of kv_tier_step's whole-step kernel (0: the step runs layer by
 * layer), shape[1] = CTAs per kv head (a thread-block cluster), shape[2] = kv heads per CTA,
 * shape[3] = the consumer design: 8 or 4 = mma.sync consumer warps per CTA, 5 = the tcgen05 /
 * TMEM consumer (4 softmax warps + the MMA-issuing warp).  Either pointer may be NULL. */
KV_TIER_API kv_tier_status kv_tier_layout(const kv_tier_ctx* ctx, int32_t* counts4, int32_t* shape4);

KV_TIER_API kv_tier_status kv_tier_end_step(kv_tier_ctx* ctx, void* stream);

/* One whole decode step: begin_step; for every layer l: [prefetch], append, decode_attention;
 * end_step.  q: device bf16 [L][B][H_q][d]; k_new, v_new: device bf16 [L][B][H_kv][d];
 * o: device [L][B][H_q][d] (fp32 or bf16 per out_fp32).  `side` carries stream-mode prefetch. */
KV_TIER_API kv_tier_status kv_tier_step(kv_tier_ctx* ctx, const void* q, const void* k_new, const void* v_new,
                                        void* o, int32_t fuse_score_update, void* stream, void* side);
/* Capture kv_tier_step over fixed buffers as a CUDA graph (stream must not be the legacy
 * default stream); kv_tier_step_graph_launch replays it as one decode step.  Kernels read
 * the step/tier counters from device memory, so one graph serves every step; the caller
 * refills q / k_new / v_new before each launch and runs classify/migrate outside it. */
KV_TIER_API kv_tier_status kv_tier_step_graph_capture(kv_tier_ctx* ctx, const void* q, const void* k_new,
                                                      const void* v_new, void* o, int32_t fuse_score_update,
                                                      void* stream, void* side);
KV_TIER_API kv_tier_status kv_tier_step_graph_launch(kv_tier_ctx* ctx, void* stream);

/* A whole decoder step in the CALLER's CUDA graph: kv_tier_capture_begin before
 * the caller begins its stream capture, the step's calls (begin_step, prefetch,
 * decode_attention per layer, end_step; no classify / migrate) on the capturing stream, and
 * kv_tier_capture_end after the capture ends: the host state machine runs once during the
 * capture and is restored.  After each replay of that graph, kv_tier_graph_advance moves the
 * host mirror on by one step (the kernels read the step and tier counters from device memory,
 * so one graph serves every step, events included).  E_STATE out of order; E_CAPACITY as
 * begin_step. */
KV_TIER_API kv_tier_status kv_tier_capture_begin(kv_tier_ctx* ctx);
KV_TIER_API kv_tier_status kv_tier_capture_end(kv_tier_ctx* ctx);
KV_TIER_API kv_tier_status kv_tier_graph_advance(kv_tier_ctx* ctx);

/* a5: per request, protected set P = [0,P) u [P,P+k_s) u [n-k_w,n); the live
 * non-protected tokens ordered by the unique key (fp32 bits of S_i, i) ascending
 * (AMB-7); n_new = bottom -> T3 (AMB-8/9), top floor(beta|surv|) -> T0, lowest
 * floor(f2 * rest) -> T2, remainder -> T1 (Alg. 1).  Idempotent until migrate.
 * The ranking key is the scorer's (kv_tier_scorer; WINDOW / RKV: the max-pooled windowed
 * score, AMB-32/33).  Waits (on `stream`) for the previous event's host offload.
 * E_STATE under KV-head or sequence sharding with world > 1 (use kv_tier_classify_gathered),
 * except a sequence-shard ctx that owns a communicator: it all-gathers S_part itself (NCCL on
 * `stream`) and classifies the sum (one owner per position: exact). */
KV_TIER_API kv_tier_status kv_tier_classify(kv_tier_ctx* ctx, void* stream);

/* a6: apply the transitions of the last classify: T0<->T1 copies, ->T2 int8
 * quantisation (AMB-12), T2-> bf16 of the dequantised row, ->T3 dropped.
 * Rows entering T1/T2 reach the pinned host store inside the migrate kernel (stream mode) or,
 * with differential staging, from their new HBM rows on the ctx's own offload stream beside the
 * following steps (the next classify waits for it; host-side readers synchronise).  One
 * cooperative launch moves every row (grid barriers; a 2 s watchdog reports E_CUDA at the next
 * sync instead of hanging).  `side` is unused.  E_STATE without a preceding classify. */
KV_TIER_API kv_tier_status kv_tier_migrate(kv_tier_ctx* ctx, void* main_stream, void* side);

/* Synchronise the device and report async errors (E_CUDA, E_NUMERIC). */
KV_TIER_API kv_tier_status kv_tier_sync(kv_tier_ctx* ctx);

/* counts: host int32 [B][4] = |T0|,|T1|,|T2|,|T3| over positions [0, n) (App. D);
 * d2h_rows: host int64, rows written to the host stores so far (may be NULL). Synchronises. */
KV_TIER_API kv_tier_status kv_tier_census(kv_tier_ctx* ctx, int32_t* counts, int64_t* d2h_rows);

/* Host-side state (no sync): current sequence length n and step t. */
KV_TIER_API kv_tier_status kv_tier_position(const kv_tier_ctx* ctx, int32_t* n, int32_t* t);

/* ---- test hooks: canonical, layout-independent exports (synchronise) -------- */
enum {
  KV_TIER_X_SCORES = 0,     /* fp32 [B][H_kv][n]   S_part (AMB-1)                        */
  KV_TIER_X_TIERS = 1,      /* u8   [B][n]                                                */
  KV_TIER_X_IDX_T0 = 2,     /* i32  [B][|T0|] positions, ascending (stores keep any order) */
  KV_TIER_X_IDX_T1 = 3,     /* i32  [B][|T1|]                                              */
  KV_TIER_X_IDX_T2 = 4,     /* i32  [B][|T2|]                                              */
  KV_TIER_X_T0_ROWS = 5,    /* bf16 [B][H_kv][|T0|][2][d]  (K,V) in ascending position     */
  KV_TIER_X_T1_ROWS = 6,    /* bf16 [B][H_kv][|T1|][2][d]  from the pinned host store      */
  KV_TIER_X_STAGING = 7,    /* bf16 [B][H_kv][|T1|][2][d]  HBM staging (differential mode) */
  KV_TIER_X_T2_CODES = 8,   /* i8   [B][H_kv][|T2|][2][d]                                  */
  KV_TIER_X_T2_SCALES = 9,  /* f32  [B][H_kv][|T2|][2]                                     */
  KV_TIER_X_REDUNDANCY = 10,/* fp32 [B][H_kv][n]   R_part (AMB-30; zeros unless REDUNDANCY/COMBINED/RKV) */
  KV_TIER_X_SNAPSHOT = 11   /* fp32 [B][H_kv][n]   S_snap (AMB-32; zeros unless WINDOW/RKV)   */
};
/* Bytes `what` needs (counts are uniform across requests). */
KV_TIER_API kv_tier_status kv_tier_export_size(kv_tier_ctx* ctx, int32_t what, size_t* bytes);
KV_TIER_API kv_tier_status kv_tier_export(kv_tier_ctx* ctx, int32_t what, int32_t layer, void* host_dst, size_t bytes);
/* Overwrite S_part with host fp32 [B][H_kv][n] (classify cross-feed, AMB-18). Synchronises. */
KV_TIER_API kv_tier_status kv_tier_import_scores(kv_tier_ctx* ctx, const float* host_S, size_t bytes);

/* Device pointer and size of this ctx's per-kv-head partial scores S_part [B][H_kv][N_max]
 * fp32 (owned by the ctx; valid until kv_tier_destroy).  For the caller's collectives. */
KV_TIER_API kv_tier_status kv_tier_scores_device(kv_tier_ctx* ctx, void** ptr, size_t* bytes);

/* a5 from gathered scores (KV-head sharding): S_all is device memory
 * [parts][B][H_kv][N_max] fp32 -- the all-gather over ranks of every rank's S_part, rank
 * order = global kv head order.  S_i = fp32 sum over the parts*H_kv heads in ascending
 * global order (AMB-1/14), then the same selection as kv_tier_classify.  S_all must stay
 * valid until the classify has run on `stream`.  E_INVAL on a null/misaligned pointer. */
KV_TIER_API kv_tier_status kv_tier_classify_gathered(kv_tier_ctx* ctx, const float* S_all, int32_t parts,
                                                     void* stream);

/* Debug: %globaltimer checkpoints [L][CTAs][16] of the last launch of every layer; n must be
 * kv_tier_debug_trace_len().  Split kernel (CTAs = B*H_kv*split): (start, after PDL wait, first
 * stage, loop done, partial written, merge released, merge resident, merge end, consumer wait
 * ns, consumer busy ns, stages, producer empty-wait ns, producer done, -, -, -).  Flat kernel
 * (CTAs = grid): (start, after PDL wait, first stage, loop done, side warp new tokens done,
 * side warp score pass done, last partial released, last unit finished, merges done, ns in
 * unit epilogues, units finished, -, ...).  Only with KVTIER_TRACE=1 at kv_tier_init. */
KV_TIER_API kv_tier_status kv_tier_debug_trace(kv_tier_ctx* ctx, uint64_t* host_dst, size_t n);
KV_TIER_API kv_tier_status kv_tier_debug_trace_len(const kv_tier_ctx* ctx, size_t* n);

KV_TIER_API const char* kv_tier_last_error(const kv_tier_ctx* ctx);
KV_TIER_API const char* kv_tier_version(void);

#ifdef __cplusplus
}
#endif
#endif /* KV_TIER_H_ */
