// a1 + a3 + a4 for EVERY layer of one decode step in one launch (kv_tier_step and the step
// graph, differential staging): PAPER.md Eq. 1, Eq. 3, Alg. 1 forward loop
// P:175-188, Prop. 1 P:416-427.
//
// Why one launch.  A layer of the 7B config moves 32 MB: 4.9 us at the measured HBM peak.  The
// per-layer kernels (decode -> merge -> next decode, attn.cu) spend ~6 us per layer in dependent
// global round trips while HBM idles.  Here a thread-block CLUSTER owns one
// request for the whole step:
//   * its K CTAs (one per SM) split the request's kv heads: s CTAs per kv head (a slice of the
//     head's rows each) or m heads per CTA;
//   * each CTA's producer warp streams K/V tiles of layer l, l+1, ... into a deep shared-memory
//     ring without waiting for the layer chain (K/V rows of layer l+1 do not depend on layer l),
//     with an L2 prefetch NST stages ahead;
//   * the partials of a kv head's s slices are exchanged through distributed shared memory: a
//     bulk copy into each peer's receive buffer completes the peer's mbarrier (no global round
//     trip); every slice merges its share of o and the head's global (M, 1/L);
//   * the dependency a decoder imposes -- q and the new token's K/V of layer l+1 are projections
//     of o(l) of the same request -- is a cluster mbarrier: q(l+1) is read only after every CTA
//     of the request has finished its part of o(l) and arrived on every peer.
// Clusters never wait on each other, so no co-residency beyond the cluster is assumed.
//
// Roles per CTA (NW consumer warps + 4):
//   producer warp  stages of up to NW 16-row groups (never straddling a head or the bf16/int8
//                  boundary) -> NST-deep ring, 1-D bulk async copies (UBLKCP) into the pre-swizzled
//                  layout ldmatrix reads.
//   consumers      S^T = K q^T and o^T += V^T p^T on the tensor cores (mma.sync m16n8k16, swap-AB:
//                  tokens = M, the G <= 8 heads = N), online softmax in fp32 (log2 domain), p split
//                  hi + lo bf16 for the P.V product; logits -> an L2-resident ring for a4; warps ->
//                  CTA partial -> DSMEM exchange -> merge -> o, (M, 1/L).
//   new-token warp the step's new token of each head (a1: its K/V row joins T0; its attention term
//                  on the CUDA cores, added by the merge).
//   score warps    a4 of layer l-1 while the consumers run layer l: S_part[b][g][pos] +=
//                  sum_{h in g} 2^(z - M_h) / L_h over this CTA's rows (one writer per entry,
//                  layer order, AMB-14).
#include "decode_common.cuh"

#ifndef KVT_TRACE
#define KVT_TRACE 0   // debug builds (-DKVT_TRACE=1): per-(layer, CTA) timeline in the ctx trace buffer
#endif

namespace kvt {

// ----------------------------------------------------------------- cluster / async-proxy PTX
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {   // local smem addr -> peer's
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// local shared -> peer shared bulk copy, completing `bytes` on the peer's mbarrier
__device__ __forceinline__ void bulk_s2peer(uint32_t dst_cl, uint32_t src, uint32_t bytes, uint32_t mbar_cl) {
  asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(dst_cl), "r"(src), "r"(bytes), "r"(mbar_cl) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ int ld_relaxed_gpu(const int* p) {
  int x;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];\n" : "=r"(x) : "l"(p) : "memory");
  return x;
}
__device__ __forceinline__ void red_relaxed_gpu(int* p, int x) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;\n" ::"l"(p), "r"(x) : "memory");
}
// CTA-local mbarrier wait that suspends until the phase completes (no issue slots while waiting)
#ifndef KVT_SPIN_CHAIN
// the layer chain's barriers and counter are polled without suspending: the hand-offs sit on the
// step's critical path (7B, same box: 254.4 vs 257.7 us/step with a 1 us suspend hint and a 64 ns
// sleep per counter poll; profiles/r02/spin_ab_r02.md).  -DKVT_SPIN_CHAIN=0 builds the suspending
// variant for A/B runs.
#define KVT_SPIN_CHAIN 1
#endif
__device__ __forceinline__ void mbar_sleep_wait(uint32_t a, uint32_t parity) {
  if (KVT_SPIN_CHAIN) mbar_wait(a, parity);
  else mbar_wait_hint(a, parity, 1000000u);
}

// ----------------------------------------------------------------- work split
// Geometry (host side, step_plan in ctx.cu): R = H_kv * s / m CTAs per request; s > 1: a
// cluster of s CTAs per kv head, slice = cluster rank; s == 1: heads [rank*m, rank*m + m) whole.
struct StepPart {
  int g, j0, j1, fnew;       // kv head, head-relative 16-row groups [j0, j1), this CTA appends the new token
};

// first group of a head whose cost range starts at or after cost x (bf16 group = 2, int8 = 1)
__device__ __forceinline__ int group_at_cost(int x, int gbf) {
  return x <= 2 * gbf ? (x + 1) >> 1 : gbf + (x - 2 * gbf);
}

struct StepIO {
  const __nv_bfloat16* q;      // [L][B][Hq][D]
  const __nv_bfloat16* knew;   // [L][B][Hkv][D]
  const __nv_bfloat16* vnew;
  void* o;                     // [L][B][Hq][D] fp32 or bf16
  int score;                   // a4 on (fuse_score_update)
};

// stage descriptor flags
constexpr int SD_FIRST = 1, SD_LAST = 2, SD_T2 = 4;
constexpr int STEP_MAXM = 8;   // kv heads per CTA when s == 1

// UM = false: consumers on the legacy tensor path (mma.sync, NW warps of 16 rows per stage).
// UM = true (d = 128, no T2 rows): the 5th-generation tensor cores -- one issuing thread runs
// S = K q^T and O = V^T P^T per 128-row stage with tcgen05.mma from the swizzled shared-memory
// tiles into TMEM; NW = 4 softmax warps (one token row, then one d row of O, per thread) keep
// the online softmax and the o accumulator.
template <int D, int NW, int NST, bool UM>
__global__ void __launch_bounds__((NW + 4 + (UM ? 1 : 0)) * 32, (NW <= 4 && !UM) ? 2 : 1)
    k_decode_step(const DevView v, const StepIO io) {
  static_assert(!UM || (D == 128 && NW == 4), "the UMMA consumer is written for d = 128, 4 softmax warps");
  constexpr int NCONS = NW * 32;
  constexpr int WPROD = NW, WNEW = NW + 1, WSC0 = NW + 2;   // + two score warps
  constexpr int WISS = NW + 4;                               // UM: the MMA-issuing warp
  constexpr int NSC = 64;                                    // score-pass threads
  constexpr int GPS = UM ? 8 : NW;                           // 16-row groups per stage
  constexpr int TILE = GPS * 16;
  constexpr int ROWB = D * 2;
  constexpr int TILEB = TILE * ROWB;
  constexpr int STAGEB = 2 * TILEB;
  constexpr int KS = D / 16;
  constexpr int OWS = D + 4;
  constexpr int NH = NW / 2;
  const int S = v.step_s, Mh = v.step_m;
  const int R = v.Hkv * S / Mh;                  // CTAs per request
  const int b = blockIdx.x / R;                  // this CTA's request
  const int rk = blockIdx.x - b * R;             // rank within the request
  int* const done_ctr = v.step_done;             // [L][B] CTAs of the request that finished layer l
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int G = v.G, L = v.L, B = v.B, Hkv = v.Hkv;
  const int U = B * Hkv;
  const int ZS = v.zring;
  const int tot = G * D;                          // o floats per kv head
  const int SL = ((tot + S - 1) / S + 3) & ~3;    // o floats per slice (s > 1)
  auto trace = [&](int l, int slot) {             // debug timeline: %globaltimer
    if (KVT_TRACE && v.trace) v.trace[((size_t)l * gridDim.x + blockIdx.x) * NTRACE + slot] = gtimer();
  };
  auto ctrace = [&](int l, int slot) {            // debug: SM clock (intra-CTA intervals)
    if (KVT_TRACE && v.trace) v.trace[((size_t)l * gridDim.x + blockIdx.x) * NTRACE + slot] = clock64();
  };

  extern __shared__ __align__(1024) unsigned char smem[];
  // UM: the swizzle atoms need 1024-byte aligned tiles
  unsigned char* ring = UM ? smem + ((1024u - (smem_u32(smem) & 1023u)) & 1023u) : smem;   // [NST][K tile | V tile]
  unsigned char* qtile = ring + NST * STAGEB;                              // UM: [16][D] q(l) of the head, swizzled
  unsigned char* ptile = qtile + (UM ? 16 * ROWB : 0);                     // UM: [2][16][TILE] p hi (rows 0-7), lo (8-15)
  unsigned char* t2w = ptile + (UM ? 2 * 16 * ROWB : 0);                   // [NW][16][D] bf16 (T2 only)
  float* ow = reinterpret_cast<float*>(t2w + (v.cap2 > 0 ? NW * 16 * ROWB : 0));   // [NH][8][OWS] combine
  float* pbuf = ow + (UM ? 0 : NH * 8 * OWS);                              // [16 + 8 D] CTA partial (m, l, o)
  float* rx = pbuf + 16 + 8 * D + 64;                                      // [2][S][16 + SL] received partials
  float* redm = rx + 2 * S * (16 + SL);                                    // [NW][8]
  float* redl = redm + NW * 8;                                             // [NW][8]
  float* ntz = redl + NW * 8;                                              // [2][8] new-token logits
  float* ntv = ntz + 16;                                                   // [2][D] new-token V row
  float* sml = ntv + 2 * D;                                                // [ZRING][STEP_MAXM][16] (M, 1/L) for a4
  float* smisc = sml + ZRING * STEP_MAXM * 16;                             // [24] merge scalars
  float* fac = smisc + 24;                                                 // [16][8] merge factors (S <= 16)
  float* wmx = fac + 16 * 8;                                               // UM: [2][NW][8] per-warp stage maxima
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(wmx + (UM ? 2 * NW * 8 : 0));
  // full[NST] empty[NST] | nfull[2] nempty[2] rxb[2] q spare | UM: sready[2] pready oready qready
  int4* sdesc = reinterpret_cast<int4*>(bars + 2 * NST + 16);              // [NST]
  StepPart* ptab = reinterpret_cast<StepPart*>(sdesc + NST);               // [STEP_MAXM] this CTA's parts
  volatile int* sc_done = reinterpret_cast<volatile int*>(ptab + STEP_MAXM);   // layers whose a4 pass is complete
  volatile int* ml_done = sc_done + 1;                                     // layers merged ((M, 1/L) in sml)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(const_cast<int*>(sc_done) + 2);   // UM: TMEM base
  volatile int* pvfresh = sc_done + 3;                                     // UM: [2] P.V of stage i starts O afresh

  const int cur = v.st->cur, sb = v.st->scur;
  Seg sg;
  sg.init(v.cnt[cur], 1, 0);                 // counts are uniform across requests
  const int gbf = sg.a2 >> 4, gq2 = (sg.n2 + 15) >> 4, ng = gbf + gq2, cu = 2 * gbf + gq2;
  const int npart = S > 1 ? 1 : Mh;
  const int slice = S > 1 ? (int)cluster_rank() : 0;   // the cluster is one kv head's S slices
  auto part_calc = [&](int k) -> StepPart {
    StepPart p;
    if (S > 1) {
      p.g = rk / S;
      p.j0 = group_at_cost(slice * cu / S, gbf);
      p.j1 = group_at_cost((slice + 1) * cu / S, gbf);
      p.fnew = slice == S - 1;
    } else {
      p.g = rk * Mh + k;
      p.j0 = 0;
      p.j1 = ng;
      p.fnew = 1;
    }
    return p;
  };
  if (tid < npart) ptab[tid] = part_calc(tid);              // constant for the step: no per-stage division
  auto part = [&](int k) -> StepPart { return ptab[k]; };

  const uint32_t ring_s = smem_u32(ring);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + NST);
  const uint32_t nfull0 = smem_u32(bars + 2 * NST), nempty0 = smem_u32(bars + 2 * NST + 2);
  const uint32_t rxb0 = smem_u32(bars + 2 * NST + 4);
  // S > 1: q(l) of the head reaches shared memory in ONE bulk copy issued by the new-token warp
  // once the layer dependency holds; its completion (phase l & 1) is also the consumers' signal
  // that q(l) may be used.  The copy lands in the receive half rx[(l + 1) & 1], which is idle
  // during layer l: its last reader was merge(l - 1) (done before the dependency of layer l can
  // hold) and its next writers are the peers' pushes of layer l + 1 (after they read q(l + 1),
  // i.e. after every CTA finished o(l)).
  const uint32_t qbar = smem_u32(bars + 2 * NST + 6);
  auto qsm = [&](int l) { return rx + ((l + 1) & 1) * S * (16 + SL); };
  // q(l) and the new token's K/V of layer l are projections of o(l-1) of the same request: wait
  // until every CTA of the request has finished its part of o(l-1) (relaxed polling: the counter
  // orders the computation; no data produced by another CTA is read after it)
  auto wait_layer = [&](int l) {
    const int* p = done_ctr + (size_t)(l - 1) * B + b;
    if (ld_relaxed_gpu(p) < R) {
      const unsigned long long t0 = gtimer();
      for (unsigned it = 1; ld_relaxed_gpu(p) < R; ++it) {
        if (!KVT_SPIN_CHAIN) __nanosleep(64);
        if ((it & 255u) == 0 && gtimer() - t0 > 2000000000ull) {   // watchdog: report, never hang the device
          atomicOr(&v.st->err, 4);
          break;
        }
      }
    }
  };
  // UM barriers: S(i) in TMEM (commit, by stage parity), P(i) in shared memory (one arrive per
  // softmax warp), P.V of stage i done (commit, by stage parity), the q tile of a layer (one
  // arrive per softmax warp)
  const uint32_t sready0 = smem_u32(bars + 2 * NST + 8), pready = smem_u32(bars + 2 * NST + 10);
  const uint32_t odone0 = smem_u32(bars + 2 * NST + 11), qready = smem_u32(bars + 2 * NST + 13);
  if (tid == 0) {
    for (int x = 0; x < NST; ++x) {
      mbar_init(full0 + 8 * x, 1);
      mbar_init(empty0 + 8 * x, UM ? 1 : NW);   // UM: the commit of the stage's P.V frees the slot
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(nfull0 + 8 * x, 1);
      mbar_init(nempty0 + 8 * x, 1);
      mbar_init(rxb0 + 8 * x, 1);               // the owner's arrive.expect_tx; peers complete tx
    }
    mbar_init(qbar, 1);
    if (UM) {
      mbar_init(sready0, 1);
      mbar_init(sready0 + 8, 1);
      mbar_init(pready, NW);
      mbar_init(odone0, 1);
      mbar_init(odone0 + 8, 1);
      mbar_init(qready, NW);
    }
    *sc_done = 0;
    *ml_done = 0;
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if constexpr (UM) {
    // stale shared memory must read as finite numbers: rows past a stage's last group enter the
    // MMAs (multiplied by p = 0 or masked), so the ring and the tiles start zeroed
    for (int i = tid; i < (NST * STAGEB + 48 * ROWB) / 16; i += blockDim.x)
      reinterpret_cast<uint4*>(ring)[i] = make_uint4(0u, 0u, 0u, 0u);
    fence_proxy_async_cta();
    if (w == WISS) {                              // TMEM: S double buffer (2 x 16 columns) + O (16)
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;\n" ::"r"(smem_u32(tmem_slot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    tc_fence_before();
  }
  __syncthreads();                              // part table, barriers, counters
  if constexpr (UM) tc_fence_after();
  const uint32_t tmem = UM ? *tmem_slot : 0u;
  if (S > 1) cluster_sync_all();                // every peer's barriers exist before any remote use
  if (KVT_TRACE && v.trace && blockIdx.x == 0 && tid == 0) v.trace[NTRACE - 1] = gridDim.x;

  // ---------------- consumer-side tail of a part, shared by both consumer designs: the CTA
  // partial (m, l, o) is in pbuf; exchange it over DSMEM, merge this CTA's share of o (+ the new
  // token), store o, publish (M, 1/L) for the score warps and count o(l) for the request.
  int nts = 0, nrx = 0;
  auto store_o = [&](int l, int g, int e, float4 val) {    // o elements [e, e+4) of kv head g
    const size_t oi = (((size_t)l * B + b) * v.Hq + g * G) * D + e;
    if (v.out_fp32) {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(io.o) + oi) = val;
    } else {
      __nv_bfloat162 lo = __floats2bfloat162_rn(val.x, val.y), hi = __floats2bfloat162_rn(val.z, val.w);
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&lo);
      pk.y = *reinterpret_cast<uint32_t*>(&hi);
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(io.o) + oi) = pk;
    }
  };
  auto merge_part = [&](int l, int kpart, int g) {
    const int par = l & 1;
    if (tid == 0 && kpart == 0) ctrace(l, 16);             // CTA partial in pbuf
    if (S > 1) {
      // ---------------- DSMEM exchange: (m, l) + o slice r of this partial -> slice r's CTA.
      // Every push carries 16 + SL floats (the last slice is padded from pbuf's tail), so each
      // receiver expects exactly S * (16 + SL) * 4 bytes per layer.
      fence_proxy_async_smem();                              // pbuf (generic stores) -> bulk copy reads
      named_sync(1, NCONS);
      if (tid == 0) {
        const uint32_t rx_s = smem_u32(rx);
        mbar_expect_tx(rxb0 + 8 * par, (uint32_t)(S * (16 + SL) * 4));
        for (int r = 0; r < S; ++r) {                       // cluster ranks = the head's slices
          const uint32_t peer = (uint32_t)r;
          const uint32_t dst = rx_s + (uint32_t)(((par * S + slice) * (16 + SL)) * 4);
          const uint32_t mb = mapa(rxb0 + 8 * par, peer);
          bulk_s2peer(mapa(dst, peer), smem_u32(pbuf), 64, mb);
          bulk_s2peer(mapa(dst + 64, peer), smem_u32(pbuf + 16 + r * SL), (uint32_t)(SL * 4), mb);
        }
        bulk_commit();
      }
    }
    // ---------------- merge: this CTA's share of o (slice, or the whole head) + the new token
    const int nslot = nts & 1;
    mbar_sleep_wait(nfull0 + 8 * nslot, (nts >> 1) & 1);   // the new token's term (every CTA of the head)
    if (tid == 0 && kpart == 0) ctrace(l, 17);             // new token ready
    if (S > 1) mbar_sleep_wait(rxb0 + 8 * par, (nrx >> 1) & 1);
    named_sync(1, NCONS);                                   // pbuf complete (S == 1)
    if (tid == 0 && kpart == 0) ctrace(l, 18);             // peers' partials landed
    const int nsrc = S > 1 ? S : 1;
    const float* src0 = S > 1 ? rx + par * S * (16 + SL) : pbuf;   // partial 0 of the merge
    const int sstride = 16 + SL;                            // between received partials
    const int e_beg = S > 1 ? slice * SL : 0;
    const int e_end = S > 1 ? min(tot, e_beg + SL) : tot;
    float* sIL = smisc;                                     // [8] 1/L
    float* sFN = smisc + 8;                                 // [8] new-token factor
    if (w == 0) {
      // warp 0: lane = (source group j = lane >> 3, head h = lane & 7); sources j, j+4, ... ;
      // max and sum over the source groups by shuffles (fixed order: deterministic)
      const int h = lane & 7, j = lane >> 3;
      const float zn = ntz[nslot * 8 + h];
      float M = zn;
      for (int x = j; x < nsrc; x += 4) M = fmaxf(M, src0[x * sstride + h]);
      M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, 8));
      M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, 16));
      float Ls = 0.f;
      for (int x = j; x < nsrc; x += 4) {
        const float m = src0[x * sstride + h];
        const float f = m == -INFINITY ? 0.f : ex2_ftz(m - M);
        fac[x * 8 + h] = f;
        Ls += f * src0[x * sstride + 8 + h];
      }
      Ls += __shfl_xor_sync(0xffffffffu, Ls, 8);
      Ls += __shfl_xor_sync(0xffffffffu, Ls, 16);
      if (j == 0) {
        const float fn = zn == -INFINITY ? 0.f : ex2_ftz(zn - M);
        Ls += fn;
        const float il = Ls > 0.f ? 1.0f / Ls : 0.f;
        sIL[h] = il;
        sFN[h] = fn;
        float* mlw = sml + ((l % ZS) * STEP_MAXM + kpart) * 16;
        mlw[h] = h < G ? M : 0.f;
        mlw[8 + h] = h < G ? il : 0.f;
      }
    }
    named_sync(1, NCONS);
    for (int e = e_beg + 4 * tid; e < e_end; e += 4 * NCONS) {
      const int h = e / D, dd = e - h * D;
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int x = 0; x < nsrc; ++x) {
        const float f = fac[x * 8 + h];
        const float4 y = *reinterpret_cast<const float4*>(src0 + x * sstride + 16 + (e - e_beg));
        acc.x += f * y.x;
        acc.y += f * y.y;
        acc.z += f * y.z;
        acc.w += f * y.w;
      }
      const float fn = sFN[h], il = sIL[h];
      const float4 nv = *reinterpret_cast<const float4*>(ntv + nslot * D + dd);
      acc.x = (acc.x + fn * nv.x) * il;
      acc.y = (acc.y + fn * nv.y) * il;
      acc.z = (acc.z + fn * nv.z) * il;
      acc.w = (acc.w + fn * nv.w) * il;
      store_o(l, g, e, acc);
    }
    named_sync(1, NCONS);                                   // o stored, rx / ntv / fac read
    if (tid == 0 && kpart == 0) ctrace(l, 19);
    if (tid == 0) {
      mbar_arrive(nempty0 + 8 * nslot);
      if (kpart == npart - 1) {
        __threadfence_block();
        *ml_done = l + 1;                                   // every part's (M, 1/L) of layer l is in sml
        // o(l) of this CTA is final: count it for the request (the q(l+1) dependency).  The
        // relaxed add orders the COMPUTATION (a fused decoder would hand o(l) to its o_proj
        // stage on chip); it deliberately does not wait for the global o stores to drain behind
        // the K/V stream -- they are visible at kernel end.
        red_relaxed_gpu(done_ctr + (size_t)l * B + b, 1);
        ctrace(l, 20);
      }
    }
    ++nts;
    if (S > 1) ++nrx;
  };

  if (w == WPROD) {
    // ================================ producer ================================
    // Stage sequence: layer-major, then this CTA's parts, then up to GPS groups per stage.  A second
    // cursor NST stages ahead prefetches into L2, so the copy that refills a ring slot hits L2.
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      struct Cur { int l, k, j; };
      auto stage_of = [&](const Cur& it, const StepPart& pp, bool& t2) {
        if (pp.j0 == pp.j1) { t2 = false; return 0; }
        t2 = it.j >= gbf;
        const int send = t2 ? pp.j1 : min(pp.j1, gbf);
        return min(GPS, send - it.j);
      };
      auto advance = [&](Cur& it) {
        const StepPart pp = part(it.k);
        bool t2;
        const int cnt = stage_of(it, pp, t2);
        it.j += cnt;
        if (cnt == 0 || it.j >= pp.j1) {
          if (++it.k == npart) { it.k = 0; ++it.l; }
          it.j = part(it.k).j0;
        }
      };
      auto issue = [&](const Cur& it, const StepPart& pp, int cnt, bool t2, uint32_t dst, uint32_t full) {
        const size_t grp = grp_of(v, it.l, b, pp.g);
        if (!t2) {
          const __nv_bfloat16* K0 = v.k0[sb] + grp * v.cap0 * D;
          const __nv_bfloat16* V0 = v.v0[sb] + grp * v.cap0 * D;
          const __nv_bfloat16* K1 = v.k1[sb] + grp * v.cap1 * D;
          const __nv_bfloat16* V1 = v.v1[sb] + grp * v.cap1 * D;
          const int ts = 16 * it.j, te = 16 * (it.j + cnt);   // virtual rows; a1 is a multiple of 16
          if (dst) mbar_expect_tx(full, 2 * (te - ts) * ROWB);
          if (ts < sg.a1) {
            const int e0 = min(te, sg.a1);
            if (dst) {
              bulk_g2s_ef(dst, K0 + (size_t)ts * D, (e0 - ts) * ROWB, full, pol);
              bulk_g2s_ef(dst + TILEB, V0 + (size_t)ts * D, (e0 - ts) * ROWB, full, pol);
            } else {
              bulk_prefetch_l2(K0 + (size_t)ts * D, (e0 - ts) * ROWB);
              bulk_prefetch_l2(V0 + (size_t)ts * D, (e0 - ts) * ROWB);
            }
          }
          if (te > sg.a1) {
            const int s0 = max(ts, sg.a1);
            if (dst) {
              bulk_g2s_ef(dst + (s0 - ts) * ROWB, K1 + (size_t)(s0 - sg.a1) * D, (te - s0) * ROWB, full, pol);
              bulk_g2s_ef(dst + TILEB + (s0 - ts) * ROWB, V1 + (size_t)(s0 - sg.a1) * D, (te - s0) * ROWB, full, pol);
            } else {
              bulk_prefetch_l2(K1 + (size_t)(s0 - sg.a1) * D, (te - s0) * ROWB);
              bulk_prefetch_l2(V1 + (size_t)(s0 - sg.a1) * D, (te - s0) * ROWB);
            }
          }
        } else {                                             // int8 codes + fp32 scales
          const size_t r0 = 16 * (size_t)(it.j - gbf);
          const int nr = 16 * cnt;
          if (dst) {
            mbar_expect_tx(full, 2 * (nr * D + nr * 4));
            bulk_g2s(dst, v.c2k[sb] + (grp * v.cap2 + r0) * D, nr * D, full);
            bulk_g2s(dst + TILE * D, v.s2k[sb] + grp * v.cap2 + r0, nr * 4, full);
            bulk_g2s(dst + TILEB, v.c2v[sb] + (grp * v.cap2 + r0) * D, nr * D, full);
            bulk_g2s(dst + TILEB + TILE * D, v.s2v[sb] + grp * v.cap2 + r0, nr * 4, full);
          } else {
            bulk_prefetch_l2(v.c2k[sb] + (grp * v.cap2 + r0) * D, nr * D);
            bulk_prefetch_l2(v.c2v[sb] + (grp * v.cap2 + r0) * D, nr * D);
          }
        }
      };
      Cur it{0, 0, part(0).j0};
      Cur ah = it;
      for (int x = 0; x < NST && ah.l < L; ++x) advance(ah);
      int i = 0;
      for (; it.l < L; ++i) {
        const int s2 = i % NST;
        if (i >= NST) mbar_sleep_wait(empty0 + 8 * s2, ((i / NST) - 1) & 1);
        if (ah.l < L) {                                       // L2 lookahead: the stage NST ahead
          const StepPart pa = part(ah.k);
          bool at2;
          const int acnt = stage_of(ah, pa, at2);
          if (acnt > 0) issue(ah, pa, acnt, at2, 0, 0);
          advance(ah);
        }
        const StepPart pp = part(it.k);
        bool t2;
        const int cnt = stage_of(it, pp, t2);
        const int fl = (it.j == pp.j0 ? SD_FIRST : 0) | ((cnt == 0 || it.j + cnt == pp.j1) ? SD_LAST : 0) |
                       (t2 ? SD_T2 : 0);
        sdesc[s2] = make_int4(it.l, it.k, it.j, fl | (cnt << 8));
        if (it.k == 0 && it.j == pp.j0) trace(it.l, 0);
        const uint32_t full = full0 + 8 * s2;
        if (cnt > 0) issue(it, pp, cnt, t2, ring_s + s2 * STAGEB, full);
        else mbar_arrive(full);                              // no cached row in this part
        advance(it);
      }
      const int s2 = i % NST;
      if (i >= NST) mbar_sleep_wait(empty0 + 8 * s2, ((i / NST) - 1) & 1);
      sdesc[s2] = make_int4(-1, 0, 0, 0);                    // sentinel
      mbar_arrive(full0 + 8 * s2);
    }
  } else if (w == WNEW) {
    // ========== new-token warp: the new token's attention term (every CTA of the head) and a1 ==========
    int nts = 0;
    constexpr int EL = D / 32;
    const float sl2 = (float)(1.4426950408889634 / __dsqrt_rn((double)D));   // log2(e)/sqrt(d)
    for (int l = 0; l < L; ++l) {
      if (l > 0) {                                           // k_new(l), q(l) follow o(l-1)
        if (lane == 0) wait_layer(l);
        __syncwarp();
      }
      if (S > 1) {                                           // q(l) of the head -> shared memory
        if (lane == 0) {
          const uint32_t qb = (uint32_t)(G * D * 2);
          mbar_expect_tx(qbar, qb);
          bulk_g2s(smem_u32(qsm(l)), io.q + (((size_t)l * B + b) * v.Hq + part(0).g * G) * D, qb, qbar);
        }
        mbar_sleep_wait(qbar, l & 1);
      }
      float* zl = v.zbuf + (size_t)(l % ZS) * U * v.zrows * 8;
      for (int k = 0; k < npart; ++k) {
        const StepPart pp = part(k);
        const int g = pp.g, u = b * Hkv + g;
        const int slot = nts & 1;
        const size_t grp = grp_of(v, l, b, g);
        const uint16_t* kin = reinterpret_cast<const uint16_t*>(io.knew) + (((size_t)l * B + b) * Hkv + g) * D;
        const uint16_t* vin = reinterpret_cast<const uint16_t*>(io.vnew) + (((size_t)l * B + b) * Hkv + g) * D;
        const uint16_t* qb0 = reinterpret_cast<const uint16_t*>(io.q) + (((size_t)l * B + b) * v.Hq + g * G) * D;
        uint16_t kb[EL], vb[EL], qb[8][EL];
        const uint16_t* qsrc = S > 1 ? reinterpret_cast<const uint16_t*>(qsm(l)) : qb0;
#pragma unroll
        for (int e2 = 0; e2 < EL; ++e2) {
          const int e = lane + 32 * e2;
          kb[e2] = __ldcg(kin + e);
          vb[e2] = __ldcg(vin + e);
#pragma unroll
          for (int h = 0; h < 8; ++h)
            qb[h][e2] = h >= G ? (uint16_t)0 : S > 1 ? qsrc[(size_t)h * D + e] : __ldcg(qsrc + (size_t)h * D + e);
        }
        float dot[8];
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          dot[h] = 0.f;
#pragma unroll
          for (int e2 = 0; e2 < EL; ++e2) dot[h] += bf16_bits_to_f(qb[h][e2]) * bf16_bits_to_f(kb[e2]);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1)
#pragma unroll
          for (int h = 0; h < 8; ++h) dot[h] += __shfl_xor_sync(0xffffffffu, dot[h], off);
        if (nts >= 2) mbar_sleep_wait(nempty0 + 8 * slot, ((nts >> 1) - 1) & 1);
#pragma unroll
        for (int e2 = 0; e2 < EL; ++e2) ntv[slot * D + lane + 32 * e2] = bf16_bits_to_f(vb[e2]);
        if (pp.fnew) {                                       // one CTA per head: a1 + its side effects
          uint16_t* K0w = reinterpret_cast<uint16_t*>(v.k0[sb]) + (grp * v.cap0 + sg.n0o) * D;
          uint16_t* V0w = reinterpret_cast<uint16_t*>(v.v0[sb]) + (grp * v.cap0 + sg.n0o) * D;
#pragma unroll
          for (int e2 = 0; e2 < EL; ++e2) {
            const int se = swz_off(sg.n0o, lane + 32 * e2, D);
            K0w[se] = kb[e2];                                // the row joins the T0 store
            V0w[se] = vb[e2];
          }
          if (v.red) redund_append(v, l, u, v.st->n - 1, kin);   // redundancy partial (AMB-30)
          if (scorer_uses_vnorm(v.scorer)) {                 // VATP: the new row's V norm
            float ss = 0.f;
#pragma unroll
            for (int e2 = 0; e2 < EL; ++e2) ss += bf16_bits_to_f(vb[e2]) * bf16_bits_to_f(vb[e2]);
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
            if (lane == 0) v.vnorm[((size_t)l * U + u) * v.Nmax + (v.st->n - 1)] = sqrtf(ss);
          }
        }
        if (lane < 8) {
          float z = 0.f;
#pragma unroll
          for (int h = 0; h < 8; ++h) z = lane == h ? dot[h] * sl2 : z;
          ntz[slot * 8 + lane] = lane < G ? z : -INFINITY;
          if (lane < G && io.score && pp.fnew) zl[((size_t)u * v.zrows + sg.a3) * 8 + lane] = z;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(nfull0 + 8 * slot);
        ++nts;
      }
    }
  } else if (w == WSC0 || w == WSC0 + 1) {
    // ====== score warps: a4 of layer l-1 while the consumers run layer l (Eq. 1, AMB-14) ======
    const int st0 = tid - WSC0 * 32;                          // 0..NSC-1
    constexpr int SB = 8;
    bool bad = false;
    for (int lp = 0; lp < L && io.score; ++lp) {
      if (st0 == 0) {
        while (*ml_done <= lp) __nanosleep(128);              // (M, 1/L) of layer lp merged
        __threadfence_block();
      }
      named_sync(2, NSC);
      const float* zb = v.zbuf + (size_t)(lp % ZS) * U * v.zrows * 8;
      for (int k = 0; k < npart; ++k) {
        const StepPart pp = part(k);
        const int u = b * Hkv + pp.g;
        const float* ml = sml + ((lp % ZS) * STEP_MAXM + k) * 16;
        float mh[8], il[8];
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          mh[h] = ml[h];
          il[h] = ml[8 + h];
        }
        // rows of the part (virtual), then the new token (row a3) in the head's appending CTA
        const int r_bf0 = 16 * min(pp.j0, gbf), r_bf1 = 16 * min(pp.j1, gbf);
        const int r_q0 = sg.a2 + 16 * (max(pp.j0, gbf) - gbf), r_q1 = sg.a2 + 16 * (max(pp.j1, gbf) - gbf);
        const int nbf = r_bf1 - r_bf0, nq = r_q1 - r_q0;
        const int ntot = nbf + nq + (pp.fnew ? 1 : 0);
        float* Sp = v.S + (size_t)u * v.Nmax;
        const float* zu = zb + (size_t)u * v.zrows * 8;
        for (int k0 = st0; k0 < ntot; k0 += NSC * SB) {
          int pos[SB];
          float4 z0[SB], z1[SB];
#pragma unroll
          for (int x = 0; x < SB; ++x) {
            const int kk = k0 + NSC * x;
            pos[x] = -1;
            if (kk < ntot) {
              const int t = kk < nbf ? r_bf0 + kk : (kk < nbf + nq ? r_q0 + (kk - nbf) : sg.a3);
              const bool ok = kk < nbf ? sg.bf16_valid(t) : (kk < nbf + nq ? (t - sg.a2 < sg.n2) : true);
              if (ok) {
                pos[x] = sg.pos(v, cur, b, t);
                z0[x] = __ldcg(reinterpret_cast<const float4*>(zu + (size_t)t * 8));
                z1[x] = __ldcg(reinterpret_cast<const float4*>(zu + (size_t)t * 8 + 4));
              }
            }
          }
          float sv[SB];
#pragma unroll
          for (int x = 0; x < SB; ++x)
            if (pos[x] >= 0) sv[x] = __ldcg(Sp + pos[x]);
#pragma unroll
          for (int x = 0; x < SB; ++x) {
            if (pos[x] < 0) continue;
            const float zz[8] = {z0[x].x, z0[x].y, z0[x].z, z0[x].w, z1[x].x, z1[x].y, z1[x].z, z1[x].w};
            float inc = 0.f;
#pragma unroll
            for (int h = 0; h < 8; ++h)
              if (h < G) inc += ex2_ftz(zz[h] - mh[h]) * il[h];
            Sp[pos[x]] = sv[x] + inc * score_weight(v, lp, u, pos[x]);
            bad |= !isfinite(inc);
          }
        }
      }
      named_sync(2, NSC);                                     // every zbuf read of layer lp is done
      if (st0 == 0) {
        __threadfence_block();
        *sc_done = lp + 1;                                    // layers 0..lp scored
        trace(lp, 5);
      }
    }
    if (bad) atomicOr(&v.st->err, 1);
  } else if (w == WISS) {
    // ========== UM: the MMA-issuing thread (tcgen05.mma, accumulators in TMEM) ==========
    // Per stage i: S(i) = K(i) q^T into TMEM S[i & 1] (commit -> sready[i & 1]); once the softmax
    // warps have written P(i) into p tile i & 1, O += V(i)^T P(i)^T into TMEM O (afresh when the
    // softmax warps say so: a part's first P.V, or the first after they folded O into registers
    // at a raised running max), commit -> odone[i & 1] and the ring slot's empty barrier.  S(i + 1)
    // is issued before the P.V of stage i (it overlaps the softmax) unless stage i + 1 opens the
    // next layer: its q waits for o(l), which needs the P.V of stage i.  Commits (never plain
    // arrives) also signal stages without rows: a commit tracks every earlier MMA of the thread.
    if constexpr (UM) {
      if (lane == 0) {
        const uint32_t idS = umma_idesc(128, 16, 0, 0), idO = umma_idesc(128, 16, 1, 0);
        const uint32_t qs = smem_u32(qtile), ps = smem_u32(ptile);
        auto koff = [](int kk) { return (uint32_t)((kk >> 2) * 1024 + (kk & 3) * 32); };
        auto issue_qk = [&](int i, int cnt) {
          if (cnt > 0) {
            const uint32_t sK = ring_s + (i % NST) * STAGEB;
#pragma unroll
            for (int kk = 0; kk < KS; ++kk)
              umma_bf16(tmem + 16 * (i & 1), umma_sdesc(sK + koff(kk), 16, 2048), umma_sdesc(qs + koff(kk), 16, 2048),
                        idS, kk > 0);
          }
          umma_commit(sready0 + 8 * (i & 1));
        };
        int nq = 0;
        bool ahead = false;
        for (int i = 0;; ++i) {
          const int s2 = i % NST;
          if (!ahead) {
            mbar_wait(full0 + 8 * s2, (i / NST) & 1);
            const int4 dsc = sdesc[s2];
            if (dsc.x < 0) { umma_commit(sready0 + 8 * (i & 1)); break; }   // wake the softmax warps
            if (dsc.w & SD_FIRST) { mbar_wait(qready, nq & 1); ++nq; }     // q(l) in the q tile
            tc_fence_after();
            issue_qk(i, dsc.w >> 8);
          }
          ahead = false;
          {
            const int i1 = i + 1;
            mbar_wait(full0 + 8 * (i1 % NST), (i1 / NST) & 1);
            const int4 d1 = sdesc[i1 % NST];
            if (d1.x >= 0 && !(d1.w & SD_FIRST)) {
              issue_qk(i1, d1.w >> 8);
              ahead = true;
            }
          }
          mbar_wait(pready, i & 1);                               // P(i) in p tile i & 1
          tc_fence_after();
          if ((sdesc[s2].w >> 8) > 0) {
            const uint32_t sV = ring_s + s2 * STAGEB + TILEB, pt = ps + (i & 1) * 16 * ROWB;
            const uint32_t fresh = (uint32_t)pvfresh[i & 1];
#pragma unroll
            for (int kk = 0; kk < TILE / 16; ++kk)
              umma_bf16(tmem + 32, umma_sdesc(sV + kk * 4096, 1024, 2048), umma_sdesc(pt + koff(kk), 16, 2048), idO,
                        (kk > 0 || !fresh) ? 1u : 0u);
          }
          umma_commit(odone0 + 8 * (i & 1));
          umma_commit(empty0 + 8 * s2);
        }
      }
    }
  } else if constexpr (UM) {
    // ========== UM: softmax warps -- thread t owns token row t of S(i) and d row t of O ==========
    // The o accumulator stays in TMEM across a part's stages; it is folded into registers only
    // when the CTA-wide running max of a head rises past its slack (rare after the first stage)
    // and at the part's end, so the softmax of stage i + 1 never waits for the P.V of stage i.
    const float sl2 = (float)(1.4426950408889634 / __dsqrt_rn((double)D));
    constexpr float RESCALE_SLACK = 8.f;
    float mref[8], lsum[8], oacc[8];
#pragma unroll
    for (int h = 0; h < 8; ++h) { mref[h] = -INFINITY; lsum[h] = 0.f; oacc[h] = 0.f; }
    float* zrow = nullptr;
    bool pend = false;                                       // a P.V of this part sits in TMEM O
    const uint32_t tq_lane = (uint32_t)(32 * w) << 16;      // TMEM lane quadrant of this warp
    auto fold_o = [&](int k) {                               // O (through the P.V of stage k) -> registers
      mbar_wait(odone0 + 8 * (k & 1), (k >> 1) & 1);
      tc_fence_after();
      uint32_t r[16];
      tmem_ld16(tmem + 32 + tq_lane, r);
      tmem_ld_wait();
#pragma unroll
      for (int h = 0; h < 8; ++h) oacc[h] += __uint_as_float(r[h]) + __uint_as_float(r[8 + h]);
    };
    auto build_q = [&](int l) {                              // q(l) of the head -> the swizzled q tile
      if (tid == 0) ctrace(l, 12);
      mbar_wait(qbar, l & 1);                          // the layer dependency held, q(l) landed
      if (tid == 0) { trace(l, 1); ctrace(l, 13); }
      const uint16_t* qsrc = reinterpret_cast<const uint16_t*>(qsm(l));
      for (int x = tid; x < 16 * (D / 8); x += NCONS) {
        const int r = x / (D / 8), c = x % (D / 8);
        const uint4 val = r < G ? *reinterpret_cast<const uint4*>(qsrc + r * D + c * 8) : make_uint4(0u, 0u, 0u, 0u);
        *reinterpret_cast<uint4*>(qtile + tile_off<D>(r, c)) = val;
      }
      fence_proxy_async_cta();                               // generic stores -> the MMA's operand reads
      __syncwarp();
      if (lane == 0) mbar_arrive(qready);
    };
    build_q(0);
    for (int i = 0;; ++i) {
      const int s2 = i % NST;
      mbar_wait(full0 + 8 * s2, (i / NST) & 1);       // acquire the stage descriptor
      const int4 dsc = sdesc[s2];
      mbar_wait(sready0 + 8 * (i & 1), (i >> 1) & 1);
      if (dsc.x < 0) break;
      const int l = dsc.x, kpart = dsc.y, j = dsc.z, fl = dsc.w & 0xFF, cnt = dsc.w >> 8;
      const int g = part(kpart).g, u = b * Hkv + g;
      if (fl & SD_FIRST) {
        if (tid == 0) ctrace(l, 14);                         // S of the layer's first stage is in TMEM
        if (lane == 0 && io.score)
          while (*sc_done < l - ZS + 1) __nanosleep(128);     // logit slot of layer l - ZS consumed
        __syncwarp();
        zrow = io.score ? v.zbuf + (size_t)(l % ZS) * U * v.zrows * 8 + (size_t)u * v.zrows * 8 : nullptr;
      }
      tc_fence_after();
      // ---- logits of token row t (log2 domain)
      const int tv = 16 * j + tid;
      const bool valid = tid < cnt * 16 && sg.bf16_valid(tv);
      float z[8];
      if (cnt > 0) {
        uint32_t r[8];
        tmem_ld8(tmem + 16 * (i & 1) + tq_lane, r);
        tmem_ld_wait();
#pragma unroll
        for (int h = 0; h < 8; ++h) z[h] = (valid && h < G) ? __uint_as_float(r[h]) * sl2 : -INFINITY;
      } else {
#pragma unroll
        for (int h = 0; h < 8; ++h) z[h] = -INFINITY;
      }
      if (zrow && valid) {
        *reinterpret_cast<float4*>(zrow + (size_t)tv * 8) = make_float4(z[0], z[1], z[2], z[3]);
        *reinterpret_cast<float4*>(zrow + (size_t)tv * 8 + 4) = make_float4(z[4], z[5], z[6], z[7]);
      }
      // ---- running max per head, CTA-wide: raised only when a logit passes it by the slack
      bool need = false;
#pragma unroll
      for (int h = 0; h < 8; ++h) need |= z[h] > mref[h] + RESCALE_SLACK;
      float* wm = wmx + (i & 1) * NW * 8;
      if (__any_sync(0xffffffffu, need)) {
        float t8[8];
#pragma unroll
        for (int h = 0; h < 8; ++h) t8[h] = z[h];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1)
#pragma unroll
          for (int h = 0; h < 8; ++h) t8[h] = fmaxf(t8[h], __shfl_xor_sync(0xffffffffu, t8[h], off));
        if (lane < 8) {
          float x = t8[0];
#pragma unroll
          for (int h = 1; h < 8; ++h) x = lane == h ? t8[h] : x;
          wm[w * 8 + lane] = x;
        }
      } else if (lane < 8) {
        wm[w * 8 + lane] = -INFINITY;
      }
      named_sync(1, NCONS);
      float mnew[8];
      bool raise = false;                                    // uniform: every thread reads the same maxima
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        float mx = wm[h];
#pragma unroll
        for (int x = 1; x < NW; ++x) mx = fmaxf(mx, wm[x * 8 + h]);
        mnew[h] = mx > mref[h] + RESCALE_SLACK ? mx : mref[h];
        raise |= mnew[h] != mref[h];
      }
      if (raise) {
        if (pend) fold_o(i - 1);                             // O so far, at the old scale
#pragma unroll
        for (int h = 0; h < 8; ++h) {
          if (mnew[h] != mref[h]) {
            const float c = mref[h] == -INFINITY ? 0.f : ex2_ftz(mref[h] - mnew[h]);
            oacc[h] *= c;
            lsum[h] *= c;
            mref[h] = mnew[h];
          }
        }
      }
      const bool fresh = !pend || raise;                     // this stage's P.V starts O afresh
      // ---- p = 2^(z - m) as two bf16 terms (hi: P rows 0-7, lo: rows 8-15), token column t
      if (i >= 2) mbar_wait(odone0 + 8 * (i & 1), ((i - 2) >> 1) & 1);   // P.V(i - 2) read this p tile
      unsigned char* pt = ptile + (i & 1) * 16 * ROWB;
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        const float p = (valid && h < G) ? ex2_ftz(z[h] - mref[h]) : 0.f;
        lsum[h] += p;
        const __nv_bfloat16 hi = __float2bfloat16_rn(p);
        const __nv_bfloat16 lo = __float2bfloat16_rn(p - __bfloat162float(hi));
        *reinterpret_cast<__nv_bfloat16*>(pt + tile_off<D>(h, tid >> 3) + (tid & 7) * 2) = hi;
        *reinterpret_cast<__nv_bfloat16*>(pt + tile_off<D>(8 + h, tid >> 3) + (tid & 7) * 2) = lo;
      }
      if (tid == 0) pvfresh[i & 1] = fresh ? 1 : 0;
      fence_proxy_async_cta();
      tc_fence_before();                                     // this warp's TMEM reads precede the next MMAs
      __syncwarp();
      if (lane == 0) mbar_arrive(pready);
      if (cnt > 0) pend = true;
      if (!(fl & SD_LAST)) continue;
      // ---- part end: the CTA partial is (m = mref, l = sum of p over the 128 token rows, o)
      if (pend) fold_o(i);
      if (tid == 0) ctrace(l, 15);
      tc_fence_before();
      pend = false;
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        float x = lsum[h];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
        lsum[h] = x;
      }
      if (lane < 8) {
        float x = lsum[0];
#pragma unroll
        for (int h = 1; h < 8; ++h) x = lane == h ? lsum[h] : x;
        redl[w * 8 + lane] = x;
      }
      if (tid == 0 && S > 1) bulk_wait_read0();              // the previous push has read pbuf
      named_sync(1, NCONS);
      if (tid < 8) {
        float Ls = 0.f, M = mref[0];
#pragma unroll
        for (int x = 0; x < NW; ++x) Ls += redl[x * 8 + tid];
#pragma unroll
        for (int h = 1; h < 8; ++h) M = tid == h ? mref[h] : M;
        pbuf[tid] = M;
        pbuf[8 + tid] = Ls;
      }
#pragma unroll
      for (int h = 0; h < 8; ++h)
        if (h < G) pbuf[16 + h * D + tid] = oacc[h];
#pragma unroll
      for (int h = 0; h < 8; ++h) { mref[h] = -INFINITY; lsum[h] = 0.f; oacc[h] = 0.f; }
      merge_part(l, kpart, g);
      if (l + 1 < L) build_q(l + 1);
    }
    if (tid == 0 && S > 1) bulk_wait_read0();
  } else {
    // ================================ consumers ================================
    const float sl2 = (float)(1.4426950408889634 / __dsqrt_rn((double)D));
    float mxa = -INFINITY, mxb = -INFINITY, la = 0.f, lb = 0.f;
    float oacc[KS][4];
    uint32_t qf[KS][2];
    float* zrow = nullptr;
    const int mi = lane >> 3, ii = lane & 7;
    constexpr float RESCALE_SLACK = 8.f;
    auto online = [&](float z00, float z01, float z10, float z11, float& p00, float& p01, float& p10, float& p11) {
      const bool grow = z00 > mxa + RESCALE_SLACK || z10 > mxa + RESCALE_SLACK ||
                        z01 > mxb + RESCALE_SLACK || z11 > mxb + RESCALE_SLACK;
      if (__any_sync(0xffffffffu, grow)) {
        float ta = fmaxf(z00, z10), tb = fmaxf(z01, z11);
#pragma unroll
        for (int off = 4; off < 32; off <<= 1) {
          ta = fmaxf(ta, __shfl_xor_sync(0xffffffffu, ta, off));
          tb = fmaxf(tb, __shfl_xor_sync(0xffffffffu, tb, off));
        }
        const float na = fmaxf(mxa, ta), nb = fmaxf(mxb, tb);
        const float ca = ex2_ftz(mxa - na), cb = ex2_ftz(mxb - nb);
        mxa = na;
        mxb = nb;
#pragma unroll
        for (int mt = 0; mt < KS; ++mt) {
          oacc[mt][0] *= ca;
          oacc[mt][2] *= ca;
          oacc[mt][1] *= cb;
          oacc[mt][3] *= cb;
        }
        la *= ca;
        lb *= cb;
      }
      p00 = ex2_ftz(z00 - mxa);
      p01 = ex2_ftz(z01 - mxb);
      p10 = ex2_ftz(z10 - mxa);
      p11 = ex2_ftz(z11 - mxb);
      la += p00 + p10;
      lb += p01 + p11;
    };
    auto qk = [&](uint32_t sK, int rowbase, float* acc) {
      constexpr int NCH = KS >= 4 ? 4 : KS;
      float ch[NCH][4];
#pragma unroll
      for (int x = 0; x < NCH; ++x) ch[x][0] = ch[x][1] = ch[x][2] = ch[x][3] = 0.f;
      const int row = rowbase + ii + ((mi & 1) << 3);
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        uint32_t a0, a1_, a2_, a3_;
        ldsm_x4(a0, a1_, a2_, a3_, sK + tile_off<D>(row, 2 * ks + (mi >> 1)));
        mma16816(ch[ks % NCH], a0, a1_, a2_, a3_, qf[ks][0], qf[ks][1]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float x = ch[0][j];
#pragma unroll
        for (int y = 1; y < NCH; ++y) x += ch[y][j];
        acc[j] += x;
      }
    };
    auto pv = [&](uint32_t sV, int rowbase, float p00, float p01, float p10, float p11) {
      uint32_t h0, l0, h1, l1;
      split_bf16x2(p00, p01, h0, l0);
      split_bf16x2(p10, p11, h1, l1);
      const uint32_t b0 = movm_t(h0), b1 = movm_t(h1), c0 = movm_t(l0), c1 = movm_t(l1);
      const int row = rowbase + ii + ((mi >> 1) << 3);
      uint32_t af[KS][4];
#pragma unroll
      for (int mt = 0; mt < KS; ++mt)
        ldsm_x4_t(af[mt][0], af[mt][1], af[mt][2], af[mt][3], sV + tile_off<D>(row, 2 * mt + (mi & 1)));
#pragma unroll
      for (int mt = 0; mt < KS; ++mt) mma16816(oacc[mt], af[mt][0], af[mt][1], af[mt][2], af[mt][3], c0, c1);
#pragma unroll
      for (int mt = 0; mt < KS; ++mt) mma16816(oacc[mt], af[mt][0], af[mt][1], af[mt][2], af[mt][3], b0, b1);
    };
    auto stage_t2_rows = [&](const int8_t* codes, unsigned char* scr) {
      for (int e = lane; e < 16 * (D / 16); e += 32) {
        const int row = e / (D / 16), j = e % (D / 16);
        const uint4 cw = *reinterpret_cast<const uint4*>(codes + (size_t)(w * 16 + row) * D + 16 * j);
        uint4 lo, hi;
        lo.x = i8pair_to_bf16x2(cw.x, 0); lo.y = i8pair_to_bf16x2(cw.x, 1);
        lo.z = i8pair_to_bf16x2(cw.y, 0); lo.w = i8pair_to_bf16x2(cw.y, 1);
        hi.x = i8pair_to_bf16x2(cw.z, 0); hi.y = i8pair_to_bf16x2(cw.z, 1);
        hi.z = i8pair_to_bf16x2(cw.w, 0); hi.w = i8pair_to_bf16x2(cw.w, 1);
        *reinterpret_cast<uint4*>(scr + tile_off<D>(row, 2 * j)) = lo;
        *reinterpret_cast<uint4*>(scr + tile_off<D>(row, 2 * j + 1)) = hi;
      }
      __syncwarp();
    };

    long long wfull = 0;                                     // debug: cycles warp 0 waited for stage data
    for (int i = 0;; ++i) {
      const int s2 = i % NST;
      const long long tw = KVT_TRACE ? clock64() : 0;
      mbar_sleep_wait(full0 + 8 * s2, (i / NST) & 1);
      if (KVT_TRACE) wfull += clock64() - tw;
      const int4 dsc = sdesc[s2];
      const int l = dsc.x;
      if (l < 0) break;
      const int kpart = dsc.y, j = dsc.z, fl = dsc.w & 0xFF, cnt = dsc.w >> 8;

      const StepPart pp = part(kpart);
      const int g = pp.g, u = b * Hkv + g;
      if (fl & SD_FIRST) {
        if (kpart == 0) {
          // q(l) is a projection of o(l-1): every CTA of this request has stored its part
          if (tid == 0) ctrace(l, 12);
          if (S > 1) mbar_sleep_wait(qbar, l & 1);          // the dependency held and q(l) landed
          if (lane == 0) {
            if (S == 1 && l > 0) wait_layer(l);
            if (io.score)
              while (*sc_done < l - ZS + 1) __nanosleep(128);   // logit slot of layer l - ZS consumed
          }
          __syncwarp();
          if (tid == 0) { trace(l, 1); ctrace(l, 13); }
        }
        if (S > 1) {
          const uint32_t* qw = reinterpret_cast<const uint32_t*>(qsm(l)) + (gq * D + 2 * tq) / 2;
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) {
            qf[ks][0] = gq < G ? qw[ks * 8] : 0u;
            qf[ks][1] = gq < G ? qw[ks * 8 + 4] : 0u;
          }
        } else {
          const __nv_bfloat16* qh = io.q + (((size_t)l * B + b) * v.Hq + g * G + gq) * D;
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) {
            if (gq < G) {
              qf[ks][0] = __ldcg(reinterpret_cast<const unsigned int*>(qh + ks * 16 + 2 * tq));
              qf[ks][1] = __ldcg(reinterpret_cast<const unsigned int*>(qh + ks * 16 + 8 + 2 * tq));
            } else {
              qf[ks][0] = 0u;
              qf[ks][1] = 0u;
            }
          }
        }
        mxa = mxb = -INFINITY;
        la = lb = 0.f;
#pragma unroll
        for (int mt = 0; mt < KS; ++mt) oacc[mt][0] = oacc[mt][1] = oacc[mt][2] = oacc[mt][3] = 0.f;
        if (tid == 0 && kpart == 0) { asm volatile("" :: "r"(qf[KS - 1][1])); ctrace(l, 14); }   // q loaded
        zrow = io.score ? v.zbuf + (size_t)(l % ZS) * U * v.zrows * 8 + (size_t)u * v.zrows * 8 : nullptr;
      }
      if (cnt > 0) {
        const bool t2 = fl & SD_T2;
        const bool wact = w < cnt;
        const int tv0 = t2 ? sg.a2 + 16 * (j - gbf + w) : 16 * (j + w);
        const int r0 = w * 16 + gq, r1 = r0 + 8;
        const int t0 = tv0 + gq, t1 = tv0 + gq + 8;
        const bool v0 = wact && (t2 ? (t0 - sg.a2 < sg.n2) : sg.bf16_valid(t0));
        const bool v1 = wact && (t2 ? (t1 - sg.a2 < sg.n2) : sg.bf16_valid(t1));
        const uint32_t sK = ring_s + s2 * STAGEB, sV = sK + TILEB;
        if (__any_sync(0xffffffffu, v0 || v1)) {
          float acc[4] = {0.f, 0.f, 0.f, 0.f};
          float fk0 = sl2, fk1 = sl2, fv0 = 1.f, fv1 = 1.f;
          unsigned char* scr = t2w + (size_t)w * 16 * ROWB;
          if (!t2) {
            qk(sK, w * 16, acc);
          } else {
            unsigned char* st = ring + s2 * STAGEB;
            const float* scK = reinterpret_cast<const float*>(st + TILE * D);
            const float* scV = reinterpret_cast<const float*>(st + TILEB + TILE * D);
            fk0 = scK[r0] * sl2; fk1 = scK[r1] * sl2;
            fv0 = scV[r0]; fv1 = scV[r1];
            stage_t2_rows(reinterpret_cast<const int8_t*>(st), scr);
            qk(smem_u32(scr), 0, acc);
          }
          const float z00 = v0 ? acc[0] * fk0 : -INFINITY, z01 = v0 ? acc[1] * fk0 : -INFINITY;
          const float z10 = v1 ? acc[2] * fk1 : -INFINITY, z11 = v1 ? acc[3] * fk1 : -INFINITY;
          if (zrow) {
            if (v0) *reinterpret_cast<float2*>(zrow + (size_t)t0 * 8 + 2 * tq) = make_float2(z00, z01);
            if (v1) *reinterpret_cast<float2*>(zrow + (size_t)t1 * 8 + 2 * tq) = make_float2(z10, z11);
          }
          float p00, p01, p10, p11;
          online(z00, z01, z10, z11, p00, p01, p10, p11);
          if (!t2) {
            pv(sV, w * 16, p00, p01, p10, p11);
          } else {
            __syncwarp();
            stage_t2_rows(reinterpret_cast<const int8_t*>(ring + s2 * STAGEB + TILEB), scr);
            pv(smem_u32(scr), 0, p00 * fv0, p01 * fv0, p10 * fv1, p11 * fv1);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty0 + 8 * s2);
      if (!(fl & SD_LAST)) continue;

      // ---------------- part end: warps -> CTA partial (m, l, o) in pbuf
      if (tid == 0 && kpart == 0) ctrace(l, 15);
      if (KVT_TRACE && v.trace && tid == 0 && kpart == 0) {
        v.trace[((size_t)l * gridDim.x + blockIdx.x) * NTRACE + 21] = (unsigned long long)wfull;
        wfull = 0;
      }
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        la += __shfl_xor_sync(0xffffffffu, la, off);
        lb += __shfl_xor_sync(0xffffffffu, lb, off);
      }
      if (tid == 0 && S > 1) bulk_wait_read0();              // the previous push has read pbuf
      // (ow / redm are free: the previous merge ended with a barrier)
      if (lane < 4) {
        redm[w * 8 + 2 * lane] = mxa;
        redm[w * 8 + 2 * lane + 1] = mxb;
        redl[w * 8 + 2 * lane] = la;
        redl[w * 8 + 2 * lane + 1] = lb;
      }
      named_sync(1, NCONS);
      {
        float Ma = -INFINITY, Mb = -INFINITY;                 // per-head max over the warps
#pragma unroll
        for (int x = 0; x < NW; ++x) {
          Ma = fmaxf(Ma, redm[x * 8 + 2 * tq]);
          Mb = fmaxf(Mb, redm[x * 8 + 2 * tq + 1]);
        }
        const float fa = mxa == -INFINITY ? 0.f : ex2_ftz(mxa - Ma), fb = mxb == -INFINITY ? 0.f : ex2_ftz(mxb - Mb);
#pragma unroll
        for (int mt = 0; mt < KS; ++mt) {
          oacc[mt][0] *= fa;
          oacc[mt][2] *= fa;
          oacc[mt][1] *= fb;
          oacc[mt][3] *= fb;
        }
      }
      // two-round tree (deterministic order): warps NH.. hand their o to warps 0.., which add it
      auto put = [&](int slot) {
#pragma unroll
        for (int mt = 0; mt < KS; ++mt) {
          float* o0 = ow + (slot * 8 + 2 * tq) * OWS + mt * 16 + gq;
          float* o1 = o0 + OWS;
          o0[0] = oacc[mt][0];
          o1[0] = oacc[mt][1];
          o0[8] = oacc[mt][2];
          o1[8] = oacc[mt][3];
        }
      };
      if (w >= NH) put(w - NH);
      named_sync(1, NCONS);
      if (w < NH) {
#pragma unroll
        for (int mt = 0; mt < KS; ++mt) {
          const float* o0 = ow + (w * 8 + 2 * tq) * OWS + mt * 16 + gq;
          const float* o1 = o0 + OWS;
          oacc[mt][0] += o0[0];
          oacc[mt][1] += o1[0];
          oacc[mt][2] += o0[8];
          oacc[mt][3] += o1[8];
        }
      }
      if (w < NH) put(w);                                    // same slot this warp just read: no barrier
      named_sync(1, NCONS);
      if (tid < 8) {
        float M = -INFINITY;
#pragma unroll
        for (int x = 0; x < NW; ++x) M = fmaxf(M, redm[x * 8 + tid]);
        float Ls = 0.f;
#pragma unroll
        for (int x = 0; x < NW; ++x) {
          const float m = redm[x * 8 + tid];
          Ls += (m == -INFINITY ? 0.f : ex2_ftz(m - M)) * redl[x * 8 + tid];
        }
        pbuf[tid] = M;
        pbuf[8 + tid] = Ls;
      }
      for (int e = tid; e < tot; e += NCONS) {
        const int h = e / D, dd = e - h * D;
        float a = 0.f;
#pragma unroll
        for (int x = 0; x < NH; ++x) a += ow[(x * 8 + h) * OWS + dd];
        pbuf[16 + e] = a;
      }
      merge_part(l, kpart, g);
    }
    if (tid == 0 && S > 1) bulk_wait_read0();
  }
  __syncwarp();
  if constexpr (UM) tc_fence_before();
  if (S > 1) cluster_sync_all();                // no peer accesses this CTA's shared memory after exit
  if constexpr (UM) {                           // (UM runs with S > 1: the cluster barrier above is CTA-wide too)
    if (w == WISS) {
      tc_fence_after();
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;\n" ::"r"(tmem));
    }
  }
}

// ----------------------------------------------------------------- host side
// Shapes: 8 consumer warps, one CTA per SM (NW = 8); 4 consumer warps, two CTAs per SM (NW = 4:
// twice the CTAs, so a request's rows are cut into twice as many slices and two requests' layer
// chains share each SM); or the tcgen05 consumer (DevView::step_um: d = 128, no T2 rows, a
// cluster per kv head; 4 softmax warps + the issuing warp, one CTA per SM, 128-row stages).
template <int D, int NW, int NST, bool UM>
static size_t step_smem_bytes_t(const DevView& v) {
  const int S = v.step_s > 0 ? v.step_s : 1;
  const int tot = v.G * D, SL = ((tot + S - 1) / S + 3) & ~3;
  constexpr int GPS = UM ? 8 : NW;
  size_t s = (size_t)NST * 2 * GPS * 16 * D * 2;                 // ring
  if (UM) s += 1024 + 3 * 16 * D * 2;                            // alignment, q tile, p tiles
  if (v.cap2 > 0) s += (size_t)NW * 16 * D * 2;                  // T2 scratch
  if (!UM) s += (size_t)(NW / 2) * 8 * (D + 4) * 4;              // ow
  s += (size_t)(16 + 8 * D + 4 * 16) * 4;                        // pbuf (+ tail read by the padded last slice)
  s += (size_t)2 * S * (16 + SL) * 4;                            // rx
  s += (size_t)2 * NW * 8 * 4 + 16 * 4 + 2 * D * 4;              // redm, redl, ntz, ntv
  s += (size_t)ZRING * STEP_MAXM * 16 * 4 + 24 * 4 + 16 * 8 * 4; // sml, merge scalars, merge factors
  if (UM) s += (size_t)2 * NW * 8 * 4;                           // stage maxima
  s += (2 * NST + 16) * 8 + NST * 16 + STEP_MAXM * sizeof(StepPart) + 32;   // barriers, descriptors, parts, counters
  return s;
}

// ring depth: as many stages as fit beside the scratch
static int step_nst(const DevView& v) {
  if (v.step_um) return 3;
  if (v.step_nw == 4) return v.D == 128 ? 2 : 4;                 // two CTAs per SM
  if (v.D == 128) return v.cap2 > 0 ? 2 : 3;
  return v.cap2 > 0 ? 5 : 6;
}

#define KVT_STEP_SHAPES(X)                                                                   \
  X(128, 8, 3, false) X(128, 8, 2, false) X(64, 8, 6, false) X(64, 8, 5, false) X(128, 4, 2, false) \
  X(64, 4, 4, false) X(128, 4, 3, true)
#define KVT_STEP_MATCH(DD, NWW, NSS, UU) \
  (v.D == DD && nst == NSS && (UU ? v.step_um != 0 : (v.step_um == 0 && v.step_nw == NWW)))

size_t step_smem_bytes(const DevView& v) {
  const int nst = step_nst(v);
#define KVT_SZ(DD, NWW, NSS, UU) \
  if (KVT_STEP_MATCH(DD, NWW, NSS, UU)) return step_smem_bytes_t<DD, NWW, NSS, UU>(v);
  KVT_STEP_SHAPES(KVT_SZ)
#undef KVT_SZ
  return ~(size_t)0;
}

template <int D, int NW, int NST, bool UM>
static cudaError_t step_conf_t(const DevView& v, int* clusters) {
  auto kern = k_decode_step<D, NW, NST, UM>;
  const size_t smem = step_smem_bytes_t<D, NW, NST, UM>(v);
  const int K = v.step_s;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(v.B * v.Hkv * v.step_s / v.step_m, 1, 1);
  cfg.blockDim = dim3((NW + 4 + (UM ? 1 : 0)) * 32, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = K;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaOccupancyMaxActiveClusters(clusters, kern, &cfg);
}

// Co-resident clusters of v.step_s CTAs of the chosen shape (0: it cannot run).
cudaError_t step_configure(const DevView& v, int* clusters) {
  *clusters = 0;
  const int nst = step_nst(v);
#define KVT_CF(DD, NWW, NSS, UU) \
  if (KVT_STEP_MATCH(DD, NWW, NSS, UU)) return step_conf_t<DD, NWW, NSS, UU>(v, clusters);
  KVT_STEP_SHAPES(KVT_CF)
#undef KVT_CF
  return cudaErrorInvalidValue;
}

template <int D, int NW, int NST, bool UM>
static cudaError_t step_launch_t(const DevView& v, const StepIO& io, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(v.step_k, 1, 1);                  // step_k = total CTAs
  cfg.blockDim = dim3((NW + 4 + (UM ? 1 : 0)) * 32, 1, 1);
  cfg.dynamicSmemBytes = step_smem_bytes_t<D, NW, NST, UM>(v);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int na = 0;
  at[na].id = cudaLaunchAttributeClusterDimension;      // one cluster per kv head (its S slices)
  at[na].val.clusterDim.x = v.step_s;
  at[na].val.clusterDim.y = 1;
  at[na].val.clusterDim.z = 1;
  ++na;
  if (v.hot_bytes > 0) {
    at[na].id = cudaLaunchAttributeAccessPolicyWindow;
    at[na].val.accessPolicyWindow.base_ptr = v.hot_base;
    at[na].val.accessPolicyWindow.num_bytes = v.hot_bytes;
    at[na].val.accessPolicyWindow.hitRatio = v.hot_hit;
    at[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    at[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, k_decode_step<D, NW, NST, UM>, v, io);
}

cudaError_t launch_decode_step(const DevView& v, const void* q, const void* knew, const void* vnew, void* o, int score,
                               cudaStream_t s) {
  StepIO io;
  io.q = reinterpret_cast<const __nv_bfloat16*>(q);
  io.knew = reinterpret_cast<const __nv_bfloat16*>(knew);
  io.vnew = reinterpret_cast<const __nv_bfloat16*>(vnew);
  io.o = o;
  io.score = score;
  const int nst = step_nst(v);
#define KVT_LN(DD, NWW, NSS, UU) \
  if (KVT_STEP_MATCH(DD, NWW, NSS, UU)) return step_launch_t<DD, NWW, NSS, UU>(v, io, s);
  KVT_STEP_SHAPES(KVT_LN)
#undef KVT_LN
  return cudaErrorInvalidValue;
}

}  // namespace kvt
