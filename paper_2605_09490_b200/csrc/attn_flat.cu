// a1 + a3 + a4, flat work distribution (default decode path): fused new-token append, GQA
// decode attention over the visible tiers, and the cumulative score update
// (Eq. 1, Eq. 3, Prop. 1).
//
// Work.  Every unit (request b, kv head g) has the same virtual row layout (Seg: counts are
// uniform across requests) cut into 16-row groups: gbf bf16 groups (T0 rows except the new
// token | pad | T1 staging | pad) then gq2 int8 groups (T2).  The groups of all units form
// one flat list; CTA c of the grid (one per SM) takes the groups whose start cost falls in
// [c*Ctot/NC, (c+1)*Ctot/NC) (bf16 group cost 2, int8 group cost 1 ~ their bytes), so every
// CTA streams the same number of bytes and a unit spans the contiguous CTA range c0(u)..c1(u).
//
//   producer warp   walks the CTA's groups as stages of <= NW groups (one unit, one kind),
//                   1-D bulk async copies (cp.async.bulk, SASS UBLKCP) into an NST-deep
//                   shared-memory ring (full/empty mbarriers).  It never waits on the previous
//                   kernel.  Once the ring is primed it requests the rest of its range, and the
//                   same range of the NEXT layer, into L2 (cp.async.bulk.prefetch.L2): HBM
//                   streams layer l+1 while layer l computes, so every layer after the first
//                   reads its rows from L2 and the per-layer dependency tail does not idle HBM.
//   consumer warps  per stage, each owns 16 rows: S^T = K q^T (mma.sync m16n8k16, swap-AB),
//                   online softmax in fp32 (log2 domain, lazy rescale), o^T += V^T p^T.  At a
//                   unit's last stage in this CTA: warps -> CTA partial (m, l, o) in a fixed
//                   order (+ the new-token term if this CTA owns it).  A unit inside one CTA is
//                   written out directly.  Otherwise the CTA owning the unit's first group
//                   merges: for it that unit is its LAST (the unit continues into the next
//                   CTAs, which process it FIRST), so the others have usually published their
//                   partial + release-add (fire and forget) by the time it checks the count;
//                   it combines its own partial (shared memory) with theirs in slot order
//                   (deterministic) and writes o and the per-head (M, 1/L).  No merge kernel,
//                   no cluster, and no round trip in any non-merging epilogue.  (The merger's
//                   wait needs every CTA of the grid resident: kv_tier_init keeps grid <= SMs.)
//   side warp       (1) appends the new token's K/V row of every unit whose last group this
//                   CTA owns (a1) and computes its logits; (2) applies the PREVIOUS launch's
//                   score update (a4) to a flat slice of (unit, token): S += sum_h exp2(z-M)/L
//                   with that launch's exact global (M, L) -- one fp32 add per (step, layer) in
//                   layer order (AMB-14), one writer per entry, off the critical path.
//
// Index arithmetic is 32-bit (kv_tier_init checks that the flat cost space times the grid fits).
#include "decode_common.cuh"

#ifndef KVT_FLAT_TRACE
#define KVT_FLAT_TRACE 0   // 1: per-stage / per-unit timing in the trace (debug builds; costs registers)
#endif

namespace kvt {

constexpr int FLAT_NNEW = 8;     // new-token terms one CTA may own (units per CTA <= 8)
constexpr int FLAT_MAXNP = 40;   // partials per unit (grid capped at 32 CTAs per unit: np <= 34)
constexpr int FLAT_SPOS = 768;   // score-pass positions the side warp prefetches before the PDL wait

struct Flat {
  uint32_t U, gbf, gq2, nu, cu, nce, ctot;
  __device__ __forceinline__ void init(const Seg& sg, int U_, int grid) {
    U = (uint32_t)U_;
    gbf = (uint32_t)max(1, sg.a2 >> 4);
    gq2 = (uint32_t)((sg.n2 + 15) >> 4);
    nu = gbf + gq2;
    cu = 2 * gbf + gq2;
    ctot = U * cu;
    nce = min(min((uint32_t)grid, 32u * U), max(1u, ctot / 2));   // width >= 2: no empty CTA
  }
  __device__ __forceinline__ uint32_t lo(uint32_t c) const { return (c * ctot + nce - 1) / nce; }
  // first linear group (u * nu + k) whose start cost is >= s
  __device__ __forceinline__ uint32_t first(uint32_t s) const {
    const uint32_t u = s / cu, r = s - u * cu;
    const uint32_t k = r <= 2 * gbf ? (r + 1) >> 1 : gbf + (r - 2 * gbf);
    return u * nu + k;
  }
  __device__ __forceinline__ int c0(int u) const { return (int)((uint32_t)u * nce / U); }
  __device__ __forceinline__ int c1(int u) const {
    const uint32_t last = gq2 > 0 ? 2 * gbf + gq2 - 1 : 2 * gbf - 2;
    return (int)(((uint32_t)u * cu + last) * nce / ctot);
  }
  // partial slots of unit u: [pbase, pbase + c1 - c0] for its CTAs, + 1 for the new token
  __device__ __forceinline__ int pbase(int u) const { return c0(u) + 2 * u; }   // disjoint ranges
};

__device__ __forceinline__ void bar_arrive_named(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void red_add_release_gpu(int* p, int x) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;\n" ::"l"(p), "r"(x) : "memory");
}
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int x;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(x) : "l"(p) : "memory");
  return x;
}

template <int D, int NW, int NST>
__global__ void __launch_bounds__((NW + 3) * 32, 1)
    k_decode_flat(const DevView v, const int layer, const __nv_bfloat16* __restrict__ q,
                  const __nv_bfloat16* __restrict__ knew, const __nv_bfloat16* __restrict__ vnew,
                  void* __restrict__ o, const int zpar, const int zprev) {
  // zpar: logits/ML ring slot of this launch (-1: no score update); zprev: slot of the previous
  // launch whose score update is still pending (-1: none)
  constexpr int NCONS = NW * 32;
  constexpr int WPROD = NW, WSIDE = NW + 1, WSIDE2 = NW + 2;   // side warps: new tokens + score pass
  constexpr int TILE = NW * 16;
  constexpr int ROWB = D * 2;
  constexpr int TILEB = TILE * ROWB;
  constexpr int STAGEB = 2 * TILEB;
  constexpr int KS = D / 16;
  constexpr int XS = D + 4;                   // padded row of the reduction slots
  constexpr int NH = NW / 2;                  // reduction slots (two-level warp combine)
  const int c = (int)blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int G = v.G;
  unsigned long long* tr = v.trace ? v.trace + ((size_t)layer * gridDim.x + c) * NTRACE : nullptr;
  if (tr && tid == 0) {
    tr[0] = gtimer();
    for (int x = 1; x < NTRACE; ++x) tr[x] = 0;
  }

  pdl_trigger();                              // the next layer's grid may be scheduled now
  const int cur = v.st->cur;
  Seg sg;
  sg.init(v.cnt[cur], v.st->nn);              // counts are uniform across requests
  Flat F;
  F.init(sg, v.B * v.Hkv, (int)gridDim.x);
  if ((uint32_t)c >= F.nce) return;
  const uint32_t gA = F.first(F.lo(c)), gB = F.first(F.lo(c + 1));
  const int uA = (int)(gA / F.nu), uB = (int)((gB - 1) / F.nu);

  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* ring = smem;                                             // [NST][K tile | V tile]
  unsigned char* t2w = ring + NST * STAGEB;                               // [NW][16][D] bf16 (T2 only)
  unsigned long long* bars =
      reinterpret_cast<unsigned long long*>(t2w + (v.cap2 > 0 ? NW * 16 * ROWB : 0));   // full, empty
  int4* sdesc = reinterpret_cast<int4*>(bars + 2 * NST);                  // [NST] stage descriptors
  float* xsl = reinterpret_cast<float*>(sdesc + NST);                     // [NH][8][XS] warp-combine slots
  float* redm = xsl + NH * 8 * XS;                                        // [NW][8] warp max
  float* redl = redm + 8 * NW;                                            // [NW][8] warp sum
  float* nz = redl + 8 * NW;                                              // [NNEW][8] new-token logits
  float* nvv = nz + 8 * FLAT_NNEW;                                        // [NNEW][D] new-token values
  float* sM = nvv + FLAT_NNEW * D;                                        // [8] CTA / unit max per head
  float* sL = sM + 8;                                                     // [8] sum (or 1/sum)
  float* smm = sL + 8;                                                    // [MAXNP][8] merge: m -> factor
  float* sml = smm + FLAT_MAXNP * 8;                                      // [MAXNP][8] merge: l
  int* spos = reinterpret_cast<int*>(sml + FLAT_MAXNP * 8);               // [SPOS] score-pass positions
  float* rml = reinterpret_cast<float*>(spos + FLAT_SPOS);                // [16] pre-merged (M, L) of the rest
  float* rfac = rml + 16;                                                 // [MAXNP][8] its per-partial factors
  float* ro = rfac + FLAT_MAXNP * 8;                                      // [8 * D] pre-merged o (unnormalised)

  const int sb = v.st->scur;
  const uint32_t ring_s = smem_u32(ring);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + NST);
  if (tid == 0) {
    for (int s2 = 0; s2 < NST; ++s2) {
      mbar_init(full0 + 8 * s2, 1);
      mbar_init(empty0 + 8 * s2, NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // units whose new token (last virtual row) this CTA owns: those whose last group is here
  const int unew0 = (F.c1(uA) == c) ? uA : uA + 1;
  const int unew1 = (F.c1(uB) == c) ? uB : uB - 1;
  const int nnew = max(0, unew1 - unew0 + 1);   // <= FLAT_NNEW (grid sized at init)
  // the unit this CTA merges (its last unit, when it starts here and continues past it)
  const int umerge = (F.c0(uB) == c && F.c1(uB) > c) ? uB : -1;

  if (w == WPROD) {
    // ============================ producer ============================
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      // request groups [g0, g1) of layer lp into L2 (whole runs of one kind of one unit)
      auto l2_range = [&](int lp, uint32_t g0, uint32_t g1, long long budget) {
        for (uint32_t gp = g0; gp < g1 && budget > 0;) {
          const int u = (int)(gp / F.nu);
          const uint32_t k0 = gp - (uint32_t)u * F.nu;
          const bool t2 = k0 >= F.gbf;
          const uint32_t run_end = min(g1, (uint32_t)u * F.nu + (t2 ? F.nu : F.gbf));
          const int ngr = (int)(run_end - gp);
          const int b = u / v.Hkv, g = u - b * v.Hkv;
          const size_t grp = grp_of(v, lp, b, g);
          if (!t2) {
            const int ts = 16 * (int)k0, te = ts + 16 * ngr;   // virtual rows [ts, te)
            const __nv_bfloat16* K0 = v.k0[sb] + grp * v.cap0 * D;
            const __nv_bfloat16* V0 = v.v0[sb] + grp * v.cap0 * D;
            const __nv_bfloat16* K1 = v.k1[sb] + grp * v.cap1 * D;
            const __nv_bfloat16* V1 = v.v1[sb] + grp * v.cap1 * D;
            const int a1e = min(te, sg.a1);
            if (a1e > ts) {
              bulk_prefetch_l2(K0 + (size_t)ts * D, (a1e - ts) * ROWB);
              bulk_prefetch_l2(V0 + (size_t)ts * D, (a1e - ts) * ROWB);
            }
            const int b0 = max(ts, sg.a1);
            if (te > b0 && !v.stream_mode) {
              bulk_prefetch_l2(K1 + (size_t)(b0 - sg.a1) * D, (te - b0) * ROWB);
              bulk_prefetch_l2(V1 + (size_t)(b0 - sg.a1) * D, (te - b0) * ROWB);
            }
            budget -= (long long)(te - ts) * 2 * ROWB;
          } else {
            const int j0 = 16 * (int)(k0 - F.gbf), nr = 16 * ngr;
            bulk_prefetch_l2(v.c2k[sb] + (grp * v.cap2 + j0) * D, nr * D);
            bulk_prefetch_l2(v.c2v[sb] + (grp * v.cap2 + j0) * D, nr * D);
            budget -= (long long)nr * 2 * D;
          }
          gp = run_end;
        }
      };
      bool pf_done = v.l2pf_bytes <= 0;
      uint32_t gcur = gA;
#if KVT_FLAT_TRACE
      unsigned long long pwait = 0;
#endif
      for (int i = 0;; ++i) {
        const int s2 = i % NST;
        if (!pf_done && (i == NST || gcur >= gB)) {      // ring primed: the rest of this layer, then
          pf_done = true;                                // this CTA's range of the next layer
          l2_range(layer, gcur, gB, v.l2pf_bytes);
          if (layer + 1 < v.L) l2_range(layer + 1, gA, gB, v.l2pf_bytes);
        }
#if KVT_FLAT_TRACE
        const unsigned long long pw0 = gtimer();
#endif
        if (i >= NST) {
          if (v.spin_hint) mbar_wait_hint(empty0 + 8 * s2, ((i / NST) - 1) & 1, (uint32_t)v.spin_hint);
          else mbar_wait(empty0 + 8 * s2, ((i / NST) - 1) & 1);
        }
#if KVT_FLAT_TRACE
        if (i >= NST) pwait += gtimer() - pw0;
#endif
        // flow control: at most v.inflight stages requested but not landed.  Bytes in flight set
        // the queueing delay every other load of the grid sees (Little: in flight / bandwidth);
        // landed-but-unconsumed stages may still fill the rest of the ring.
        if (v.inflight > 0 && i >= v.inflight) {
          const int j = i - v.inflight;
          mbar_wait(full0 + 8 * (j % NST), (j / NST) & 1);
        }
        const uint32_t full = full0 + 8 * s2, dst = ring_s + s2 * STAGEB;
        if (gcur >= gB) {
#if KVT_FLAT_TRACE
          if (tr) { tr[16] = pwait; tr[23] = gtimer(); }
#endif
          sdesc[s2] = make_int4(-1, 0, 0, 0);
          mbar_arrive(full);                  // sentinel stage (no data)
          break;
        }
        const int u = (int)(gcur / F.nu);
        const int k0 = (int)(gcur - (uint32_t)u * F.nu);
        const bool t2 = k0 >= (int)F.gbf;
        const uint32_t uend = (uint32_t)u * F.nu + F.nu;
        const uint32_t lim = min(gB, (uint32_t)u * F.nu + (t2 ? F.nu : F.gbf));
        const int ng = (int)min((uint32_t)NW, lim - gcur);
        const bool last = gcur + ng == min(gB, uend);
        sdesc[s2] = make_int4(u, k0, ng | (t2 ? 256 : 0) | (last ? 512 : 0), 0);
        const int b = u / v.Hkv, g = u - b * v.Hkv;
        const size_t grp = grp_of(v, layer, b, g);
        const int nrows = 16 * ng;
        if (!t2) {
          const __nv_bfloat16* K0 = v.k0[sb] + grp * v.cap0 * D;
          const __nv_bfloat16* V0 = v.v0[sb] + grp * v.cap0 * D;
          const __nv_bfloat16 *K1, *V1;
          if (v.stream_mode) {
            const size_t sgi = ((size_t)(layer & 1) * v.B + b) * v.Hkv + g;
            K1 = v.k1[0] + sgi * v.cap1 * D;
            V1 = v.v1[0] + sgi * v.cap1 * D;
          } else {
            K1 = v.k1[sb] + grp * v.cap1 * D;
            V1 = v.v1[sb] + grp * v.cap1 * D;
          }
          const int ts = 16 * k0;
          mbar_expect_tx(full, 2 * nrows * ROWB);
          if (ts < sg.a1) {                   // a1 is a multiple of 16: the T1 part starts at T1 row 0
            const int n0r = min(nrows, sg.a1 - ts);
            bulk_g2s_ef(dst, K0 + (size_t)ts * D, n0r * ROWB, full, pol);
            bulk_g2s_ef(dst + TILEB, V0 + (size_t)ts * D, n0r * ROWB, full, pol);
            if (n0r < nrows) {
              bulk_g2s_ef(dst + n0r * ROWB, K1, (nrows - n0r) * ROWB, full, pol);
              bulk_g2s_ef(dst + TILEB + n0r * ROWB, V1, (nrows - n0r) * ROWB, full, pol);
            }
          } else {
            bulk_g2s_ef(dst, K1 + (size_t)(ts - sg.a1) * D, nrows * ROWB, full, pol);
            bulk_g2s_ef(dst + TILEB, V1 + (size_t)(ts - sg.a1) * D, nrows * ROWB, full, pol);
          }
        } else {                              // T2: int8 codes + fp32 scales
          const int j0 = 16 * (k0 - (int)F.gbf);
          const int8_t* CK = v.c2k[sb] + (grp * v.cap2 + j0) * D;
          const int8_t* CV = v.c2v[sb] + (grp * v.cap2 + j0) * D;
          const float* SK = v.s2k[sb] + grp * v.cap2 + j0;
          const float* SV = v.s2v[sb] + grp * v.cap2 + j0;
          mbar_expect_tx(full, 2 * (nrows * D + nrows * 4));
          bulk_g2s(dst, CK, nrows * D, full);
          bulk_g2s(dst + TILE * D, SK, nrows * 4, full);
          bulk_g2s(dst + TILEB, CV, nrows * D, full);
          bulk_g2s(dst + TILEB + TILE * D, SV, nrows * 4, full);
        }
        gcur += ng;
      }
    }
    return;
  }

  // score-pass slice of the side warp: (unit, virtual token) entries [si0, si1) of the previous
  // launch.  Positions come from the index lists (not written by the previous kernel), so they
  // are fetched before the PDL wait.
  const uint32_t nvirt = (uint32_t)sg.nvirt;
  const uint32_t sE = F.U * nvirt;
  const uint32_t sc0 = (uint32_t)(((unsigned long long)c * sE) / F.nce);
  const uint32_t sc1 = (uint32_t)(((unsigned long long)(c + 1) * sE) / F.nce);
  const uint32_t si0 = sc0, si1 = sc1;                    // side warp 1's score slice
  int* wpos = spos;
  if (w == WSIDE && zprev >= 0) {
    const int np0 = (int)min((uint32_t)FLAT_SPOS, si1 - si0);
    for (int j = lane; j < np0; j += 32) {
      const uint32_t i = si0 + j;
      const int u = (int)(i / nvirt), t = (int)(i - (uint32_t)u * nvirt);
      wpos[j] = sg.valid(t) ? sg.pos(v, cur, u / v.Hkv, t) : -1;
    }
    __syncwarp();
  }

  // ---------------------------------------------------------------- dependent inputs
  pdl_wait();
  if (tr && tid == 0) tr[1] = gtimer();
  const float sl2 = (float)(1.4426950408889634 / __dsqrt_rn((double)D));   // log2(e)/sqrt(d)

  if (w == WSIDE2) {
    // ============================ side warp 2: pre-merge ============================
    // The other CTAs of the unit this CTA merges process it FIRST and the new-token partial is
    // published right after the PDL wait, so while this CTA's consumers stream, this warp
    // waits for those npt - 1 partials and combines them in slot order (deterministic) into
    // (rml, ro); the consumers' epilogue then only folds in their own partial (slot 0).
    if (umerge >= 0) {
      const int npt = F.c1(umerge) - F.c0(umerge) + 2;   // CTAs + the new token
      while (ld_acquire_gpu(v.unit_ctr + umerge) < npt - 1) __nanosleep(64);
      __syncwarp();
      if (lane == 0) v.unit_ctr[umerge] = 0;   // every add has landed; next launch after this grid
      const float* P = v.part + (size_t)F.pbase(umerge) * v.part_stride;
      for (int i = lane; i < (npt - 1) * 8; i += 32) {
        const int p = 1 + (i >> 3), h = i & 7;
        rfac[p * 8 + h] = __ldcg(P + (size_t)p * v.part_stride + h);
        sml[p * 8 + h] = __ldcg(P + (size_t)p * v.part_stride + 8 + h);
      }
      __syncwarp();
      if (lane < 8) {
        float M = -INFINITY;
        for (int p = 1; p < npt; ++p) M = fmaxf(M, rfac[p * 8 + lane]);
        float Ls = 0.f;
        for (int p = 1; p < npt; ++p) {
          const float m = rfac[p * 8 + lane];
          const float f = m == -INFINITY ? 0.f : ex2_ftz(m - M);
          rfac[p * 8 + lane] = f;
          Ls += f * sml[p * 8 + lane];
        }
        rml[lane] = M;
        rml[8 + lane] = Ls;
      }
      __syncwarp();
      const int tot4 = G * D / 4;
      constexpr int NE = (8 * D / 4 + 31) / 32, MB = 3;   // float4s per lane, partials per batch
      float4 acc[NE];
#pragma unroll
      for (int k = 0; k < NE; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int p0 = 1; p0 < npt; p0 += MB) {
        float4 x[MB][NE];
#pragma unroll
        for (int p = 0; p < MB; ++p)
#pragma unroll
          for (int k = 0; k < NE; ++k)
            if (p0 + p < npt && lane + 32 * k < tot4)
              x[p][k] = __ldcg(reinterpret_cast<const float4*>(P + (size_t)(p0 + p) * v.part_stride + 16) + lane + 32 * k);
#pragma unroll
        for (int p = 0; p < MB; ++p)
#pragma unroll
          for (int k = 0; k < NE; ++k)
            if (p0 + p < npt && lane + 32 * k < tot4) {
              const float f = rfac[(p0 + p) * 8 + (4 * (lane + 32 * k)) / D];
              acc[k].x += f * x[p][k].x;
              acc[k].y += f * x[p][k].y;
              acc[k].z += f * x[p][k].z;
              acc[k].w += f * x[p][k].w;
            }
      }
#pragma unroll
      for (int k = 0; k < NE; ++k)
        if (lane + 32 * k < tot4) reinterpret_cast<float4*>(ro)[lane + 32 * k] = acc[k];
      __syncwarp();
      bar_arrive_named(3, NCONS + 32);        // pre-merged remainder ready
    }
    if (tr && lane == 0) tr[6] = gtimer();
    return;
  }
  if (w == WSIDE) {
    // ============================ side warp 1 ============================
    // (1) side warp 1, new tokens: append the K/V row to T0 row n0o (swizzled); the token's
    //     attention term (m = z, l = 1, o = v) is published as the unit's last partial (slot
    //     c1 - c0 + 1) when the unit spans several CTAs, else handed to this CTA's consumers;
    //     logits also go to zbuf.
#if KVT_FLAT_TRACE
    if (tr && w == WSIDE) {                   // probe: one dependent L2/HBM round trip now
      const unsigned long long p0 = gtimer();
      const int probe = __ldcg(&v.st->n);
      const unsigned long long p1 = gtimer();
      if (lane == 0) { tr[11] = p1 - p0 + (probe < -1000000 ? 1 : 0); }
    }
    unsigned long long tn0 = 0, tn1 = 0, tn2 = 0;
#endif
    for (int j = 0; j < nnew; ++j) {
#if KVT_FLAT_TRACE
      if (j == 0) tn0 = gtimer();
#endif
      const int u = unew0 + j, b = u / v.Hkv, g = u - b * v.Hkv;
      const size_t grp = grp_of(v, layer, b, g);
      uint16_t* K0w = reinterpret_cast<uint16_t*>(v.k0[sb]) + (grp * v.cap0 + sg.n0o) * D;
      uint16_t* V0w = reinterpret_cast<uint16_t*>(v.v0[sb]) + (grp * v.cap0 + sg.n0o) * D;
      const uint16_t* kin = knew ? reinterpret_cast<const uint16_t*>(knew) + ((size_t)b * v.Hkv + g) * D : nullptr;
      const uint16_t* vin = vnew ? reinterpret_cast<const uint16_t*>(vnew) + ((size_t)b * v.Hkv + g) * D : nullptr;
      constexpr int EL = D / 32;
      uint16_t kb[EL], vb[EL], qb[8][EL];
      const uint16_t* qbase = reinterpret_cast<const uint16_t*>(q) + ((size_t)b * v.Hq + g * G) * D;
#pragma unroll
      for (int k = 0; k < EL; ++k) {
        const int e = lane + 32 * k;
        const int se = swz_off(sg.n0o, e);
        kb[k] = kin ? kin[e] : K0w[se];
        vb[k] = vin ? vin[e] : V0w[se];
#pragma unroll
        for (int h = 0; h < 8; ++h) qb[h][k] = h < G ? qbase[(size_t)h * D + e] : (uint16_t)0;
      }
      float dot[8];
#if KVT_FLAT_TRACE
      if (j == 0) { tn1 = gtimer(); if (bf16_bits_to_f(kb[0]) == 12345.f && bf16_bits_to_f(qb[0][0]) == 1.f) tn1 += 1; }
#endif
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        dot[h] = 0.f;
#pragma unroll
        for (int k = 0; k < EL; ++k) dot[h] += bf16_bits_to_f(qb[h][k]) * bf16_bits_to_f(kb[k]);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1)
#pragma unroll
        for (int h = 0; h < 8; ++h) dot[h] += __shfl_xor_sync(0xffffffffu, dot[h], off);
#pragma unroll
      for (int k = 0; k < EL; ++k) {
        const int e = lane + 32 * k;
        const int se = swz_off(sg.n0o, e);
        if (kin) K0w[se] = kb[k];
        if (vin) V0w[se] = vb[k];
        nvv[j * D + e] = bf16_bits_to_f(vb[k]);
      }
      float z = -INFINITY;
#pragma unroll
      for (int h = 0; h < 8; ++h) z = (lane == h && h < G) ? dot[h] * sl2 : z;
      if (lane < 8) {
        nz[j * 8 + lane] = z;
        if (zpar >= 0 && lane < G)
          v.zbuf[(((size_t)zpar * v.B * v.Hkv + u) * v.zrows + sg.a3) * 8 + lane] = z;
      }
#if KVT_FLAT_TRACE
      if (j == 0) tn2 = gtimer();
#endif
      if (F.c0(u) != c) {                     // unit spans CTAs: the term is a partial of its own
        float* part = v.part + (size_t)(F.pbase(u) + F.c1(u) - F.c0(u) + 1) * v.part_stride;
        if (lane < 8) {
          part[lane] = z;
          part[8 + lane] = lane < G ? 1.f : 0.f;
        }
#pragma unroll
        for (int k = 0; k < EL; ++k)
          for (int h = 0; h < G; ++h) part[16 + h * D + lane + 32 * k] = bf16_bits_to_f(vb[k]);
        __syncwarp();
        if (lane == 0) red_add_release_gpu(v.unit_ctr + u, 1);
      }
    }
    if (nnew > 0) bar_arrive_named(2, NCONS + 32);   // new-token terms ready
    if (tr && lane == 0) tr[4] = gtimer();
#if KVT_FLAT_TRACE
    if (tr && lane == 0 && nnew > 0) { tr[12] = tn1 - tn0; tr[13] = tn2 - tn1; tr[14] = tr[4] - tn2; }
#endif
    // (2) the previous launch's score update over this CTA's flat slice of (unit, token):
    //     S_part[u][pos] += sum_h exp2(z_h - M_h) / L_h, all loads of a batch at once
    if (zprev >= 0) {
      const float* zb = v.zbuf + (size_t)zprev * v.B * v.Hkv * v.zrows * 8;
      const float* mlb = v.ml + (size_t)zprev * v.B * v.Hkv * 16;
      constexpr int SB = 8;
      bool bad = false;
      int mu = -1;                            // unit whose (M, 1/L) sit in mM / mI
      float mM[8], mI[8];
      for (uint32_t base = si0 + lane; base < si1; base += 32 * SB) {
        int pos[SB], uu[SB], tt[SB];
#pragma unroll
        for (int k = 0; k < SB; ++k) {
          const uint32_t i = base + 32 * k;
          pos[k] = -1;
          uu[k] = 0;
          tt[k] = 0;
          if (i < si1) {
            const int u = (int)(i / nvirt), t = (int)(i - (uint32_t)u * nvirt);
            uu[k] = u;
            tt[k] = t;
            const uint32_t j = i - si0;
            pos[k] = j < (uint32_t)FLAT_SPOS ? wpos[j] : (sg.valid(t) ? sg.pos(v, cur, u / v.Hkv, t) : -1);
          }
        }
        float sv[SB];
        float4 za[SB], zc[SB];
#pragma unroll
        for (int k = 0; k < SB; ++k) {
          if (pos[k] >= 0) {
            sv[k] = v.S[(size_t)uu[k] * v.Nmax + pos[k]];
            const float* z = zb + ((size_t)uu[k] * v.zrows + tt[k]) * 8;
            za[k] = *reinterpret_cast<const float4*>(z);
            zc[k] = *reinterpret_cast<const float4*>(z + 4);
          }
        }
#pragma unroll
        for (int k = 0; k < SB; ++k) {
          if (pos[k] < 0) continue;
          if (uu[k] != mu) {
            mu = uu[k];
            const float4* ml4 = reinterpret_cast<const float4*>(mlb + (size_t)mu * 16);
            const float4 a0 = ml4[0], a1 = ml4[1], a2 = ml4[2], a3 = ml4[3];
            mM[0] = a0.x; mM[1] = a0.y; mM[2] = a0.z; mM[3] = a0.w;
            mM[4] = a1.x; mM[5] = a1.y; mM[6] = a1.z; mM[7] = a1.w;
            mI[0] = a2.x; mI[1] = a2.y; mI[2] = a2.z; mI[3] = a2.w;
            mI[4] = a3.x; mI[5] = a3.y; mI[6] = a3.z; mI[7] = a3.w;
          }
          const float zz[8] = {za[k].x, za[k].y, za[k].z, za[k].w, zc[k].x, zc[k].y, zc[k].z, zc[k].w};
          float inc = 0.f;
#pragma unroll
          for (int h = 0; h < 8; ++h)
            if (h < G) inc += ex2_ftz(zz[h] - mM[h]) * mI[h];
          v.S[(size_t)uu[k] * v.Nmax + pos[k]] = sv[k] + inc;
          bad |= !isfinite(inc);
        }
      }
      if (bad) atomicOr(&v.st->err, 1);
    }
    if (tr && lane == 0) tr[5] = gtimer();
    return;
  }

  // ============================ consumers ============================
  float mxa = -INFINITY, mxb = -INFINITY;   // per-warp running max, heads 2tq, 2tq+1 (log2)
  float la = 0.f, lb = 0.f;                 // per-thread partial sums
  float oacc[KS][4];
  uint32_t qf[KS][2], qn[KS][2];            // q fragments of the current / the next unit
  auto load_q = [&](int u, uint32_t (&dst)[KS][2]) {
    const int b = u / v.Hkv, g = u - b * v.Hkv;
    const __nv_bfloat16* qh = q + ((size_t)b * v.Hq + g * G + gq) * D;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      dst[ks][0] = gq < G ? *reinterpret_cast<const uint32_t*>(qh + ks * 16 + 2 * tq) : 0u;
      dst[ks][1] = gq < G ? *reinterpret_cast<const uint32_t*>(qh + ks * 16 + 8 + 2 * tq) : 0u;
    }
  };
  // both loads right after the PDL wait: one round trip for the CTA's first two units
  load_q(uA, qf);
  int qf_u = uA, qn_u = -1;
  if (uB > uA) {
    load_q(uA + 1, qn);
    qn_u = uA + 1;
  }
  int ucur = -1;
  float* zrow = nullptr;
  bool new_ready = false;
#if KVT_FLAT_TRACE
  unsigned long long cwait = 0, cbusy = 0, tw1 = 0, tf_sum = 0, n_units = 0;
#endif

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
  const int mi = lane >> 3, ii = lane & 7;
  auto qk = [&](uint32_t sK, int rowbase, float* acc) {
    constexpr int NCH = KS >= 4 ? 4 : KS;
    float ch[NCH][4];
#pragma unroll
    for (int cc = 0; cc < NCH; ++cc) ch[cc][0] = ch[cc][1] = ch[cc][2] = ch[cc][3] = 0.f;
    const int row = rowbase + ii + ((mi & 1) << 3);
    uint32_t af[KS][4];                     // every fragment load first: one shared-memory latency
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
      ldsm_x4(af[ks][0], af[ks][1], af[ks][2], af[ks][3], sK + row * ROWB + (((2 * ks + (mi >> 1)) ^ (row & 7)) << 4));
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
      mma16816(ch[ks % NCH], af[ks][0], af[ks][1], af[ks][2], af[ks][3], qf[ks][0], qf[ks][1]);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float x = ch[0][j];
#pragma unroll
      for (int cc = 1; cc < NCH; ++cc) x += ch[cc][j];
      acc[j] += x;
    }
  };
  auto pv = [&](uint32_t sV, int rowbase, float p00, float p01, float p10, float p11) {
    uint32_t h0, l0, h1, l1;                  // p = hi + lo (split_bf16x2)
    split_bf16x2(p00, p01, h0, l0);
    split_bf16x2(p10, p11, h1, l1);
    const uint32_t b0 = movm_t(h0), b1 = movm_t(h1), c0 = movm_t(l0), c1 = movm_t(l1);
    const int row = rowbase + ii + ((mi >> 1) << 3);
    uint32_t af[KS][4];
#pragma unroll
    for (int mt = 0; mt < KS; ++mt)
      ldsm_x4_t(af[mt][0], af[mt][1], af[mt][2], af[mt][3], sV + row * ROWB + (((2 * mt + (mi & 1)) ^ (row & 7)) << 4));
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
      *reinterpret_cast<uint4*>(scr + row * ROWB + (((2 * j) ^ (row & 7)) << 4)) = lo;
      *reinterpret_cast<uint4*>(scr + row * ROWB + (((2 * j + 1) ^ (row & 7)) << 4)) = hi;
    }
    __syncwarp();
  };

  // end of unit u's groups in this CTA: warps -> CTA partial (fixed order, + new token), publish;
  // the CTA completing the unit's count merges every partial of the unit in slot order
  auto finish_unit = [&](int u) {
#if KVT_FLAT_TRACE
    const unsigned long long tf0 = tr ? gtimer() : 0ull;
#endif
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      la += __shfl_xor_sync(0xffffffffu, la, off);
      lb += __shfl_xor_sync(0xffffffffu, lb, off);
    }
    const int jn = u - unew0;                 // new-token term index (if owned here and the
    const bool hasnew = jn >= 0 && jn < nnew && F.c0(u) == c;   // unit lies inside this CTA)
    if (hasnew && !new_ready) {
      named_sync(2, NCONS + 32);
      new_ready = true;
    }
    if (lane < 4) {
      redm[w * 8 + 2 * lane] = mxa;
      redm[w * 8 + 2 * lane + 1] = mxb;
      redl[w * 8 + 2 * lane] = la;
      redl[w * 8 + 2 * lane + 1] = lb;
    }
    named_sync(1, NCONS);
    // per-head CTA max over the warps (and the new token): heads 2tq, 2tq+1 for this thread
    float Ma = hasnew ? nz[jn * 8 + 2 * tq] : -INFINITY, Mb = hasnew ? nz[jn * 8 + 2 * tq + 1] : -INFINITY;
#pragma unroll
    for (int x = 0; x < NW; ++x) {
      Ma = fmaxf(Ma, redm[x * 8 + 2 * tq]);
      Mb = fmaxf(Mb, redm[x * 8 + 2 * tq + 1]);
    }
    const float fa = mxa == -INFINITY ? 0.f : ex2_ftz(mxa - Ma), fb = mxb == -INFINITY ? 0.f : ex2_ftz(mxb - Mb);
    // two-level combine (fixed order): slot s = o_s + o_{s+NH} for s < NH, then sum of slots
    float* o0 = xsl + (size_t)(w % NH) * 8 * XS + (2 * tq) * XS + gq;
    if (w >= NH) {
#pragma unroll
      for (int mt = 0; mt < KS; ++mt) {
        o0[mt * 16] = fa * oacc[mt][0];
        o0[XS + mt * 16] = fb * oacc[mt][1];
        o0[mt * 16 + 8] = fa * oacc[mt][2];
        o0[XS + mt * 16 + 8] = fb * oacc[mt][3];
      }
    }
    named_sync(1, NCONS);
    if (w < NH) {
      float t[KS][4];
#pragma unroll
      for (int mt = 0; mt < KS; ++mt) {
        t[mt][0] = o0[mt * 16];
        t[mt][1] = o0[XS + mt * 16];
        t[mt][2] = o0[mt * 16 + 8];
        t[mt][3] = o0[XS + mt * 16 + 8];
      }
#pragma unroll
      for (int mt = 0; mt < KS; ++mt) {
        o0[mt * 16] = fa * oacc[mt][0] + t[mt][0];
        o0[XS + mt * 16] = fb * oacc[mt][1] + t[mt][1];
        o0[mt * 16 + 8] = fa * oacc[mt][2] + t[mt][2];
        o0[XS + mt * 16 + 8] = fb * oacc[mt][3] + t[mt][3];
      }
    }
    // per-head CTA (M, L) incl. the new token -> sM / sL
    const int b = u / v.Hkv, g = u - b * v.Hkv;
    const int np = F.c1(u) - F.c0(u) + 1;
    const int tot = G * D;
    if (tid < 8) {
      const int h = tid;
      float M = hasnew ? nz[jn * 8 + h] : -INFINITY;
      for (int x = 0; x < NW; ++x) M = fmaxf(M, redm[x * 8 + h]);
      float Ls = 0.f;
      for (int x = 0; x < NW; ++x) {
        const float m = redm[x * 8 + h];
        Ls += (m == -INFINITY ? 0.f : ex2_ftz(m - M)) * redl[x * 8 + h];
      }
      if (hasnew && h < G) Ls += ex2_ftz(nz[jn * 8 + h] - M);
      sM[h] = h < G ? M : -INFINITY;
      sL[h] = h < G ? Ls : 0.f;
    }
    named_sync(1, NCONS);
    auto put_o = [&](int e, float val) {
      const int h = e / D, dd = e - h * D;
      const size_t oi = ((size_t)b * v.Hq + g * G + h) * D + dd;
      if (v.out_fp32) reinterpret_cast<float*>(o)[oi] = val;
      else reinterpret_cast<__nv_bfloat16*>(o)[oi] = __float2bfloat16_rn(val);
    };
    auto cta_o = [&](int e) {                // this CTA's o (+ new token), unnormalised
      const int h = e / D, dd = e - h * D;
      float a = xsl[h * XS + dd];
#pragma unroll
      for (int s = 1; s < NH; ++s) a += xsl[(size_t)s * 8 * XS + h * XS + dd];
      if (hasnew) a += ex2_ftz(nz[jn * 8 + h] - sM[h]) * nvv[jn * D + dd];
      return a;
    };
    if (np == 1) {                            // the whole unit is in this CTA: write o directly
      for (int e = tid; e < tot; e += NCONS) put_o(e, cta_o(e) * (1.0f / sL[e / D]));
      if (tid < G && zpar >= 0) {
        float* ml = v.ml + ((size_t)zpar * v.B * v.Hkv + u) * 16;
        ml[tid] = sM[tid];
        ml[8 + tid] = 1.0f / sL[tid];
      }
    } else if (F.c0(u) != c) {                // publish slot c - c0 and move on (no round trip)
      float* part = v.part + (size_t)(F.pbase(u) + c - F.c0(u)) * v.part_stride;
      if (tid < 16) part[tid] = tid < 8 ? sM[tid] : sL[tid - 8];
      for (int e = tid; e < tot; e += NCONS) part[16 + e] = cta_o(e);
      named_sync(1, NCONS);                   // every partial store precedes the release below
      if (tid == 0) red_add_release_gpu(v.unit_ctr + u, 1);
    } else {
      // merger: fold this CTA's partial (slot 0) into the other partials' pre-merged remainder
      named_sync(3, NCONS + 32);
      if (tid < 8) {
        const int h = tid;
        const float M = fmaxf(sM[h], rml[h]);
        const float f0 = sM[h] == -INFINITY ? 0.f : ex2_ftz(sM[h] - M);
        const float f1 = rml[h] == -INFINITY ? 0.f : ex2_ftz(rml[h] - M);
        const float Ls = f0 * sL[h] + f1 * rml[8 + h];
        smm[h] = f0;
        smm[8 + h] = f1;
        sml[h] = 1.0f / Ls;
        if (h < G && zpar >= 0) {
          float* ml = v.ml + ((size_t)zpar * v.B * v.Hkv + u) * 16;
          ml[h] = M;
          ml[8 + h] = 1.0f / Ls;
        }
      }
      named_sync(1, NCONS);
      for (int e = tid; e < tot; e += NCONS) {
        const int h = e / D;
        put_o(e, (smm[h] * cta_o(e) + smm[8 + h] * ro[e]) * sml[h]);
      }
    }
    named_sync(1, NCONS);                     // slots / red* free for the next unit
#if KVT_FLAT_TRACE
    if (tr) {
      tf_sum += gtimer() - tf0;
      n_units += 1;
    }
#endif
  };

  for (int i = 0;; ++i) {
    const int s2 = i % NST;
#if KVT_FLAT_TRACE
    const unsigned long long tw0 = gtimer();
    if (i > 0) cbusy += tw0 - tw1;
#endif
    if (v.spin_hint) mbar_wait_hint(full0 + 8 * s2, (i / NST) & 1, (uint32_t)v.spin_hint);
    else mbar_wait(full0 + 8 * s2, (i / NST) & 1);
#if KVT_FLAT_TRACE
    tw1 = gtimer();
    cwait += tw1 - tw0;
#endif
    const int4 dsc = sdesc[s2];
    if (dsc.x < 0) break;
    if (tr && tid == 0 && i == 0) tr[2] = gtimer();
    const int u = dsc.x, k0 = dsc.y, ng = dsc.z & 255;
    const bool t2 = (dsc.z & 256) != 0, last = (dsc.z & 512) != 0;
    if (u != ucur) {                          // first stage of a unit: its q and fresh state
      ucur = u;
      if (u != qf_u) {
        if (u == qn_u) {
#pragma unroll
          for (int ks = 0; ks < KS; ++ks) {
            qf[ks][0] = qn[ks][0];
            qf[ks][1] = qn[ks][1];
          }
        } else {
          load_q(u, qf);
        }
        qf_u = u;
      }
#pragma unroll
      for (int mt = 0; mt < KS; ++mt) oacc[mt][0] = oacc[mt][1] = oacc[mt][2] = oacc[mt][3] = 0.f;
      mxa = mxb = -INFINITY;
      la = lb = 0.f;
      zrow = zpar >= 0 ? v.zbuf + ((size_t)zpar * v.B * v.Hkv + u) * v.zrows * 8 : nullptr;
    }
    const uint32_t sK = ring_s + s2 * STAGEB, sV = sK + TILEB;
    const bool wact = w < ng;
    const int tv0 = t2 ? sg.a2 + 16 * (k0 - (int)F.gbf) : 16 * k0;
    const int r0 = w * 16 + gq, r1 = r0 + 8;
    const int t0 = tv0 + r0, t1 = tv0 + r1;
    const bool v0 = wact && (t2 ? (t0 - sg.a2 < sg.n2) : sg.bf16_valid(t0));
    const bool v1 = wact && (t2 ? (t1 - sg.a2 < sg.n2) : sg.bf16_valid(t1));
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
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * s2);
    if (last) finish_unit(u);
  }
  if (tr && tid == 0) tr[3] = gtimer();
#if KVT_FLAT_TRACE
  if (tr && tid == 0) { tr[9] = tf_sum; tr[10] = n_units; tr[21] = cwait; tr[22] = cbusy; }
#endif
}

// ----------------------------------------------------------------------------------- host side
struct FVariant { int nw, nst; };
static constexpr FVariant kFVariants[] = {{8, 3}, {8, 2}, {4, 3}, {4, 6}, {8, 1}};
constexpr int kNumFVariants = sizeof(kFVariants) / sizeof(kFVariants[0]);

size_t flat_smem_bytes(const DevView& v) {
  const FVariant vr = kFVariants[v.fvariant];
  const int tile = 16 * vr.nw;
  size_t b = (size_t)vr.nst * 2 * tile * v.D * 2;                 // ring
  if (v.cap2 > 0) b += (size_t)vr.nw * 16 * v.D * 2;              // T2 scratch
  b += (size_t)2 * vr.nst * 8 + (size_t)vr.nst * 16;              // barriers, descriptors
  b += (size_t)(vr.nw / 2) * 8 * (v.D + 4) * 4 + (size_t)2 * 8 * vr.nw * 4;   // combine slots, warp (m, l)
  b += (size_t)FLAT_NNEW * (8 + v.D) * 4 + 16 * 4;                // new tokens, sM, sL
  b += (size_t)2 * FLAT_MAXNP * 8 * 4 + 16;                        // merge (m, l), flag
  b += (size_t)FLAT_SPOS * 4;                                      // score-pass positions
  b += (size_t)(16 + FLAT_MAXNP * 8 + 8 * v.D) * 4;                // merger's pre-merged remainder
  return b;
}

#define KVT_FVARIANTS(X, D) X(D, 8, 3) X(D, 8, 2) X(D, 4, 3) X(D, 4, 6) X(D, 8, 1)

cudaError_t flat_configure(const DevView& v) {
  if (v.fvariant < 0 || v.fvariant >= kNumFVariants) return cudaErrorInvalidValue;
  const FVariant vr = kFVariants[v.fvariant];
#define KVT_FCONF(DD, NWW, NSS)                                                                   \
  if (v.D == DD && vr.nw == NWW && vr.nst == NSS)                                                 \
    return cudaFuncSetAttribute(k_decode_flat<DD, NWW, NSS>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                (int)flat_smem_bytes(v));
  KVT_FVARIANTS(KVT_FCONF, 128)
  KVT_FVARIANTS(KVT_FCONF, 64)
#undef KVT_FCONF
  return cudaErrorInvalidValue;
}

int flat_num_variants() { return kNumFVariants; }

cudaError_t launch_decode_flat(const DevView& v, int layer, const void* q, const void* knew, const void* vnew,
                               void* o, int zpar, int zprev, int pdl, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(v.nc, 1, 1);
  cfg.dynamicSmemBytes = flat_smem_bytes(v);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (v.hot_bytes > 0) {
    at[na].id = cudaLaunchAttributeAccessPolicyWindow;
    at[na].val.accessPolicyWindow.base_ptr = v.hot_base;
    at[na].val.accessPolicyWindow.num_bytes = v.hot_bytes;
    at[na].val.accessPolicyWindow.hitRatio = v.hot_hit;
    at[na].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    at[na].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    ++na;
  }
  if (pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  const FVariant vr = kFVariants[v.fvariant];
  const __nv_bfloat16* qb = reinterpret_cast<const __nv_bfloat16*>(q);
  const __nv_bfloat16* kb = reinterpret_cast<const __nv_bfloat16*>(knew);
  const __nv_bfloat16* vb = reinterpret_cast<const __nv_bfloat16*>(vnew);
#define KVT_FLAUNCH(DD, NWW, NSS)                                                                  \
  if (v.D == DD && vr.nw == NWW && vr.nst == NSS) {                                                \
    cfg.blockDim = dim3((NWW + 3) * 32, 1, 1);                                                     \
    return cudaLaunchKernelEx(&cfg, k_decode_flat<DD, NWW, NSS>, v, layer, qb, kb, vb, o, zpar, zprev); \
  }
  KVT_FVARIANTS(KVT_FLAUNCH, 128)
  KVT_FVARIANTS(KVT_FLAUNCH, 64)
#undef KVT_FLAUNCH
  return cudaErrorInvalidValue;
}

}  // namespace kvt
