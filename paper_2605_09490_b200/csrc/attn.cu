// a1 + a3 + a4: fused new-token append, GQA decode attention over the visible tiers, and the
// cumulative score update (Eq. 1, Eq. 3, Prop. 1).
//
// C CTAs per unit (request b, kv head g).  The unit's visible rows are laid out virtually as
// [T0 rows except the new token | pad | T1 staging | pad | T2 int8 | pad | new token],
// segments starting at multiples of 16.  Each CTA owns a contiguous range of whole stages
// (NW 16-row groups) of the bf16 part and one of the int8 part (stage counts differ by <= 1).
//
//   producer warp   streams its stages (NW groups = one per consumer warp) with 1-D bulk async
//                   copies (cp.async.bulk) into an NST-deep shared-memory ring guarded by
//                   full/empty mbarriers.  Rows are stored pre-swizzled in HBM (16-B chunk c of
//                   store row j at c ^ (j & 7)), so a linear copy is the conflict-free layout.
//                   The whole ring is issued before griddepcontrol.wait: it overlaps the
//                   previous kernel's tail.
//   consumer warps  each owns 16 rows of a stage: S^T = K q^T on the tensor cores (mma.sync
//                   m16n8k16 bf16, swap-AB: tokens = M, the G <= 8 heads of the group = N),
//                   per-warp online softmax in fp32, o^T += V^T p^T (movmatrix.trans turns the
//                   C fragment into the B fragment).  Logits (log2 domain) go to an
//                   L2-resident buffer for the score update.
//   side warp       rank 0: appends the new token's K/V row (a1) and computes its attention
//                   term on the CUDA cores as one more partial (m = z, l = 1, o = v_new).
//   merge           warps -> CTA partial (m, l, o) in shared memory -> a global partial slot,
//                   merged in rank order by the PDL-chained k_decode_merge, which also publishes
//                   the per-head (M, 1/L); the score update (a4) then runs as k_score_flush on the
//                   library's score stream.
// This is the per-layer path (kv_tier_decode_attention[_lse], sequence shards, stream mode,
// host-T1); kv_tier_step runs every layer in one launch (step.cu).
//
#include "decode_common.cuh"

namespace kvt {

// Variants (consumer warps NW, pipeline stages NST): a tile is 16 tokens per consumer warp.

__device__ __forceinline__ int atom_add_acqrel_gpu(int* p, int x) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], %2;\n" : "=r"(old) : "l"(p), "r"(x) : "memory");
  return old;
}

template <int D, int NW, int NST>
__global__ void __launch_bounds__((NW + 2) * 32, (NW == 4 ? 2 : 1))
    k_decode_attn(const DevView v, const int layer, const __nv_bfloat16* __restrict__ q,
                  const __nv_bfloat16* __restrict__ knew, const __nv_bfloat16* __restrict__ vnew,
                  void* __restrict__ o, const int zpar) {
  // zpar: logits/ML ring slot of this launch (-1: no score update)
  constexpr int NCONS = NW * 32;              // consumer threads
  constexpr int WPROD = NW, WSCORE = NW + 1;
  constexpr int TILE = NW * 16;
  constexpr int ROWB = D * 2;
  constexpr int TILEB = TILE * ROWB;
  constexpr int STAGEB = 2 * TILEB;           // K tile + V tile
  constexpr int KS = D / 16;
  constexpr int OWS = D + 4;
  const int C = (int)gridDim.x;
  const int r = (int)blockIdx.x;
  const int unit = blockIdx.y;
  const int b = unit / v.Hkv, g = unit - b * v.Hkv;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int G = v.G;
  unsigned long long* tr = v.trace ? v.trace + (((size_t)layer * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x) * NTRACE : nullptr;
  if (tr && tid == 0) { tr[0] = gtimer(); for (int x = 8; x < NTRACE; ++x) tr[x] = 0; }

  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* ring = smem;                                             // [NST][K tile | V tile]
  unsigned char* t2w = ring + NST * STAGEB;                               // [NW][16][D] bf16 (T2 only)
  unsigned long long* bars =
      reinterpret_cast<unsigned long long*>(t2w + (v.cap2 > 0 ? NW * 16 * ROWB : 0));   // full, empty
  int* stile = reinterpret_cast<int*>(bars + 2 * NST);                    // [NST] tile of each stage
  float* redm = reinterpret_cast<float*>(stile + NST + 4);               // [NW][8] warp max
  float* redl = redm + 8 * NW;                                            // [NW][8] warp sum

  // ---------------------------------------------------------------- prologue (pre-PDL-wait)
  const int cur = v.st->cur;
  Seg sg;
  sg.init(v.cnt[cur] + b * CNT_STRIDE, v.st->nn, v.host_t1);
  // This CTA's work: stages of up to NW 16-row groups (one per consumer warp) from the unit's
  // groups [bf16 segment [0, a2) | int8 segment [a2, a2 + n2)]; whole stages are dealt round-robin
  // over the unit's C CTAs (static: the fp32 summation order never depends on timing; measured
  // faster than dealing single groups or cutting contiguous ranges).
  // stage_at(i) -> kind, groups in the stage; group_of(i, w) -> the segment-relative index of
  // warp w's group.
  const int gbf = sg.a2 >> 4, gq2 = (sg.n2 + 15) >> 4;
  const int sbf = (gbf + NW - 1) / NW, ns_all = sbf + (gq2 + NW - 1) / NW;
  const int cs0 = r, cstr = C;
  const int nstage = ns_all > r ? (ns_all - r + C - 1) / C : 0;
  auto stage_at = [&](int i, bool& t2, int& ng) {          // this CTA's i-th stage
    const int gs = cs0 + i * cstr;
    t2 = gs >= sbf;
    const int g0 = (t2 ? gs - sbf : gs) * NW;
    ng = min(NW, (t2 ? gq2 : gbf) - g0);
  };
  auto group_of = [&](int i, int wi) {                      // segment-relative group index
    const int gs = cs0 + i * cstr;
    return (gs >= sbf ? gs - sbf : gs) * NW + wi;
  };
  const bool has_new = r == 0 && sg.nn;                      // rank 0 handles the new token

  const int sb = v.st->scur;                                 // row-store buffer
  const size_t grp = grp_of(v, layer, b, g);
  const __nv_bfloat16* K0 = v.k0[sb] + grp * v.cap0 * D;
  const __nv_bfloat16* V0 = v.v0[sb] + grp * v.cap0 * D;
  const __nv_bfloat16* K1;
  const __nv_bfloat16* V1;
  if (v.stream_mode) {
    const size_t sgi = ((size_t)(layer & 1) * v.B + b) * v.Hkv + g;
    K1 = v.k1[0] + sgi * v.cap1 * D;
    V1 = v.v1[0] + sgi * v.cap1 * D;
  } else {
    K1 = v.k1[sb] + grp * v.cap1 * D;
    V1 = v.v1[sb] + grp * v.cap1 * D;
  }
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

  if (w == WPROD) {
    // ============================ producer ============================
    // streams this CTA's stages (static ranges: the fp32 summation order never depends on timing).
    // It never waits for the previous kernel: K/V rows of this layer do not depend on it, only
    // their consumption (q, the new token) does, and the consumers wait (griddepcontrol.wait).
    if (lane == 0) {
      const uint64_t pol = evict_first_policy();
      for (int i = 0;; ++i) {
        const int s2 = i % NST;
        if (i >= NST) mbar_wait(empty0 + 8 * s2, ((i / NST) - 1) & 1);
        const uint32_t full = full0 + 8 * s2, dst = ring_s + s2 * STAGEB;
        if (i >= nstage) {
          stile[s2] = -1;
          mbar_arrive(full);          // sentinel stage (no data)
          break;
        }
        stile[s2] = i;
        bool st2;
        int ng;
        stage_at(i, st2, ng);
        const int nrows = 16 * ng;
        if (!st2) {                   // bf16 rows: T0 (pad rows beyond n0o are stale but finite), T1
          mbar_expect_tx(full, 2 * nrows * ROWB);
          for (int wi = 0; wi < ng;) {               // runs of consecutive groups in one store
            const int gi = group_of(i, wi);
            const int ts = 16 * gi;                  // a1 is a multiple of 16: no group straddles
            int run = 1;
            while (wi + run < ng && group_of(i, wi + run) == gi + run && (ts < sg.a1) == (ts + 16 * run < sg.a1)) ++run;
            const __nv_bfloat16* ks = ts < sg.a1 ? K0 + (size_t)ts * D : K1 + (size_t)(ts - sg.a1) * D;
            const __nv_bfloat16* vs = ts < sg.a1 ? V0 + (size_t)ts * D : V1 + (size_t)(ts - sg.a1) * D;
            bulk_g2s_ef(dst + wi * 16 * ROWB, ks, run * 16 * ROWB, full, pol);
            bulk_g2s_ef(dst + TILEB + wi * 16 * ROWB, vs, run * 16 * ROWB, full, pol);
            wi += run;
          }
        } else {                      // T2: int8 codes + fp32 scales (canonical layout; rows < cap2)
          mbar_expect_tx(full, 2 * (nrows * D + nrows * 4));
          for (int wi = 0; wi < ng; ++wi) {
            const int j0 = 16 * group_of(i, wi);
            bulk_g2s(dst + wi * 16 * D, v.c2k[sb] + (grp * v.cap2 + j0) * D, 16 * D, full);
            bulk_g2s(dst + TILE * D + wi * 16 * 4, v.s2k[sb] + grp * v.cap2 + j0, 16 * 4, full);
            bulk_g2s(dst + TILEB + wi * 16 * D, v.c2v[sb] + (grp * v.cap2 + j0) * D, 16 * D, full);
            bulk_g2s(dst + TILEB + TILE * D + wi * 16 * 4, v.s2v[sb] + grp * v.cap2 + j0, 16 * 4, full);
          }
        }
      }
    }
    __syncwarp();
    return;
  }
  pdl_trigger();
  // ---------------------------------------------------------------- dependent inputs
  pdl_wait();
  if (tr && tid == 0) tr[1] = gtimer();

  if (w == WSCORE) {
    // ============================ side warp ============================
    // (1) rank 0: the new token (a1 fused): append its K/V row to T0 row n0-1 (swizzled) and
    //     publish its attention term as the unit's partial number C: m = z, l = 1, o = v_new.
    if (has_new) {
      uint16_t* K0w = reinterpret_cast<uint16_t*>(v.k0[sb]) + (grp * v.cap0 + sg.n0o) * D;
      uint16_t* V0w = reinterpret_cast<uint16_t*>(v.v0[sb]) + (grp * v.cap0 + sg.n0o) * D;
      const uint16_t* kin = knew ? reinterpret_cast<const uint16_t*>(knew) + ((size_t)b * v.Hkv + g) * D : nullptr;
      const uint16_t* vin = vnew ? reinterpret_cast<const uint16_t*>(vnew) + ((size_t)b * v.Hkv + g) * D : nullptr;
      float* part = v.part + ((size_t)unit * (C + 1) + C) * v.part_stride;
      constexpr int EL = D / 32;
      const float sl2 = (float)(1.4426950408889634 / __dsqrt_rn((double)D));
      uint16_t kb[EL], vb[EL], qb[8][EL];
      const uint16_t* qbase = reinterpret_cast<const uint16_t*>(q) + ((size_t)b * v.Hq + g * G) * D;
#pragma unroll
      for (int k = 0; k < EL; ++k) {          // every load of the new-token work issued at once
        const int e = lane + 32 * k;
        const int se = swz_off(sg.n0o, e, D);
        kb[k] = kin ? kin[e] : K0w[se];
        vb[k] = vin ? vin[e] : V0w[se];
#pragma unroll
        for (int h = 0; h < 8; ++h) qb[h][k] = h < G ? qbase[(size_t)h * D + e] : (uint16_t)0;
      }
      float* zrow = zpar >= 0 ? v.zbuf + ((size_t)zpar * v.B * v.Hkv + unit) * v.zrows * 8 : nullptr;
      float dot[8];
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
        const int se = swz_off(sg.n0o, e, D);
        if (kin) K0w[se] = kb[k];
        if (vin) V0w[se] = vb[k];
        const float vf = bf16_bits_to_f(vb[k]);
        for (int h = 0; h < G; ++h) part[16 + h * D + e] = vf;
      }
      if (v.red && kin) redund_append(v, layer, unit, v.st->n - 1, kin);   // redundancy (fused append only)
      if (scorer_uses_vnorm(v.scorer)) {   // VATP: the new token's V-row norm for this layer
        float ss = 0.f;
#pragma unroll
        for (int k = 0; k < EL; ++k) ss += bf16_bits_to_f(vb[k]) * bf16_bits_to_f(vb[k]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
        if (lane == 0) v.vnorm[((size_t)layer * v.B * v.Hkv + unit) * v.Nmax + (v.st->n - 1)] = sqrtf(ss);
      }
      if (lane < G) {
        float z = 0.f;
#pragma unroll
        for (int h = 0; h < 8; ++h) z = lane == h ? dot[h] * sl2 : z;
        part[lane] = z;
        part[8 + lane] = 1.f;
        if (zrow) zrow[(size_t)sg.a3 * 8 + lane] = z;
      }
      if (lane >= G && lane < 8) {       // unused heads of the partial
        part[lane] = -INFINITY;
        part[8 + lane] = 0.f;
      }
    }
    if (r == 0 && !sg.nn) {     // sequence shard without the new token: neutral partial C
      float* part = v.part + ((size_t)unit * (C + 1) + C) * v.part_stride;
      for (int e = lane; e < 16 + G * D; e += 32) part[e] = e < 8 ? -INFINITY : 0.f;
      // redundancy: every shard tracks the globally previous key and R_part of every position
      // (identical on all shards, so each classifies from its own copy)
      if (v.red && knew) redund_append(v, layer, unit, v.st->n - 1,
                                       reinterpret_cast<const uint16_t*>(knew) + ((size_t)b * v.Hkv + g) * D);
    }
    return;
  }

  // ============================ consumers ============================
  float mxa = -INFINITY, mxb = -INFINITY;   // per-warp running max, heads 2tq, 2tq+1 (log2)
  float la = 0.f, lb = 0.f;                 // per-thread partial sums
  float oacc[KS][4];
#pragma unroll
  for (int mt = 0; mt < KS; ++mt) oacc[mt][0] = oacc[mt][1] = oacc[mt][2] = oacc[mt][3] = 0.f;
  uint32_t qf[KS][2];
  {
    const __nv_bfloat16* qh = q + ((size_t)b * v.Hq + g * G + gq) * D;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      if (gq < G) {
        qf[ks][0] = *reinterpret_cast<const uint32_t*>(qh + ks * 16 + 2 * tq);
        qf[ks][1] = *reinterpret_cast<const uint32_t*>(qh + ks * 16 + 8 + 2 * tq);
      } else {
        qf[ks][0] = 0u;
        qf[ks][1] = 0u;
      }
    }
  }
  const float sl2 = (float)(1.4426950408889634 / __dsqrt_rn((double)D));   // log2(e)/sqrt(d)
  float* zrow = zpar >= 0 ? v.zbuf + ((size_t)zpar * v.B * v.Hkv + unit) * v.zrows * 8 : nullptr;

  // one warp-slice (16 rows) of a stage: logits, online softmax, P.V.  Lazy rescale: the running
  // max of a head only moves (warp reduction + rescale of o and l) when some logit exceeds it
  // by more than RESCALE_SLACK (log2 units); otherwise p = exp2(z - m) <= 2^RESCALE_SLACK is
  // accumulated against the stale max -- the same softmax, without the shuffle chain.
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
      const float na = fmaxf(mxa, ta), nb = fmaxf(mxb, tb);     // finite: some row is valid
      const float ca = ex2_ftz(mxa - na), cb = ex2_ftz(mxb - nb);   // 0 when the old max is -inf
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
  // K slice . q^T: KS independent-ish MMAs in NCH accumulator chains (short dependency depth:
  // the per-stage critical path is latency, not tensor throughput)
  auto qk = [&](uint32_t sK, int rowbase, float* acc) {
    constexpr int NCH = KS >= 4 ? 4 : KS;
    float ch[NCH][4];
#pragma unroll
    for (int c = 0; c < NCH; ++c) ch[c][0] = ch[c][1] = ch[c][2] = ch[c][3] = 0.f;
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
      for (int c = 1; c < NCH; ++c) x += ch[c][j];
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
      ldsm_x4_t(af[mt][0], af[mt][1], af[mt][2], af[mt][3], sV + tile_off<D>(row, 2 * mt + (mi & 1)));
#pragma unroll
    for (int mt = 0; mt < KS; ++mt) mma16816(oacc[mt], af[mt][0], af[mt][1], af[mt][2], af[mt][3], c0, c1);
#pragma unroll
    for (int mt = 0; mt < KS; ++mt) mma16816(oacc[mt], af[mt][0], af[mt][1], af[mt][2], af[mt][3], b0, b1);
  };
  // this warp's 16 rows of int8 codes -> exact bf16 into its scratch (swizzled by row)
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

  for (int i = 0;; ++i) {
    const int s2 = i % NST;
    mbar_wait(full0 + 8 * s2, (i / NST) & 1);
    const int k = stile[s2];
    if (k < 0) break;
    if (tr && tid == 0 && i == 0) tr[2] = gtimer();
    const uint32_t sK = ring_s + s2 * STAGEB, sV = sK + TILEB;
    bool t2;
    int ng;
    stage_at(k, t2, ng);
    const bool wact = w < ng;                                 // this warp's group is in the stage
    const int tv0 = (t2 ? sg.a2 : 0) + 16 * (wact ? group_of(k, w) : 0);   // warp's first virtual row
    const int r0 = w * 16 + gq, r1 = r0 + 8;                  // rows within the stage tile
    const int t0 = tv0 + gq, t1 = tv0 + gq + 8;
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
      } else {                    // o += p * scale_v * code (codes exact in bf16)
        __syncwarp();
        stage_t2_rows(reinterpret_cast<const int8_t*>(ring + s2 * STAGEB + TILEB), scr);
        pv(smem_u32(scr), 0, p00 * fv0, p01 * fv0, p10 * fv1, p11 * fv1);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(empty0 + 8 * s2);
  }
  if (tr && tid == 0) tr[3] = gtimer();

  // ---- warps -> CTA partial (ring reused as [NW][8][D+4] fp32)
#pragma unroll
  for (int off = 4; off < 32; off <<= 1) {
    la += __shfl_xor_sync(0xffffffffu, la, off);
    lb += __shfl_xor_sync(0xffffffffu, lb, off);
  }
  named_sync(1, NCONS);                // every consumer is done with the ring
  float* ow = reinterpret_cast<float*>(ring);
  if (lane < 4) {
    redm[w * 8 + 2 * lane] = mxa;
    redm[w * 8 + 2 * lane + 1] = mxb;
    redl[w * 8 + 2 * lane] = la;
    redl[w * 8 + 2 * lane + 1] = lb;
  }
#pragma unroll
  for (int mt = 0; mt < KS; ++mt) {
    float* o0 = ow + (w * 8 + 2 * tq) * OWS + mt * 16 + gq;
    float* o1 = o0 + OWS;
    o0[0] = oacc[mt][0];
    o1[0] = oacc[mt][1];
    o0[8] = oacc[mt][2];
    o1[8] = oacc[mt][3];
  }
  named_sync(1, NCONS);
  const int tot = G * D;
  // publish straight to the global slot (visible to the merge kernel once this grid completes):
  // every thread forms its elements' per-head max and warp factors itself
  float* part = v.part + ((size_t)unit * (C + 1) + r) * v.part_stride;
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
    part[tid] = M;
    part[8 + tid] = Ls;
  }
  for (int e = tid; e < tot; e += NCONS) {
    const int h = e / D, dd = e - h * D;
    float mw[NW], M = -INFINITY;
#pragma unroll
    for (int x = 0; x < NW; ++x) {
      mw[x] = redm[x * 8 + h];
      M = fmaxf(M, mw[x]);
    }
    float a = 0.f;
#pragma unroll
    for (int x = 0; x < NW; ++x) a += (mw[x] == -INFINITY ? 0.f : ex2_ftz(mw[x] - M)) * ow[(x * 8 + h) * OWS + dd];
    part[16 + e] = a;
  }
  if (tr && tid == 0) tr[4] = gtimer();
}

// Merge of the C per-CTA partials (+ the new-token partial) of every unit, in rank order
// (deterministic): o and the per-head (max, 1/sum) for the deferred score pass.  Launched right
// behind the decode kernel with programmatic dependent launch: its CTAs are resident early and
// start when it completes.  One CTA per unit, one float4 of o per thread; each thread issues its
// partial loads right after the wait, the per-head (M, 1/L) and the factors exp2(m_c - M) are
// computed once (shared memory) in the same round trip, and o goes out as one vector store.
template <int D>
__global__ void __launch_bounds__(256) k_decode_merge(const DevView v, const int layer, void* __restrict__ o,
                                                      const int zpar, float* __restrict__ lse) {
  // lse (optional) [B][Hq][2]: this ctx's (max, sum) per head, log2 domain (sequence sharding)
  constexpr int MAXP = 9, MAXNP = 65;      // split <= 8: one batch
  __shared__ float sf[MAXNP * 8], sl[MAXNP * 8], sI[8];
  const int unit = blockIdx.x, tid = threadIdx.x;
  const int b = unit / v.Hkv, g = unit - b * v.Hkv;
  const int G = v.G, NP = v.split + 1, tot4 = G * D / 4;
  unsigned long long* tr = v.trace ? v.trace + (((size_t)layer * v.B * v.Hkv + unit) * v.split) * NTRACE : nullptr;
  if (tr && tid == 0) tr[6] = gtimer();
  pdl_trigger();
  pdl_wait();
  if (tr && tid == 0) tr[5] = gtimer();
  const float* P = v.part + (size_t)unit * NP * v.part_stride;
  const bool act = tid < tot4;
  float4 x[MAXP];
#pragma unroll
  for (int c = 0; c < MAXP; ++c)
    if (act && c < NP) x[c] = __ldcg(reinterpret_cast<const float4*>(P + (size_t)c * v.part_stride + 16) + tid);
  for (int i = tid; i < NP * 8; i += blockDim.x) {
    sf[i] = __ldcg(P + (size_t)(i >> 3) * v.part_stride + (i & 7));
    sl[i] = __ldcg(P + (size_t)(i >> 3) * v.part_stride + 8 + (i & 7));
  }
  __syncthreads();
  if (unit == 0 && tid == 0 && zpar >= 0) v.zlayer[zpar] = layer;   // the slot's layer (VATP weights)
  if (tid < 8) {
    const int h = tid;
    float M = -INFINITY;
    for (int c = 0; c < NP; ++c) M = fmaxf(M, sf[c * 8 + h]);
    float Ls = 0.f;
    for (int c = 0; c < NP; ++c) {
      const float mc = sf[c * 8 + h];
      const float f = mc == -INFINITY ? 0.f : ex2_ftz(mc - M);
      sf[c * 8 + h] = f;
      Ls += f * sl[c * 8 + h];
    }
    const float invL = Ls > 0.f ? 1.0f / Ls : 0.f;   // 0: a sequence shard with no visible token
    sI[h] = invL;
    if (h < G && lse) {
      lse[(((size_t)b * v.Hq + g * G + h) << 1)] = M;
      lse[(((size_t)b * v.Hq + g * G + h) << 1) + 1] = Ls;
    }
    if (h < G && zpar >= 0 && !lse) {  // publish (M, 1/L) for the deferred score pass (with lse:
                                       // the caller's global values, kv_tier_score_update_lse)
      float* ml = v.ml + ((size_t)zpar * v.B * v.Hkv + unit) * 16;
      ml[h] = M;
      ml[8 + h] = invL;
    }
  }
  __syncthreads();
  if (act) {
    const int h = (4 * tid) / D;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int c0 = 0; c0 < NP; c0 += MAXP) {
      if (c0 > 0) {                    // split > 15: next batch of partials
#pragma unroll
        for (int c = 0; c < MAXP; ++c)
          if (c0 + c < NP) x[c] = __ldcg(reinterpret_cast<const float4*>(P + (size_t)(c0 + c) * v.part_stride + 16) + tid);
      }
#pragma unroll
      for (int c = 0; c < MAXP; ++c)
        if (c0 + c < NP) {
          const float f = sf[(c0 + c) * 8 + h];
          acc.x += f * x[c].x;
          acc.y += f * x[c].y;
          acc.z += f * x[c].z;
          acc.w += f * x[c].w;
        }
    }
    const float il = sI[h];
    const size_t oi = ((size_t)b * v.Hq + g * G) * D + 4 * tid;
    if (v.out_fp32) {
      *reinterpret_cast<float4*>(reinterpret_cast<float*>(o) + oi) = make_float4(acc.x * il, acc.y * il, acc.z * il, acc.w * il);
    } else {
      __nv_bfloat162 lo = __floats2bfloat162_rn(acc.x * il, acc.y * il), hi = __floats2bfloat162_rn(acc.z * il, acc.w * il);
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&lo);
      pk.y = *reinterpret_cast<uint32_t*>(&hi);
      *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(o) + oi) = pk;
    }
  }
  if (tr && tid == 0) tr[7] = gtimer();
}

size_t merge_smem_bytes(const DevView& v) { (void)v; return 0; }

// a4: the score update of nz consecutive decode_attention launches (ring slots zfirst..), on
// the library's score stream, off the attention critical path.
__global__ void __launch_bounds__(256) k_score_flush(const DevView v, const int zfirst, const int nz) {
  const int cur = v.st->cur;
  Seg sg;
  sg.init(v.cnt[cur], v.st->nn, v.host_t1);   // counts are uniform across requests
  const long long tot = (long long)v.B * v.Hkv * sg.nvirt;
  bool bad = false;
  score_range(v, sg, cur, zfirst, nz, 0, tot, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x, bad);
  if (bad) atomicOr(&v.st->err, 1);
}

// Sequence shards: a shard's tier counts differ per request, so every unit decodes its own
// virtual layout (one thread per (unit, virtual row) over the zrows-wide logit rows).
__global__ void __launch_bounds__(256) k_score_flush_req(const DevView v, const int zfirst, const int nz) {
  const int cur = v.st->cur, nn = v.st->nn;
  const size_t zslot = (size_t)v.B * v.Hkv * v.zrows * 8, mslot = (size_t)v.B * v.Hkv * 16;
  const long long tot = (long long)v.B * v.Hkv * v.zrows;
  bool bad = false;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < tot; i += (long long)gridDim.x * blockDim.x) {
    const int u = (int)(i / v.zrows), t = (int)(i - (long long)u * v.zrows), b = u / v.Hkv;
    Seg sg;
    sg.init(v.cnt[cur] + b * CNT_STRIDE, nn, v.host_t1);
    if (t >= sg.nvirt || !sg.valid(t)) continue;
    const int pos = sg.pos(v, cur, b, t);
    float s = v.S[(size_t)u * v.Nmax + pos];
    for (int j = 0; j < nz; ++j) {                 // launches in layer order
      const int slot = zslot_of(v, zfirst + j);
      const float* z = v.zbuf + slot * zslot + ((size_t)u * v.zrows + t) * 8;
      const float* ml = v.ml + slot * mslot + (size_t)u * 16;
      float inc = 0.f;
      for (int h = 0; h < v.G; ++h) inc += ex2_ftz(z[h] - ml[h]) * ml[8 + h];
      s = s + inc * score_weight(v, v.scorer ? v.zlayer[slot] : 0, u, pos);
      bad |= !isfinite(inc);
    }
    v.S[(size_t)u * v.Nmax + pos] = s;
  }
  if (bad) atomicOr(&v.st->err, 1);
}

cudaError_t launch_score_flush(const DevView& v, int zfirst, int nz, cudaStream_t s) {
  if (v.seq_w > 1) k_score_flush_req<<<148, 256, 0, s>>>(v, zfirst, nz);
  else k_score_flush<<<v.score_grid, 256, 0, s>>>(v, zfirst, nz);
  return cudaGetLastError();
}

// (consumer warps, stages) variants; DevView::variant selects one (0 = default)
struct Variant { int nw, nst; };
static constexpr Variant kVariants[] = {{4, 3}, {4, 4}, {8, 2}, {8, 3}, {4, 2}, {4, 6}};
constexpr int kNumVariants = sizeof(kVariants) / sizeof(kVariants[0]);

size_t attn_smem_bytes(const DevView& v) {
  const Variant vr = kVariants[v.variant];
  const int tile = 16 * vr.nw;
  const size_t ringb = (size_t)vr.nst * 2 * tile * v.D * 2 + (2 * vr.nst) * 8 + (vr.nst + 4) * 4 + 16;
  const size_t xob = (size_t)8 * v.D * 4 + (8 + 8 + 16 * vr.nw + 16 + 2 * v.D + 8) * 4;
  const size_t t2 = (v.cap2 > 0) ? (size_t)vr.nw * 16 * v.D * 2 : 0;
  size_t total = ringb + xob + t2;
  const size_t ow = (size_t)vr.nw * 8 * (v.D + 4) * 4 + vr.nw * 8 * 4;   // end-of-kernel reuse of the ring
  if (ow > (size_t)vr.nst * 2 * tile * v.D * 2) total += ow;   // (never for the shipped variants)
  return total;
}

template <int D, int NW, int NST>
static cudaError_t configure_k(const DevView& v) {
  return cudaFuncSetAttribute(k_decode_attn<D, NW, NST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)attn_smem_bytes(v));
}

template <int D, int NW, int NST>
static cudaError_t launch_k(const DevView& v, cudaLaunchConfig_t& cfg, int layer, const void* q, const void* knew,
                            const void* vnew, void* o, int zpar) {
  cfg.blockDim = dim3((NW + 2) * 32, 1, 1);
  return cudaLaunchKernelEx(&cfg, k_decode_attn<D, NW, NST>, v, layer, reinterpret_cast<const __nv_bfloat16*>(q),
                            reinterpret_cast<const __nv_bfloat16*>(knew), reinterpret_cast<const __nv_bfloat16*>(vnew),
                            o, zpar);
}

#define KVT_VARIANTS(X, D) X(D, 4, 3) X(D, 4, 4) X(D, 8, 2) X(D, 8, 3) X(D, 4, 2) X(D, 4, 6)

cudaError_t attn_configure(const DevView& v) {
  if (v.variant < 0 || v.variant >= kNumVariants) return cudaErrorInvalidValue;
  {
    cudaError_t e = v.D == 128 ? cudaFuncSetAttribute(k_decode_merge<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                      (int)merge_smem_bytes(v))
                               : cudaFuncSetAttribute(k_decode_merge<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                      (int)merge_smem_bytes(v));
    if (e != cudaSuccess) return e;
  }
  const Variant vr = kVariants[v.variant];
#define KVT_CONF(DD, NWW, NSS) \
  if (v.D == DD && vr.nw == NWW && vr.nst == NSS) return configure_k<DD, NWW, NSS>(v);
  KVT_VARIANTS(KVT_CONF, 128)
  KVT_VARIANTS(KVT_CONF, 64)
#undef KVT_CONF
  return cudaErrorInvalidValue;
}

static cudaError_t launch_decode_main(const DevView& v, int layer, const void* q, const void* knew,
                                      const void* vnew, void* o, int zpar, int pdl, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(v.split, v.B * v.Hkv, 1);
  cfg.dynamicSmemBytes = attn_smem_bytes(v);
  cfg.stream = s;
  cudaLaunchAttribute at[3];
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
  const Variant vr = kVariants[v.variant];
#define KVT_LAUNCH(DD, NWW, NSS)                          \
  if (v.D == DD && vr.nw == NWW && vr.nst == NSS)         \
    return launch_k<DD, NWW, NSS>(v, cfg, layer, q, knew, vnew, o, zpar);
  KVT_VARIANTS(KVT_LAUNCH, 128)
  KVT_VARIANTS(KVT_LAUNCH, 64)
#undef KVT_LAUNCH
  return cudaErrorInvalidValue;
}

static cudaError_t launch_merge(const DevView& v, int layer, void* o, int zpar, int pdl, cudaStream_t s, float* lse) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(v.B * v.Hkv, 1, 1);
  cfg.blockDim = dim3(256, 1, 1);
  cfg.dynamicSmemBytes = merge_smem_bytes(v);
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
  if (v.D == 128) return cudaLaunchKernelEx(&cfg, k_decode_merge<128>, v, layer, o, zpar, lse);
  return cudaLaunchKernelEx(&cfg, k_decode_merge<64>, v, layer, o, zpar, lse);
}

cudaError_t launch_decode_attn(const DevView& v, int layer, const void* q, const void* knew, const void* vnew,
                               void* o, int zpar, int pdl, cudaStream_t s, float* lse) {
  cudaError_t e = launch_decode_main(v, layer, q, knew, vnew, o, zpar, pdl, s);
  if (e != cudaSuccess) return e;
  return launch_merge(v, layer, o, zpar, 1, s, lse);
}

// (M, 1/L) of every (unit, head) for score slot zslot from the caller's global (M, L)
// [B][Hq][2] (sequence sharding: the ranks' partial sums combined, kv_tier_score_update_lse)
__global__ void k_set_ml(const DevView v, const int zslot, const float* __restrict__ lse) {
  const int unit = blockIdx.x, h = threadIdx.x;
  const int b = unit / v.Hkv, g = unit - b * v.Hkv;
  if (h >= 8) return;
  float* ml = v.ml + ((size_t)zslot * v.B * v.Hkv + unit) * 16;
  if (h < v.G) {
    const size_t i = ((size_t)b * v.Hq + g * v.G + h) << 1;
    ml[h] = lse[i];
    ml[8 + h] = 1.0f / lse[i + 1];
  } else {
    ml[h] = -INFINITY;
    ml[8 + h] = 0.f;
  }
}

// Rank combine of sequence-shard partials (kv_tier_lse_combine): one thread per (row, 4 lanes
// of d), ranks in order.
// ml (optional): the score pass's (M, 1/L) ring slot [B*H_kv][16], written here instead of by a
// separate k_set_ml (rows = b * H_q + h, kv head h / G)
__global__ void k_lse_combine(const float* __restrict__ op, const float* __restrict__ lp, const int world,
                              const int rows, const int d, float* __restrict__ oo, float* __restrict__ lo,
                              float* __restrict__ ml, const int G, const size_t rs_o, const size_t rs_l) {
  // PDL (sequence step): the next layer's decode may launch now (its K/V prologue does not read o);
  // the parts are read after the producer grid (merge or the all-gather) has completed
  pdl_trigger();
  pdl_wait();
  const int d4 = d / 4;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)rows * d4) return;
  const int row = (int)(i / d4), j = (int)(i - (long long)row * d4);
  float M = -INFINITY;
  for (int r = 0; r < world; ++r) M = fmaxf(M, lp[r * rs_l + (size_t)row * 2]);
  float L = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int r = 0; r < world; ++r) {
    const float m = lp[r * rs_l + (size_t)row * 2], l = lp[r * rs_l + (size_t)row * 2 + 1];
    const float wr = m == -INFINITY ? 0.f : ex2_ftz(m - M) * l;
    const float4 x = reinterpret_cast<const float4*>(op + r * rs_o + (size_t)row * d)[j];
    L += wr;
    acc.x += wr * x.x;
    acc.y += wr * x.y;
    acc.z += wr * x.z;
    acc.w += wr * x.w;
  }
  const float il = L > 0.f ? 1.0f / L : 0.f;
  reinterpret_cast<float4*>(oo + (size_t)row * d)[j] = make_float4(acc.x * il, acc.y * il, acc.z * il, acc.w * il);
  if (j == 0) {
    lo[(size_t)row * 2] = M;
    lo[(size_t)row * 2 + 1] = L;
    if (ml) {
      const int unit = row / G, hh = row - unit * G;     // rows of one kv head are consecutive
      float* m = ml + (size_t)unit * 16;
      m[hh] = M;
      m[8 + hh] = 1.0f / L;
      if (hh == 0)
        for (int x = G; x < 8; ++x) { m[x] = -INFINITY; m[8 + x] = 0.f; }
    }
  }
}

cudaError_t launch_lse_combine(const float* op, const float* lp, int world, int rows, int d, float* oo, float* lo,
                               cudaStream_t s, float* ml, int G, size_t rs_o, size_t rs_l, int pdl) {
  const long long n = (long long)rows * (d / 4);
  if (!rs_o) rs_o = (size_t)rows * d;
  if (!rs_l) rs_l = (size_t)rows * 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((n + 255) / 256), 1, 1);
  cfg.blockDim = dim3(256, 1, 1);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_lse_combine, op, lp, world, rows, d, oo, lo, ml, G, rs_o, rs_l);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_set_ml(const DevView& v, int zslot, const float* lse, cudaStream_t s) {
  k_set_ml<<<v.B * v.Hkv, 32, 0, s>>>(v, zslot, lse);
  return cudaGetLastError();
}

}  // namespace kvt
