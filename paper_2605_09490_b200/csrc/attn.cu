// a1 + a3 + a4: fused new-token append, GQA decode attention over the visible tiers, and the
// cumulative score update (Eq. 1, Eq. 3, Prop. 1).
//
// One thread-block cluster of C CTAs per (request b, kv head g).  The visible rows of the
// unit are laid out virtually as [T0 rows except the new token | pad | T1 staging | pad |
// T2 int8 | pad | new token] (segments start at multiples of 16); CTA r of the cluster owns
// a contiguous 1/C chunk.  Warp NW is the producer: it streams the chunk's K tiles, then its
// V tiles, with 1-D bulk async copies (cp.async.bulk, one or two per tile) into an NST-deep
// shared-memory ring guarded by full/empty mbarriers.  Rows are stored pre-swizzled in HBM
// (16-B chunk c of store row j at c ^ (j & 7)), so a linear copy is the conflict-free layout.
//
//   prologue  (before griddepcontrol.wait, overlaps the previous layer's kernel under PDL)
//            counters, the first tiles in flight, positions of the chunk -> SMEM
//   phase A  K tiles -> S^T = K q^T on the tensor cores
//            (mma.sync m16n8k16 bf16, swap-AB: tokens = M, heads = N = 8); logits (log2
//            domain) stay in SMEM for the whole chunk; running max per head
//   phase B  V tiles -> p = exp2(z - m_local) -> o^T += V^T p^T (movmatrix.trans turns the
//            C fragment into the B fragment; ldmatrix.trans reads V^T)
//   merge    (m, l, o) of the C CTAs through distributed shared memory; CTA r writes 1/C of o
//   score    exact p_i = exp2(z_i - M)/L from the SMEM logits; S_part[b][g][pos_i] += sum over
//            the group's heads (one fp32 add per layer, AMB-14); each (b,g,pos) belongs to one
//            CTA -> no atomics, bit-reproducible
//
// HBM traffic per launch = algorithmic bytes: every visible K/V row once, q, o, the new row
// (read + written), and 8 B of score read+write per visible token per kv head.
#include "kv_internal.cuh"
#include <cooperative_groups.h>

namespace cg = cooperative_groups;

namespace kvt {

// Variants (consumer warps NW, pipeline stages NST): a tile is 16 tokens per consumer warp.

__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok)
                 : "r"(a), "r"(parity)
                 : "memory");
  } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ int ru16(int x) { return (x + 15) & ~15; }
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
constexpr int NTRACE = 8;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int nbytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(nbytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::); }

__device__ __forceinline__ void ldsm_x4(uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& a3, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t& a0, uint32_t& a1, uint32_t& a2, uint32_t& a3, uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3)
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t movm_t(uint32_t x) {
  uint32_t y;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;\n" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);   // .x (low 16 bits) = lo
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ uint32_t i8pair_to_bf16x2(uint32_t word, int k) {
  const float lo = (float)(int8_t)((word >> (16 * k)) & 0xFF);   // exact: |code| <= 127
  const float hi = (float)(int8_t)((word >> (16 * k + 8)) & 0xFF);
  return pack_bf16(lo, hi);
}
__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

template <int D, int NW, int NST>
__global__ void __launch_bounds__((NW + 1) * 32, (NW == 4 ? 2 : 1))
    k_decode_attn(const DevView v, const int layer, const __nv_bfloat16* __restrict__ q,
                  const __nv_bfloat16* __restrict__ knew, const __nv_bfloat16* __restrict__ vnew,
                  void* __restrict__ o, const int fuse) {
  constexpr int NCONS = NW * 32;              // consumer threads
  constexpr int NTHR = NCONS + 32;            // + producer warp
  constexpr int TILE = NW * 16;
  constexpr int ROWB = D * 2;
  constexpr int TILEB = TILE * ROWB;
  constexpr int KS = D / 16;
  cg::cluster_group cluster = cg::this_cluster();
  const int C = (int)cluster.num_blocks();
  const int r = (int)cluster.block_rank();
  const int unit = blockIdx.y;
  const int b = unit / v.Hkv, g = unit - b * v.Hkv;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int G = v.G;

  unsigned long long* tr = v.trace ? v.trace + ((size_t)blockIdx.y * gridDim.x + blockIdx.x) * NTRACE : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = gtimer();
  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* ring = smem;
  unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + NST * TILEB);   // full[NST], empty[NST]
  float* zs = reinterpret_cast<float*>(bars + 2 * NST + 2);     // [chunk_max][8] logits (log2)
  int* spos = reinterpret_cast<int*>(zs + (size_t)v.chunk_max * 8);   // [chunk_max] positions (-1: pad)
  float* sS = reinterpret_cast<float*>(spos + v.chunk_max);     // [chunk_max] S_part values
  float* xo = sS + v.chunk_max;                                 // [8][D]  exchange: o partial
  float* xm = xo + 8 * D;                                       // [8]     exchange: max (log2)
  float* xl = xm + 8;                                           // [8]     exchange: sum
  float* red = xl + 8;                                          // [2][NW][8] warp max / warp l
  float* sML = red + 16 * NW;                                   // [16] merged M, 1/L
  float* nrow = sML + 16;                                       // [2][D] new token K, V (fp32)
  float* t2sc = nrow + 2 * D;                                   // [TILE] T2 row scales
  unsigned char* t2buf = reinterpret_cast<unsigned char*>(t2sc + TILE);   // [TILE][D] bf16

  // ---------------------------------------------------------------- prologue (pre-PDL-wait)
  const int cur = v.st->cur;
  const int* cn = v.cnt[cur] + b * CNT_STRIDE;
  const int n0 = cn[0], n1 = cn[1], n2 = cn[2];
  const int n0o = n0 - 1;                                  // T0 rows before the new token
  const int a1 = ru16(n0o), a2 = ru16(a1 + n1), a3 = ru16(a2 + n2);   // segment starts
  const int nvirt = a3 + 1;
  const int chunk = ru16((nvirt + C - 1) / C);
  const int vbeg = min(r * chunk, nvirt), vend = min(vbeg + chunk, nvirt);
  const int aend = min(vend, a2);                          // bf16 tiles cover [vbeg, aend)
  const int t2beg = max(vbeg, a2), t2end = min(vend, a2 + n2);
  const bool has_new = vbeg <= a3 && a3 < vend;
  const int nb = max(0, aend - vbeg);
  const int nt = (nb + TILE - 1) / TILE;
  const int total = 2 * nt;
  auto bf16_valid = [&](int t) { return t < n0o || (t >= a1 && t < a1 + n1); };

  const size_t grp = grp_of(v, layer, b, g);
  const __nv_bfloat16* K0 = v.k0[cur] + grp * v.cap0 * D;
  const __nv_bfloat16* V0 = v.v0[cur] + grp * v.cap0 * D;
  const __nv_bfloat16* K1;
  const __nv_bfloat16* V1;
  if (v.stream_mode) {
    const size_t sg = ((size_t)(layer & 1) * v.B + b) * v.Hkv + g;
    K1 = v.k1[0] + sg * v.cap1 * D;
    V1 = v.v1[0] + sg * v.cap1 * D;
  } else {
    K1 = v.k1[cur] + grp * v.cap1 * D;
    V1 = v.v1[cur] + grp * v.cap1 * D;
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

  if (w == NW) {
    // ============================ producer warp ============================
    if (lane == 0) {
      for (int i = 0; i < total; ++i) {
        const int s2 = i % NST;
        if (i >= NST) mbar_wait(empty0 + 8 * s2, ((i / NST) - 1) & 1);
        const bool isV = i >= nt;
        const int ts = vbeg + (isV ? i - nt : i) * TILE;
        const uint32_t full = full0 + 8 * s2, dst = ring_s + s2 * TILEB;
        mbar_expect_tx(full, TILEB);
        if (ts < a1) {   // T0 rows [ts, min(ts+TILE, a1)) (pad rows beyond n0o are stale but finite)
          const int nrows = min(TILE, a1 - ts);
          bulk_g2s(dst, (isV ? V0 : K0) + (size_t)ts * D, nrows * ROWB, full);
          if (nrows < TILE)
            bulk_g2s(dst + nrows * ROWB, isV ? V1 : K1, (TILE - nrows) * ROWB, full);
        } else {
          bulk_g2s(dst, (isV ? V1 : K1) + (size_t)(ts - a1) * D, TILEB, full);
        }
      }
    }
    __syncwarp();
    pdl_trigger();
  } else {
    // ============================ consumer warps ============================
    // positions of the chunk (for the score update), cp.async: no stall
    if (fuse) {
      const int* I0 = v.idx[cur][0] + (size_t)b * v.cap0;
      const int* I1 = v.idx[cur][1] + (size_t)b * v.cap1;
      const int* I2 = v.idx[cur][2] + (size_t)b * v.cap2;
      for (int j = tid; j < vend - vbeg; j += NCONS) {
        const int t = vbeg + j;
        const int* src = t < n0o ? I0 + t
                       : (t >= a1 && t < a1 + n1) ? I1 + (t - a1)
                       : (t >= a2 && t < a2 + n2) ? I2 + (t - a2)
                       : t == a3 ? I0 + n0o : nullptr;
        if (src) cp_async4(smem_u32(spos + j), src);
        else spos[j] = -1;
      }
      cp_commit();
    }
    pdl_trigger();
  }
  // ---------------------------------------------------------------- dependent inputs
  pdl_wait();
  if (tr && tid == 0) tr[1] = gtimer();
  if (w == NW) {
    // the producer warp only joins the CTA-wide barriers below
  } else {
    if (fuse) {   // S_part values of the chunk's tokens (written by the previous layer)
      cp_wait<0>();
      float* Sg = v.S + ((size_t)b * v.Hkv + g) * v.Nmax;
      for (int j = tid; j < vend - vbeg; j += NCONS) {
        const int pos = spos[j];
        if (pos >= 0) cp_async4(smem_u32(sS + j), Sg + pos);
      }
      cp_commit();
    }
  }

  uint32_t qf[KS][2];
  const float sl2 = (float)(1.4426950408889634 / __dsqrt_rn((double)D));   // log2(e)/sqrt(d)
  float mx0 = -INFINITY, mx1 = -INFINITY;    // running max, heads 2tq, 2tq+1
  float l0 = 0.f, l1 = 0.f;
  float oacc[KS][4];
#pragma unroll
  for (int mt = 0; mt < KS; ++mt) oacc[mt][0] = oacc[mt][1] = oacc[mt][2] = oacc[mt][3] = 0.f;
  float m2a = 0.f, m2b = 0.f;   // CTA max for heads 2tq, 2tq+1

  if (w < NW) {
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
    // new token (a1): append its K/V row to T0 row n0-1 (swizzled) and keep it in SMEM (fp32)
    if (has_new) {
      uint16_t* K0w = reinterpret_cast<uint16_t*>(v.k0[cur]) + (grp * v.cap0 + n0o) * D;
      uint16_t* V0w = reinterpret_cast<uint16_t*>(v.v0[cur]) + (grp * v.cap0 + n0o) * D;
      const uint16_t* kin = knew ? reinterpret_cast<const uint16_t*>(knew) + ((size_t)b * v.Hkv + g) * D : nullptr;
      const uint16_t* vin = vnew ? reinterpret_cast<const uint16_t*>(vnew) + ((size_t)b * v.Hkv + g) * D : nullptr;
      for (int e = tid; e < D; e += NCONS) {
        const int se = swz_off(n0o, e);
        const uint16_t kb = kin ? kin[e] : K0w[se];
        const uint16_t vb = vin ? vin[e] : V0w[se];
        nrow[e] = bf16_bits_to_f(kb);
        nrow[D + e] = bf16_bits_to_f(vb);
        if (kin) K0w[se] = kb;
        if (vin) V0w[se] = vb;
      }
    }

    auto qk_warp = [&](uint32_t sbase, int tv0, int tend, const float* rsc, bool t2seg) {
      if (tv0 + w * 16 >= tend) return;
      float acc[4] = {0.f, 0.f, 0.f, 0.f}, acc2[4] = {0.f, 0.f, 0.f, 0.f};
      const int mi = lane >> 3, ii = lane & 7;
      const int row = w * 16 + ii + ((mi & 1) << 3);
#pragma unroll
      for (int ks = 0; ks < KS; ks += 2) {
        uint32_t a0, a1_, a2_, a3_;
        ldsm_x4(a0, a1_, a2_, a3_, sbase + row * ROWB + (((2 * ks + (mi >> 1)) ^ (row & 7)) << 4));
        mma16816(acc, a0, a1_, a2_, a3_, qf[ks][0], qf[ks][1]);
        ldsm_x4(a0, a1_, a2_, a3_, sbase + row * ROWB + (((2 * ks + 2 + (mi >> 1)) ^ (row & 7)) << 4));
        mma16816(acc2, a0, a1_, a2_, a3_, qf[ks + 1][0], qf[ks + 1][1]);
      }
      const int r0 = w * 16 + gq, r1 = r0 + 8;
      const int t0 = tv0 + r0, t1 = tv0 + r1;
      if (t0 < tend && (t2seg || bf16_valid(t0))) {
        const float f = rsc ? rsc[r0] * sl2 : sl2;
        const float z0 = (acc[0] + acc2[0]) * f, z1 = (acc[1] + acc2[1]) * f;
        *reinterpret_cast<float2*>(&zs[(t0 - vbeg) * 8 + 2 * tq]) = make_float2(z0, z1);
        mx0 = fmaxf(mx0, z0);
        mx1 = fmaxf(mx1, z1);
      }
      if (t1 < tend && (t2seg || bf16_valid(t1))) {
        const float f = rsc ? rsc[r1] * sl2 : sl2;
        const float z0 = (acc[2] + acc2[2]) * f, z1 = (acc[3] + acc2[3]) * f;
        *reinterpret_cast<float2*>(&zs[(t1 - vbeg) * 8 + 2 * tq]) = make_float2(z0, z1);
        mx0 = fmaxf(mx0, z0);
        mx1 = fmaxf(mx1, z1);
      }
    };
    auto pv_warp = [&](uint32_t sbase, int tv0, int tend, const float* rsc, bool t2seg) {
      if (tv0 + w * 16 >= tend) return;
      const int r0 = w * 16 + gq, r1 = r0 + 8;
      const int t0 = tv0 + r0, t1 = tv0 + r1;
      float p00 = 0.f, p01 = 0.f, p10 = 0.f, p11 = 0.f;
      if (t0 < tend && (t2seg || bf16_valid(t0))) {
        const float2 z = *reinterpret_cast<const float2*>(&zs[(t0 - vbeg) * 8 + 2 * tq]);
        p00 = exp2f(z.x - m2a);
        p01 = exp2f(z.y - m2b);
      }
      if (t1 < tend && (t2seg || bf16_valid(t1))) {
        const float2 z = *reinterpret_cast<const float2*>(&zs[(t1 - vbeg) * 8 + 2 * tq]);
        p10 = exp2f(z.x - m2a);
        p11 = exp2f(z.y - m2b);
      }
      l0 += p00 + p10;
      l1 += p01 + p11;
      if (rsc) {   // T2: o += p * scale_v * code  (codes are exact in bf16)
        p00 *= rsc[r0]; p01 *= rsc[r0];
        p10 *= rsc[r1]; p11 *= rsc[r1];
      }
      const uint32_t b0 = movm_t(pack_bf16(p00, p01));
      const uint32_t b1 = movm_t(pack_bf16(p10, p11));
      const int mi = lane >> 3, ii = lane & 7;
      const int row = w * 16 + ii + ((mi >> 1) << 3);
#pragma unroll
      for (int mt = 0; mt < KS; ++mt) {
        const int ch = 2 * mt + (mi & 1);
        uint32_t a0, a1_, a2_, a3_;
        ldsm_x4_t(a0, a1_, a2_, a3_, sbase + row * ROWB + ((ch ^ (row & 7)) << 4));
        mma16816(oacc[mt], a0, a1_, a2_, a3_, b0, b1);
      }
    };
    auto stage_t2 = [&](int tv0, bool isV) {   // int8 codes -> exact bf16 (canonical codes, swizzled in SMEM)
      const int8_t* C2 = (isV ? v.c2v[cur] : v.c2k[cur]) + grp * v.cap2 * D;
      const float* S2 = (isV ? v.s2v[cur] : v.s2k[cur]) + grp * v.cap2;
      for (int e = tid; e < TILE * (D / 16); e += NCONS) {
        const int row = e / (D / 16), j = e % (D / 16);
        const int tok = tv0 + row;
        uint4 cw = make_uint4(0u, 0u, 0u, 0u);
        if (tok < t2end) cw = *reinterpret_cast<const uint4*>(C2 + (size_t)(tok - a2) * D + 16 * j);
        uint4 lo, hi;
        lo.x = i8pair_to_bf16x2(cw.x, 0); lo.y = i8pair_to_bf16x2(cw.x, 1);
        lo.z = i8pair_to_bf16x2(cw.y, 0); lo.w = i8pair_to_bf16x2(cw.y, 1);
        hi.x = i8pair_to_bf16x2(cw.z, 0); hi.y = i8pair_to_bf16x2(cw.z, 1);
        hi.z = i8pair_to_bf16x2(cw.w, 0); hi.w = i8pair_to_bf16x2(cw.w, 1);
        *reinterpret_cast<uint4*>(t2buf + row * ROWB + (((2 * j) ^ (row & 7)) << 4)) = lo;
        *reinterpret_cast<uint4*>(t2buf + row * ROWB + (((2 * j + 1) ^ (row & 7)) << 4)) = hi;
      }
      for (int row = tid; row < TILE; row += NCONS) {
        const int tok = tv0 + row;
        t2sc[row] = tok < t2end ? S2[tok - a2] : 0.f;
      }
    };

    // ---- phase A on T2 rows (rare; synchronous, consumer barrier 1)
    for (int tv0 = t2beg; tv0 < t2end; tv0 += TILE) {
      named_sync(1, NCONS);
      stage_t2(tv0, false);
      named_sync(1, NCONS);
      qk_warp(smem_u32(t2buf), tv0, t2end, t2sc, true);
    }
    // ---- phase A on the new token (CUDA cores, fp32): warp 0 computes all heads' logits
    if (has_new) named_sync(1, NCONS);   // nrow visible
    if (has_new && w == 0) {
      float part = 0.f;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        const int d0 = ks * 16 + 2 * tq;
        part += bf16lo(qf[ks][0]) * nrow[d0] + bf16hi(qf[ks][0]) * nrow[d0 + 1];
        part += bf16lo(qf[ks][1]) * nrow[d0 + 8] + bf16hi(qf[ks][1]) * nrow[d0 + 9];
      }
      part += __shfl_xor_sync(0xffffffffu, part, 1);
      part += __shfl_xor_sync(0xffffffffu, part, 2);
      if (tq == 0) zs[(a3 - vbeg) * 8 + gq] = part * sl2;
    }

    auto write_warp_max = [&]() {
      float a = mx0, c = mx1;
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        a = fmaxf(a, __shfl_xor_sync(0xffffffffu, a, off));
        c = fmaxf(c, __shfl_xor_sync(0xffffffffu, c, off));
      }
      if (lane < 4) {
        red[w * 8 + 2 * lane] = a;
        red[w * 8 + 2 * lane + 1] = c;
      }
    };
    auto reduce_max = [&]() {   // after a consumer barrier: CTA max incl. the new token
      float nz0 = -INFINITY, nz1 = -INFINITY;
      if (has_new) {
        nz0 = zs[(a3 - vbeg) * 8 + 2 * tq];
        nz1 = zs[(a3 - vbeg) * 8 + 2 * tq + 1];
      }
      m2a = nz0;
      m2b = nz1;
#pragma unroll
      for (int ww = 0; ww < NW; ++ww) {
        m2a = fmaxf(m2a, red[ww * 8 + 2 * tq]);
        m2b = fmaxf(m2b, red[ww * 8 + 2 * tq + 1]);
      }
      if (tid < 8) {
        float m = has_new ? zs[(a3 - vbeg) * 8 + tid] : -INFINITY;
#pragma unroll
        for (int ww = 0; ww < NW; ++ww) m = fmaxf(m, red[ww * 8 + tid]);
        xm[tid] = m;
      }
      if (m2a == -INFINITY) m2a = 0.f;
      if (m2b == -INFINITY) m2b = 0.f;
    };

    // ---- phases A (K tiles) and B (V tiles) from the bulk-copy ring
    for (int i = 0; i < total; ++i) {
      const int s2 = i % NST;
      if (i == nt) {                 // every warp's max of phase A is in `red`
        named_sync(1, NCONS);
        reduce_max();
      }
      mbar_wait(full0 + 8 * s2, (i / NST) & 1);
      if (tr && tid == 0 && i == 0) tr[2] = gtimer();
      if (tr && tid == 0 && i == nt) tr[3] = gtimer();
      const uint32_t sbase = ring_s + s2 * TILEB;
      if (i < nt) {
        qk_warp(sbase, vbeg + i * TILE, aend, nullptr, false);
        if (i == nt - 1) write_warp_max();
      } else {
        pv_warp(sbase, vbeg + (i - nt) * TILE, aend, nullptr, false);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty0 + 8 * s2);
    }
    if (nt == 0) {
      write_warp_max();
      named_sync(1, NCONS);
      reduce_max();
    }
    // ---- phase B on T2 rows
    for (int tv0 = t2beg; tv0 < t2end; tv0 += TILE) {
      named_sync(1, NCONS);
      stage_t2(tv0, true);
      named_sync(1, NCONS);
      pv_warp(smem_u32(t2buf), tv0, t2end, t2sc, true);
    }
    // ---- phase B on the new token: rank-1 update of warp 0's o^T fragments
    if (has_new && w == 0) {
      const float* zr = zs + (a3 - vbeg) * 8;
      const float pa = exp2f(zr[2 * tq] - m2a), pb = exp2f(zr[2 * tq + 1] - m2b);
      if (gq == 0) { l0 += pa; l1 += pb; }          // counted once per head (lanes 0..3)
#pragma unroll
      for (int mt = 0; mt < KS; ++mt) {
        const float va = nrow[D + mt * 16 + gq], vb = nrow[D + mt * 16 + gq + 8];
        oacc[mt][0] += pa * va;
        oacc[mt][1] += pb * va;
        oacc[mt][2] += pa * vb;
        oacc[mt][3] += pb * vb;
      }
    }
#pragma unroll
    for (int off = 4; off < 32; off <<= 1) {
      l0 += __shfl_xor_sync(0xffffffffu, l0, off);
      l1 += __shfl_xor_sync(0xffffffffu, l1, off);
    }
  }

  // ---- CTA reduction of l and o (ring reused as [NW warps][8 heads][D+4] fp32, padded rows)
  if (tr && tid == 0) tr[4] = gtimer();
  constexpr int OWS = D + 4;
  __syncthreads();
  float* ow = reinterpret_cast<float*>(ring);
  if (w < NW) {
    if (lane < 4) {
      red[8 * NW + w * 8 + 2 * lane] = l0;
      red[8 * NW + w * 8 + 2 * lane + 1] = l1;
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
  }
  __syncthreads();
  for (int e = tid; e < G * D; e += NTHR) {
    const int h = e / D, dd = e - h * D;
    float a = ow[h * OWS + dd];
#pragma unroll
    for (int ww = 1; ww < NW; ++ww) a += ow[(ww * 8 + h) * OWS + dd];
    xo[e] = a;
  }
  if (tid < 8) {
    float a = red[8 * NW + tid];
#pragma unroll
    for (int ww = 1; ww < NW; ++ww) a += red[8 * NW + ww * 8 + tid];
    xl[tid] = a;
  }

  // ---- cluster merge through distributed shared memory (all remote reads issued in parallel)
  cluster.sync();
  if (tr && tid == 0) tr[5] = gtimer();
  float* gm = ow;                 // [16][8] peers' m    (ring is free now)
  float* gl = ow + 128;           // [16][8] peers' l
  float* gf = ow + 256;           // [16][8] merge factors exp2(m_c - M) / L
  if (tid < 8 * C) {
    const int c = tid >> 3, h = tid & 7;
    gm[tid] = cluster.map_shared_rank(xm, c)[h];
    gl[tid] = cluster.map_shared_rank(xl, c)[h];
  }
  __syncthreads();
  if (tid < 8) {
    float M = -INFINITY;
    for (int c = 0; c < C; ++c) M = fmaxf(M, gm[c * 8 + tid]);
    float Ls = 0.f;
    for (int c = 0; c < C; ++c) {
      const float mc = gm[c * 8 + tid];
      if (mc != -INFINITY) Ls += gl[c * 8 + tid] * exp2f(mc - M);
    }
    sML[tid] = M;
    sML[8 + tid] = 1.0f / Ls;
  }
  __syncthreads();
  if (tid < 8 * C) {
    const int h = tid & 7;
    const float mc = gm[tid];
    gf[tid] = mc == -INFINITY ? 0.f : exp2f(mc - sML[h]) * sML[8 + h];
  }
  __syncthreads();
  {
    const int tot = G * D;
    const int per = (tot + C - 1) / C;
    const int e1 = min(tot, (r + 1) * per);
    for (int e = r * per + tid; e < e1; e += NTHR) {
      const int h = e / D;
      float part[16];
#pragma unroll
      for (int c = 0; c < 16; ++c)
        if (c < C) part[c] = cluster.map_shared_rank(xo, c)[e];
      float acc = 0.f;
#pragma unroll
      for (int c = 0; c < 16; ++c)
        if (c < C) acc += gf[c * 8 + h] * part[c];
      const int dd = e - h * D;
      const size_t oi = ((size_t)b * v.Hq + g * G + h) * D + dd;
      if (v.out_fp32) reinterpret_cast<float*>(o)[oi] = acc;
      else reinterpret_cast<__nv_bfloat16*>(o)[oi] = __float2bfloat16_rn(acc);
    }
  }
  // done reading peers' shared memory: arrive now, wait before exit (score work overlaps)
  if (tr && tid == 0) tr[6] = gtimer();
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  if (fuse && w < NW) {
    cp_wait<0>();                    // this thread's S_part values are in sS
    float* Sg = v.S + ((size_t)b * v.Hkv + g) * v.Nmax;
    bool bad = false;
    for (int j = tid; j < vend - vbeg; j += NCONS) {
      const int pos = spos[j];
      if (pos < 0) continue;
      const float* zr = zs + j * 8;
      float inc = 0.f;
      for (int h = 0; h < G; ++h) inc += exp2f(zr[h] - sML[h]) * sML[8 + h];
      Sg[pos] = sS[j] + inc;
      bad |= !isfinite(inc);
    }
    if (bad) atomicOr(&v.st->err, 1);
  }
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  if (tr && tid == 0) tr[7] = gtimer();
}

// (warps, stages) variants; DevView::variant selects one (0 = default)
struct Variant { int nw, nst; };
static constexpr Variant kVariants[] = {{4, 4}, {4, 6}, {8, 3}, {8, 4}, {4, 5}, {8, 6}};
constexpr int kNumVariants = sizeof(kVariants) / sizeof(kVariants[0]);

size_t attn_smem_bytes(const DevView& v) {
  const Variant vr = kVariants[v.variant];
  const int tile = 16 * vr.nw;
  const size_t ringb = (size_t)vr.nst * tile * v.D * 2 + (2 * vr.nst + 2) * 8;
  const size_t zsb = (size_t)v.chunk_max * 8 * 4 + (size_t)v.chunk_max * 8;
  const size_t xob = (size_t)8 * v.D * 4;
  const size_t misc = (size_t)(8 + 8 + 16 * vr.nw + 16 + 2 * v.D + tile) * 4;
  const size_t t2 = (v.cap2 > 0) ? (size_t)tile * v.D * 2 : 0;
  return ringb + zsb + xob + misc + t2;
}

template <int D, int NW, int NST>
static cudaError_t configure_k(const DevView& v) {
  cudaError_t e = cudaFuncSetAttribute(k_decode_attn<D, NW, NST>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)attn_smem_bytes(v));
  if (e != cudaSuccess) return e;
  if (v.split > 8)
    e = cudaFuncSetAttribute(k_decode_attn<D, NW, NST>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  return e;
}

template <int D, int NW, int NST>
static cudaError_t launch_k(const DevView& v, cudaLaunchConfig_t& cfg, int layer, const void* q, const void* knew,
                            const void* vnew, void* o, int fuse) {
  cfg.blockDim = dim3((NW + 1) * 32, 1, 1);
  return cudaLaunchKernelEx(&cfg, k_decode_attn<D, NW, NST>, v, layer, reinterpret_cast<const __nv_bfloat16*>(q),
                            reinterpret_cast<const __nv_bfloat16*>(knew), reinterpret_cast<const __nv_bfloat16*>(vnew),
                            o, fuse);
}

#define KVT_VARIANTS(X, D) X(D, 4, 4) X(D, 4, 6) X(D, 8, 3) X(D, 8, 4) X(D, 4, 5) X(D, 8, 6)

cudaError_t attn_configure(const DevView& v) {
  if (v.variant < 0 || v.variant >= kNumVariants) return cudaErrorInvalidValue;
  const Variant vr = kVariants[v.variant];
#define KVT_CONF(DD, NWW, NSS) \
  if (v.D == DD && vr.nw == NWW && vr.nst == NSS) return configure_k<DD, NWW, NSS>(v);
  KVT_VARIANTS(KVT_CONF, 128)
  KVT_VARIANTS(KVT_CONF, 64)
#undef KVT_CONF
  return cudaErrorInvalidValue;
}

cudaError_t launch_decode_attn(const DevView& v, int layer, const void* q, const void* knew, const void* vnew,
                               void* o, int fuse, int pdl, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(v.split, v.B * v.Hkv, 1);
  cfg.dynamicSmemBytes = attn_smem_bytes(v);
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = v.split;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl ? 2 : 1;
  const Variant vr = kVariants[v.variant];
#define KVT_LAUNCH(DD, NWW, NSS) \
  if (v.D == DD && vr.nw == NWW && vr.nst == NSS) return launch_k<DD, NWW, NSS>(v, cfg, layer, q, knew, vnew, o, fuse);
  KVT_VARIANTS(KVT_LAUNCH, 128)
  KVT_VARIANTS(KVT_LAUNCH, 64)
#undef KVT_LAUNCH
  return cudaErrorInvalidValue;
}

}  // namespace kvt
