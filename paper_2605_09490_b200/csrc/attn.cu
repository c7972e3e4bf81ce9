// a1 + a3 + a4: fused new-token append, GQA decode attention over the visible tiers, and the
// cumulative score update (Eq. 1, Eq. 3, Prop. 1).
//
// One thread-block cluster of C CTAs per (request b, kv head g).  The visible rows of the
// unit are ordered [T0 rows except the new token | T1 staging | T2 int8 | new token]; CTA r
// of the cluster owns a contiguous 1/C chunk.
//
//   prologue  (before griddepcontrol.wait, overlaps the previous layer's kernel under PDL)
//            counters, positions of the chunk -> SMEM, first K tiles in flight
//   phase A  K tiles (cp.async ring, XOR-swizzled SMEM) -> S^T = K q^T on the tensor cores
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

// Variants (warps per CTA NW, pipeline stages NST): a tile is 16 tokens per warp.

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
__global__ void __launch_bounds__(NW * 32, (NW == 4 ? 3 : 2))
    k_decode_attn(const DevView v, const int layer, const __nv_bfloat16* __restrict__ q,
                  const __nv_bfloat16* __restrict__ knew, const __nv_bfloat16* __restrict__ vnew,
                  void* __restrict__ o, const int fuse) {
  constexpr int ATT_THREADS = NW * 32;
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

  extern __shared__ __align__(128) unsigned char smem[];
  unsigned char* ring = smem;
  float* zs = reinterpret_cast<float*>(smem + NST * TILEB);   // [chunk_max][8] logits (log2)
  int* spos = reinterpret_cast<int*>(zs + (size_t)v.chunk_max * 8);   // [chunk_max] positions
  float* xo = reinterpret_cast<float*>(spos + v.chunk_max);    // [8][D]  exchange: o partial
  float* xm = xo + 8 * D;                                      // [8]     exchange: max (log2)
  float* xl = xm + 8;                                          // [8]     exchange: sum
  float* red = xl + 8;                                         // [2][NW][8] warp max / warp l
  float* sML = red + 16 * NW;                                  // [16] merged M, 1/L
  float* nrow = sML + 16;                                      // [2][D] new token K, V (fp32)
  float* t2sc = nrow + 2 * D;                                  // [TILE] T2 row scales
  unsigned char* t2buf = reinterpret_cast<unsigned char*>(t2sc + TILE);   // [TILE][D] bf16

  // ---------------------------------------------------------------- prologue (pre-PDL-wait)
  const int cur = v.st->cur;
  const int* cn = v.cnt[cur] + b * CNT_STRIDE;
  const int n0 = cn[0], n1 = cn[1], n2 = cn[2];
  const int n0o = n0 - 1;                           // T0 rows before the new token
  const int n01 = n0o + n1, n012 = n01 + n2, nvis = n012 + 1;
  const int chunk = (nvis + C - 1) / C;
  const int vbeg = min(r * chunk, nvis), vend = min(vbeg + chunk, nvis);
  const int aend = min(vend, n01);                  // bf16 segment [vbeg, aend)
  const int t2beg = max(vbeg, n01), t2end = min(vend, n012);   // int8 segment
  const bool has_new = vend == nvis && nvis > vbeg; // this CTA owns the new token
  const int nb = max(0, aend - vbeg);
  const int nt = (nb + TILE - 1) / TILE;

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

  auto load_tile = [&](int i) {
    const bool isV = i >= nt;
    const int tv0 = vbeg + (isV ? i - nt : i) * TILE;
    const __nv_bfloat16* S0 = isV ? V0 : K0;
    const __nv_bfloat16* S1 = isV ? V1 : K1;
    const uint32_t sbase = smem_u32(ring + (i % NST) * TILEB);
    constexpr int CPR = D / 8;                // 16-B chunks per row
    constexpr int RPP = ATT_THREADS / CPR;    // rows per pass
    const int c = tid % CPR, r0 = tid / CPR;
#pragma unroll
    for (int p = 0; p < TILE / RPP; ++p) {
      const int row = r0 + p * RPP;
      const int tok = tv0 + row;
      const __nv_bfloat16* src = S0;
      int nbytes = 0;
      if (tok < aend) {
        nbytes = 16;
        src = tok < n0o ? S0 + (size_t)tok * D : S1 + (size_t)(tok - n0o) * D;
      }
      cp_async16(sbase + row * ROWB + ((c ^ (row & 7)) << 4), src + c * 8, nbytes);
    }
  };
  const int total = 2 * nt;
#pragma unroll
  for (int s = 0; s < NST - 1; ++s) {
    if (s < total) load_tile(s);
    cp_commit();
  }
  // positions of the chunk's tokens (for the score update)
  if (fuse) {
    const int* I0 = v.idx[cur][0] + (size_t)b * v.cap0;
    const int* I1 = v.idx[cur][1] + (size_t)b * v.cap1;
    const int* I2 = v.idx[cur][2] + (size_t)b * v.cap2;
    for (int j = tid; j < vend - vbeg; j += ATT_THREADS) {
      const int tok = vbeg + j;
      spos[j] = tok < n0o ? I0[tok] : tok < n01 ? I1[tok - n0o] : tok < n012 ? I2[tok - n01] : I0[n0o];
    }
  }
  pdl_trigger();
  // ---------------------------------------------------------------- dependent inputs
  pdl_wait();

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

  // new token (a1): append its K/V row to T0 row n0-1 and keep it in SMEM (fp32)
  if (has_new) {
    uint16_t* K0w = reinterpret_cast<uint16_t*>(v.k0[cur]) + (grp * v.cap0 + n0o) * D;
    uint16_t* V0w = reinterpret_cast<uint16_t*>(v.v0[cur]) + (grp * v.cap0 + n0o) * D;
    const uint16_t* ks_ = knew ? reinterpret_cast<const uint16_t*>(knew) + ((size_t)b * v.Hkv + g) * D : K0w;
    const uint16_t* vs_ = vnew ? reinterpret_cast<const uint16_t*>(vnew) + ((size_t)b * v.Hkv + g) * D : V0w;
    for (int e = tid; e < D; e += ATT_THREADS) {
      const uint16_t kb = ks_[e], vb = vs_[e];
      nrow[e] = bf16_bits_to_f(kb);
      nrow[D + e] = bf16_bits_to_f(vb);
      if (knew) K0w[e] = kb;
      if (vnew) V0w[e] = vb;
    }
  }

  float mx0 = -INFINITY, mx1 = -INFINITY;    // running max, heads 2tq, 2tq+1
  float l0 = 0.f, l1 = 0.f;
  float oacc[KS][4];
#pragma unroll
  for (int mt = 0; mt < KS; ++mt) oacc[mt][0] = oacc[mt][1] = oacc[mt][2] = oacc[mt][3] = 0.f;

  auto qk_warp = [&](uint32_t sbase, int tv0, int tend, const float* rsc) {
    if (tv0 + w * 16 >= tend) return;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    const int mi = lane >> 3, ii = lane & 7;
    const int row = w * 16 + ii + ((mi & 1) << 3);
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int ch = 2 * ks + (mi >> 1);
      uint32_t a0, a1, a2, a3;
      ldsm_x4(a0, a1, a2, a3, sbase + row * ROWB + ((ch ^ (row & 7)) << 4));
      mma16816(acc, a0, a1, a2, a3, qf[ks][0], qf[ks][1]);
    }
    const int r0 = w * 16 + gq, r1 = r0 + 8;
    const int t0 = tv0 + r0, t1 = tv0 + r1;
    if (t0 < tend) {
      const float f = rsc ? rsc[r0] * sl2 : sl2;
      const float z0 = acc[0] * f, z1 = acc[1] * f;
      *reinterpret_cast<float2*>(&zs[(t0 - vbeg) * 8 + 2 * tq]) = make_float2(z0, z1);
      mx0 = fmaxf(mx0, z0);
      mx1 = fmaxf(mx1, z1);
    }
    if (t1 < tend) {
      const float f = rsc ? rsc[r1] * sl2 : sl2;
      const float z0 = acc[2] * f, z1 = acc[3] * f;
      *reinterpret_cast<float2*>(&zs[(t1 - vbeg) * 8 + 2 * tq]) = make_float2(z0, z1);
      mx0 = fmaxf(mx0, z0);
      mx1 = fmaxf(mx1, z1);
    }
  };
  float m2a = 0.f, m2b = 0.f;   // CTA max for heads 2tq, 2tq+1
  auto pv_warp = [&](uint32_t sbase, int tv0, int tend, const float* rsc) {
    if (tv0 + w * 16 >= tend) return;
    const int r0 = w * 16 + gq, r1 = r0 + 8;
    const int t0 = tv0 + r0, t1 = tv0 + r1;
    float p00 = 0.f, p01 = 0.f, p10 = 0.f, p11 = 0.f;
    if (t0 < tend) {
      const float2 z = *reinterpret_cast<const float2*>(&zs[(t0 - vbeg) * 8 + 2 * tq]);
      p00 = exp2f(z.x - m2a);
      p01 = exp2f(z.y - m2b);
    }
    if (t1 < tend) {
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
      uint32_t a0, a1, a2, a3;
      ldsm_x4_t(a0, a1, a2, a3, sbase + row * ROWB + ((ch ^ (row & 7)) << 4));
      mma16816(oacc[mt], a0, a1, a2, a3, b0, b1);
    }
  };
  auto stage_t2 = [&](int tv0, bool isV) {
    const int8_t* C2 = (isV ? v.c2v[cur] : v.c2k[cur]) + grp * v.cap2 * D;
    const float* S2 = (isV ? v.s2v[cur] : v.s2k[cur]) + grp * v.cap2;
    for (int e = tid; e < TILE * (D / 16); e += ATT_THREADS) {
      const int row = e / (D / 16), j = e % (D / 16);
      const int tok = tv0 + row;
      uint4 cw = make_uint4(0u, 0u, 0u, 0u);
      if (tok < t2end) cw = *reinterpret_cast<const uint4*>(C2 + (size_t)(tok - n01) * D + 16 * j);
      uint4 lo, hi;
      lo.x = i8pair_to_bf16x2(cw.x, 0); lo.y = i8pair_to_bf16x2(cw.x, 1);
      lo.z = i8pair_to_bf16x2(cw.y, 0); lo.w = i8pair_to_bf16x2(cw.y, 1);
      hi.x = i8pair_to_bf16x2(cw.z, 0); hi.y = i8pair_to_bf16x2(cw.z, 1);
      hi.z = i8pair_to_bf16x2(cw.w, 0); hi.w = i8pair_to_bf16x2(cw.w, 1);
      *reinterpret_cast<uint4*>(t2buf + row * ROWB + (((2 * j) ^ (row & 7)) << 4)) = lo;
      *reinterpret_cast<uint4*>(t2buf + row * ROWB + (((2 * j + 1) ^ (row & 7)) << 4)) = hi;
    }
    for (int row = tid; row < TILE; row += ATT_THREADS) {
      const int tok = tv0 + row;
      t2sc[row] = tok < t2end ? S2[tok - n01] : 0.f;
    }
  };

  // ---- phase A on T2 rows (rare; synchronous)
  for (int tv0 = t2beg; tv0 < t2end; tv0 += TILE) {
    __syncthreads();
    stage_t2(tv0, false);
    __syncthreads();
    qk_warp(smem_u32(t2buf), tv0, t2end, t2sc);
  }
  // ---- phase A on the new token (CUDA cores, fp32): warp 0 computes all G logits
  __syncthreads();   // nrow visible
  if (has_new && w == 0) {
    float part = 0.f;   // head gq, dims of this lane's q fragments
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int d0 = ks * 16 + 2 * tq;
      part += bf16lo(qf[ks][0]) * nrow[d0] + bf16hi(qf[ks][0]) * nrow[d0 + 1];
      part += bf16lo(qf[ks][1]) * nrow[d0 + 8] + bf16hi(qf[ks][1]) * nrow[d0 + 9];
    }
    part += __shfl_xor_sync(0xffffffffu, part, 1);
    part += __shfl_xor_sync(0xffffffffu, part, 2);
    if (tq == 0) zs[(nvis - 1 - vbeg) * 8 + gq] = part * sl2;
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
  auto reduce_max = [&]() {   // after a barrier: CTA max incl. the new token
    float nz0 = -INFINITY, nz1 = -INFINITY;
    if (has_new) {
      nz0 = zs[(nvis - 1 - vbeg) * 8 + 2 * tq];
      nz1 = zs[(nvis - 1 - vbeg) * 8 + 2 * tq + 1];
    }
    m2a = nz0;
    m2b = nz1;
#pragma unroll
    for (int ww = 0; ww < NW; ++ww) {
      m2a = fmaxf(m2a, red[ww * 8 + 2 * tq]);
      m2b = fmaxf(m2b, red[ww * 8 + 2 * tq + 1]);
    }
    if (tid < 8) {
      float m = has_new ? zs[(nvis - 1 - vbeg) * 8 + tid] : -INFINITY;
#pragma unroll
      for (int ww = 0; ww < NW; ++ww) m = fmaxf(m, red[ww * 8 + tid]);
      xm[tid] = m;
    }
    if (m2a == -INFINITY) m2a = 0.f;
    if (m2b == -INFINITY) m2b = 0.f;
  };

  // ---- phases A (K tiles) and B (V tiles) through the cp.async ring
  for (int i = 0; i < total; ++i) {
    cp_wait<NST - 2>();
    __syncthreads();
    if (i + NST - 1 < total) load_tile(i + NST - 1);
    cp_commit();
    if (i == nt) reduce_max();
    const uint32_t sbase = smem_u32(ring + (i % NST) * TILEB);
    if (i < nt) {
      qk_warp(sbase, vbeg + i * TILE, aend, nullptr);
      if (i == nt - 1) write_warp_max();
    } else {
      pv_warp(sbase, vbeg + (i - nt) * TILE, aend, nullptr);
    }
  }
  cp_wait<0>();
  if (nt == 0) {
    write_warp_max();
    __syncthreads();
    reduce_max();
  }
  // ---- phase B on T2 rows
  for (int tv0 = t2beg; tv0 < t2end; tv0 += TILE) {
    __syncthreads();
    stage_t2(tv0, true);
    __syncthreads();
    pv_warp(smem_u32(t2buf), tv0, t2end, t2sc);
  }
  // ---- phase B on the new token: rank-1 update of this thread's o^T fragments
  if (has_new && w == 0) {
    const float* zr = zs + (nvis - 1 - vbeg) * 8;
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

  // ---- CTA reduction of l and o (ring reused as [NW warps][8 heads][D] fp32)
#pragma unroll
  for (int off = 4; off < 32; off <<= 1) {
    l0 += __shfl_xor_sync(0xffffffffu, l0, off);
    l1 += __shfl_xor_sync(0xffffffffu, l1, off);
  }
  __syncthreads();
  float* ow = reinterpret_cast<float*>(ring);
  if (lane < 4) {
    red[8 * NW + w * 8 + 2 * lane] = l0;
    red[8 * NW + w * 8 + 2 * lane + 1] = l1;
  }
#pragma unroll
  for (int mt = 0; mt < KS; ++mt) {
    float* o0 = ow + (w * 8 + 2 * tq) * D + mt * 16 + gq;
    float* o1 = ow + (w * 8 + 2 * tq + 1) * D + mt * 16 + gq;
    o0[0] = oacc[mt][0];
    o1[0] = oacc[mt][1];
    o0[8] = oacc[mt][2];
    o1[8] = oacc[mt][3];
  }
  __syncthreads();
  for (int e = tid; e < 8 * D; e += ATT_THREADS) {
    float a = ow[e];
#pragma unroll
    for (int ww = 1; ww < NW; ++ww) a += ow[ww * 8 * D + e];
    xo[e] = a;
  }
  if (tid < 8) {
    float a = red[8 * NW + tid];
#pragma unroll
    for (int ww = 1; ww < NW; ++ww) a += red[8 * NW + ww * 8 + tid];
    xl[tid] = a;
  }

  // ---- cluster merge through distributed shared memory
  cluster.sync();
  if (tid < 8) {
    float M = -INFINITY;
    for (int c = 0; c < C; ++c) M = fmaxf(M, cluster.map_shared_rank(xm, c)[tid]);
    float Ls = 0.f;
    for (int c = 0; c < C; ++c) {
      const float mc = cluster.map_shared_rank(xm, c)[tid];
      if (mc != -INFINITY) Ls += cluster.map_shared_rank(xl, c)[tid] * exp2f(mc - M);
    }
    sML[tid] = M;
    sML[8 + tid] = 1.0f / Ls;
  }
  __syncthreads();
  {
    const int tot = G * D;
    const int per = (tot + C - 1) / C;
    const int e1 = min(tot, (r + 1) * per);
    for (int e = r * per + tid; e < e1; e += ATT_THREADS) {
      const int h = e / D, dd = e - h * D;
      float acc = 0.f;
      for (int c = 0; c < C; ++c) {
        const float mc = cluster.map_shared_rank(xm, c)[h];
        if (mc != -INFINITY) acc += exp2f(mc - sML[h]) * cluster.map_shared_rank(xo, c)[h * D + dd];
      }
      const float val = acc * sML[8 + h];
      const size_t oi = ((size_t)b * v.Hq + g * G + h) * D + dd;
      if (v.out_fp32) reinterpret_cast<float*>(o)[oi] = val;
      else reinterpret_cast<__nv_bfloat16*>(o)[oi] = __float2bfloat16_rn(val);
    }
  }
  // done reading peers' shared memory: arrive now, wait before exit (score work overlaps)
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  if (fuse) {
    float* Sg = v.S + ((size_t)b * v.Hkv + g) * v.Nmax;
    bool bad = false;
    for (int j = tid; j < vend - vbeg; j += ATT_THREADS) {
      const float* zr = zs + j * 8;
      float inc = 0.f;
      for (int h = 0; h < G; ++h) inc += exp2f(zr[h] - sML[h]) * sML[8 + h];
      const int pos = spos[j];
      Sg[pos] = Sg[pos] + inc;
      bad |= !isfinite(inc);
    }
    if (bad) atomicOr(&v.st->err, 1);
  }
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// (warps, stages) variants; DevView::variant selects one (0 = default)
struct Variant { int nw, nst; };
static constexpr Variant kVariants[] = {{4, 3}, {4, 4}, {8, 3}, {8, 4}, {4, 6}, {8, 6}};
constexpr int kNumVariants = sizeof(kVariants) / sizeof(kVariants[0]);

size_t attn_smem_bytes(const DevView& v) {
  const Variant vr = kVariants[v.variant];
  const int tile = 16 * vr.nw;
  const size_t ringb = (size_t)vr.nst * tile * v.D * 2;
  const size_t zsb = (size_t)v.chunk_max * 8 * 4 + (size_t)v.chunk_max * 4;
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
  cfg.blockDim = dim3(NW * 32, 1, 1);
  return cudaLaunchKernelEx(&cfg, k_decode_attn<D, NW, NST>, v, layer, reinterpret_cast<const __nv_bfloat16*>(q),
                            reinterpret_cast<const __nv_bfloat16*>(knew), reinterpret_cast<const __nv_bfloat16*>(vnew),
                            o, fuse);
}

#define KVT_VARIANTS(X, D) X(D, 4, 3) X(D, 4, 4) X(D, 8, 3) X(D, 8, 4) X(D, 4, 6) X(D, 8, 6)

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
