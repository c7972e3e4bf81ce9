// PTX helpers, the virtual-token layout and the deferred score pass shared by the decode
// kernels of libkvtier.so (attn.cu: split-per-unit kernel, attn_flat.cu: flat kernel).
#pragma once
#include "kv_internal.cuh"

namespace kvt {

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
// wait with a suspend-time hint (ns): the thread sleeps until the phase completes or the hint
// expires instead of re-polling the barrier
__device__ __forceinline__ void mbar_wait_hint(uint32_t a, uint32_t parity, uint32_t hint_ns) {
  uint32_t ok = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok)
                 : "r"(a), "r"(parity), "r"(hint_ns)
                 : "memory");
  } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar) : "memory");
}
// L2 prefetch of a contiguous byte range (no shared-memory destination)
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}
// streamed K/V rows are read once per layer: evict them first so the hot data stays in L2
__device__ __forceinline__ uint64_t evict_first_policy() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_ef(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar, uint64_t pol) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(mbar), "l"(pol) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ int ru16(int x) { return (x + 15) & ~15; }

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
// register-only: not volatile, so the scheduler may overlap it with later shared-memory loads
__device__ __forceinline__ void mma16816(float* c, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// 2^x on the SFU without the subnormal range fix-up exp2f adds (results below 2^-126 flush to
// 0: p of a token 126 log2 units under the running max is below fp32 resolution of l anyway)
__device__ __forceinline__ float ex2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t movm_t(uint32_t x) {
  uint32_t y;
  asm("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;\n" : "=r"(y) : "r"(x));
  return y;
}
// p (fp32) as the B operand of o^T += V^T p^T in two bf16 terms, p ~= hi + lo with
// hi = bf16(p), lo = bf16(p - hi): the P.V product keeps ~16 mantissa bits of p instead of 8
// (a lone bf16 p costs up to 2^-9 relative per term: 2.4e-3 abs at |v| ~ 4 for a dominant token).
__device__ __forceinline__ void split_bf16x2(float x, float y, uint32_t& hi, uint32_t& lo) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(x, y);
  const float2 hf = __bfloat1622float2(h);
  const __nv_bfloat162 l = __floats2bfloat162_rn(x - hf.x, y - hf.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
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

// ----------------------------------------------------------------- tcgen05 (UMMA) + TMEM, sm_100a
// Operands in shared memory in the 128-byte swizzle atom the stores use (kv_internal.cuh):
// 8-row groups of 2 KB ([8 rows x 128 B column block 0 | column block 1]), chunk c of row j at
// c ^ (j & 7).  Conventions checked on a B200 by scripts/micro/umma_check.cu:
//   K-major operand (contiguous dim = the MMA's K): LBO 16, SBO 2048, the k-th 16-element step
//     starts at (k >> 2) * 1024 + (k & 3) * 32;
//   MN-major operand (contiguous dim = M): the k-th 16-row step starts at k * 4096, LBO 1024,
//     SBO 2048.
// Shared-memory matrix descriptor: start >> 4 [0,14), LBO >> 4 [16,30), SBO >> 4 [32,46),
// version 1 [46,48), layout SWIZZLE_128B (2) [61,64).
__device__ __forceinline__ uint64_t umma_sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
// instruction descriptor of kind::f16: fp32 accumulate, bf16 A and B, operand majors, N, M
__host__ __device__ constexpr uint32_t umma_idesc(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
               " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
               ::"r"(tmem_d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// mbarrier arrive (one) when every previously issued tcgen05.mma of this thread has completed
__device__ __forceinline__ void umma_commit(uint32_t mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(mbar) : "memory");
}
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
// 32 lanes x 8 / 16 consecutive 32-bit columns; warp w of the CTA reads lanes 32 (w % 4) + lane
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(taddr));
}
__device__ __forceinline__ void fence_proxy_async_cta() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// Virtual-token bookkeeping shared by the decode kernel and the score pass.
struct Seg {
  int n0o, n1, n2, a1, a2, a3, nvirt, nn;
  // nn: the step's new token is the last T0 row of this ctx (DevState::nn)
  // skip1: host-T1 mode: the host cores attend T1, the GPU skips it
  __device__ __forceinline__ void init(const int* cn, int nn_ = 1, int skip1 = 0) {
    nn = nn_;
    n0o = cn[0] - nn;
    n1 = skip1 ? 0 : cn[1];
    n2 = cn[2];
    a1 = ru16(n0o);
    a2 = ru16(a1 + n1);
    a3 = ru16(a2 + n2);
    nvirt = a3 + 1;
  }
  __device__ __forceinline__ bool bf16_valid(int t) const { return t < n0o || (t >= a1 && t < a1 + n1); }
  __device__ __forceinline__ bool valid(int t) const {
    return t < n0o || (t >= a1 && t < a1 + n1) || (t >= a2 && t < a2 + n2) || (nn && t == a3);
  }
  // position of virtual token t (valid t only)
  __device__ __forceinline__ int pos(const DevView& v, int cur, int b, int t) const {
    if (t < n0o) return v.idx[cur][0][(size_t)b * v.cap0 + t];
    if (t < a2) return v.idx[cur][1][(size_t)b * v.cap1 + (t - a1)];
    if (t < a3) return v.idx[cur][2][(size_t)b * v.cap2 + (t - a2)];
    return v.idx[cur][0][(size_t)b * v.cap0 + n0o];
  }
};

// Score pass over virtual tokens [i0, i1) of the flattened (unit, token) space for nz <= ZBATCH
// consecutive launches (ring slots zfirst, zfirst+1, ...), applied in launch (= layer) order:
// S <- fp32(S + inc_l) per launch, the same adds one pass per launch would do.  Every load of a
// token batch is hoisted (three dependent round trips: position, then S_part + logits, then
// the store).
__device__ __forceinline__ void score_range(const DevView& v, const Seg& sg, int cur, int zfirst, int nz,
                                            long long i0, long long i1, int lane0, int stride, bool& bad) {
  constexpr int SB = 8 / ZBATCH;
  const size_t zslot = (size_t)v.B * v.Hkv * v.zrows * 8, mslot = (size_t)v.B * v.Hkv * 16;
  for (long long base = i0 + lane0; base < i1; base += (long long)stride * SB) {
    int pos[SB], uu[SB], tt[SB];
#pragma unroll
    for (int k = 0; k < SB; ++k) {
      const long long i = base + (long long)k * stride;
      pos[k] = -1;
      uu[k] = 0;
      tt[k] = 0;
      if (i < i1) {
        const int u = (int)(i / sg.nvirt), t = (int)(i - (long long)u * sg.nvirt);
        uu[k] = u;
        tt[k] = t;
        if (sg.valid(t)) pos[k] = sg.pos(v, cur, u / v.Hkv, t);
      }
    }
    float sv[SB];
    float4 z0[SB][ZBATCH], z1[SB][ZBATCH];
#pragma unroll
    for (int k = 0; k < SB; ++k) {
      if (pos[k] >= 0) {
        sv[k] = v.S[(size_t)uu[k] * v.Nmax + pos[k]];     // S_part[b][g] rows are unit-major
#pragma unroll
        for (int j = 0; j < ZBATCH; ++j) {
          if (j < nz) {
            const int slot = zslot_of(v, zfirst + j);
            const float* z = v.zbuf + slot * zslot + ((size_t)uu[k] * v.zrows + tt[k]) * 8;
            z0[k][j] = *reinterpret_cast<const float4*>(z);
            z1[k][j] = *reinterpret_cast<const float4*>(z + 4);
          }
        }
      }
    }
#pragma unroll
    for (int k = 0; k < SB; ++k) {
      if (pos[k] < 0) continue;
      float s = sv[k];
#pragma unroll
      for (int j = 0; j < ZBATCH; ++j) {
        if (j >= nz) break;
        const int slot = zslot_of(v, zfirst + j);
        const float wgt = score_weight(v, v.scorer ? v.zlayer[slot] : 0, uu[k], pos[k]);
        const float* ml = v.ml + slot * mslot + (size_t)uu[k] * 16;
        const float zz[8] = {z0[k][j].x, z0[k][j].y, z0[k][j].z, z0[k][j].w,
                             z1[k][j].x, z1[k][j].y, z1[k][j].z, z1[k][j].w};
        float inc = 0.f;
#pragma unroll
        for (int h = 0; h < 8; ++h)
          if (h < v.G) inc += ex2_ftz(zz[h] - ml[h]) * ml[8 + h];
        s = s + inc * wgt;
        bad |= !isfinite(inc);
      }
      v.S[(size_t)uu[k] * v.Nmax + pos[k]] = s;
    }
  }
}

}  // namespace kvt
