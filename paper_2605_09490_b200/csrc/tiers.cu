// Tier management kernels of libkvtier.so:
//   a1 append / step bookkeeping, a4 standalone score update, a5 classify
//   (radix select + compaction), a6 migrate (gather / quantise / offload), a2 stream
//   prefetch.  Citations: PAPER.md Alg. 1, §3.2-3.4 P:143-211.
#include "kv_internal.cuh"
#include <algorithm>

namespace kvt {

// ------------------------------------------------------------------ step bookkeeping
// New position n joins T0 at the end of the T0 list (ascending order is kept since
// n exceeds every stored position); it is inside the window, hence protected.
// Sequence sharding: only the rank owning position n stores it; every rank marks it T0.
__global__ void k_begin_step(const DevView v) {
  const int b = threadIdx.x;
  const int cur = v.st->cur;
  const int n = v.st->n;
  const bool own = seq_own(v.seq_w, v.seq_r, n);
  if (b < v.B) {
    int* cn = v.cnt[cur] + b * CNT_STRIDE;
    v.tier[cur][(size_t)b * v.Nmax + n] = T0;
    if (own) {
      const int r = cn[0];
      v.idx[cur][0][(size_t)b * v.cap0 + r] = n;
      v.rowof[cur][(size_t)b * v.Nmax + n] = r;
      cn[0] = r + 1;
    } else {
      v.rowof[cur][(size_t)b * v.Nmax + n] = -1;
    }
  }
  if (v.step_k > 0)                            // whole-step kernel: fresh layer counters
    for (int i = threadIdx.x; i < v.L * v.B; i += blockDim.x) v.step_done[i] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    v.st->n = n + 1;
    v.st->nn = own ? 1 : 0;
  }
}

// Windowed / R-KV scorers (AMB-32): at the start of step t with (t + w - 1) % Delta == 0,
// w = min(8, Delta), S_snap = S_part over positions [0, n), so that the event of step t + w - 1
// ranks S(after that step) - S_snap = the probability mass of its last w steps.
// Launched before k_begin_step on the step's stream (graph-static: t is read from the device).
__global__ void k_snapshot(const DevView v) {
  const int t = v.st->t, n = v.st->n;
  const int w = v.interval < RKV_ALPHA ? v.interval : RKV_ALPHA;
  if ((t + w - 1) % v.interval != 0) return;
  const size_t base = (size_t)blockIdx.y * v.Nmax;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    v.snap[base + i] = v.S[base + i];
}

__global__ void k_end_step(const DevView v) {
  if (threadIdx.x == 0) v.st->t += 1;
}

// a1: K/V row of the new token for one layer -> T0 store row |T0|-1.
__global__ void k_append(const DevView v, const int layer, const uint16_t* __restrict__ k,
                         const uint16_t* __restrict__ vv) {
  const int unit = blockIdx.x;               // b * Hkv + g
  const int b = unit / v.Hkv, g = unit % v.Hkv;
  const int cur = v.st->cur;
  if (v.red && threadIdx.x >= 32 && threadIdx.x < 64)   // redundancy: cos with the previous key (every shard)
    redund_append(v, layer, unit, v.st->n - 1, k + (size_t)unit * v.D);
  if (!v.st->nn) return;                     // another sequence shard holds the new token
  const int row = v.cnt[cur][b * CNT_STRIDE + 0] - 1;
  const size_t dst = (grp_of(v, layer, b, g) * v.cap0 + row) * v.D;
  const int sb = v.st->scur;
  uint16_t* K = reinterpret_cast<uint16_t*>(v.k0[sb]);
  uint16_t* V = reinterpret_cast<uint16_t*>(v.v0[sb]);
  for (int e = threadIdx.x; e < v.D; e += blockDim.x) {
    K[dst + swz_off(row, e, v.D)] = k[(size_t)unit * v.D + e];
    V[dst + swz_off(row, e, v.D)] = vv[(size_t)unit * v.D + e];
  }
  if (scorer_uses_vnorm(v.scorer) && threadIdx.x < 32) {   // VATP: V-row norm of the appended token
    float ss = 0.f;
    for (int e = threadIdx.x; e < v.D; e += 32) {
      const float x = bf16_bits_to_f(vv[(size_t)unit * v.D + e]);
      ss += x * x;
    }
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    if (threadIdx.x == 0) v.vnorm[((size_t)layer * v.B * v.Hkv + unit) * v.Nmax + (v.st->n - 1)] = sqrtf(ss);
  }
}

// VATP: fp32 L2 norm of every prefix token's V row of one layer (one warp per row); positions
// of a sequence shard's own rows only.
__global__ void k_vnorm_prefix(const DevView v, const int layer, const uint16_t* __restrict__ vv, const int n0) {
  const int unit = blockIdx.y, lane = threadIdx.x & 31;
  const int nown = seq_owned_below(v.seq_w, v.seq_r, n0);
  for (int j = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); j < nown; j += gridDim.x * (blockDim.x / 32)) {
    const int p = seq_pos_of(v.seq_w, v.seq_r, j);
    const uint16_t* row = vv + ((size_t)unit * n0 + p) * v.D;
    float ss = 0.f;
    for (int e = lane; e < v.D; e += 32) {
      const float x = bf16_bits_to_f(row[e]);
      ss += x * x;
    }
    for (int off = 16; off > 0; off >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, off);
    if (lane == 0) v.vnorm[((size_t)layer * v.B * v.Hkv + unit) * v.Nmax + p] = sqrtf(ss);
  }
}

// Redundancy (AMB-30): c_p = cos(k_p, k_{p-1}) of every prefix row of one layer added to R_part
// (one warp per row, c_0 = 0), and the last prefix key becomes the unit's previous key.
__global__ void k_redund_prefix(const DevView v, const int layer, const uint16_t* __restrict__ k, const int n0) {
  const int unit = blockIdx.y, lane = threadIdx.x & 31;
  for (int p = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); p < n0; p += gridDim.x * (blockDim.x / 32)) {
    const uint16_t* row = k + ((size_t)unit * n0 + p) * v.D;
    float dot = 0.f, na = 0.f, nb = 0.f;
    if (p > 0) {
      for (int e = lane; e < v.D; e += 32) {
        const float a = bf16_bits_to_f(row[e]), q = bf16_bits_to_f(row[e - v.D]);
        dot = fmaf(a, q, dot);
        na = fmaf(a, a, na);
        nb = fmaf(q, q, nb);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        dot += __shfl_xor_sync(0xffffffffu, dot, off);
        na += __shfl_xor_sync(0xffffffffu, na, off);
        nb += __shfl_xor_sync(0xffffffffu, nb, off);
      }
    }
    if (lane == 0) {
      const float c = (na > 0.f && nb > 0.f) ? __fdiv_rn(dot, __fsqrt_rn(__fmul_rn(na, nb))) : 0.f;
      float* r = v.red + (size_t)unit * v.Nmax + p;
      *r = __fadd_rn(*r, c);
    }
    if (p == n0 - 1)
      for (int e = lane; e < v.D; e += 32) v.lastk[((size_t)layer * v.B * v.Hkv + unit) * v.D + e] = row[e];
  }
}

// N1 host-T1 mode: S_part[b][g][idx1[b][j]] += inc[b][g][j] for the T1 tokens the host attended
// (inc: [B][H_kv][cap1] fp32 in mapped pinned memory, store order of the T1 index list).
__global__ void k_t1_score_add(const DevView v, const float* __restrict__ inc) {
  const int unit = blockIdx.y, b = unit / v.Hkv;
  const int cur = v.st->cur;
  const int n1 = v.cnt[cur][b * CNT_STRIDE + 1];
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n1; j += gridDim.x * blockDim.x) {
    const float x = inc[(size_t)unit * v.cap1 + j];
    float* S = v.S + (size_t)unit * v.Nmax + v.idx[cur][1][(size_t)b * v.cap1 + j];
    *S = *S + x;
    if (!isfinite(x)) atomicOr(&v.st->err, 1);
  }
}

cudaError_t launch_t1_score_add(const DevView& v, const float* inc, cudaStream_t s) {
  dim3 grid((unsigned)std::max(1, std::min(64, (v.cap1 + 255) / 256)), v.B * v.Hkv);
  k_t1_score_add<<<grid, 256, 0, s>>>(v, inc);
  return cudaGetLastError();
}

cudaError_t launch_redund_prefix(const DevView& v, int layer, const void* k, int n0, cudaStream_t s) {
  dim3 grid((unsigned)std::max(1, std::min(1024, (n0 + 7) / 8)), v.B * v.Hkv);
  k_redund_prefix<<<grid, 256, 0, s>>>(v, layer, reinterpret_cast<const uint16_t*>(k), n0);
  return cudaGetLastError();
}

cudaError_t launch_vnorm_prefix(const DevView& v, int layer, const void* vv, int n0, cudaStream_t s) {
  dim3 grid((unsigned)std::max(1, std::min(1024, (n0 + 7) / 8)), v.B * v.Hkv);
  k_vnorm_prefix<<<grid, 256, 0, s>>>(v, layer, reinterpret_cast<const uint16_t*>(vv), n0);
  return cudaGetLastError();
}

// Prefill rows [0, n0) of one layer (Alg. 1).  The first c0_load owned positions fill the
// T0 store; a prefix longer than that (T0 is sized for the steady state, |P| + n_hbm + Delta, not
// for the whole chain: DESIGN.md AMB-26) places the rest in T1 -- the pinned host store and, in
// differential mode, the HBM staging -- until the first manage event sorts the chain.  Attention
// reads T0 and T1 alike, so step 0 is unchanged.  A sequence shard keeps its own positions only
// (store row j = its j-th owned position).
__global__ void k_load_prefix(const DevView v, const int layer, const uint16_t* __restrict__ k,
                              const uint16_t* __restrict__ vv, const int n0) {
  const int unit = blockIdx.y;
  const int b = unit / v.Hkv, g = unit % v.Hkv;
  const size_t grp = grp_of(v, layer, b, g);
  uint16_t* K = reinterpret_cast<uint16_t*>(v.k0[0]);
  uint16_t* V = reinterpret_cast<uint16_t*>(v.v0[0]);
  uint16_t* K1 = reinterpret_cast<uint16_t*>(v.k1[0]);
  uint16_t* V1 = reinterpret_cast<uint16_t*>(v.v1[0]);
  const int n0own = seq_owned_below(v.seq_w, v.seq_r, n0);
  const size_t tot = (size_t)n0own * v.D;
  const size_t in_tot = (size_t)n0 * v.D;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (size_t)gridDim.x * blockDim.x) {
    const int j = (int)(e / v.D), el = (int)(e % v.D);
    const int p = seq_pos_of(v.seq_w, v.seq_r, j);
    const uint16_t kx = k[(size_t)unit * in_tot + (size_t)p * v.D + el];
    const uint16_t vx = vv[(size_t)unit * in_tot + (size_t)p * v.D + el];
    if (j < v.c0_load) {
      const size_t dst = (grp * v.cap0 + j) * v.D + swz_off(j, el, v.D);
      K[dst] = kx;
      V[dst] = vx;
    } else {
      const int r = j - v.c0_load;                             // T1 row (store order = position order)
      const size_t hdst = host_row(v, grp, p) * v.D + el;      // pinned host store: canonical layout
      reinterpret_cast<uint16_t*>(v.hk1)[hdst] = kx;
      reinterpret_cast<uint16_t*>(v.hv1)[hdst] = vx;
      if (!v.stream_mode) {
        const size_t dst = (grp * v.cap1 + r) * v.D + swz_off(r, el, v.D);
        K1[dst] = kx;
        V1[dst] = vx;
      }
    }
  }
}

// The n0 prefix tokens with S = 0 (Alg. 1): the first c0_load owned positions in T0,
// the rest in T1 (k_load_prefix).
__global__ void k_init_meta(const DevView v, const int n0) {
  const int b = blockIdx.y;
  const int n0own = seq_owned_below(v.seq_w, v.seq_r, n0);
  const int c0 = min(n0own, v.c0_load);
  for (int pos = blockIdx.x * blockDim.x + threadIdx.x; pos < v.Nmax; pos += gridDim.x * blockDim.x) {
    const bool own = seq_own(v.seq_w, v.seq_r, pos);
    const int j = seq_owned_below(v.seq_w, v.seq_r, pos);      // owned index of pos (if owned)
    const bool in1 = pos < n0 && own && j >= c0;
    for (int buf = 0; buf < 2; ++buf) {
      v.tier[buf][(size_t)b * v.Nmax + pos] = pos < n0 ? (in1 ? T1 : T0) : T3;
      v.rowof[buf][(size_t)b * v.Nmax + pos] = pos < n0 && own ? (in1 ? j - c0 : j) : -1;
      v.idxvis[buf][(size_t)b * v.Nmax + pos] = seq_pos_of(v.seq_w, v.seq_r, pos);
    }
    if (pos < n0 && own) {
      if (in1) v.idx[0][1][(size_t)b * v.cap1 + (j - c0)] = pos;
      else v.idx[0][0][(size_t)b * v.cap0 + j] = pos;
    }
    for (int g = 0; g < v.Hkv; ++g) v.S[((size_t)b * v.Hkv + g) * v.Nmax + pos] = 0.f;
    if (v.snap)                                  // windowed scorers: no window before step 0
      for (int g = 0; g < v.Hkv; ++g) v.snap[((size_t)b * v.Hkv + g) * v.Nmax + pos] = 0.f;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    for (int buf = 0; buf < 2; ++buf) {
      int* cn = v.cnt[buf] + b * CNT_STRIDE;
      cn[0] = buf == 0 ? c0 : 0;
      cn[1] = buf == 0 ? n0own - c0 : 0;
      cn[2] = cn[3] = 0;
      cn[4] = buf == 0 ? n0own : 0;
      cn[5] = cn[6] = cn[7] = 0;
    }
    if (b == 0) {
      v.st->n = n0;
      v.st->t = 0;
      v.st->cur = 0;
      v.st->n_event = n0;
      v.st->err = 0;
      v.st->scur = 0;
      v.st->d2h_rows = 0ull;
      v.st->nn = 1;
    }
  }
}

// ------------------------------------------------------------------ a4 standalone
// probs [B][Hq][n_vis] in ascending visible order; visible list = idxvis at the last
// event followed by the positions appended since (all T0, ascending).
__global__ void k_score_update(const DevView v, const int layer, const float* __restrict__ probs) {
  const int unit = blockIdx.y;
  const int b = unit / v.Hkv, g = unit % v.Hkv;
  const int cur = v.st->cur;
  const int nve = v.cnt[cur][b * CNT_STRIDE + 4];
  const int n_event = v.st->n_event;
  const int nvis = nve + (v.st->n - n_event);
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nvis) return;
  const int pos = j < nve ? v.idxvis[cur][(size_t)b * v.Nmax + j] : n_event + (j - nve);
  float inc = 0.f;
  for (int h = g * v.G; h < (g + 1) * v.G; ++h) inc += probs[((size_t)b * v.Hq + h) * nvis + j];
  float* S = v.S + ((size_t)b * v.Hkv + g) * v.Nmax + pos;
  *S = *S + inc * score_weight(v, layer, unit, pos);
  if (!isfinite(inc)) atomicOr(&v.st->err, 1);
}

// ------------------------------------------------------------------ a5 classify
// One 1024-thread CTA per request.  Keys (bits(S_i) << 32 | i) are unique, so the
// tier of every live token is decided by comparing its key with the keys at three
// ranks, found by an 8-pass MSB radix select (histograms in shared memory).
constexpr int CLS_THREADS = 1024;

// order-preserving fp32 -> uint32 (negatives below positives; raw bits order on S >= 0, AMB-7/31)
__device__ __forceinline__ unsigned ord_bits(float f) {
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// Sx: per-kv-head partial scores [parts][B][H_kv][N_max] -- the ctx's own S_part (parts = 1)
// or the all-gathered S_part of `parts` KV-head shards (global kv head = part * H_kv + g).
// snapx (windowed scorers): the S_part snapshots in Sx's layout (the all-gathered ones of every
// sequence shard), or the ctx's own (parts = 1)
__global__ void __launch_bounds__(CLS_THREADS) k_classify(const DevView v, const float* __restrict__ Sx, const int parts,
                                                          const float* __restrict__ snapx) {
  const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int cur = v.st->cur, nxt = cur ^ 1, n = v.st->n;
  const uint8_t* told = v.tier[cur] + (size_t)b * v.Nmax;
  float* fS = v.fS + (size_t)b * v.Nmax;
  const int prot_lo = v.P + v.ks;          // [0,P) u [P,P+k_s)  (positions < n)
  const int prot_hi = n - v.kw;            // window [n-k_w, n)

  __shared__ int s_cnt[2];
  __shared__ unsigned int s_smax;
  __shared__ unsigned int hist[3][256];
  __shared__ unsigned long long s_prefix[3];
  __shared__ long long s_rank[3];
  __shared__ int s_active[3];
  __shared__ int s_wsum[4][32];
  __shared__ int s_tot[4];
  __shared__ int s_base[4];

  if (tid < 2) s_cnt[tid] = 0;
  if (tid == 0) s_smax = 0u;
  __syncthreads();
  // S_i = fp32 sum over kv heads in ascending order (AMB-1/14)
  int c_live = 0, c_t3 = 0;
  unsigned smax = 0u;                      // max S over the live set (bits; S >= 0)
  bool bad = false;
  const bool win = v.snap != nullptr;      // windowed / R-KV (AMB-32); parts == 1 (classify_gathered refuses)
  for (int pos = tid; pos < n; pos += CLS_THREADS) {
    float s = Sx[((size_t)b * v.Hkv) * v.Nmax + pos];
    for (int gg = 1; gg < parts * v.Hkv; ++gg) {     // ascending global kv head
      const int part = gg / v.Hkv, g = gg - part * v.Hkv;
      s = __fadd_rn(s, Sx[(((size_t)part * v.B + b) * v.Hkv + g) * v.Nmax + pos]);
    }
    if (win) {                             // W_i = fp32(sum_g S) - fp32(sum_g S_snap), same summation order
      float s0 = snapx[((size_t)b * v.Hkv) * v.Nmax + pos];
      for (int gg = 1; gg < parts * v.Hkv; ++gg) {
        const int part = gg / v.Hkv, g = gg - part * v.Hkv;
        s0 = __fadd_rn(s0, snapx[(((size_t)part * v.B + b) * v.Hkv + g) * v.Nmax + pos]);
      }
      s = __fsub_rn(s, s0);
    }
    fS[pos] = s;
    bad |= !(s >= 0.f) || isinf(s);
    if (told[pos] == T3) ++c_t3;
    else if (pos >= prot_lo && pos < prot_hi) {
      ++c_live;
      smax = max(smax, __float_as_uint(s));
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    c_live += __shfl_xor_sync(0xffffffffu, c_live, off);
    c_t3 += __shfl_xor_sync(0xffffffffu, c_t3, off);
  }
  if (lane == 0) {
    atomicAdd(&s_cnt[0], c_live);
    atomicAdd(&s_cnt[1], c_t3);
  }
  if (v.red && !win) atomicMax(&s_smax, smax);
  if (bad) atomicOr(&v.st->err, 1);
  __syncthreads();
  if (win) {
    // max-pool (kernel 7, stride 1) over the non-T3 positions in ascending order (P:976 / AMB-32).
    // The order is built from the tier array, which every sequence shard holds for all positions:
    // compact W into pool[0..nvis) (prefix sums over the block), keep each position's index.
    float* cw = v.pool + (size_t)b * v.Nmax;
    int* cix = reinterpret_cast<int*>(v.pool + (size_t)v.B * v.Nmax) + (size_t)b * v.Nmax;
    if (tid == 0) s_base[0] = 0;
    __syncthreads();
    for (int base = 0; base < n; base += CLS_THREADS) {
      const int pos = base + tid;
      const bool f = pos < n && told[pos] != T3;
      const unsigned m = __ballot_sync(0xffffffffu, f);
      if (lane == 0) s_wsum[0][w] = __popc(m);
      __syncthreads();
      if (w == 0) {
        const int x = s_wsum[0][lane];
        int inc = x;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, inc, off);
          if (lane >= off) inc += y;
        }
        s_wsum[0][lane] = inc - x;
        if (lane == 31) s_tot[0] = inc;
      }
      __syncthreads();
      if (f) {
        const int k = s_base[0] + s_wsum[0][w] + __popc(m & ((1u << lane) - 1u));
        cw[k] = fS[pos];
        cix[pos] = k;
      }
      __syncthreads();
      if (tid == 0) s_base[0] += s_tot[0];
      __syncthreads();
    }
    const int nvis = s_base[0];
    unsigned pmax = 0u;
    for (int pos = tid; pos < n; pos += CLS_THREADS) {
      if (told[pos] == T3) continue;
      const int k = cix[pos];
      float m = cw[k];
      for (int x = max(0, k - RKV_HALF_POOL); x <= min(nvis - 1, k + RKV_HALF_POOL); ++x) m = fmaxf(m, cw[x]);
      fS[pos] = m;
      if (pos >= prot_lo && pos < prot_hi) pmax = max(pmax, __float_as_uint(m));
    }
    if (v.red) atomicMax(&s_smax, pmax);
    __syncthreads();
  }
  if (v.red) {
    // redundancy / combined (AMB-31): rank by I - rho, I = S / S_max, rho = mean_{l,g} cos
    const float fmax = __uint_as_float(s_smax);
    const float lh = (float)(v.L * v.Hkv);
    for (int pos = tid; pos < n; pos += CLS_THREADS) {
      const float* r = v.red + (size_t)b * v.Hkv * v.Nmax + pos;
      float rs = r[0];
      for (int g = 1; g < v.Hkv; ++g) rs = __fadd_rn(rs, r[(size_t)g * v.Nmax]);
      const float I = fmax > 0.f ? __fdiv_rn(fS[pos], fmax) : 0.f;
      const float rho = __fdiv_rn(rs, lh);
      fS[pos] = v.scorer == 5 ? __fsub_rn(__fmul_rn(0.07f, I), __fmul_rn(0.93f, rho))   // R-KV (AMB-33)
                              : __fsub_rn(I, rho);
    }
    __syncthreads();
  }
  if (tid == 0) {
    // Alg. 1 floor arithmetic in integer basis points (AMB-8/9/11), or the
    // pure-eviction baselines' counts (tier policy)
    const long long nl = s_cnt[0], n3 = s_cnt[1];
    const long long n_prot = (long long)min(prot_lo, n) + (n - max(max(prot_hi, 0), min(prot_lo, n)));
    long long n_new, n_hbm, n_t2;
    policy_counts(v.policy, v.budget, v.hbm_bp, v.evict_bp, v.t2_bp, v.evict_mode, n_prot, nl, n3, &n_new, &n_hbm, &n_t2);
    const long long rk[3] = {n_new, n_new + n_t2, nl - n_hbm};
    for (int k = 0; k < 3; ++k) {
      s_active[k] = rk[k] < nl;
      s_rank[k] = rk[k];
      s_prefix[k] = 0ull;
    }
  }
  __syncthreads();

  // radix select: key at rank s_rank[k] among the live keys
  for (int shift = 56; shift >= 0; shift -= 8) {
    for (int i = tid; i < 3 * 256; i += CLS_THREADS) (&hist[0][0])[i] = 0u;
    __syncthreads();
    for (int pos = tid; pos < n; pos += CLS_THREADS) {
      if (told[pos] == T3 || pos < prot_lo || pos >= prot_hi) continue;
      const unsigned long long key = ((unsigned long long)(v.policy == 3 ? random_key32(v.policy_seed, b, pos)
                                                                          : ord_bits(fS[pos])) << 32) | (unsigned)pos;
      const unsigned dig = (unsigned)(key >> shift) & 255u;
#pragma unroll
      for (int k = 0; k < 3; ++k)
        if (s_active[k] && (shift == 56 || (key >> (shift + 8)) == (s_prefix[k] >> (shift + 8))))
          atomicAdd(&hist[k][dig], 1u);
    }
    __syncthreads();
    if (w < 3 && s_active[w]) {
      const long long rank = s_rank[w];
      unsigned loc[8], sum = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        loc[j] = hist[w][lane * 8 + j];
        sum += loc[j];
      }
      unsigned inc = sum;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += y;
      }
      const unsigned excl = inc - sum;
      __syncwarp();
      if ((long long)excl <= rank && rank < (long long)inc) {
        unsigned c = excl;
        int j = 0;
        while (c + loc[j] <= rank) c += loc[j++];
        s_rank[w] = rank - c;
        s_prefix[w] |= ((unsigned long long)(lane * 8 + j)) << shift;
      }
    }
    __syncthreads();
  }
  const unsigned long long thr_e = s_active[0] ? s_prefix[0] : ~0ull;   // keys below -> T3
  const unsigned long long thr_2 = s_active[1] ? s_prefix[1] : ~0ull;   // keys below -> T2
  const unsigned long long thr_1 = s_active[2] ? s_prefix[2] : ~0ull;   // keys below -> T1, else T0

  // assign + ascending compaction of T0 / T1 / T2 / visible lists
  if (tid < 4) s_base[tid] = 0;
  __syncthreads();
  uint8_t* tnew = v.tier[nxt] + (size_t)b * v.Nmax;
  int* rnew = v.rowof[nxt] + (size_t)b * v.Nmax;
  const int caps[3] = {v.cap0, v.cap1, v.cap2};
  for (int base = 0; base < n; base += CLS_THREADS) {
    const int pos = base + tid;
    int t = -1;
    if (pos < n) {
      const int to = told[pos];
      if (to == T3) t = T3;
      else if (pos < prot_lo || pos >= prot_hi) t = T0;
      else {
        const unsigned long long key = ((unsigned long long)(v.policy == 3 ? random_key32(v.policy_seed, b, pos)
                                                                            : ord_bits(fS[pos])) << 32) | (unsigned)pos;
        t = key < thr_e ? T3 : key < thr_2 ? T2 : key < thr_1 ? T1 : T0;
      }
      tnew[pos] = (uint8_t)t;
      if (t == T3 || !seq_own(v.seq_w, v.seq_r, pos)) rnew[pos] = -1;
    }
    const bool own = pos < n && seq_own(v.seq_w, v.seq_r, pos);   // lists hold own positions only
    unsigned m[4];
#pragma unroll
    for (int L4 = 0; L4 < 4; ++L4) {
      const bool f = own && (L4 < 3 ? (t == L4) : (t >= 0 && t != T3));
      m[L4] = __ballot_sync(0xffffffffu, f);
      if (lane == 0) s_wsum[L4][w] = __popc(m[L4]);
    }
    __syncthreads();
    if (w < 4) {
      const int x = s_wsum[w][lane];
      int inc = x;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += y;
      }
      s_wsum[w][lane] = inc - x;
      if (lane == 31) s_tot[w] = inc;
    }
    __syncthreads();
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int L4 = 0; L4 < 4; ++L4) {
      if (m[L4] & (1u << lane)) {
        const int off = s_base[L4] + s_wsum[L4][w] + __popc(m[L4] & lt);
        if (L4 < 3) {
          if (off < caps[L4]) {           // never past a store (sequence shards size T1/T2 by share)
            v.idx[nxt][L4][(size_t)b * caps[L4] + off] = pos;
            rnew[pos] = off;
          } else {
            atomicOr(&v.st->err, 2);
          }
        } else {
          v.idxvis[nxt][(size_t)b * v.Nmax + off] = pos;
        }
      }
    }
    __syncthreads();
    if (tid < 4) s_base[tid] += s_tot[tid];
    __syncthreads();
  }
  if (tid == 0) {
    int* cn = v.cnt[nxt] + b * CNT_STRIDE;
    cn[0] = min(s_base[0], caps[0]);   // an overflow (flagged above) stays inside the stores
    cn[1] = min(s_base[1], caps[1]);
    cn[2] = min(s_base[2], caps[2]);
    cn[3] = seq_owned_below(v.seq_w, v.seq_r, n) - s_base[3];
    cn[4] = s_base[3];
  }
}

// ------------------------------------------------------------------ a6 migrate
// Rows of one lane: D/32 bf16 (D = 64 or 128).
template <int D>
struct RowIO {
  static constexpr int E = D / 32;
};

__device__ __forceinline__ void load_bits(uint16_t* x, const uint16_t* src, int e) {
  if (e == 4) {
    const uint2 u = *reinterpret_cast<const uint2*>(src);
    x[0] = u.x & 0xFFFF; x[1] = u.x >> 16; x[2] = u.y & 0xFFFF; x[3] = u.y >> 16;
  } else {
    const uint32_t u = *reinterpret_cast<const uint32_t*>(src);
    x[0] = u & 0xFFFF; x[1] = u >> 16;
  }
}
__device__ __forceinline__ void store_bits(uint16_t* dst, const uint16_t* x, int e) {
  if (e == 4) {
    *reinterpret_cast<uint2*>(dst) = make_uint2((uint32_t)x[0] | ((uint32_t)x[1] << 16),
                                                (uint32_t)x[2] | ((uint32_t)x[3] << 16));
  } else {
    *reinterpret_cast<uint32_t*>(dst) = (uint32_t)x[0] | ((uint32_t)x[1] << 16);
  }
}

// Source row (bf16 bit pattern, canonical element order) of position `pos` of layer/group
// `grp` in tier `ot`, store row `orow` of the row-store buffer `sb`.  T2 sources return
// bf16(dequant) (AMB-12); stream-mode T1 rows come from the pinned host store.
template <int D>
__device__ __forceinline__ void source_row(const DevView& v, int sb, int kv, size_t grp, int ot, int orow,
                                           int pos, int lane, uint16_t* x) {
  constexpr int E = D / 32;
  if (ot == T0) {
    const uint16_t* s = reinterpret_cast<const uint16_t*>(kv ? v.v0[sb] : v.k0[sb]) + (grp * v.cap0 + orow) * D;
    load_bits(x, s + swz_off(orow, lane * E, D), E);
  } else if (ot == T1) {
    if (v.stream_mode) {
      const uint16_t* s = reinterpret_cast<const uint16_t*>(kv ? v.hv1 : v.hk1) + host_row(v, grp, pos) * D;
      load_bits(x, s + lane * E, E);   // pinned host store: canonical layout
    } else {
      const uint16_t* s = reinterpret_cast<const uint16_t*>(kv ? v.v1[sb] : v.k1[sb]) + (grp * v.cap1 + orow) * D;
      load_bits(x, s + swz_off(orow, lane * E, D), E);
    }
  } else {
    const int8_t* c = (kv ? v.c2v[sb] : v.c2k[sb]) + (grp * v.cap2 + orow) * D + lane * E;
    const float sc = (kv ? v.s2v[sb] : v.s2k[sb])[grp * v.cap2 + orow];
#pragma unroll
    for (int k = 0; k < E; ++k) x[k] = f_to_bf16_bits(__fmul_rn((float)c[k], sc));
  }
}

// per-row symmetric int8: scale = fp32(absmax/127), code = clamp(rint(x/scale)) (AMB-12)
template <int D>
__device__ __forceinline__ void quantize_row(const uint16_t* x, int8_t* codes, float* scale, int lane) {
  constexpr int E = D / 32;
  float f[E];
  float amax = 0.f;
#pragma unroll
  for (int k = 0; k < E; ++k) {
    f[k] = bf16_bits_to_f(x[k]);
    amax = fmaxf(amax, fabsf(f[k]));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, off));
  const float sc = amax == 0.f ? 1.0f : __fdiv_rn(amax, 127.0f);
#pragma unroll
  for (int k = 0; k < E; ++k) {
    float qv = amax == 0.f ? 0.f : rintf(__fdiv_rn(f[k], sc));
    qv = fminf(127.f, fmaxf(-127.f, qv));
    codes[k] = (int8_t)qv;
  }
  *scale = sc;
}

// ------------------------------------------------------------------ a6 plan
// New row layout of every tier store after a classify (one CTA per request).  Tokens that
// stay in a store keep their row when it is below the new count; the free rows below the
// new count ("holes", ascending) are filled first with the store's own tail rows, then
// with the tokens entering the store (ascending position).  Emits the store-order index
// lists and rowof of the nxt metadata buffer and the list of row moves; a move list longer
// than mcap switches this migrate to a full rebuild into the other row-store buffer.
constexpr int PLAN_THREADS = 1024;

template <typename Flag, typename Act>
__device__ __forceinline__ int block_compact(int lo, int hi, int* s_wsum, int* s_tot, Flag flag, Act act) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  int base = 0;
  for (int c0 = lo; c0 < hi; c0 += PLAN_THREADS) {
    const int i = c0 + tid;
    const bool f = i < hi && flag(i);
    const unsigned m = __ballot_sync(0xffffffffu, f);
    if (lane == 0) s_wsum[w] = __popc(m);
    __syncthreads();
    if (w == 0) {
      const int x = s_wsum[lane];
      int inc = x;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, off);
        if (lane >= off) inc += y;
      }
      s_wsum[lane] = inc - x;
      if (lane == 31) *s_tot = inc;
    }
    __syncthreads();
    if (f) act(i, base + s_wsum[w] + __popc(m & ((1u << lane) - 1u)));
    base += *s_tot;
    __syncthreads();
  }
  return base;
}

__global__ void __launch_bounds__(PLAN_THREADS) k_plan(const DevView v) {
  const int b = blockIdx.x, tid = threadIdx.x;
  const int cur = v.st->cur, nxt = cur ^ 1, n = v.st->n;
  const uint8_t* told = v.tier[cur] + (size_t)b * v.Nmax;
  const uint8_t* tnew = v.tier[nxt] + (size_t)b * v.Nmax;
  const int* rold = v.rowof[cur] + (size_t)b * v.Nmax;
  int* rnew = v.rowof[nxt] + (size_t)b * v.Nmax;
  int* hole = v.scratch + (size_t)b * v.Nmax;
  int4* mv = v.moves + (size_t)b * v.mcap;
  __shared__ int s_wsum[32], s_tot, s_nm;
  if (tid == 0) s_nm = 0;
  __syncthreads();
  const int caps[3] = {v.cap0, v.cap1, v.cap2};
  for (int X = 0; X < 3; ++X) {
    const int cap = caps[X];
    if (cap == 0) continue;
    const int c_old = v.cnt[cur][b * CNT_STRIDE + X], c_new = v.cnt[nxt][b * CNT_STRIDE + X];
    const int* iold = v.idx[cur][X] + (size_t)b * cap;
    int* inew = v.idx[nxt][X] + (size_t)b * cap;
    auto kept = [&](int r) { return r < c_old && tnew[iold[r]] == X; };
    // holes below the new count, ascending
    block_compact(0, c_new, s_wsum, &s_tot, [&](int r) { return !kept(r); }, [&](int r, int k) { hole[k] = r; });
    // kept in place
    for (int r = tid; r < min(c_old, c_new); r += PLAN_THREADS)
      if (kept(r)) {
        inew[r] = iold[r];
        rnew[iold[r]] = r;
      }
    __syncthreads();
    const int m0 = s_nm;
    // tail rows of the store -> holes
    const int ntk = block_compact(c_new, c_old, s_wsum, &s_tot, [&](int r) { return kept(r); },
                                  [&](int r, int k) {
                                    const int pos = iold[r], dst = hole[k];
                                    inew[dst] = pos;
                                    rnew[pos] = dst;
                                    if (m0 + k < v.mcap) mv[m0 + k] = make_int4(X, r, X | (dst << 2), pos);
                                  });
    // tokens entering the store -> remaining holes
    const int nin = block_compact(0, n, s_wsum, &s_tot,
                                  [&](int p) { return tnew[p] == X && told[p] != X && seq_own(v.seq_w, v.seq_r, p); },
                                  [&](int p, int k) {
                                    const int dst = hole[ntk + k];
                                    inew[dst] = p;
                                    rnew[p] = dst;
                                    if (m0 + ntk + k < v.mcap)
                                      mv[m0 + ntk + k] = make_int4(told[p], rold[p], X | (dst << 2), p);
                                  });
    if (tid == 0) s_nm = m0 + ntk + nin;
    __syncthreads();
  }
  for (int p = tid; p < n; p += PLAN_THREADS)
    if (tnew[p] == T3) rnew[p] = -1;
  if (tid == 0) {
    if (b == 0) *v.gbar = 0u;                                 // k_migrate_rows' grid barrier
    v.mcount[b] = min(s_nm, v.mcap);
    if (s_nm > v.mcap) atomicOr(&v.st->err, 2);              // cannot happen: moves <= n <= mcap
  }
}

// Migrate (a6) in ONE cooperative launch: every moved row of every (layer, kv head) pair.  The
// stores are updated in place, so the moved rows of a chunk of pairs are all gathered into
// mtemp (destination format: bf16 canonical, or int8 codes + scale for T2) before any is
// scattered; the chunk holds as many pairs as mtemp fits at this event's largest move count
// (pairs are independent: a move never crosses layers or heads).  Rows newly in T1 / T2 are
// written to the pinned host stores in the gather phase (zero-copy stores over the host link:
// "Offload T1 entries").  Work items = (pair, request, move), one warp each; grid-wide
// barriers between the phases (all CTAs co-resident: cudaLaunchAttributeCooperative).
__device__ __forceinline__ bool grid_barrier(unsigned* ctr, unsigned target) {
  bool ok = true;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    const unsigned long long t0 = gtimer();
    for (;;) {
      unsigned x;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(x) : "l"(ctr) : "memory");
      if (x >= target) break;
      if (gtimer() - t0 > 2000000000ull) { ok = false; break; }   // watchdog: report, never hang
      __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
  return ok;
}

template <int D>
__global__ void __launch_bounds__(256) k_migrate_rows(const DevView v) {
  constexpr int E = D / 32;
  const int lane = threadIdx.x & 31;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const int B = v.B, npairs = v.L * v.Hkv;
  int mmax = 0;
  for (int b = 0; b < B; ++b) mmax = max(mmax, v.mcount[b]);
  if (mmax == 0) return;                                      // uniform over the grid: no barrier reached
  const long long cap_rows = (long long)B * v.mcap * v.mchunk;
  const int K = (int)max(1ll, min((long long)npairs, cap_rows / ((long long)B * mmax)));
  const int sb = v.st->scur;
  unsigned gen = 0;
  bool ok = true;
  for (int c0 = 0; c0 < npairs; c0 += K) {
    const long long items = (long long)min(K, npairs - c0) * B * mmax;
    // ---- phase 1: gather (+ host offload)
    for (long long i = gw; i < items; i += nw) {
      const int m = (int)(i % mmax);
      const long long r = i / mmax;
      const int b = (int)(r % B), lg = c0 + (int)(r / B), l = lg / v.Hkv, g = lg % v.Hkv;
      if (m >= v.mcount[b]) continue;
      const int4 mv = v.moves[(size_t)b * v.mcap + m];
      const int st = mv.x, srow = mv.y, dt = mv.z & 3, pos = mv.w;
      if (st == T1 && dt == T1 && v.stream_mode) continue;   // list-only move (rows live on the host)
      const size_t grp = grp_of(v, l, b, g);
      // stream mode: the pinned store is T1's only home, so a row entering T1/T2 is written there
      // now; differential staging keeps it in HBM and k_offload_rows copies it out afterwards
      const bool off = (v.stream_mode || KVT_INLINE_OFFLOAD) && st != dt && (dt == T1 || (dt == T2 && v.hc2k != nullptr));
      uint16_t* tmp = reinterpret_cast<uint16_t*>(v.mtemp) + (size_t)i * 2 * D;
      for (int kv = 0; kv < 2; ++kv) {
        uint16_t* tk = tmp + kv * D;
        if (dt == T2 && st == T2) {       // T2 -> T2: codes and scale verbatim
          const int8_t* c = (kv ? v.c2v[sb] : v.c2k[sb]) + (grp * v.cap2 + srow) * D + lane * E;
          int8_t* o = reinterpret_cast<int8_t*>(tk) + lane * E;
#pragma unroll
          for (int k = 0; k < E; ++k) o[k] = c[k];
          if (lane == 0) *reinterpret_cast<float*>(reinterpret_cast<int8_t*>(tk) + D) = (kv ? v.s2v[sb] : v.s2k[sb])[grp * v.cap2 + srow];
          continue;
        }
        uint16_t x[E];
        source_row<D>(v, sb, kv, grp, st, srow, pos, lane, x);
        if (dt == T2) {
          int8_t codes[E];
          float sc;
          quantize_row<D>(x, codes, &sc, lane);
          int8_t* o = reinterpret_cast<int8_t*>(tk) + lane * E;
#pragma unroll
          for (int k = 0; k < E; ++k) o[k] = codes[k];
          if (lane == 0) *reinterpret_cast<float*>(reinterpret_cast<int8_t*>(tk) + D) = sc;
          if (off) {
            int8_t* dc = (kv ? v.hc2v : v.hc2k) + host_row(v, grp, pos) * D + lane * E;
#pragma unroll
            for (int k = 0; k < E; ++k) dc[k] = codes[k];
            if (lane == 0) (kv ? v.hs2v : v.hs2k)[host_row(v, grp, pos)] = sc;
          }
        } else {
          store_bits(tk + lane * E, x, E);
          if (off) store_bits(reinterpret_cast<uint16_t*>(kv ? v.hv1 : v.hk1) + host_row(v, grp, pos) * D + lane * E, x, E);
        }
      }
      if (off && lane == 0) atomicAdd(&v.st->d2h_rows, 2ull);
    }
    ok &= grid_barrier(v.gbar, ++gen * gridDim.x);
    // ---- phase 2: scatter into the destination rows
    for (long long i = gw; i < items; i += nw) {
      const int m = (int)(i % mmax);
      const long long r = i / mmax;
      const int b = (int)(r % B), lg = c0 + (int)(r / B), l = lg / v.Hkv, g = lg % v.Hkv;
      if (m >= v.mcount[b]) continue;
      const int4 mv = v.moves[(size_t)b * v.mcap + m];
      const int dt = mv.z & 3, drow = mv.z >> 2;
      if (dt == T1 && v.stream_mode) continue;               // T1 rows live on the host
      const size_t grp = grp_of(v, l, b, g);
      const uint16_t* tmp = reinterpret_cast<const uint16_t*>(v.mtemp) + (size_t)i * 2 * D;
      for (int kv = 0; kv < 2; ++kv) {
        const uint16_t* tk = tmp + kv * D;
        if (dt == T2) {
          const int8_t* c = reinterpret_cast<const int8_t*>(tk) + lane * E;
          int8_t* o = (kv ? v.c2v[sb] : v.c2k[sb]) + (grp * v.cap2 + drow) * D + lane * E;
#pragma unroll
          for (int k = 0; k < E; ++k) o[k] = c[k];
          if (lane == 0) (kv ? v.s2v[sb] : v.s2k[sb])[grp * v.cap2 + drow] = *reinterpret_cast<const float*>(reinterpret_cast<const int8_t*>(tk) + D);
        } else {
          uint16_t x[E];
          load_bits(x, tk + lane * E, E);
          uint16_t* dst = dt == T0
              ? reinterpret_cast<uint16_t*>(kv ? v.v0[sb] : v.k0[sb]) + (grp * v.cap0 + drow) * D
              : reinterpret_cast<uint16_t*>(kv ? v.v1[sb] : v.k1[sb]) + (grp * v.cap1 + drow) * D;
          store_bits(dst + swz_off(drow, lane * E, D), x, E);
        }
      }
    }
    if (c0 + K < npairs) ok &= grid_barrier(v.gbar, ++gen * gridDim.x);   // mtemp is reused
  }
  if (!ok && threadIdx.x == 0) atomicOr(&v.st->err, 4);
}

__global__ void k_commit(const DevView v) {
  if (threadIdx.x == 0) {
    DevState* s = v.st;
    s->cur ^= 1;
    s->n_event = s->n;
  }
}

// a2 stream mode: T1 rows of `layer` from pinned host memory -> HBM ring slot layer&1.
template <int D>
__global__ void __launch_bounds__(256) k_prefetch(const DevView v, const int layer) {
  constexpr int E = D / 32;
  const int unit = blockIdx.y;
  const int b = unit / v.Hkv, g = unit % v.Hkv;
  const int cur = v.st->cur;
  const int n1 = v.cnt[cur][b * CNT_STRIDE + 1];
  const size_t grp = grp_of(v, layer, b, g);
  const size_t sg = ((size_t)(layer & 1) * v.B + b) * v.Hkv + g;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j0 = blockIdx.x * 32;
  const int j1 = min(j0 + 32, n1);
  for (int j = j0 + w; j < j1; j += 8) {
    const int pos = v.idx[cur][1][(size_t)b * v.cap1 + j];
    for (int kv = 0; kv < 2; ++kv) {
      const uint16_t* s = reinterpret_cast<const uint16_t*>(kv ? v.hv1 : v.hk1) + host_row(v, grp, pos) * D;
      uint16_t* d = reinterpret_cast<uint16_t*>(kv ? v.v1[0] : v.k1[0]) + (sg * v.cap1 + j) * D;
      uint16_t x[E];
      load_bits(x, s + lane * E, E);
      store_bits(d + swz_off(j, lane * E, D), x, E);
    }
  }
}

// ------------------------------------------------------------------ launchers
cudaError_t launch_begin_step(const DevView& v, cudaStream_t s) {
  if (v.snap) {                                  // windowed / R-KV scorers: the window may start here
    k_snapshot<<<dim3(64, v.B * v.Hkv), 256, 0, s>>>(v);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  k_begin_step<<<1, ((v.B + 31) / 32) * 32, 0, s>>>(v);
  return cudaGetLastError();
}
cudaError_t launch_end_step(const DevView& v, cudaStream_t s) {
  k_end_step<<<1, 32, 0, s>>>(v);
  return cudaGetLastError();
}
cudaError_t launch_append(const DevView& v, int layer, const void* k, const void* vv, cudaStream_t s) {
  k_append<<<v.B * v.Hkv, 64, 0, s>>>(v, layer, reinterpret_cast<const uint16_t*>(k),
                                      reinterpret_cast<const uint16_t*>(vv));
  return cudaGetLastError();
}
cudaError_t launch_load_prefix(const DevView& v, int layer, const void* k, const void* vv, int n0, cudaStream_t s) {
  dim3 grid(64, v.B * v.Hkv);
  k_load_prefix<<<grid, 256, 0, s>>>(v, layer, reinterpret_cast<const uint16_t*>(k),
                                    reinterpret_cast<const uint16_t*>(vv), n0);
  return cudaGetLastError();
}
cudaError_t launch_init_meta(const DevView& v, int n0, cudaStream_t s) {
  dim3 grid((v.Nmax + 255) / 256, v.B);
  k_init_meta<<<grid, 256, 0, s>>>(v, n0);
  return cudaGetLastError();
}
cudaError_t launch_score_update(const DevView& v, int layer, const float* probs, cudaStream_t s) {
  dim3 grid((v.Nmax + 255) / 256, v.B * v.Hkv);
  k_score_update<<<grid, 256, 0, s>>>(v, layer, probs);
  return cudaGetLastError();
}
cudaError_t launch_classify(const DevView& v, const float* Sx, int parts, cudaStream_t s, const float* snapx) {
  k_classify<<<v.B, CLS_THREADS, 0, s>>>(v, Sx ? Sx : v.S, Sx ? parts : 1, snapx ? snapx : v.snap);
  return cudaGetLastError();
}
cudaError_t launch_plan(const DevView& v, cudaStream_t s) {
  k_plan<<<v.B, PLAN_THREADS, 0, s>>>(v);
  return cudaGetLastError();
}
// Differential staging: the rows that entered T1 / T2 at the last migrate, from their new HBM rows
// (staging / T2 store) to the pinned host stores ("Offload T1 entries"), on the ctx's
// offload stream while the next steps run: the next classify waits for it (the move list and the
// rows may change then), and every host-side reader of the pinned stores synchronises first.
template <int D>
__global__ void __launch_bounds__(256) k_offload_rows(const DevView v) {
  constexpr int E = D / 32;
  const int lane = threadIdx.x & 31;
  const long long gw = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const int B = v.B, npairs = v.L * v.Hkv, sb = v.st->scur;
  int mmax = 0;
  for (int b = 0; b < B; ++b) mmax = max(mmax, v.mcount[b]);
  const long long items = (long long)npairs * B * mmax;
  for (long long i = gw; i < items; i += nw) {
    const int m = (int)(i % mmax);
    const long long r = i / mmax;
    const int b = (int)(r % B), lg = (int)(r / B), l = lg / v.Hkv, g = lg % v.Hkv;
    if (m >= v.mcount[b]) continue;
    const int4 mv = v.moves[(size_t)b * v.mcap + m];
    const int st = mv.x, dt = mv.z & 3, drow = mv.z >> 2, pos = mv.w;
    if (st == dt || !(dt == T1 || (dt == T2 && v.hc2k != nullptr))) continue;
    const size_t grp = grp_of(v, l, b, g);
    const size_t hr = host_row(v, grp, pos);
    for (int kv = 0; kv < 2; ++kv) {
      if (dt == T1) {
        uint16_t x[E];
        const uint16_t* s = reinterpret_cast<const uint16_t*>(kv ? v.v1[sb] : v.k1[sb]) + (grp * v.cap1 + drow) * D;
        load_bits(x, s + swz_off(drow, lane * E, D), E);
        store_bits(reinterpret_cast<uint16_t*>(kv ? v.hv1 : v.hk1) + hr * D + lane * E, x, E);
      } else {
        const int8_t* c = (kv ? v.c2v[sb] : v.c2k[sb]) + (grp * v.cap2 + drow) * D + lane * E;
        int8_t* dc = (kv ? v.hc2v : v.hc2k) + hr * D + lane * E;
#pragma unroll
        for (int k = 0; k < E; ++k) dc[k] = c[k];
        if (lane == 0) (kv ? v.hs2v : v.hs2k)[hr] = (kv ? v.s2v[sb] : v.s2k[sb])[grp * v.cap2 + drow];
      }
    }
    if (lane == 0) atomicAdd(&v.st->d2h_rows, 2ull);
  }
}
// 16 CTAs: the whole-step kernel holds one CTA per SM on 128 of the 148 SMs and needs every
// cluster resident; an offload that stays under the 20 free SMs never displaces it, and 16 SMs of
// zero-copy stores already fill the host link
cudaError_t launch_offload_rows(const DevView& v, cudaStream_t s) {
  if (v.D == 128) k_offload_rows<128><<<16, 256, 0, s>>>(v);
  else k_offload_rows<64><<<16, 256, 0, s>>>(v);
  return cudaGetLastError();
}

// every moved row of the event: one cooperative launch, as many CTAs as are co-resident (<= 2 per SM)
template <int D>
static cudaError_t migrate_rows_t(const DevView& v, cudaStream_t s) {
  constexpr int MAXDEV = 64;
  static int grids[MAXDEV] = {};                 // per device: co-resident CTAs (<= 2 per SM)
  int dev = 0;
  cudaError_t e0 = cudaGetDevice(&dev);
  if (e0 != cudaSuccess) return e0;
  int& grid = grids[dev < MAXDEV ? dev : MAXDEV - 1];
  if (grid == 0 || dev >= MAXDEV) {
    int sms = 0, per = 0;
    cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_migrate_rows<D>, 256, 0);
    if (e != cudaSuccess) return e;
    grid = sms * std::max(1, std::min(per, 2));
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid, 1, 1);
  cfg.blockDim = dim3(256, 1, 1);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_migrate_rows<D>, v);
}
cudaError_t launch_migrate_rows(const DevView& v, cudaStream_t s) {
  return v.D == 128 ? migrate_rows_t<128>(v, s) : migrate_rows_t<64>(v, s);
}
cudaError_t launch_commit(const DevView& v, cudaStream_t s) {
  k_commit<<<1, 32, 0, s>>>(v);
  return cudaGetLastError();
}
cudaError_t launch_prefetch(const DevView& v, int layer, cudaStream_t s) {
  if (v.cap1 == 0) return cudaSuccess;
  dim3 grid((v.cap1 + 31) / 32, v.B * v.Hkv);
  if (v.D == 128) k_prefetch<128><<<grid, 256, 0, s>>>(v, layer);
  else k_prefetch<64><<<grid, 256, 0, s>>>(v, layer);
  return cudaGetLastError();
}

}  // namespace kvt
