// Fused tcgen05 attention for 128 < s <= 512 (GPT-2-style causal decoder,
// s = 512; ViT, s = 197): the reference's attention / vjp_attention
// (blocks.cpp:142-236; softmax_rows / vjp_softmax_rows, tensor.cpp:310-342)
// streamed over 128-key blocks.
//
// The probabilities are never stored: the forward keeps two per-row
// statistics (the row max m of the scaled, masked scores and 1/l with l the
// row sum of exp(s - m)) in the P slot of the activation arena, and the
// backward recomputes P = exp(s - m) / l from Q, K and those statistics (same
// MMAs, same order, same exponential as the forward's P~ = exp(s - m)). The
// backward also keeps t_i = dO_i . O_i there ([2 sq + i]).
//
//   forward  (CTA per member, batch, head, 128-query block)
//     pass A: per key block S = Q K^T (3-pass split MMA) -> row max m only
//     pass B: per key block S again -> P~ = exp(S*scale - m) -> O += P~ V,
//             l += sum P~; the epilogue writes O / l
//   backward, two deterministic kernels (no atomics, no split-K reductions):
//     dK/dV  (CTA per 128-key block): loops over the query blocks that see it,
//            dV += P^T dO, dK += dS^T Q accumulated in TMEM
//     dQ     (CTA per 128-query block): loops over key blocks, dQ += dS K
//   with dS = P (dP - t), dP = dO V^T and t_i = sum_j dP_ij P_ij = dO_i . O_i
//   (O = P V), so no pass over whole rows of dP is needed.
// Causal problems skip the key blocks above the diagonal entirely.
#include "attn_common.cuh"

namespace mglp {

using namespace tc;
using namespace attn;

namespace {

constexpr int kThreads = 256;  // warp w: TMEM lanes 32 (w & 3), key-column half w >> 2
constexpr int STG = 128 * 64 * 4;  // fp32 staging of one [128][64] block

struct LongSmem {
  uint32_t stg, t0, t1, t2, t3, t4;  // staging + five tiles (t4 is a 64 KB pair128)
  uint64_t* bars;                    // [0] TMA, [1] MMA
  float* xch;                        // [2][128] row-statistic exchange
  uint32_t* tslot;
};

__device__ __forceinline__ LongSmem carve(uint8_t* smem_raw) {
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  LongSmem L;
  const uint32_t base = smem_u32(smem);
  L.stg = base;
  L.t0 = base + STG;
  L.t1 = L.t0 + PAIR64;
  L.t2 = L.t1 + PAIR64;
  L.t3 = L.t2 + PAIR64;
  L.t4 = L.t3 + PAIR64;
  L.bars = reinterpret_cast<uint64_t*>(smem + STG + 4 * PAIR64 + PAIR128);
  L.xch = reinterpret_cast<float*>(L.bars + 4);
  L.tslot = reinterpret_cast<uint32_t*>(L.xch + 256);
  return L;
}
constexpr int kLongSmem = 1024 + STG + 4 * PAIR64 + PAIR128 + 32 + 256 * 4 + 16;

__device__ __forceinline__ Opnd pair64(uint32_t t, bool mn) { return Opnd{t, t + TILE64, 128, mn}; }
__device__ __forceinline__ Opnd pair128(uint32_t t, bool mn) {
  return Opnd{t, t + 2 * TILE64, 128, mn};
}

// one thread issues a [128][dh] box (rows row0.. of operand `which`) into the
// staging; a head-split pre-split operand arrives as its hi and lo' tiles
// (two [128][32] SWIZZLE_128B boxes, the same 32 KiB)
__device__ __forceinline__ void issue(const LongSmem& L, const AttnTma& tm, int which, int g, int b,
                                      int h, int row0, int dh) {
  mbar_expect_tx(&L.bars[0], (uint32_t)(128 * dh * 4));
  if ((tm.hs_mask >> which) & 1) {
    tma_box(L.stg, tm, which, g, b, h, &L.bars[0], row0, 0);
    tma_box(L.stg + TILE64, tm, which, g, b, h, &L.bars[0], row0, 32);
  } else {
    tma_box(L.stg, tm, which, g, b, h, &L.bars[0], row0);
  }
}
// the staged operand `which` -> its tile pair: converted (fp32) or copied
// (pre-split: the staging already holds the two tiles in their layout)
__device__ __forceinline__ void land(const LongSmem& L, const AttnTma& tm, int which, uint32_t thi,
                                     uint32_t tlo, int dh, int tid, float& amax) {
  if ((tm.hs_mask >> which) & 1) {
    for (int c = tid; c < 2048; c += kThreads) {
      const uint32_t off = (uint32_t)(c & 1023) * 16;
      sts128((c < 1024 ? thi : tlo) + off, lds128u(L.stg + (c < 1024 ? 0 : TILE64) + off));
    }
  } else {
    conv_rows(L.stg, 128, 128, dh, thi, tlo, tid, kThreads, amax);
  }
}

struct Phase {
  uint32_t st = 0, mm = 0;
};
__device__ __forceinline__ void wait_stage(const LongSmem& L, Phase& ph) {
  mbar_wait(&L.bars[0], ph.st);
  ph.st ^= 1;
}
__device__ __forceinline__ void mma_done(const LongSmem& L, Phase& ph) {
  mbar_wait(&L.bars[1], ph.mm);
  ph.mm ^= 1;
  tc_after();
}
__device__ __forceinline__ void sync_all() {
  tc_before();
  __syncthreads();
  tc_after();
}

// 64 combined score columns [c0, c0 + 64) of this thread's row
__device__ __forceinline__ void read64(uint32_t trow, int c0, float* v) {
#pragma unroll
  for (int c = 0; c < 64; c += 16) tmem_pair16(trow + c0 + c, trow + 128 + c0 + c, v + c);
}

// index of the (query block, key block) dS tile of a head in AttnArgs::dS
__device__ __forceinline__ long long ds_pair(const AttnArgs& a, int qb, int kb, int nkb) {
  return a.causal ? (long long)qb * (qb + 1) / 2 + kb : (long long)qb * nkb + kb;
}

// number of valid keys of query q among keys [key0, key0 + 64): j < skv and,
// causal, j <= q (one compare per key in the loops)
__device__ __forceinline__ int key_limit(int q, int key0, int skv, bool causal, bool live) {
  return live ? (causal ? min(skv, q + 1) : skv) - key0 : 0;
}

// P = exp(S * scale - m) * inv for keys (kb*128 + c0 + e), masked -> 0
__device__ __forceinline__ void probs(float* v, int q, int key0, int skv, bool causal, bool live,
                                      float scale, float m, float inv) {
  const int lim = key_limit(q, key0, skv, causal, live);
#pragma unroll
  for (int e = 0; e < 64; ++e) v[e] = e < lim ? fast_exp(v[e] * scale - m) * inv : 0.f;
}

// ---- forward -----------------------------------------------------------------------
// smem (no staging: TMA lands fp32 in a tile region, converted in place):
//   Q | K[2] | V[2] | P (pair128); K and V double-buffered so the next block's
//   load is in flight while the current one computes.
// TMEM: S [0,256), O [256,..)/[384,..)
constexpr int kFwdLongSmem = 1024 + 5 * PAIR64 + PAIR128 + 8 * 8 + 256 * 4 + 16;

__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_long_kernel(const __grid_constant__ AttnTma tm, const AttnArgs a, const int* active) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  if (active && *(volatile const int*)active == 0) return;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const uint32_t base = smem_u32(smem);
  const uint32_t tQ = base, tK[2] = {base + PAIR64, base + 2 * PAIR64},
                 tV[2] = {base + 3 * PAIR64, base + 4 * PAIR64}, tP = base + 5 * PAIR64;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 5 * PAIR64 + PAIR128);
  uint64_t* bQ = &bars[0];
  uint64_t* bK = &bars[1];  // [2]
  uint64_t* bV = &bars[3];  // [2]
  uint64_t* bM = &bars[5];
  float* xch = reinterpret_cast<float*>(bars + 8);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(xch + 256);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q4 = warp & 3, half = warp >> 2, c0 = half * 64;
  const int sq = a.sq, skv = a.skv, dh = a.dh;
  const int nqb = (sq + 127) >> 7, nkb = (skv + 127) >> 7;
  const int nprob = a.G * a.Bb * a.H * nqb;
  const uint32_t box = (uint32_t)(128 * dh * 4);
  const Opnd Qk = pair64(tQ, false), Pk = pair128(tP, false);
  if (tid == 0) {
    for (int i = 0; i < 6; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tslot, 512);
  sync_all();
  const uint32_t tmem = *tslot;
  const uint32_t trow = tmem + ((uint32_t)(q4 * 32) << 16);
  const int i = q4 * 32 + lane;
  float amax = 0.f;
  // completed-load counts per buffer (-> mbarrier phases), identical in every thread
  uint32_t nq = 0, nk[2] = {0, 0}, nv[2] = {0, 0}, nm = 0;
  auto coords = [&](int z, int& g, int& b, int& h, int& qb) {
    qb = z % nqb;
    int r = z / nqb;
    h = r % a.H;
    r /= a.H;
    b = r % a.Bb;
    g = r / a.Bb;
  };
  auto load = [&](uint32_t dst, uint64_t* bar, int which, int g, int b, int h, int row0) {
    mbar_expect_tx(bar, box);
    tma_box(dst, tm, which, g, b, h, bar, row0);
  };
  auto mma_wait = [&]() {
    mbar_wait(bM, nm & 1);
    ++nm;
    tc_after();
  };
  if (tid == 0 && (int)blockIdx.x < nprob) {
    int g, b, h, qb;
    coords(blockIdx.x, g, b, h, qb);
    load(tQ, bQ, TQ, g, b, h, qb * 128);
    load(tK[0], &bK[0], TK, g, b, h, 0);
  }
  for (int z = blockIdx.x; z < nprob; z += gridDim.x) {
    int g, b, h, qb;
    coords(z, g, b, h, qb);
    const int q = qb * 128 + i;  // this thread's query
    const int kend = a.causal ? min(nkb, qb + 1) : nkb;
    mbar_wait(bQ, nq & 1);
    ++nq;
    conv_inplace(tQ, 128, 128, dh, tid, kThreads, amax);
    float m = -INFINITY, l = 0.f, inv = 0.f;
    // steps 0..kend-1: pass A (row statistics); kend..2 kend-1: pass B
    for (int st = 0; st < 2 * kend; ++st) {
      const bool pb = st >= kend;
      const int kb = pb ? st - kend : st, kbuf = st & 1;
      mbar_wait(&bK[kbuf], nk[kbuf] & 1);
      ++nk[kbuf];
      conv_inplace(tK[kbuf], 128, 128, dh, tid, kThreads, amax);
      fence_async_smem();
      sync_all();
      if (tid == 0) {
        // the other K buffer held the block of step st-1, whose S is done
        if (st + 1 < 2 * kend) {
          const int nb = st + 1 < kend ? st + 1 : st + 1 - kend;
          load(tK[(st + 1) & 1], &bK[(st + 1) & 1], TK, g, b, h, nb * 128);
        }
        // V one step ahead: V_0 during the last statistics step, V_kb+1 during pass-B step kb
        if (st == kend - 1) load(tV[0], &bV[0], TV, g, b, h, 0);
        if (pb && kb + 1 < kend) load(tV[(kb + 1) & 1], &bV[(kb + 1) & 1], TV, g, b, h, (kb + 1) * 128);
        mma3(tmem, tmem + 128, Qk, pair64(tK[kbuf], false), 128, dh >> 4);  // S = Q K^T
        mma_commit<1>(bM);
      }
      mma_wait();
      float v[64];
      read64(trow, c0, v);
      if (!pb) {
        // pass A: the row max of the scaled, masked scores only
        const int lim = key_limit(q, kb * 128 + c0, skv, a.causal != 0, true);
        float mh = -INFINITY;
#pragma unroll
        for (int e = 0; e < 64; ++e) mh = fmaxf(mh, e < lim ? v[e] * a.scale : -INFINITY);
        xch[half * 128 + i] = mh;
        sync_all();
        m = fmaxf(m, fmaxf(xch[i], xch[128 + i]));
        sync_all();  // xch reads done; S consumed
      } else {
        // pass B: P~ = exp(S*scale - m) (the final row max: no rescaling) ->
        // tile; O += P~ V; l += sum P~; O is normalised by 1/l at the end
        const int vbuf = kb & 1;
        mbar_wait(&bV[vbuf], nv[vbuf] & 1);
        ++nv[vbuf];
        conv_inplace(tV[vbuf], 128, 128, dh, tid, kThreads, amax);
        probs(v, q, kb * 128 + c0, skv, a.causal != 0, q < sq, a.scale, m, 1.f);
#pragma unroll
        for (int e = 0; e < 64; ++e) l += v[e];
#pragma unroll
        for (int c = 0; c < 8; ++c) put8(Pk.hi, Pk.lo, 128, i, half * 8 + c, v + c * 8, amax);
        fence_async_smem();
        sync_all();
        if (tid == 0) {
          mma3(tmem + 256, tmem + 384, Pk, pair64(tV[vbuf], true), dh, 8, kb > 0);
          mma_commit<1>(bM);
        }
        mma_wait();
      }
    }
    // Q and both K buffers are free: the next problem's first loads overlap the epilogue
    if (tid == 0 && z + (int)gridDim.x < nprob) {
      int g2, b2, h2, qb2;
      coords(z + gridDim.x, g2, b2, h2, qb2);
      load(tQ, bQ, TQ, g2, b2, h2, qb2 * 128);
      load(tK[0], &bK[0], TK, g2, b2, h2, 0);
    }
    // l = the row sum of P~ over both key-column halves; O = (P~ V) / l
    xch[half * 128 + i] = l;
    sync_all();
    l = xch[i] + xch[128 + i];
    inv = l > 0.f ? 1.f / l : 0.f;
    {
      const long long ld = a.Ohl.ok() ? a.Ohl.ld : a.O.ld;
      rows_out_hl(trow + 256, trow + 384,
                  a.O.ok() ? a.O.at(g, b, h) + (long long)qb * 128 * ld : nullptr,
                  a.Ohl.ok() ? a.Ohl.at(g, b, h) + (long long)qb * 128 * ld : nullptr, ld, i,
                  sq - qb * 128, half * (dh >> 1), dh >> 1, inv, amax);
    }
    if (half == 0 && q < sq) {
      float* stp = a.P.at(g, b, h) + 2LL * q;
      stp[0] = m;
      stp[1] = inv;
    }
    sync_all();
  }
  if (amax >= 65520.f && amax <= FLT_MAX && a.range_flag) atomicOr(a.range_flag, 1);
  sync_all();
  if (warp == 0) tmem_free(tmem, 512);
}

// t_i = dO_i . O_i (the softmax-VJP row constant), fixed order
__device__ __forceinline__ float row_dot(const float* x, const float* y, int n) {
  float t = 0.f;
  for (int e = 0; e < n; e += 4) {
    const float4 u = *reinterpret_cast<const float4*>(x + e);
    const float4 w = *reinterpret_cast<const float4*>(y + e);
    t += u.x * w.x;
    t += u.y * w.y;
    t += u.z * w.z;
    t += u.w * w.w;
  }
  return t;
}

// ---- backward: dK, dV per 128-key block ------------------------------------------
// tiles: t0 = K, t1 = V, t2 = Q, t3 = dO, t4 = P then dS;
// TMEM: S / dP [0,256), dV [256,..)/[320,..), dK [384,..)/[448,..)
__global__ void __launch_bounds__(kThreads, 1)
    attn_bwd_dkdv_kernel(const __grid_constant__ AttnTma tm, const AttnArgs a, const int* active) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  if (active && *(volatile const int*)active == 0) return;
  const LongSmem L = carve(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q4 = warp & 3, half = warp >> 2, c0 = half * 64;
  const int sq = a.sq, skv = a.skv, dh = a.dh;
  const int nqb = (sq + 127) >> 7, nkb = (skv + 127) >> 7;
  const int nprob = a.G * a.Bb * a.H * nkb;
  const Opnd Kk = pair64(L.t0, false), Vk = pair64(L.t1, false);
  const Opnd Qm = pair64(L.t2, true), dOk = pair64(L.t3, false), dOm = pair64(L.t3, true);
  const Opnd Pm = pair128(L.t4, true);
  if (tid == 0) {
    mbar_init(&L.bars[0], 1);
    mbar_init(&L.bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(L.tslot, 512);
  sync_all();
  const uint32_t tmem = *L.tslot;
  const uint32_t trow = tmem + ((uint32_t)(q4 * 32) << 16);
  const int i = q4 * 32 + lane;
  float amax = 0.f;
  Phase ph;
  auto kv_problem = [&](int z, int& kb, int& g, int& b, int& h) {
    kb = z % nkb;
    int r = z / nkb;
    h = r % a.H;
    r /= a.H;
    b = r % a.Bb;
    g = r / a.Bb;
  };
  if (tid == 0 && (int)blockIdx.x < nprob) {
    int kb, g, b, h;
    kv_problem(blockIdx.x, kb, g, b, h);
    issue(L, tm, TK, g, b, h, kb * 128, dh);
  }
  for (int z = blockIdx.x; z < nprob; z += gridDim.x) {
    int kb, g, b, h;
    kv_problem(z, kb, g, b, h);
    const int qb0 = a.causal ? kb : 0;
    const float* stats = a.P.at(g, b, h);
    wait_stage(L, ph);
    land(L, tm, TK, Kk.hi, Kk.lo, dh, tid, amax);
    fence_async_smem();
    sync_all();
    if (tid == 0) issue(L, tm, TV, g, b, h, kb * 128, dh);
    wait_stage(L, ph);
    land(L, tm, TV, Vk.hi, Vk.lo, dh, tid, amax);
    fence_async_smem();
    sync_all();
    if (tid == 0) issue(L, tm, TQ, g, b, h, qb0 * 128, dh);
    for (int qb = qb0; qb < nqb; ++qb) {
      const bool first = qb == qb0;
      const int q = qb * 128 + i;
      const bool live = q < sq;
      wait_stage(L, ph);
      land(L, tm, TQ, Qm.hi, Qm.lo, dh, tid, amax);
      fence_async_smem();
      sync_all();
      if (tid == 0) {
        issue(L, tm, TDO, g, b, h, qb * 128, dh);
        mma3(tmem, tmem + 128, Opnd{Qm.hi, Qm.lo, 128, false}, Kk, 128, dh >> 4);  // S = Q K^T
        mma_commit<1>(&L.bars[1]);
      }
      const float mi = live ? stats[2LL * q] : 0.f;
      const float inv = live ? stats[2LL * q + 1] : 0.f;
      mma_done(L, ph);
      float p[64];
      read64(trow, c0, p);
      probs(p, q, kb * 128 + c0, skv, a.causal != 0, live, a.scale, mi, inv);
#pragma unroll
      for (int c = 0; c < 8; ++c) put8(Pm.hi, Pm.lo, 128, i, half * 8 + c, p + c * 8, amax);
      wait_stage(L, ph);
      land(L, tm, TDO, dOk.hi, dOk.lo, dh, tid, amax);
      fence_async_smem();
      sync_all();
      if (tid == 0) {
        if (qb + 1 < nqb) issue(L, tm, TQ, g, b, h, (qb + 1) * 128, dh);
        mma3(tmem + 256, tmem + 320, Pm, dOm, dh, 8, !first);  // dV += P^T dO
        mma3(tmem, tmem + 128, dOk, Vk, 128, dh >> 4);         // dP = dO V^T
        mma_commit<1>(&L.bars[1]);
      }
      const float t = live ? stats[2LL * sq + q] : 0.f;  // dO . O, written by the dQ kernel
      mma_done(L, ph);
      float dp[64];
      read64(trow, c0, dp);
#pragma unroll
      for (int e = 0; e < 64; ++e) dp[e] = p[e] * (dp[e] - t);  // dS (0 where P is 0)
#pragma unroll
      for (int c = 0; c < 8; ++c) put8(Pm.hi, Pm.lo, 128, i, half * 8 + c, dp + c * 8, amax);
      fence_async_smem();
      sync_all();
      if (tid == 0) {
        mma3(tmem + 384, tmem + 448, Pm, Qm, dh, 8, !first);  // dK += dS^T Q
        mma_commit<1>(&L.bars[1]);
        // the dQ kernel's operand: this dS tile, pre-split (async)
        if (a.dS.ok()) bulk_store(a.dS.at(g, b, h) + ds_pair(a, qb, kb, nkb) * (long long)(128 * 128),
                                  Pm.hi, 4 * TILE64);
      }
      mma_done(L, ph);
      if (tid == 0 && a.dS.ok()) bulk_store_wait_read();  // Pm is rewritten next step
    }
    // the staging is free: the next problem's K streams in under this epilogue
    if (tid == 0 && z + (int)gridDim.x < nprob) {
      int kb2, g2, b2, h2;
      kv_problem(z + gridDim.x, kb2, g2, b2, h2);
      issue(L, tm, TK, g2, b2, h2, kb2 * 128, dh);
    }
    const int nv = skv - kb * 128;
    {
      const long long ldv = a.dVhl.ok() ? a.dVhl.ld : a.dV.ld;
      const long long ldk = a.dKhl.ok() ? a.dKhl.ld : a.dK.ld;
      const long long ov = (long long)kb * 128 * ldv, ok = (long long)kb * 128 * ldk;
      rows_out_hl(trow + 256, trow + 320, a.dV.ok() ? a.dV.at(g, b, h) + ov : nullptr,
                  a.dVhl.ok() ? a.dVhl.at(g, b, h) + ov : nullptr, ldv, i, nv, half * (dh >> 1),
                  dh >> 1, 1.f, amax);
      rows_out_hl(trow + 384, trow + 448, a.dK.ok() ? a.dK.at(g, b, h) + ok : nullptr,
                  a.dKhl.ok() ? a.dKhl.at(g, b, h) + ok : nullptr, ldk, i, nv, half * (dh >> 1),
                  dh >> 1, a.scale, amax);
    }
    sync_all();
  }
  if (amax >= 65520.f && amax <= FLT_MAX && a.range_flag) atomicOr(a.range_flag, 1);
  if (tid == 0 && a.dS.ok()) bulk_store_wait();
  sync_all();
  if (warp == 0) tmem_free(tmem, 512);
}

// ---- backward: t_i = dO_i . O_i for every query row (before dK/dV when the
// dQ kernel reads the stored dS tiles) --------------------------------------------
__global__ void __launch_bounds__(256) attn_rowdot_kernel(const AttnArgs a, const int* active) {
  pdl_wait();
  pdl_trigger();
  if (active && *(volatile const int*)active == 0) return;
  const long long n = (long long)a.G * a.Bb * a.H * a.sq;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int q = (int)(i % a.sq);
  long long r = i / a.sq;
  const int h = (int)(r % a.H);
  r /= a.H;
  const int b = (int)(r % a.Bb), g = (int)(r / a.Bb);
  a.P.at(g, b, h)[2LL * a.sq + q] =
      row_dot(a.dO.at(g, b, h) + (long long)q * a.dO.ld, a.O.at(g, b, h) + (long long)q * a.O.ld,
              a.dh);
}

// ---- backward: dQ per 128-query block from the stored dS tiles ------------------------
// tiles: t2 = K, t4 = dS (bulk-loaded pre-split); TMEM: dQ [256,..)/[384,..)
__global__ void __launch_bounds__(kThreads, 1)
    attn_bwd_dq_ds_kernel(const __grid_constant__ AttnTma tm, const AttnArgs a, const int* active) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  if (active && *(volatile const int*)active == 0) return;
  const LongSmem L = carve(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q4 = warp & 3, half = warp >> 2;
  const int sq = a.sq, skv = a.skv, dh = a.dh;
  const int nqb = (sq + 127) >> 7, nkb = (skv + 127) >> 7;
  const int nprob = a.G * a.Bb * a.H * nqb;
  const Opnd Kk = pair64(L.t2, false), Km = pair64(L.t2, true);
  const Opnd dSk = pair128(L.t4, false);
  uint64_t* dsb = &L.bars[2];
  if (tid == 0) {
    mbar_init(&L.bars[0], 1);
    mbar_init(&L.bars[1], 1);
    mbar_init(dsb, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(L.tslot, 512);
  sync_all();
  const uint32_t tmem = *L.tslot;
  const uint32_t trow = tmem + ((uint32_t)(q4 * 32) << 16);
  const int i = q4 * 32 + lane;
  float amax = 0.f;
  Phase ph;
  uint32_t dsp = 0;
  (void)Kk;
  for (int z = blockIdx.x; z < nprob; z += gridDim.x) {
    const int qb = z % nqb;
    int r = z / nqb;
    const int h = r % a.H;
    r /= a.H;
    const int b = r % a.Bb, g = r / a.Bb;
    const int kend = a.causal ? min(nkb, qb + 1) : nkb;
    const float* ds0 = a.dS.at(g, b, h);
    if (tid == 0) issue(L, tm, TK, g, b, h, 0, dh);
    for (int kb = 0; kb < kend; ++kb) {
      if (tid == 0) {
        mbar_expect_tx(dsb, 4 * TILE64);
        bulk_load(L.t4, ds0 + ds_pair(a, qb, kb, nkb) * (long long)(128 * 128), 4 * TILE64, dsb);
      }
      wait_stage(L, ph);
      land(L, tm, TK, Km.hi, Km.lo, dh, tid, amax);
      fence_async_smem();
      mbar_wait(dsb, dsp);
      dsp ^= 1;
      sync_all();
      if (tid == 0) {
        if (kb + 1 < kend) issue(L, tm, TK, g, b, h, (kb + 1) * 128, dh);
        mma3(tmem + 256, tmem + 384, dSk, Km, dh, 8, kb > 0);  // dQ += dS K
        mma_commit<1>(&L.bars[1]);
      }
      mma_done(L, ph);
    }
    {
      const long long ldq = a.dQhl.ok() ? a.dQhl.ld : a.dQ.ld;
      const long long oq = (long long)qb * 128 * ldq;
      rows_out_hl(trow + 256, trow + 384, a.dQ.ok() ? a.dQ.at(g, b, h) + oq : nullptr,
                  a.dQhl.ok() ? a.dQhl.at(g, b, h) + oq : nullptr, ldq, i, sq - qb * 128,
                  half * (dh >> 1), dh >> 1, a.scale, amax);
    }
    sync_all();
  }
  if (amax >= 65520.f && amax <= FLT_MAX && a.range_flag) atomicOr(a.range_flag, 1);
  sync_all();
  if (warp == 0) tmem_free(tmem, 512);
}

// ---- backward: dQ per 128-query block ---------------------------------------------
// tiles: t0 = Q, t1 = dO, t2 = K, t3 = V, t4 = dS; TMEM: S / dP [0,256), dQ [256,..)/[384,..)
__global__ void __launch_bounds__(kThreads, 1)
    attn_bwd_dq_kernel(const __grid_constant__ AttnTma tm, const AttnArgs a, const int* active) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  if (active && *(volatile const int*)active == 0) return;
  const LongSmem L = carve(smem_raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q4 = warp & 3, half = warp >> 2, c0 = half * 64;
  const int sq = a.sq, skv = a.skv, dh = a.dh;
  const int nqb = (sq + 127) >> 7, nkb = (skv + 127) >> 7;
  const int nprob = a.G * a.Bb * a.H * nqb;
  const Opnd Qk = pair64(L.t0, false), dOk = pair64(L.t1, false);
  const Opnd Kk = pair64(L.t2, false), Km = pair64(L.t2, true), Vk = pair64(L.t3, false);
  const Opnd dSk = pair128(L.t4, false);
  if (tid == 0) {
    mbar_init(&L.bars[0], 1);
    mbar_init(&L.bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(L.tslot, 512);
  sync_all();
  const uint32_t tmem = *L.tslot;
  const uint32_t trow = tmem + ((uint32_t)(q4 * 32) << 16);
  const int i = q4 * 32 + lane;
  float amax = 0.f;
  Phase ph;
  auto q_problem = [&](int z, int& qb, int& g, int& b, int& h) {
    qb = z % nqb;
    int r = z / nqb;
    h = r % a.H;
    r /= a.H;
    b = r % a.Bb;
    g = r / a.Bb;
  };
  if (tid == 0 && (int)blockIdx.x < nprob) {
    int qb, g, b, h;
    q_problem(blockIdx.x, qb, g, b, h);
    issue(L, tm, TQ, g, b, h, qb * 128, dh);
  }
  for (int z = blockIdx.x; z < nprob; z += gridDim.x) {
    int qb, g, b, h;
    q_problem(z, qb, g, b, h);
    const int q = qb * 128 + i;
    const bool live = q < sq;
    const int kend = a.causal ? min(nkb, qb + 1) : nkb;
    const float* stats = a.P.at(g, b, h);
    wait_stage(L, ph);
    land(L, tm, TQ, Qk.hi, Qk.lo, dh, tid, amax);
    fence_async_smem();
    sync_all();
    if (tid == 0) issue(L, tm, TDO, g, b, h, qb * 128, dh);
    wait_stage(L, ph);
    land(L, tm, TDO, dOk.hi, dOk.lo, dh, tid, amax);
    fence_async_smem();
    sync_all();
    if (tid == 0) issue(L, tm, TK, g, b, h, 0, dh);
    const float mi = live ? stats[2LL * q] : 0.f;
    const float inv = live ? stats[2LL * q + 1] : 0.f;
    const float t = live ? row_dot(a.dO.at(g, b, h) + (long long)q * a.dO.ld,
                                   a.O.at(g, b, h) + (long long)q * a.O.ld, dh)
                         : 0.f;
    // published for the dK/dV kernel (launched after this one) next to the row statistics
    if (live && half == 0) const_cast<float*>(stats)[2LL * sq + q] = t;
    for (int kb = 0; kb < kend; ++kb) {
      wait_stage(L, ph);
      land(L, tm, TK, Kk.hi, Kk.lo, dh, tid, amax);
      fence_async_smem();
      sync_all();
      if (tid == 0) {
        issue(L, tm, TV, g, b, h, kb * 128, dh);
        mma3(tmem, tmem + 128, Qk, Kk, 128, dh >> 4);  // S = Q K^T
        mma_commit<1>(&L.bars[1]);
      }
      mma_done(L, ph);
      float p[64];
      read64(trow, c0, p);
      probs(p, q, kb * 128 + c0, skv, a.causal != 0, live, a.scale, mi, inv);
      wait_stage(L, ph);
      land(L, tm, TV, Vk.hi, Vk.lo, dh, tid, amax);
      fence_async_smem();
      sync_all();
      if (tid == 0) {
        if (kb + 1 < kend) issue(L, tm, TK, g, b, h, (kb + 1) * 128, dh);
        mma3(tmem, tmem + 128, dOk, Vk, 128, dh >> 4);  // dP = dO V^T
        mma_commit<1>(&L.bars[1]);
      }
      mma_done(L, ph);
      float dp[64];
      read64(trow, c0, dp);
#pragma unroll
      for (int e = 0; e < 64; ++e) dp[e] = p[e] * (dp[e] - t);
#pragma unroll
      for (int c = 0; c < 8; ++c) put8(dSk.hi, dSk.lo, 128, i, half * 8 + c, dp + c * 8, amax);
      fence_async_smem();
      sync_all();
      if (tid == 0) {
        mma3(tmem + 256, tmem + 384, dSk, Km, dh, 8, kb > 0);  // dQ += dS K
        mma_commit<1>(&L.bars[1]);
      }
      mma_done(L, ph);
    }
    // the staging is free: the next problem's Q streams in under this epilogue
    if (tid == 0 && z + (int)gridDim.x < nprob) {
      int qb2, g2, b2, h2;
      q_problem(z + gridDim.x, qb2, g2, b2, h2);
      issue(L, tm, TQ, g2, b2, h2, qb2 * 128, dh);
    }
    {
      const long long ldq = a.dQhl.ok() ? a.dQhl.ld : a.dQ.ld;
      const long long oq = (long long)qb * 128 * ldq;
      rows_out_hl(trow + 256, trow + 384, a.dQ.ok() ? a.dQ.at(g, b, h) + oq : nullptr,
                  a.dQhl.ok() ? a.dQhl.at(g, b, h) + oq : nullptr, ldq, i, sq - qb * 128,
                  half * (dh >> 1), dh >> 1, a.scale, amax);
    }
    sync_all();
  }
  if (amax >= 65520.f && amax <= FLT_MAX && a.range_flag) atomicOr(a.range_flag, 1);
  sync_all();
  if (warp == 0) tmem_free(tmem, 512);
}

bool aligned(const Mat& m) {
  return !m.ok() || ((reinterpret_cast<uintptr_t>(m.ptr) & 15) == 0 && m.ld % 4 == 0 &&
                     m.slot_stride % 4 == 0 && m.bstride % 4 == 0 && m.hstride % 4 == 0);
}

AttnTma long_maps(const AttnArgs& a, bool backward) {
  AttnTma t{};
  t.hs_mask = (a.qkv_hs ? (1 << TQ) | (1 << TK) | (1 << TV) : 0) | (a.do_hs ? 1 << TDO : 0);
  auto mk = [&](int which, const Mat& m, int rows) {
    t.m[which] = ((t.hs_mask >> which) & 1)
                     ? tc_make_map(m, a.G, a.Bb, a.H, rows, 64, 128, 32, true, &t.op[which])
                     : tc_make_map(m, a.G, a.Bb, a.H, rows, a.dh, 128, a.dh, false, &t.op[which]);
  };
  mk(TQ, a.Q, a.sq);
  mk(TK, a.K, a.skv);
  mk(TV, a.V, a.skv);
  if (backward) mk(TDO, a.dO, a.sq);
  return t;
}

int sms() {
  static int n = 0;
  if (!n) MGLP_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, 0));
  return n;
}

template <typename K>
void launch_long(K kernel, const AttnTma& t, const AttnArgs& a, long long nprob, const int* active,
                 cudaStream_t s, int smem = kLongSmem) {
  if (nprob == 0) return;
  const int grid = (int)std::min<long long>(nprob, sms());
  launch_k(kernel, dim3(grid), dim3(kThreads), smem, s, 1, t, a, active);
  MGLP_CUDA(cudaGetLastError());
}

}  // namespace

bool attn_long_supported(const AttnArgs& a, bool backward) {
  if (!backward && (a.qkv_hs || a.do_hs)) return attn_flash_supported(a, backward);
  if (backward && a.do_hs) return attn_flash_supported(a, true);
  if (a.do_hs) return false;  // the row dot t_i = dO_i . O_i reads fp32 dO
  if (a.qkv_hs && a.dh != 64) return false;
  if (a.sq < 128 || a.skv < 128 || a.sq > 512 || a.skv > 512) return false;
  if (a.dh != 32 && a.dh != 64) return false;
  if (!a.P.ok() || !aligned(a.Q) || !aligned(a.K) || !aligned(a.V) || !aligned(a.O) ||
      !aligned(a.P))
    return false;
  if (backward && (!aligned(a.dO) || !aligned(a.dQ) || !aligned(a.dK) || !aligned(a.dV)))
    return false;
  return true;
}

void launch_attn_fwd_long(const AttnArgs& a, const int* active, cudaStream_t s) {
  if (a.qkv_hs) return launch_attn_fwd_flash(a, active, s);  // pre-split operands: attn_flash.cu
  if (!attn_long_supported(a, false)) throw ContractViolation("attn_fwd_long: unsupported shape");
  static bool attr = [] {
    MGLP_CUDA(cudaFuncSetAttribute(attn_fwd_long_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, kFwdLongSmem));
    return true;
  }();
  (void)attr;
  launch_long(attn_fwd_long_kernel, long_maps(a, false), a,
              (long long)a.G * a.Bb * a.H * ((a.sq + 127) / 128), active, s, kFwdLongSmem);
}

void launch_attn_bwd_long(const AttnArgs& a, const int* active, cudaStream_t s) {
  if (a.do_hs) return launch_attn_bwd_flash(a, active, s);  // pre-split dO: attn_flash.cu
  if (!attn_long_supported(a, true)) throw ContractViolation("attn_bwd_long: unsupported shape");
  static bool attr = [] {
    MGLP_CUDA(cudaFuncSetAttribute(attn_bwd_dkdv_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, kLongSmem));
    MGLP_CUDA(cudaFuncSetAttribute(attn_bwd_dq_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, kLongSmem));
    return true;
  }();
  (void)attr;
  const AttnTma t = long_maps(a, true);
  const long long heads = (long long)a.G * a.Bb * a.H;
  if (a.dS.ok()) {
    static bool attr2 = [] {
      MGLP_CUDA(cudaFuncSetAttribute(attn_bwd_dq_ds_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, kLongSmem));
      return true;
    }();
    (void)attr2;
    // t_i first; dK/dV stores every dS tile; dQ = sum over key blocks of dS K
    const long long rows = heads * a.sq;
    launch_k(attn_rowdot_kernel, dim3((unsigned)((rows + 255) / 256)), dim3(256), 0, s, 1, a,
             active);
    launch_long(attn_bwd_dkdv_kernel, t, a, heads * ((a.skv + 127) / 128), active, s);
    launch_long(attn_bwd_dq_ds_kernel, t, a, heads * ((a.sq + 127) / 128), active, s);
    return;
  }
  // dQ first: it also publishes t_i = dO_i . O_i (at P + 2 sq + i) for dK / dV
  launch_long(attn_bwd_dq_kernel, t, a, heads * ((a.sq + 127) / 128), active, s);
  launch_long(attn_bwd_dkdv_kernel, t, a, heads * ((a.skv + 127) / 128), active, s);
}

}  // namespace mglp
