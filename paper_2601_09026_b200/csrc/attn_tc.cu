// Fused multi-head attention on tcgen05 for sequences of <= 128 tokens: the
// device form of the reference's attention / vjp_attention
// (blocks.cpp:142-236; softmax_rows / vjp_softmax_rows, tensor.cpp:310-342).
//
// Persistent kernels, one CTA per SM, looping over the (member g, batch b,
// head h) problems of a family. Every operand is split into fp16 hi / lo'
// exactly as in gemm_tc.cu (same ~22-bit operand precision; main and
// correction products in separate TMEM accumulators), but the whole per-head
// problem stays on chip:
//   forward   S = Q K^T (TMEM) -> softmax (one thread per query row and half
//             of the keys; the reference's scale, -inf causal mask,
//             max-subtracted exp and 1/sum) -> P (hi/lo' in smem; for the
//             backward either fp32 rows or, at s = 128, the hi/lo' tiles
//             themselves, bulk-copied out: AttnArgs::p_hl) -> O = P V (TMEM)
//             -> O (fp32 and/or pre-split for the O-projection)
//   backward  dP = dO V^T and dV = P^T dO (TMEM) -> dS = P (dP - rowsum(dP P))
//             (hi/lo' in smem; P read back from its hi/lo' tiles) ->
//             dQ = dS K / sqrt(dh), dK = dS^T Q / sqrt(dh) (fp32 and/or
//             pre-split for the QKV dgrad)
// replacing 2 + 4 tensor-core GEMM launches and 2 softmax row kernels (and the
// S / dS round trips through HBM) per attention evaluation.
//
// Data movement: rows are fetched with cp.async.bulk into an fp32 staging
// buffer (completion on an mbarrier, no register cost, the next problem's
// first operands prefetched while the current one computes) and converted
// smem -> smem. Every operand is kept ONCE, in its natural row-major
// orientation, as a pair of fp16 SWIZZLE_128B tiles (hi, lo'): [rows][64
// columns] blocks, 16-byte chunk c of row r at (c ^ (r & 7)). The same tile
// is a K-major operand (rows = M/N, K = columns) for one MMA and an MN-major
// operand (rows = K, columns = M/N; UMMA descriptor LBO = block stride, major
// bit set in the instruction descriptor) for another, so nothing is ever
// transposed: Q (S: A, K-major; dK: B, MN-major), K (S: B, K; dQ: B, MN),
// V (PV: B, MN; dP: B, K), dO (dP: A, K; dV: B, MN), P (PV: A, K; dV: A, MN),
// dS (dQ: A, K; dK: A, MN).
#include <cfloat>

#include "attn_common.cuh"

namespace mglp {

using namespace tc;
using namespace attn;

namespace {

constexpr int kThreads = 256;  // 8 warps; warp w owns TMEM lanes 32 (w & 3), column half w >> 2

// ---- forward -------------------------------------------------------------------
// smem (96 KB, two CTAs per SM): [Q | K] (each TMA-staged fp32, converted in
// place to its hi/lo tile pair; P's two 64-key blocks overlay both after S)
// | V | barriers. The next problem's loads go out as soon as O = P V has
// consumed the tiles, so they overlap this problem's epilogue and the other
// CTA's work.
constexpr int kFwdSmem = 1024 + PAIR128 + PAIR64 + 64 + 256 * 4 + 16;

__global__ void __launch_bounds__(kThreads, 2) attn_fwd_kernel(const __grid_constant__ AttnTma tm, const AttnArgs a, const int* active) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  if (active && *(volatile const int*)active == 0) return;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q4 = warp & 3, half = warp >> 2;
  const int sq = a.sq, skv = a.skv, dh = a.dh;
  const int skv16 = rup(skv, 16);
  const uint32_t base = smem_u32(smem);
  const Opnd Qt{base, base + TILE64, 128, false};
  const Opnd Kt{base + PAIR64, base + PAIR64 + TILE64, 128, false};
  const Opnd Pt{base, base + 2 * TILE64, 128, false};  // over [Q | K]: hi blocks 0-1, lo blocks 0-1
  const Opnd Vt{base + PAIR128, base + PAIR128 + TILE64, 128, true};
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + PAIR128 + PAIR64);
  uint64_t* st_full = &bars[0];
  uint64_t* s_bar = &bars[1];
  uint64_t* o_bar = &bars[2];
  float* xch = reinterpret_cast<float*>(bars + 4);  // [2][128] row max / sum exchange
  uint32_t* tslot = reinterpret_cast<uint32_t*>(xch + 256);
  const int nprob = a.G * a.Bb * a.H;

  const bool hs = a.qkv_hs != 0;
  auto issue_loads = [&](int z) {  // one thread
    int g, b, h;
    problem_of(a, z, g, b, h);
    if (hs) {  // pre-split: straight into the tiles (rows >= s zero-filled)
      mbar_expect_tx(st_full, 3 * kHsBytes);
      tma_pair(Qt, tm, TQ, g, b, h, st_full);
      tma_pair(Kt, tm, TK, g, b, h, st_full);
      tma_pair(Vt, tm, TV, g, b, h, st_full);
      return;
    }
    mbar_expect_tx(st_full, (uint32_t)((sq + 2 * skv) * dh * 4));
    tma_box(Qt.hi, tm, TQ, g, b, h, st_full);
    tma_box(Kt.hi, tm, TK, g, b, h, st_full);
    tma_box(Vt.hi, tm, TV, g, b, h, st_full);
  };

  if (tid == 0) {
    mbar_init(st_full, 1);
    mbar_init(s_bar, 1);
    mbar_init(o_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tslot, 256);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = *tslot;
  const uint32_t trow = tmem + ((uint32_t)(q4 * 32) << 16);
  const int i = q4 * 32 + lane;  // query row = TMEM lane
  float amax = 0.f;
  if (tid == 0 && (int)blockIdx.x < nprob) issue_loads(blockIdx.x);

  int it = 0;
  for (int z = blockIdx.x; z < nprob; z += gridDim.x, ++it) {
    int g, b, h;
    problem_of(a, z, g, b, h);
    const uint32_t ph = it & 1;
    mbar_wait(st_full, ph);
    if (!hs) {
      conv_inplace(Qt.hi, sq, 128, dh, tid, kThreads, amax);
      conv_inplace(Kt.hi, skv, skv16, dh, tid, kThreads, amax);
      conv_inplace(Vt.hi, skv, skv16, dh, tid, kThreads, amax);
      fence_async_smem();
      tc_before();
      __syncthreads();
      tc_after();
    }
    if (tid == 0) {
      mma3(tmem, tmem + 128, Qt, Kt, skv16, dh >> 4);  // S
      mma_commit<1>(s_bar);
    }
    // ---- softmax_rows(S * scale) with the causal mask (tensor.cpp:310-326,
    // blocks.cpp:160-166): row i, keys [64 half, 64 half + 64) ----
    mbar_wait(s_bar, ph);
    tc_after();
    const int c0 = half * 64;
    const bool any = c0 < skv16;  // warp-uniform
    float v[64];
    float m = -INFINITY;
    if (any) {
#pragma unroll
      for (int c = 0; c < 64; c += 16) {
        if (c0 + c < skv16) {
          tmem_pair16(trow + c0 + c, trow + 128 + c0 + c, v + c);
        } else {
#pragma unroll
          for (int e = 0; e < 16; ++e) v[c + e] = 0.f;
        }
      }
      // valid keys of this row: j < lim (causal: j <= i), one compare per key
      const int lim = (a.causal ? min(skv, i + 1) : skv) - c0;
#pragma unroll
      for (int e = 0; e < 64; ++e) {
        v[e] = e < lim ? v[e] * a.scale : -INFINITY;
        m = fmaxf(m, v[e]);
      }
    }
    xch[half * 128 + i] = m;
    tc_before();
    __syncthreads();
    m = fmaxf(xch[i], xch[128 + i]);
    float sum = 0.f;
    if (any) {
#pragma unroll
      for (int e = 0; e < 64; ++e) {
        v[e] = v[e] == -INFINITY ? 0.f : fast_exp(v[e] - m);
        sum += v[e];
      }
    }
    __syncthreads();  // every max read before the sums overwrite xch
    xch[half * 128 + i] = sum;
    __syncthreads();
    const float inv = 1.f / (xch[i] + xch[128 + i]);
    if (any) {
#pragma unroll
      for (int e = 0; e < 64; ++e) v[e] *= inv;
      if (a.P.ok() && !a.p_hl && i < sq) {
        float* prow = a.P.at(g, b, h) + i * (long long)a.P.ld + c0;
#pragma unroll
        for (int e = 0; e < 64; e += 4)
          if (c0 + e < skv) *reinterpret_cast<float4*>(prow + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
      }
      // P (row i, K = keys) as the A operand of O = P V; zero beyond skv
#pragma unroll
      for (int c = 0; c < 8; ++c)
        if (c0 + c * 8 < skv16) put8(Pt.hi, Pt.lo, 128, i, half * 8 + c, v + c * 8, amax);
    }
    fence_async_smem();
    tc_before();
    __syncthreads();
    if (tid == 0) {
      tc_after();
      mma3(tmem, tmem + 128, Pt, Vt, dh, skv16 >> 4);  // O
      mma_commit<1>(o_bar);
      // P for the backward: the hi|lo' tiles themselves (async, coalesced)
      if (a.P.ok() && a.p_hl) bulk_store(a.P.at(g, b, h), Pt.hi, 4 * TILE64);
    }
    mbar_wait(o_bar, ph);
    tc_after();
    // the tiles are free (once the P copy has read them): the next problem's
    // loads overlap this epilogue
    if (tid == 0 && z + (int)gridDim.x < nprob) {
      bulk_store_wait_read();
      issue_loads(z + gridDim.x);
    }
    rows_out_hl(trow, trow + 128, a.O.ok() ? a.O.at(g, b, h) : nullptr,
                a.Ohl.ok() ? a.Ohl.at(g, b, h) : nullptr, a.Ohl.ok() ? a.Ohl.ld : a.O.ld, i, sq,
                half * (dh >> 1), dh >> 1, 1.f, amax);
    tc_before();
    __syncthreads();  // TMEM free for the next problem
  }
  if (amax >= 65520.f && amax <= FLT_MAX && a.range_flag) atomicOr(a.range_flag, 1);
  if (tid == 0) bulk_store_wait();
  tc_before();
  __syncthreads();
  if (warp == 0) tmem_free(tmem, 256);
}

// ---- backward ------------------------------------------------------------------
// smem: staging fp32 64 KB ([dO | V], then P, then [Q | K]) | tiles:
//   T0 = [dO | V] (-> dS), T1 = P (-> [Q | K]) | barriers
// TMEM: dP main [0,128) corr [128,256); dV main [256,..) corr [384,..);
//       dQ main [0,..) corr [64,..); dK main [128,..) corr [192,..)
__global__ void __launch_bounds__(kThreads, 1) attn_bwd_kernel(const __grid_constant__ AttnTma tm, const AttnArgs a, const int* active) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  if (active && *(volatile const int*)active == 0) return;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q4 = warp & 3, half = warp >> 2;
  const int sq = a.sq, skv = a.skv, dh = a.dh;
  const int skv16 = rup(skv, 16), sq16 = rup(sq, 16);
  const uint32_t base = smem_u32(smem);
  const uint32_t stg = base;                    // 64 KB
  const uint32_t st2 = base + 128 * 64 * 4;     // second half of the staging
  const uint32_t T0 = base + 2 * 128 * 64 * 4;  // 64 KB
  const uint32_t T1 = T0 + PAIR128;             // 64 KB
  // [dO | V] -> dS region of problem `it`: T0, or -- when every operand
  // arrives pre-split and P too (the staging is then unused) -- T0 and the
  // staging alternately, so the next problem's dO / V load under this one
  const bool pp2 = a.qkv_hs && a.do_hs && a.p_hl && a.pingpong;
  auto rbase = [&](int it) -> uint32_t { return (pp2 && (it & 1)) ? stg : T0; };
  auto dOk_ = [&](int it) { return Opnd{rbase(it), rbase(it) + TILE64, 128, false}; };  // dP: A
  auto Vk_ = [&](int it) {
    return Opnd{rbase(it) + PAIR64, rbase(it) + PAIR64 + TILE64, 128, false};  // dP: B
  };
  const Opnd Pm{T1, T1 + 2 * TILE64, 128, true};          // dV: A
  const Opnd Qm{T1, T1 + TILE64, 128, true};              // dK: B
  const Opnd Km{T1 + PAIR64, T1 + PAIR64 + TILE64, 128, true};  // dQ: B
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * 128 * 64 * 4 + 2 * PAIR128);
  uint64_t* st_full = &bars[0];
  uint64_t* m_bar = &bars[1];
  uint64_t* p_full = &bars[2];  // p_hl: the pre-split P tiles landed in T1
  uint64_t* dov_full = &bars[3];  // [2] (pp2) dO / V landed in region it & 1
  float* xch = reinterpret_cast<float*>(bars + 8);  // [2][128] row-sum exchange
  uint32_t* tslot = reinterpret_cast<uint32_t*>(xch + 256);
  const int nprob = a.G * a.Bb * a.H;

  // pre-split operands (qkv_hs / do_hs) land straight in their tiles, once
  // those are free; fp32 ones go through the staging and are converted
  const bool hsq = a.qkv_hs != 0, hsd = a.do_hs != 0;
  auto load_dov = [&](int z, int it) {
    int g, b, h;
    problem_of(a, z, g, b, h);
    if (lane == 0) {
      uint64_t* bar = pp2 ? &dov_full[it & 1] : st_full;
      mbar_expect_tx(bar, (hsd ? kHsBytes : (uint32_t)(sq * dh * 4)) +
                              (hsq ? kHsBytes : (uint32_t)(skv * dh * 4)));
      if (hsd) tma_pair(dOk_(it), tm, TDO, g, b, h, bar);
      else tma_box(stg, tm, TDO, g, b, h, bar);
      if (hsq) tma_pair(Vk_(it), tm, TV, g, b, h, bar);
      else tma_box(st2, tm, TV, g, b, h, bar);
    }
    __syncwarp();
  };
  auto load_qk = [&](int g, int b, int h) {
    if (lane == 0) {
      if (hsq) {
        mbar_expect_tx(st_full, 2 * kHsBytes);
        tma_pair(Qm, tm, TQ, g, b, h, st_full);
        tma_pair(Km, tm, TK, g, b, h, st_full);
      } else {
        mbar_expect_tx(st_full, (uint32_t)((sq + skv) * dh * 4));
        tma_box(stg, tm, TQ, g, b, h, st_full);
        tma_box(st2, tm, TK, g, b, h, st_full);
      }
    }
    __syncwarp();
  };

  const bool phl = a.p_hl != 0;
  auto load_p = [&](int z) {  // one thread: T1 is free
    int g, b, h;
    problem_of(a, z, g, b, h);
    mbar_expect_tx(p_full, 4 * TILE64);
    bulk_load(T1, a.P.at(g, b, h), 4 * TILE64, p_full);
  };

  if (tid == 0) {
    mbar_init(st_full, 1);
    mbar_init(m_bar, 1);
    mbar_init(p_full, 1);
    mbar_init(&dov_full[0], 1);
    mbar_init(&dov_full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tslot, 512);
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = *tslot;
  const uint32_t trow = tmem + ((uint32_t)(q4 * 32) << 16);
  const int r = q4 * 32 + lane;  // TMEM lane: query row (dP, dQ) or key row (dV, dK)
  float amax = 0.f;
  if (warp == 0 && (int)blockIdx.x < nprob) load_dov(blockIdx.x, 0);
  if (phl && tid == 0 && (int)blockIdx.x < nprob) load_p(blockIdx.x);

  uint32_t stp = 0, mp = 0, pp = 0;  // barrier phases
  int it = 0;
  for (int z = blockIdx.x; z < nprob; z += gridDim.x, ++it) {
    int g, b, h;
    problem_of(a, z, g, b, h);
    const bool next = z + (int)gridDim.x < nprob;
    const Opnd dOk = dOk_(it), Vk = Vk_(it);
    const Opnd dOm{dOk.hi, dOk.lo, 128, true};                      // dV: B
    const Opnd dSk{rbase(it), rbase(it) + 2 * TILE64, 128, false};  // dQ: A
    const Opnd dSm{rbase(it), rbase(it) + 2 * TILE64, 128, true};   // dK: A
    // (1) dO, V -> this problem's region
    if (pp2) {
      mbar_wait(&dov_full[it & 1], (it >> 1) & 1);
      // the other region's dS was consumed by the previous problem's dQ / dK
      // MMAs: the next problem's dO / V stream in under this whole problem
      if (warp == 0 && next) load_dov(z + gridDim.x, it + 1);
    } else {
      mbar_wait(st_full, stp);
      stp ^= 1;
    }
    if (!hsd) conv_rows(stg, sq, 128, dh, dOk.hi, dOk.lo, tid, kThreads, amax);
    if (!hsq) conv_rows(st2, skv, skv16, dh, Vk.hi, Vk.lo, tid, kThreads, amax);
    fence_async_smem();  // staging reads ordered before the bulk copies that reuse it
    __syncthreads();
    if (phl) {
      // (2') P arrives pre-split in T1 (sq = skv = 128: no padding rows)
      mbar_wait(p_full, pp);
      pp ^= 1;
    } else {
      if (warp == 0) {
        if (lane == 0) {
          mbar_expect_tx(st_full, (uint32_t)(sq * skv * 4));
          tma_box(stg, tm, TP, g, b, h, st_full);
        }
        __syncwarp();
      }
      // (2) P -> T1 (rows >= sq zero: K padding of dV)
      mbar_wait(st_full, stp);
      stp ^= 1;
      conv_rows(stg, sq, 128, skv, Pm.hi, Pm.lo, tid, kThreads, amax);
      fence_async_smem();
    }
    tc_before();
    __syncthreads();
    tc_after();
    if (warp == 0 && !hsq) load_qk(g, b, h);  // into the staging
    if (tid == 0) {
      mma3(tmem, tmem + 128, dOk, Vk, skv16, dh >> 4);        // dP = dO V^T
      mma3(tmem + 256, tmem + 384, Pm, dOm, dh, sq16 >> 4);  // dV = P^T dO
      mma_commit<1>(m_bar);
    }
    mbar_wait(m_bar, mp);
    mp ^= 1;
    tc_after();
    // (3) vjp_softmax_rows (tensor.cpp:328-342): dS = P (dP - sum_j dP_j P_j),
    // row r = query, keys [64 half, +64)
    {
      const int c0 = half * 64;
      const bool any = c0 < skv16;
      const bool live = r < sq;
      // this half-row of P (zero beyond skv and for rows >= sq) from the
      // hi/lo' tiles just converted for the dV MMA: p = hi + 2^-11 lo', the
      // operand value the MMAs use (<= 2^-22 relative from the stored fp32 P;
      // no second read of P from global memory)
      const int lim = live ? skv - c0 : 0;
      float pv[64];
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {
        if (cc * 8 < lim) {
          const uint32_t off = chunk_off(128, r, half * 8 + cc);
          const uint4 h4 = lds128u(Pm.hi + off), l4 = lds128u(Pm.lo + off);
          const uint32_t hw[4] = {h4.x, h4.y, h4.z, h4.w}, lw[4] = {l4.x, l4.y, l4.z, l4.w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float2 hf = __half22float2(*reinterpret_cast<const __half2*>(&hw[k]));
            const float2 lf = __half22float2(*reinterpret_cast<const __half2*>(&lw[k]));
            pv[cc * 8 + 2 * k] = fmaf(lf.x, kLoInv, hf.x);
            pv[cc * 8 + 2 * k + 1] = fmaf(lf.y, kLoInv, hf.y);
          }
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) pv[cc * 8 + e] = 0.f;
        }
      }
      // every P half-row is in registers and the dV MMA (m_bar) has read P:
      // pre-split Q, K go straight into T1, their load under the dP reads
      if (hsq) {
        __syncthreads();
        if (warp == 0) load_qk(g, b, h);
      }
      float dp[64];
      float t = 0.f;
      if (any) {
#pragma unroll
        for (int c = 0; c < 64; c += 16) {
          if (c0 + c < skv16) {
            tmem_pair16(trow + c0 + c, trow + 128 + c0 + c, dp + c);
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) dp[c + e] = 0.f;
          }
        }
#pragma unroll
        for (int e = 0; e < 64; ++e) t += dp[e] * pv[e];
      }
      xch[half * 128 + r] = t;
      tc_before();
      __syncthreads();  // also: dP / dV MMAs done -> T0 may take dS
      t = xch[r] + xch[128 + r];
      if (any) {
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if (c0 + c * 8 < skv16) {
            float ds[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) ds[e] = pv[c * 8 + e] * (dp[c * 8 + e] - t);
            put8(dSk.hi, dSk.lo, 128, r, half * 8 + c, ds, amax);
          }
        }
      }
    }
    // (4) Q, K -> T1 (the dV MMA is done)
    mbar_wait(st_full, stp);
    stp ^= 1;
    if (!hsq) {
      conv_rows(stg, sq, sq16, dh, Qm.hi, Qm.lo, tid, kThreads, amax);
      conv_rows(st2, skv, skv16, dh, Km.hi, Km.lo, tid, kThreads, amax);
    }
    fence_async_smem();
    tc_before();
    __syncthreads();
    tc_after();
    // the staging is free (and T0 is not: the dS tiles feed dQ / dK)
    if (warp == 0 && next && !hsq && !hsd) load_dov(z + gridDim.x, it + 1);
    if (tid == 0) {
      mma3(tmem, tmem + 64, dSk, Km, dh, skv16 >> 4);         // dQ = dS K
      mma3(tmem + 128, tmem + 192, dSm, Qm, dh, sq16 >> 4);   // dK = dS^T Q
      mma_commit<1>(m_bar);
    }
    // dV rows (keys) under the dQ / dK MMAs (disjoint TMEM columns)
    rows_out_hl(trow + 256, trow + 384, a.dV.ok() ? a.dV.at(g, b, h) : nullptr,
                a.dVhl.ok() ? a.dVhl.at(g, b, h) : nullptr, a.dVhl.ok() ? a.dVhl.ld : a.dV.ld, r,
                skv, half * (dh >> 1), dh >> 1, 1.f, amax);
    mbar_wait(m_bar, mp);
    mp ^= 1;
    tc_after();
    // T0 (dS) is free: pre-split dO / V go straight in under this epilogue
    if (warp == 0 && next && (hsq || hsd) && !pp2) load_dov(z + gridDim.x, it + 1);
    // T1 (Q | K) is free: the next problem's P streams in under this epilogue
    if (phl && tid == 0 && next) load_p(z + gridDim.x);
    rows_out_hl(trow, trow + 64, a.dQ.ok() ? a.dQ.at(g, b, h) : nullptr,
                a.dQhl.ok() ? a.dQhl.at(g, b, h) : nullptr, a.dQhl.ok() ? a.dQhl.ld : a.dQ.ld, r,
                sq, half * (dh >> 1), dh >> 1, a.scale, amax);
    rows_out_hl(trow + 128, trow + 192, a.dK.ok() ? a.dK.at(g, b, h) : nullptr,
                a.dKhl.ok() ? a.dKhl.at(g, b, h) : nullptr, a.dKhl.ok() ? a.dKhl.ld : a.dK.ld, r,
                skv, half * (dh >> 1), dh >> 1, a.scale, amax);
    tc_before();
    __syncthreads();
  }
  if (amax >= 65520.f && amax <= FLT_MAX && a.range_flag) atomicOr(a.range_flag, 1);
  tc_before();
  __syncthreads();
  if (warp == 0) tmem_free(tmem, 512);
}

constexpr int kBwdSmem = 1024 + 2 * 128 * 64 * 4 + 2 * PAIR128 + 64 + 256 * 4 + 16;

bool aligned(const Mat& m) {
  return !m.ok() || ((reinterpret_cast<uintptr_t>(m.ptr) & 15) == 0 && m.ld % 4 == 0 &&
                     m.slot_stride % 4 == 0 && m.bstride % 4 == 0 && m.hstride % 4 == 0);
}

int num_sms() {
  static int sms = 0;
  if (!sms) MGLP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  return sms;
}

AttnTma maps(const AttnArgs& a, bool backward) {
  AttnTma t{};
  auto mk = [&](int which, const Mat& m, int rows, int cols, bool hs) {
    // head-split pre-split: [128][32] boxes (hi, lo' halves) in the tiles'
    // SWIZZLE_128B layout; rows >= s arrive zero-filled
    t.m[which] = hs ? tc_make_map(m, a.G, a.Bb, a.H, rows, cols, 128, 32, true, &t.op[which])
                    : tc_make_map(m, a.G, a.Bb, a.H, rows, cols, rows, cols, false, &t.op[which]);
  };
  mk(TQ, a.Q, a.sq, a.dh, a.qkv_hs);
  mk(TK, a.K, a.skv, a.dh, a.qkv_hs);
  mk(TV, a.V, a.skv, a.dh, a.qkv_hs);
  if (backward) {
    mk(TP, a.P, a.sq, a.skv, false);
    mk(TDO, a.dO, a.sq, a.dh, a.do_hs);
  }
  return t;
}

}  // namespace

bool attn_tc_supported(const AttnArgs& a, bool backward) {
  if (a.sq < 1 || a.skv < 1 || a.sq > 128 || a.skv > 128) return false;
  if (a.sq % 8 || a.skv % 8) return false;
  if (a.dh != 32 && a.dh != 64) return false;
  if ((a.qkv_hs || a.do_hs) && a.dh != 64) return false;
  if (!aligned(a.Q) || !aligned(a.K) || !aligned(a.V) || !aligned(a.O) || !aligned(a.P))
    return false;
  if (backward && (!aligned(a.dO) || !aligned(a.dQ) || !aligned(a.dK) || !aligned(a.dV) || !a.P.ok()))
    return false;
  // pre-split P: 128 x 128 problems whose P slots are 64 KiB apart
  if (a.p_hl && a.P.ok() &&
      (a.sq != 128 || a.skv != 128 || a.P.ld != 128 || (a.Bb > 1 && a.P.bstride % (128 * 128)) ||
       (a.H > 1 && a.P.hstride != 128 * 128)))
    return false;
  return true;
}

void launch_attn_fwd(const AttnArgs& a, const int* active, cudaStream_t s) {
  if (!attn_tc_supported(a, false)) throw ContractViolation("attn_fwd: unsupported shape");
  static bool attr = [] {
    MGLP_CUDA(cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kFwdSmem));
    return true;
  }();
  (void)attr;
  const long long n = (long long)a.G * a.Bb * a.H;
  if (n == 0) return;
  const int grid = (int)std::min<long long>(n, 2 * num_sms());
  AttnTma t = maps(a, false);
  launch_k(attn_fwd_kernel, dim3(grid), dim3(kThreads), kFwdSmem, s, 1, t, a, active);
  MGLP_CUDA(cudaGetLastError());
}

void launch_attn_bwd(const AttnArgs& a_in, const int* active, cudaStream_t s) {
  // MGLP_ATTN_PINGPONG=0 (A/B): one dO / V region, loaded under the epilogue
  static const int pingpong = [] {
    const char* e = getenv("MGLP_ATTN_PINGPONG");
    return (e && atoi(e) == 0) ? 0 : 1;
  }();
  AttnArgs a = a_in;
  a.pingpong = pingpong;
  if (!attn_tc_supported(a, true)) throw ContractViolation("attn_bwd: unsupported shape");
  static bool attr = [] {
    MGLP_CUDA(cudaFuncSetAttribute(attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   kBwdSmem));
    return true;
  }();
  (void)attr;
  const long long n = (long long)a.G * a.Bb * a.H;
  if (n == 0) return;
  const int grid = (int)std::min<long long>(n, num_sms());
  AttnTma t = maps(a, true);
  launch_k(attn_bwd_kernel, dim3(grid), dim3(kThreads), kBwdSmem, s, 1, t, a, active);
  MGLP_CUDA(cudaGetLastError());
}

}  // namespace mglp
