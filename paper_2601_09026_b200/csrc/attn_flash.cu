// Single-pass streamed attention for 128 < s <= 512 with head-split pre-split
// operands (AttnArgs::qkv_hs / do_hs, dh = 64): the GPT-2-style causal decoder
// (s = 512) and ViT (s = 197). The reference's attention / vjp_attention
// (blocks.cpp:142-236; softmax_rows / vjp_softmax_rows, tensor.cpp:310-342).
//
// Forward (CTA = one (member, batch, head, 128-query block); two CTAs per SM,
// 96 KB of shared memory and 256 TMEM columns each, so one CTA's softmax runs
// under the other's MMAs):
//   Q (hi|lo' tiles) once; 64-key blocks j of K and V double-buffered, all
//   TMA'd straight into their tiles (no staging, no conversion);
//   S_j = Q K_j^T -> TMEM [0,128) (main | 2^-11 correction);
//   online softmax with a lazy max: the reference max m of a row moves only
//   when a block raises the row max by more than kLazy (then O and the row
//   sum are rescaled by exp(m_old - m_new)); P~_j = exp(S scale - m) split
//   hi|lo' and written back into TMEM over S_j (fp16x2 packed columns);
//   O += P~_j V_j with A = P~ from TMEM (tcgen05.mma ... [a-tmem]) -> TMEM
//   [128,256); the epilogue writes O / l (fp32 and/or pre-split) and the row
//   statistics (m, 1/l) the backward recomputes P = exp(S scale - m) / l from.
// S is computed once (the two-pass form computed it twice) and no probability
// tile ever goes through shared memory.
#include "attn_common.cuh"

namespace mglp {

using namespace tc;
using namespace attn;

namespace {

constexpr int kThreads = 256;  // warp w: TMEM lanes 32 (w & 3), key / column half w >> 2
constexpr int KB = 64;         // keys per block
constexpr int KT = KB * 128;   // one 64-row hi (or lo') tile: 8 KiB
constexpr float kLazy = 8.f;   // natural-log headroom before the reference max moves

// tcgen05.mma with A in TMEM (fp16x2 packed columns, row = lane)
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t db, uint32_t id,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t"
      "}" ::"r"(d),
      "r"(a_tmem), "l"(db), "r"(id), "r"(accumulate));
}

// D = A . B^T, A (M = 128 rows, K = nk16 * 16) in TMEM: hi at a_hi, lo' at
// a_lo (8 columns per K step), B a smem tile pair; 3-pass split
__device__ __forceinline__ void mma3_ts(uint32_t tm, uint32_t tcor, uint32_t a_hi, uint32_t a_lo,
                                        const Opnd& B, int N, int nk16, bool acc_in) {
  const uint32_t id = idesc(N, false, B.mn);
  for (int k = 0; k < nk16; ++k) {
    const uint32_t ob = B.at(k);
    const uint64_t dbh = desc_sw128(B.hi + ob, B.lbo()), dbl = desc_sw128(B.lo + ob, B.lbo());
    const uint32_t acc = (k > 0 || acc_in) ? 1u : 0u;
    mma_ts(tm, a_hi + 8 * k, dbh, id, acc);
    mma_ts(tcor, a_lo + 8 * k, dbh, id, acc);
    mma_ts(tcor, a_hi + 8 * k, dbl, id, 1u);
  }
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),
      "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st_wait() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void bar_sync() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// ---- forward ---------------------------------------------------------------------
// One accumulator per product: the 2^-11 of the split's correction terms is
// folded into an operand instead of a second TMEM accumulator,
//   S = Q_hi K_hi + Q_lo'' K_hi + Q_hi'' K_lo',   O += P_hi V_hi + P_lo'' V_hi + P_hi'' V_lo'
// with X_lo'' = fp16(X_lo' 2^-11) = fp16(x - x_hi) and X_hi'' = fp16(x_hi 2^-11)
// (Q's formed once per problem in shared memory, P~'s in registers). Below the
// fp16 normal range these round to subnormals: an ABSOLUTE error <= 2^-25 per
// operand value, against S (|q| |k| sums over 64 terms) and O (weights p of a
// normalised row, l >= 1) negligible next to the split's own 2^-22 relative;
// tests/test_attention.py holds the kernel to the fp64 reference.
//
// Warp roles: 0-7 softmax (two threads per query row, 32 keys each), 8 MMA
// issue, 9 TMA. TMEM (256 columns): two S / P~ buffers of 96 columns (S_j:
// 64 fp32 columns; then P~_j as hi | lo'' | hi'' fp16x2-packed, 32 columns
// each, over it) and O (64), so S_{j+1} is computed while the softmax of
// block j runs. Two CTAs per SM.
constexpr int kFwdThreads = 320;
__device__ __forceinline__ uint32_t kbuf(int s) { return s ? 160u : 0u; }
constexpr uint32_t kO = 96;
// smem: Q_hi | Q_lo'' | Q_hi'' (16 KiB each) | K[2] (hi|lo', 16 KiB each) | V (16 KiB)
constexpr int kQKV = 6 * 16384;
constexpr int kFwdSmem = 1024 + kQKV + 128 + 3 * 256 * 4 + 16;
constexpr float kLo2 = 1.f / 2048.f;

__device__ __forceinline__ void named_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void mma_ss(uint32_t d, const Opnd& A, bool a_lo, const Opnd& B, bool b_lo,
                                       int k, uint32_t id, uint32_t acc) {
  const uint32_t oa = A.at(k), ob = B.at(k);
  mma_f16<1>(d, desc_sw128((a_lo ? A.lo : A.hi) + oa, A.lbo()),
             desc_sw128((b_lo ? B.lo : B.hi) + ob, B.lbo()), id, acc);
}

__global__ void __launch_bounds__(kFwdThreads, 2)
    attn_fwd_flash_kernel(const __grid_constant__ AttnTma tm, const AttnArgs a, const int* active) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  if (active && *(volatile const int*)active == 0) return;
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  const uint32_t base = smem_u32(smem);
  const uint32_t qhi = base, qlo = base + 16384, qhi2 = base + 32768;
  const Opnd Qa{qhi, qlo, 128, false};    // hi / lo''
  const Opnd Qb{qhi2, qhi2, 128, false};  // hi''
  auto Kt = [&](int s) {
    return Opnd{base + 49152 + s * 16384, base + 49152 + s * 16384 + KT, 64, false};
  };
  const Opnd Vt{base + 81920, base + 81920 + KT, 64, true};
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kQKV);
  uint64_t* bQ = &bars[0];   // Q landed (TMA)
  uint64_t* bQc = &bars[1];  // Q_lo'' / Q_hi'' formed (256 arrivals)
  uint64_t* bK = &bars[2];   // [2] K_j landed (K buffer j & 1)
  uint64_t* bV = &bars[4];   // V_j landed
  uint64_t* bS = &bars[5];   // [2] S_j done (S / P~ buffer j & 1)
  uint64_t* bP = &bars[7];   // P~_j written (256 arrivals)
  uint64_t* bO = &bars[8];   // PV_j done (every PV: the softmax warps and the loader)
  // PV_j done, by parity of j: the MMA thread waits for PV_{j-2} while PV_{j-1}
  // may already be complete (one barrier would have moved two phases on)
  uint64_t* bO2 = &bars[9];  // [2]
  // row-max exchange [block parity][key half][128] (a thread may run one block
  // ahead of its row partner), row-sum exchange [key half][128]
  float* xch = reinterpret_cast<float*>(smem + kQKV + 128);
  float* lxch = xch + 512;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(xch + 768);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int sq = a.sq, skv = a.skv;
  const int nqb = (sq + 127) >> 7, nkb = (skv + KB - 1) / KB;
  const int nprob = a.G * a.Bb * a.H * nqb;
  if (tid == 0) {
    for (int k = 0; k < 11; ++k) mbar_init(&bars[k], (k == 1 || k == 7) ? 256 : 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tslot, 256);
  bar_sync();
  const uint32_t tmem = *tslot;
  float amax = 0.f;
  auto coords = [&](int z, int& g, int& b, int& h, int& qb) {
    qb = nqb - 1 - z % nqb;  // heavier (later) causal query blocks first
    int r = z / nqb;
    h = r % a.H;
    r /= a.H;
    b = r % a.Bb;
    g = r / a.Bb;
  };
  auto nblocks = [&](int qb) { return a.causal ? min(nkb, (qb * 128 + 127) / KB + 1) : nkb; };
  auto load = [&](const Opnd& X, int which, int g, int b, int h, int row0, uint64_t* bar,
                  uint32_t bytes) {
    mbar_expect_tx(bar, bytes);
    tma_box(X.hi, tm, which, g, b, h, bar, row0, 0);
    tma_box(X.lo, tm, which, g, b, h, bar, row0, 32);
  };
  // Completion counts are deterministic (n blocks per problem), so a waiter
  // waits for exactly the operation it needs: a parity wait is safe when the
  // phase before it is known complete and the phase after it cannot complete
  // before the wait.
  if (warp == 9) {
    // ================= TMA loads (one thread) =================
    if (lane == 0) {
      uint32_t cs[2] = {0, 0}, co = 0;  // S per buffer / PV, before this problem
      for (int z = blockIdx.x; z < nprob; z += gridDim.x) {
        int g, b, h, qb;
        coords(z, g, b, h, qb);
        const int n = nblocks(qb);
        if (co > 0) mbar_wait(bO, (co - 1) & 1);  // previous problem: every MMA done
        load(Qa, TQ, g, b, h, qb * 128, bQ, kHsBytes);
        load(Kt(0), TK, g, b, h, 0, &bK[0], 2 * KT);
        if (n > 1) load(Kt(1), TK, g, b, h, KB, &bK[1], 2 * KT);
        load(Vt, TV, g, b, h, 0, bV, 2 * KT);
        for (int j = 1; j < n; ++j) {
          if (j + 1 < n) {  // K_{j+1} once S_{j-1} has read its buffer
            const int bj = (j - 1) & 1;
            mbar_wait(&bS[bj], (cs[bj] + (j - 1) / 2) & 1);
            load(Kt((j + 1) & 1), TK, g, b, h, (j + 1) * KB, &bK[(j + 1) & 1], 2 * KT);
          }
          mbar_wait(bO, (co + j - 1) & 1);  // V_j once PV_{j-1} has read V_{j-1}
          load(Vt, TV, g, b, h, j * KB, bV, 2 * KT);
        }
        cs[0] += (n + 1) / 2;
        cs[1] += n / 2;
        co += n;
      }
      if (co > 0) mbar_wait(bO, (co - 1) & 1);
    }
    __syncwarp();
  } else if (warp == 8) {
    // ================= MMA issue (one thread) =================
    if (lane == 0) {
      uint32_t nqc = 0, nk[2] = {0, 0}, nv = 0, np = 0, co = 0;
      const uint32_t idS = idesc(KB, false, false), idO = idesc(64, false, true);
      for (int z = blockIdx.x; z < nprob; z += gridDim.x) {
        int g, b, h, qb;
        coords(z, g, b, h, qb);
        const int n = nblocks(qb);
        mbar_wait(bQc, nqc & 1);  // Q landed and the softmax warps formed Q_lo'' / Q_hi''
        ++nqc;
        for (int j = 0; j <= n; ++j) {
          if (j < n) {
            // S_j = Q K_j^T into buffer j & 1 (free once PV_{j-2} is done)
            mbar_wait(&bK[j & 1], nk[j & 1] & 1);
            ++nk[j & 1];
            if (j >= 2) {
              const uint32_t k2 = co + j - 2;  // PV index; the (k2 / 2)-th on bO2[k2 & 1]
              mbar_wait(&bO2[k2 & 1], (k2 >> 1) & 1);
            }
            tc_after();
            const uint32_t d = tmem + kbuf(j & 1);
            const Opnd K = Kt(j & 1);
            for (int k = 0; k < 4; ++k) {
              mma_ss(d, Qa, false, K, false, k, idS, k > 0 ? 1u : 0u);
              mma_ss(d, Qa, true, K, false, k, idS, 1u);
              mma_ss(d, Qb, false, K, true, k, idS, 1u);
            }
            mma_commit<1>(&bS[j & 1]);
          }
          if (j >= 1) {
            // O += P~_{j-1} V_{j-1} (A = P~ from TMEM)
            mbar_wait(bP, np & 1);
            ++np;
            mbar_wait(bV, nv & 1);
            ++nv;
            tc_after();
            const uint32_t pa = tmem + kbuf((j - 1) & 1);
            for (int k = 0; k < 4; ++k) {
              const uint32_t ob = Vt.at(k);
              const uint64_t dvh = desc_sw128(Vt.hi + ob, Vt.lbo()),
                             dvl = desc_sw128(Vt.lo + ob, Vt.lbo());
              mma_ts(tmem + kO, pa + 8 * k, dvh, idO, (j > 1 || k > 0) ? 1u : 0u);
              mma_ts(tmem + kO, pa + 32 + 8 * k, dvh, idO, 1u);
              mma_ts(tmem + kO, pa + 64 + 8 * k, dvl, idO, 1u);
            }
            mma_commit<1>(bO);
            mma_commit<1>(&bO2[(co + j - 1) & 1]);
          }
        }
        co += n;
      }
    }
    __syncwarp();
  } else {
    // ================= softmax warps 0-7 =================
    const int q4 = warp & 3, kh = warp >> 2;
    const uint32_t lanes = (uint32_t)(q4 * 32) << 16;
    const int i = q4 * 32 + lane;  // query row within the block = TMEM lane
    uint32_t nq = 0, ns[2] = {0, 0}, no = 0;
    for (int z = blockIdx.x; z < nprob; z += gridDim.x) {
      int g, b, h, qb;
      coords(z, g, b, h, qb);
      const int n = nblocks(qb);
      const int q = qb * 128 + i;
      const int qlim = a.causal ? min(q + 1, skv) : skv;  // valid keys: < qlim
      // ---- Q_lo' -> Q_lo'' in place, Q_hi'' = Q_hi 2^-11 (16-byte chunks) ----
      mbar_wait(bQ, nq & 1);
      ++nq;
      {
        const __half2 sc = __float2half2_rn(kLo2);
        for (int c = tid; c < 1024; c += 256) {
          const uint32_t off = (uint32_t)c * 16;
          uint4 hv = lds128u(qhi + off), lv = lds128u(qlo + off);
          uint32_t* hp = &hv.x;
          uint32_t* lp = &lv.x;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const __half2 l2 = __hmul2(*reinterpret_cast<const __half2*>(&lp[e]), sc);
            const __half2 h2 = __hmul2(*reinterpret_cast<const __half2*>(&hp[e]), sc);
            lp[e] = *reinterpret_cast<const uint32_t*>(&l2);
            hp[e] = *reinterpret_cast<const uint32_t*>(&h2);
          }
          sts128(qlo + off, lv);
          sts128(qhi2 + off, hv);
        }
      }
      fence_async_smem();
      mbar_arrive(bQc);
      float m = -INFINITY, l = 0.f;
      for (int j = 0; j < n; ++j) {
        const uint32_t buf = tmem + kbuf(j & 1);
        mbar_wait(&bS[j & 1], ns[j & 1] & 1);
        ++ns[j & 1];
        tc_after();
        float v[32];
        {
          uint32_t r[32];
          tmem_ld16(buf + lanes + kh * 32, r);
          tmem_ld16(buf + lanes + kh * 32 + 16, r + 16);
          tmem_wait();
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = __uint_as_float(r[e]);
        }
        const int lim = qlim - (j * KB + kh * 32);  // valid: e < lim
        float mb = -INFINITY;
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          v[e] = e < lim ? v[e] * a.scale : -INFINITY;
          mb = fmaxf(mb, v[e]);
        }
        float* xb = xch + (j & 1) * 256;
        xb[kh * 128 + i] = mb;
        named_sync(1, 256);  // also: every S_j read is done (P~_j overwrites it)
        mb = fmaxf(xb[i], xb[128 + i]);
        float alpha = 1.f;
        if (mb > m + kLazy) {
          alpha = m == -INFINITY ? 0.f : fast_exp(m - mb);
          m = mb;
        }
        float ls = 0.f;
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          v[e] = e < lim ? fast_exp(v[e] - m) : 0.f;
          ls += v[e];
        }
        l = l * alpha + ls;
        // P~ hi, lo'' = fp16(p - hi), hi'' = fp16(hi 2^-11) -> this buffer
        // (key pairs packed per column; this thread's 32 keys = 16 columns)
        {
          uint32_t ph[16], pl[16];
          const __half2 sc = __float2half2_rn(kLo2);
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const __half2 hh = __floats2half2_rn(v[e], v[e + 1]);
            const float2 hf = __half22float2(hh);
            const __half2 ll = __floats2half2_rn(v[e] - hf.x, v[e + 1] - hf.y);
            ph[e >> 1] = *reinterpret_cast<const uint32_t*>(&hh);
            pl[e >> 1] = *reinterpret_cast<const uint32_t*>(&ll);
          }
          tmem_st16(buf + lanes + kh * 16, ph);
          tmem_st16(buf + lanes + 32 + kh * 16, pl);
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const __half2 h2 = __hmul2(*reinterpret_cast<const __half2*>(&ph[e]), sc);
            ph[e] = *reinterpret_cast<const uint32_t*>(&h2);
          }
          tmem_st16(buf + lanes + 64 + kh * 16, ph);
        }
        // PV_{j-1} done (then the O rescale when this row's reference max
        // moved); also keeps P~_j's arrival after PV_{j-1}'s issue
        if (j > 0) {
          mbar_wait(bO, no & 1);
          ++no;
          tc_after();
          if (__any_sync(0xffffffffu, alpha != 1.f)) {
            uint32_t r[32];
            tmem_ld16(tmem + kO + lanes + kh * 32, r);
            tmem_ld16(tmem + kO + lanes + kh * 32 + 16, r + 16);
            tmem_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * alpha);
            tmem_st16(tmem + kO + lanes + kh * 32, r);
            tmem_st16(tmem + kO + lanes + kh * 32 + 16, r + 16);
          }
        }
        tmem_st_wait();
        tc_before();
        mbar_arrive(bP);
      }
      // ---- epilogue: O / l ----
      mbar_wait(bO, no & 1);
      ++no;
      tc_after();
      lxch[kh * 128 + i] = l;
      named_sync(1, 256);
      l = lxch[i] + lxch[128 + i];
      const float inv = l > 0.f ? 1.f / l : 0.f;
      {
        const long long ld = a.Ohl.ok() ? a.Ohl.ld : a.O.ld;
        float* orow = a.O.ok() ? a.O.at(g, b, h) + (long long)qb * 128 * ld : nullptr;
        float* hrow = a.Ohl.ok() ? a.Ohl.at(g, b, h) + (long long)qb * 128 * ld : nullptr;
        const bool live = i < sq - qb * 128;
#pragma unroll
        for (int c = 0; c < 32; c += 16) {
          uint32_t r[16];
          tmem_ld16(tmem + kO + lanes + kh * 32 + c, r);
          tmem_wait();
          float v[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) v[e] = __uint_as_float(r[e]) * inv;
          if (live) {
            const int col = kh * 32 + c;
            if (orow) {
#pragma unroll
              for (int e = 0; e < 16; e += 4)
                *reinterpret_cast<float4*>(orow + i * ld + col + e) =
                    make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
            }
            if (hrow) {
#pragma unroll
              for (int e = 0; e < 16; e += 8) {
                uint4 hi, lo;
                split8(v + e, hi, lo, amax);
                char* p = reinterpret_cast<char*>(hrow + i * ld) + ((col + e) >> 5) * 128 +
                          ((col + e) & 31) * 2;
                *reinterpret_cast<uint4*>(p) = hi;
                *reinterpret_cast<uint4*>(p + 64) = lo;
              }
            }
          }
        }
        if (kh == 0 && live) {
          float* stp = a.P.at(g, b, h) + 2LL * q;
          stp[0] = m;
          stp[1] = inv;
        }
      }
      tc_before();
      // O and lxch read before the next problem's PV_0 / exchanges
      named_sync(1, 256);
    }
  }
  if (amax >= 65520.f && amax <= FLT_MAX && a.range_flag) atomicOr(a.range_flag, 1);
  bar_sync();
  if (warp == 0) tmem_free(tmem, 256);
}

AttnTma flash_maps(const AttnArgs& a, bool backward) {
  AttnTma t{};
  // head-split pre-split operands: [rows][32] fp32-sized boxes (hi, lo'
  // halves) in the tiles' SWIZZLE_128B layout; rows >= s arrive zero-filled
  auto mk = [&](int which, const Mat& m, int rows, int box_rows) {
    t.m[which] = tc_make_map(m, a.G, a.Bb, a.H, rows, 64, box_rows, 32, true, &t.op[which]);
  };
  mk(TQ, a.Q, a.sq, 128);
  mk(TK, a.K, a.skv, KB);
  mk(TV, a.V, a.skv, KB);
  if (backward) mk(TDO, a.dO, a.sq, 128);
  return t;
}

int n_sms() {
  static int n = 0;
  if (!n) MGLP_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, 0));
  return n;
}

}  // namespace

bool attn_flash_supported(const AttnArgs& a, bool backward) {
  if (backward) return false;  // backward: not yet
  return a.qkv_hs && a.dh == 64 && a.sq > 128 && a.skv > 128 && a.sq <= 512 && a.skv <= 512 &&
         a.P.ok();
}

void launch_attn_fwd_flash(const AttnArgs& a, const int* active, cudaStream_t s) {
  if (!attn_flash_supported(a, false)) throw ContractViolation("attn_fwd_flash: unsupported");
  static bool attr = [] {
    MGLP_CUDA(cudaFuncSetAttribute(attn_fwd_flash_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, kFwdSmem));
    return true;
  }();
  (void)attr;
  const long long nprob = (long long)a.G * a.Bb * a.H * ((a.sq + 127) / 128);
  if (nprob == 0) return;
  const int grid = (int)std::min<long long>(nprob, 2LL * n_sms());
  launch_k(attn_fwd_flash_kernel, dim3(grid), dim3(kFwdThreads), kFwdSmem, s, 1,
           flash_maps(a, false), a, active);
  MGLP_CUDA(cudaGetLastError());
}

}  // namespace mglp
