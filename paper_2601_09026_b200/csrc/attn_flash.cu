// Single-pass streamed attention for 128 <= s <= 512 with head-split
// pre-split operands (AttnArgs::qkv_hs / do_hs, dh = 64): the GPT-2-style
// causal decoder (s = 512) and ViT (s = 197). The reference's attention /
// vjp_attention (blocks.cpp:142-236; softmax_rows / vjp_softmax_rows,
// tensor.cpp:310-342).
//
// Forward (attn_fwd_flash_kernel): CTA = one (member, batch, head, 128-query
// block), two CTAs per SM; warps 0-7 softmax (two threads per query row),
// warp 8 MMA issue, warp 9 TMA. Q once, 64-key blocks of K (double-buffered)
// and V TMA'd straight into their tiles; S_j = Q K_j^T into one of two TMEM
// buffers; online softmax with a lazy reference max (it moves only when a
// block raises the row max by more than kLazy; O and l are then rescaled);
// P~_j = exp(S scale - m) written back into TMEM over S_j as fp16x2 columns
// and used as the A operand of O += P~_j V_j (tcgen05.mma ... [a-tmem]); the
// epilogue writes O / l and the row statistics (m, 1/l). S is computed once
// and no probability tile goes through shared memory. The split's 2^-11
// correction terms are folded into operands (one accumulator per product:
// see the forward section below).
//
// Backward: flash_rowdot_kernel (t_q = dO_q . O_q), attn_bwd_kv_flash_kernel
// (dK, dV per 128-key block with keys as TMEM lanes; every dS tile stored
// pre-split), attn_bwd_q_flash_kernel (dQ = sum dS K per 128-query block).
// Deterministic: no atomics.
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
// Problem z of a persistent CTA (z = blockIdx + round * grid) -> (head, block).
// The blocks of one head are consecutive problems, so CTAs running at the
// same time share that head's K / V (or Q / dO) rows in L2, and the block
// index is rotated by the round z / R (R = the grid rounded down to whole
// heads), so every CTA cycles through all block indices: under the causal
// mask the blocks carry 1..n units of work, and a CTA that kept one block
// index (z mod n with a grid that is a multiple of n) ran up to 8/5 of the
// mean. A bijection for any grid (R is a multiple of nblk).
__device__ __forceinline__ void head_block(int z, int nblk, int& head, int& blk) {
  const int R = max(nblk, ((int)gridDim.x / nblk) * nblk);
  head = z / nblk;
  blk = (z % nblk + z / R) % nblk;
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
    int r;
    head_block(z, nqb, r, qb);
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
              float* o = orow + i * ld + col;
              if ((reinterpret_cast<uintptr_t>(o) & 31) == 0) {  // 256-bit stores
#pragma unroll
                for (int e = 0; e < 16; e += 8)
                  st_v8(o + e, __float_as_uint(v[e]), __float_as_uint(v[e + 1]), __float_as_uint(v[e + 2]),
                        __float_as_uint(v[e + 3]), __float_as_uint(v[e + 4]), __float_as_uint(v[e + 5]),
                        __float_as_uint(v[e + 6]), __float_as_uint(v[e + 7]));
              } else {
#pragma unroll
                for (int e = 0; e < 16; e += 4)
                  *reinterpret_cast<float4*>(o + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
              }
            }
            if (hrow) {
              uint4 hi[2], lo[2];
#pragma unroll
              for (int e = 0; e < 2; ++e) split8(v + 8 * e, hi[e], lo[e], amax);
              // col % 16 == 0: hi at p, p + 16, lo' at p + 64, p + 80
              char* p = reinterpret_cast<char*>(hrow + i * ld) + (col >> 5) * 128 + (col & 31) * 2;
              if ((reinterpret_cast<uintptr_t>(p) & 31) == 0) {
                st_v8(p, hi[0].x, hi[0].y, hi[0].z, hi[0].w, hi[1].x, hi[1].y, hi[1].z, hi[1].w);
                st_v8(p + 64, lo[0].x, lo[0].y, lo[0].z, lo[0].w, lo[1].x, lo[1].y, lo[1].z, lo[1].w);
              } else {
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                  *reinterpret_cast<uint4*>(p + 16 * e) = hi[e];
                  *reinterpret_cast<uint4*>(p + 64 + 16 * e) = lo[e];
                }
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

// ---- backward ---------------------------------------------------------------------
// Deterministic two-kernel form (no atomics): per 128-key block, dK and dV
// accumulate over 64-query blocks in TMEM and every dS tile is stored
// pre-split for the dQ kernel, which sums dQ = dS K per 128-query block.
// Keys are the TMEM lanes (S^T = K Q^T, M = 128 keys, N = 64 queries):
//   S^T  = K_hi Q_hi + 2^-11 (K_lo' Q_hi + K_hi Q_lo')       one accumulator each: the
//   dP^T = V_hi dO_hi + 2^-11 (V_lo' dO_hi + V_hi dO_lo')    correction products go
//          first and the first main MMA scales them (tcgen05.mma scale-input-d = 11:
//          D = A B + D 2^-11), so K, V are used exactly as TMA lands them
//   P^T  = exp(S^T scale - m_q) / l_q (the forward's row statistics), dS^T = P^T (dP^T - t_q)
//   dV  += P_hi dO_hi + 2^-11 (P_lo' dO_hi + P_hi dO_lo')    (A = P^T from TMEM; main and
//   dK  += dS_hi Q_hi + 2^-11 (dS_lo' Q_hi + dS_hi Q_lo')     correction accumulators)
// t_q = dO_q . O_q comes from flash_rowdot_kernel first.
//
// Pipeline: one step = one 64-query block of one problem; steps are numbered
// globally over the CTA's problems (k), so every barrier phase is a function
// of k and nothing drains between problems: the next K, V land once the last
// S^T / dP^T of the current problem have read theirs (under its last softmax
// step), and the dV / dK epilogue of a problem runs while the next problem's
// first S^T / dP^T are computed. Four query stages (Q, dO, statistics): step
// k's loads go out once step k-4's gradient MMAs are done.
constexpr int kKvThreads = 576;  // warps 0-15 compute, 16 MMA issue, 17 TMA
constexpr int kQB = 64;          // queries per step
constexpr int QT = kQB * 128;    // one 64-row hi (or lo') tile: 8 KiB
constexpr int kSt = 4;           // query stages
// smem: K hi | lo' (16 KiB each) | V likewise | Q[4] (hi|lo', 16 KiB) | dO[4] | stats[4]
constexpr int kKvOff = 4 * 16384 + kSt * 4 * QT;
constexpr int kKvSmem = 1024 + kKvOff + kSt * 1024 + 256 + 16;
// TMEM: S/P~ [0,64) [64,128); dP/dS [128,192) [192,256); dV main [256,320), corr [320,384);
//       dK main [384,448), corr [448,512)
__device__ __forceinline__ uint32_t tsb(int s) { return s ? 64u : 0u; }
__device__ __forceinline__ uint32_t tdb(int s) { return s ? 192u : 128u; }
constexpr uint32_t kTdV = 256, kTdVc = 320, kTdK = 384, kTdKc = 448;

// D = A . B^T + D 2^-11 (scale-input-d), both operands in shared memory
__device__ __forceinline__ void mma_ss_scaled(uint32_t d, const Opnd& A, const Opnd& B, int k,
                                              uint32_t id) {
  const uint32_t oa = A.at(k), ob = B.at(k);
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.eq.u32 p, 1, 1;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p, 11;\n\t"
      "}" ::"r"(d),
      "l"(desc_sw128(A.hi + oa, A.lbo())), "l"(desc_sw128(B.hi + ob, B.lbo())), "r"(id));
}

// 32 lanes x 8 columns into TMEM (this warp's lane quarter)
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

// MGLP_FLASH_TRACE (diagnostics): clock64 stamps of CTA 0 of the dK/dV kernel
#ifdef MGLP_FLASH_TRACE
__device__ long long g_flash_trace[4096];
#define FTRACE(slot) \
  do { if (blockIdx.x == 0 && (slot) < 4096) g_flash_trace[(slot)] = clock64(); } while (0)
#else
#define FTRACE(slot) do { } while (0)
#endif

// the t_q offset in a head's P slot (after the forward's [sq][2] statistics)
__device__ __host__ __forceinline__ long long t_off(int sq) { return 2LL * ((sq + 63) & ~63); }

// t_q = dO_q . O_q with dO head-split pre-split (d = hi + 2^-11 lo', the value
// the MMAs use) and O fp32, fixed order
__global__ void __launch_bounds__(256) flash_rowdot_kernel(const AttnArgs a, const int* active) {
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
  const __half* d = reinterpret_cast<const __half*>(a.dO.at(g, b, h) + (long long)q * a.dO.ld);
  const float* o = a.O.at(g, b, h) + (long long)q * a.O.ld;
  float t = 0.f;
  // a thread reads its own row: 256-bit loads where the rows allow (the same
  // values in the same order as the 128-bit form below)
  if (((reinterpret_cast<uintptr_t>(d) | reinterpret_cast<uintptr_t>(o)) & 31) == 0) {
#pragma unroll
    for (int e = 0; e < 64; e += 16) {
      uint32_t hw[8], lw[8];
      float ov[16];
      asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(hw[0]), "=r"(hw[1]), "=r"(hw[2]), "=r"(hw[3]), "=r"(hw[4]), "=r"(hw[5]),
                     "=r"(hw[6]), "=r"(hw[7])
                   : "l"(d + e));
      asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(lw[0]), "=r"(lw[1]), "=r"(lw[2]), "=r"(lw[3]), "=r"(lw[4]), "=r"(lw[5]),
                     "=r"(lw[6]), "=r"(lw[7])
                   : "l"(d + 64 + e));
#pragma unroll
      for (int hh = 0; hh < 2; ++hh)
        asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(ov[8 * hh]), "=f"(ov[8 * hh + 1]), "=f"(ov[8 * hh + 2]), "=f"(ov[8 * hh + 3]),
                       "=f"(ov[8 * hh + 4]), "=f"(ov[8 * hh + 5]), "=f"(ov[8 * hh + 6]), "=f"(ov[8 * hh + 7])
                     : "l"(o + e + 8 * hh));
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float2 hf = __half22float2(*reinterpret_cast<const __half2*>(&hw[k]));
        const float2 lf = __half22float2(*reinterpret_cast<const __half2*>(&lw[k]));
        t += fmaf(lf.x, kLo2, hf.x) * ov[2 * k];
        t += fmaf(lf.y, kLo2, hf.y) * ov[2 * k + 1];
      }
    }
    a.P.at(g, b, h)[t_off(a.sq) + q] = t;
    return;
  }
  for (int e = 0; e < 64; e += 8) {
    const uint4 hv = *reinterpret_cast<const uint4*>(d + e);
    const uint4 lv = *reinterpret_cast<const uint4*>(d + 64 + e);
    const float4 o0 = *reinterpret_cast<const float4*>(o + e);
    const float4 o1 = *reinterpret_cast<const float4*>(o + e + 4);
    const float ov[8] = {o0.x, o0.y, o0.z, o0.w, o1.x, o1.y, o1.z, o1.w};
    const uint32_t hw[4] = {hv.x, hv.y, hv.z, hv.w}, lw[4] = {lv.x, lv.y, lv.z, lv.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 hf = __half22float2(*reinterpret_cast<const __half2*>(&hw[k]));
      const float2 lf = __half22float2(*reinterpret_cast<const __half2*>(&lw[k]));
      t += fmaf(lf.x, kLo2, hf.x) * ov[2 * k];
      t += fmaf(lf.y, kLo2, hf.y) * ov[2 * k + 1];
    }
  }
  a.P.at(g, b, h)[t_off(a.sq) + q] = t;
}

__global__ void __launch_bounds__(kKvThreads, 1)
    attn_bwd_kv_flash_kernel(const __grid_constant__ AttnTma tm, const AttnArgs a, const int* active) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  if (active && *(volatile const int*)active == 0) return;
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  const uint32_t base = smem_u32(smem);
  const uint32_t khi = base, klo = base + 16384, vhi = base + 32768, vlo = base + 49152;
  const Opnd Ka{khi, klo, 128, false}, Va{vhi, vlo, 128, false};
  auto Qt = [&](int s, bool mn) {
    const uint32_t q0 = base + 65536 + s * 2 * QT;
    return Opnd{q0, q0 + QT, 64, mn};
  };
  auto dOt = [&](int s, bool mn) {
    const uint32_t q0 = base + 65536 + kSt * 2 * QT + s * 2 * QT;
    return Opnd{q0, q0 + QT, 64, mn};
  };
  float* stats = reinterpret_cast<float*>(smem + kKvOff);  // [kSt][256]: m, inv pairs | t
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kKvOff + kSt * 1024);
  uint64_t* bKV = &bars[0];  // K, V of the problem landed
  uint64_t* bQ = &bars[1];   // [kSt] Q_k, dO_k, stats_k landed (stage k % kSt)
  uint64_t* bSD = &bars[5];  // [2] S_k, dP_k done (TMEM buffer k & 1)
  uint64_t* bPD = &bars[7];  // [2] P~_k, dS_k written (512 arrivals)
  uint64_t* bM = &bars[9];   // [kSt] step k's dV / dK MMAs done (by k % kSt)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 13);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int sq = a.sq, skv = a.skv;
  const int nkb = (skv + 127) >> 7, nq64 = (sq + kQB - 1) / kQB;
  const int nprob = a.G * a.Bb * a.H * nkb;
  if (tid == 0) {
    for (int k = 0; k < 13; ++k) mbar_init(&bars[k], (k == 7 || k == 8) ? 512 : 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tslot, 512);
  bar_sync();
  const uint32_t tmem = *tslot;
  float amax = 0.f;
  auto coords = [&](int z, int& g, int& b, int& h, int& kb) {
    int r;
    head_block(z, nkb, r, kb);
    h = r % a.H;
    r /= a.H;
    b = r % a.Bb;
    g = r / a.Bb;
  };
  auto first_q = [&](int kb) { return a.causal ? (kb * 128) / kQB : 0; };
  // Every role walks the same problems and steps, so a parity wait is for
  // exactly the phase it needs: the phase before it is complete and the one
  // after it cannot complete before the wait (checked per barrier below).
  if (warp == 17) {
    // ================= TMA loads (one thread) =================
    if (lane == 0) {
      uint32_t k = 0;       // global step
      int klast = -1;       // last step of the previous problem
      int pi = 0;           // problems (trace slots)
      for (int z = blockIdx.x; z < nprob; z += gridDim.x, ++pi) {
        int g, b, h, kb;
        coords(z, g, b, h, kb);
        const int q0 = first_q(kb), n = nq64 - q0;
        if (n <= 0) continue;
        const float* st = a.P.at(g, b, h);
        for (int j = 0; j < n; ++j, ++k) {
          const int s = (int)(k % kSt);
          // stage s: step k - kSt's gradient MMAs done (bM's next phase is step
          // k's, which needs this load)
          if (k >= (uint32_t)kSt) mbar_wait(&bM[s], ((k - kSt) / kSt) & 1);
          const int qr = (q0 + j) * kQB;
          FTRACE((k) < 256 ? 8 * (k) + 6 : 4096);
          mbar_expect_tx(&bQ[s], 4 * QT + 768);
          const Opnd Q = Qt(s, false), D = dOt(s, false);
          tma_box(Q.hi, tm, TQ, g, b, h, &bQ[s], qr, 0);
          tma_box(Q.lo, tm, TQ, g, b, h, &bQ[s], qr, 32);
          tma_box(D.hi, tm, TDO, g, b, h, &bQ[s], qr, 0);
          tma_box(D.lo, tm, TDO, g, b, h, &bQ[s], qr, 32);
          bulk_load(smem_u32(stats + s * 256), st + 2LL * qr, 512, &bQ[s]);  // m, 1/l
          bulk_load(smem_u32(stats + s * 256 + 128), st + t_off(sq) + qr, 256, &bQ[s]);
          if (j == 0) {
            // K, V once the previous problem's last S^T / dP^T have read theirs
            // (bSD's next phase is step klast + 2's, which needs these K, V)
            if (klast >= 0) mbar_wait(&bSD[klast & 1], ((uint32_t)klast >> 1) & 1);
            mbar_expect_tx(bKV, 4 * 16384);
            tma_box(khi, tm, TK, g, b, h, bKV, kb * 128, 0);
            tma_box(klo, tm, TK, g, b, h, bKV, kb * 128, 32);
            tma_box(vhi, tm, TV, g, b, h, bKV, kb * 128, 0);
            tma_box(vlo, tm, TV, g, b, h, bKV, kb * 128, 32);
            FTRACE(2048 + 4 * pi + 0);
          }
        }
        klast = (int)k - 1;
      }
    }
    __syncwarp();
  } else if (warp == 16) {
    // ================= MMA issue (one thread) =================
    if (lane == 0) {
      uint32_t k = 0, np = 0;  // global step base of the problem, problems
      const uint32_t idN64 = idesc(64, false, false), idG = idesc(64, false, true);
      for (int z = blockIdx.x; z < nprob; z += gridDim.x) {
        int g, b, h, kb;
        coords(z, g, b, h, kb);
        const int n = nq64 - first_q(kb);
        if (n <= 0) continue;
        // K, V of this problem (the next load needs this problem's last S^T)
        mbar_wait(bKV, np & 1);
        FTRACE(2048 + 4 * np + 3);
        ++np;
        for (int j = 0; j <= n; ++j) {
          if (j < n) {
            const uint32_t kk = k + j;
            const int s = (int)(kk & 1), q = (int)(kk % kSt);
            mbar_wait(&bQ[q], (kk / kSt) & 1);
            FTRACE((kk) < 256 ? 8 * (kk) + 0 : 4096);
            // TMEM buffers s: step kk-2's gradient MMAs have read its P~ / dS
            if (kk >= 2) mbar_wait(&bM[(kk - 2) % kSt], ((kk - 2) / kSt) & 1);
            FTRACE((kk) < 256 ? 8 * (kk) + 1 : 4096);
            tc_after();
            const Opnd Q = Qt(q, false), D = dOt(q, false);
            const uint32_t dS_ = tmem + tsb(s), dD = tmem + tdb(s);
            for (int c = 0; c < 4; ++c) {  // corrections (2^11 domain)
              mma_ss(dS_, Ka, true, Q, false, c, idN64, c > 0 ? 1u : 0u);  // S^T = K Q^T
              mma_ss(dS_, Ka, false, Q, true, c, idN64, 1u);
              mma_ss(dD, Va, true, D, false, c, idN64, c > 0 ? 1u : 0u);   // dP^T = V dO^T
              mma_ss(dD, Va, false, D, true, c, idN64, 1u);
            }
            mma_ss_scaled(dS_, Ka, Q, 0, idN64);
            mma_ss_scaled(dD, Va, D, 0, idN64);
            for (int c = 1; c < 4; ++c) {
              mma_ss(dS_, Ka, false, Q, false, c, idN64, 1u);
              mma_ss(dD, Va, false, D, false, c, idN64, 1u);
            }
            mma_commit<1>(&bSD[s]);
          }
          if (j >= 1) {
            const uint32_t kk = k + j - 1;
            const int s = (int)(kk & 1), q = (int)(kk % kSt);
            mbar_wait(&bPD[s], (kk >> 1) & 1);
            FTRACE((kk) < 256 ? 8 * (kk) + 2 : 4096);
            tc_after();
            const Opnd Qm = Qt(q, true), Dm = dOt(q, true);
            const uint32_t pa = tmem + tsb(s), da = tmem + tdb(s);
            const bool first = j == 1;
            for (int c = 0; c < 4; ++c) {
              const uint32_t oq = Qm.at(c), od = Dm.at(c);
              const uint64_t dqh = desc_sw128(Qm.hi + oq, Qm.lbo()), dql = desc_sw128(Qm.lo + oq, Qm.lbo());
              const uint64_t ddh = desc_sw128(Dm.hi + od, Dm.lbo()), ddl = desc_sw128(Dm.lo + od, Dm.lbo());
              const uint32_t acc = (!first || c > 0) ? 1u : 0u;
              mma_ts(tmem + kTdV, pa + 8 * c, ddh, idG, acc);  // dV += P^T dO
              mma_ts(tmem + kTdVc, pa + 32 + 8 * c, ddh, idG, acc);
              mma_ts(tmem + kTdVc, pa + 8 * c, ddl, idG, 1u);
              mma_ts(tmem + kTdK, da + 8 * c, dqh, idG, acc);  // dK += dS^T Q
              mma_ts(tmem + kTdKc, da + 32 + 8 * c, dqh, idG, acc);
              mma_ts(tmem + kTdKc, da + 8 * c, dql, idG, 1u);
            }
            mma_commit<1>(&bM[kk % kSt]);
          }
        }
        k += n;
      }
    }
    __syncwarp();
  } else {
    // ================= compute warps 0-15 =================
    // warp w: key rows 32 (w & 3) + lane (TMEM lanes), queries 16 (w >> 2) .. + 16
    const int q4 = warp & 3, qq = warp >> 2;
    const uint32_t lanes = (uint32_t)(q4 * 32) << 16;
    const int r = q4 * 32 + lane;  // key row within the block
    uint32_t k = 0;
    int pi = 0;  // problems (trace slots)
    for (int z = blockIdx.x; z < nprob; z += gridDim.x, ++pi) {
      int g, b, h, kb;
      coords(z, g, b, h, kb);
      const int q0 = first_q(kb), n = nq64 - q0;
      if (n <= 0) continue;
      const int key = kb * 128 + r;
      float* dsg = a.dS.at(g, b, h);
      const bool ds_v8 = (reinterpret_cast<uintptr_t>(dsg) & 31) == 0;  // 256-bit stores
      for (int j = 0; j < n; ++j, ++k) {
        const int s = (int)(k & 1);
        if (tid == 0) FTRACE((k) < 256 ? 8 * (k) + 3 : 4096);
        // bSD's next phase is step k+2's S^T, which needs this step's bPD
        mbar_wait(&bSD[s], (k >> 1) & 1);
        if (tid == 0) FTRACE((k) < 256 ? 8 * (k) + 4 : 4096);
        tc_after();
        float sv[16], dp[16];
        {
          uint32_t u[16], w[16];
          tmem_ld16(tmem + tsb(s) + lanes + qq * 16, u);
          tmem_ld16(tmem + tdb(s) + lanes + qq * 16, w);
          tmem_wait();
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            sv[e] = __uint_as_float(u[e]);
            dp[e] = __uint_as_float(w[e]);
          }
        }
        // P~ and dS overwrite S / dP columns the other three warps of these
        // TMEM lanes read: they all have read theirs first
        named_sync(2 + q4, 128);
        const float* st = stats + (k % kSt) * 256;
        const int qa = (q0 + j) * kQB + qq * 16;  // this thread's first query
        uint32_t ph[8], pl[8], dh[8], dl[8];
#pragma unroll
        for (int e = 0; e < 16; e += 2) {
          float p[2], ds[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int ql = qq * 16 + e + u, q = qa + e + u;
            const bool ok = q < sq && key < skv && (!a.causal || key <= q);
            const float m = st[2 * ql], inv = st[2 * ql + 1], t = st[128 + ql];
            p[u] = ok ? fast_exp(sv[e + u] * a.scale - m) * inv : 0.f;
            ds[u] = ok ? p[u] * (dp[e + u] - t) : 0.f;
          }
          const __half2 hh = __floats2half2_rn(p[0], p[1]);
          const float2 hf = __half22float2(hh);
          const __half2 ll = __floats2half2_rn((p[0] - hf.x) * kLoScale, (p[1] - hf.y) * kLoScale);
          ph[e >> 1] = *reinterpret_cast<const uint32_t*>(&hh);
          pl[e >> 1] = *reinterpret_cast<const uint32_t*>(&ll);
          const __half2 dhh = __floats2half2_rn(ds[0], ds[1]);
          const float2 dhf = __half22float2(dhh);
          const __half2 dll = __floats2half2_rn((ds[0] - dhf.x) * kLoScale, (ds[1] - dhf.y) * kLoScale);
          dh[e >> 1] = *reinterpret_cast<const uint32_t*>(&dhh);
          dl[e >> 1] = *reinterpret_cast<const uint32_t*>(&dll);
          amax = fmaxf(amax, fmaxf(fabsf(ds[0]), fabsf(ds[1])));
        }
        // P~ -> buffer s (hi | lo'), dS -> dP buffer s (hi | lo'): 8 columns each
        tmem_st8(tmem + tsb(s) + lanes + qq * 8, ph);
        tmem_st8(tmem + tsb(s) + lanes + 32 + qq * 8, pl);
        tmem_st8(tmem + tdb(s) + lanes + qq * 8, dh);
        tmem_st8(tmem + tdb(s) + lanes + 32 + qq * 8, dl);
        // dS for the dQ kernel: the (64-query block, 128-key block) tile pair
        // image [128 key rows][64 queries] hi | lo', SWIZZLE_128B layout
#ifndef MGLP_DIAG_NO_DS_STORE
        {
          char* img = reinterpret_cast<char*>(dsg + ((long long)(q0 + j) * nkb + kb) * 8192);
          const int c0 = qq * 2;  // this thread's two 16-byte chunks of its row
          if (ds_v8) {
            // chunks c0, c0 + 1 (c0 even) land at (c0 ^ x), (c0 ^ x) ^ 1, x = r & 7:
            // one aligned 32-byte sector, in swapped order when x is odd
            const uint32_t off = (uint32_t)(r * 128 + (((c0 ^ (r & 7)) & ~1) << 4));
            const bool sw = r & 1;
            uint32_t h8[8], l8[8];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              h8[e] = sw ? dh[4 + e] : dh[e];
              h8[4 + e] = sw ? dh[e] : dh[4 + e];
              l8[e] = sw ? dl[4 + e] : dl[e];
              l8[4 + e] = sw ? dl[e] : dl[4 + e];
            }
            st_v8(img + off, h8[0], h8[1], h8[2], h8[3], h8[4], h8[5], h8[6], h8[7]);
            st_v8(img + 16384 + off, l8[0], l8[1], l8[2], l8[3], l8[4], l8[5], l8[6], l8[7]);
          } else {
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              const uint32_t off = (uint32_t)(r * 128 + (((c0 + c) ^ (r & 7)) << 4));
              *reinterpret_cast<uint4*>(img + off) = make_uint4(dh[4 * c], dh[4 * c + 1], dh[4 * c + 2], dh[4 * c + 3]);
              *reinterpret_cast<uint4*>(img + 16384 + off) =
                  make_uint4(dl[4 * c], dl[4 * c + 1], dl[4 * c + 2], dl[4 * c + 3]);
            }
          }
        }
#endif
        tmem_st_wait();
        tc_before();
        if (tid == 0) FTRACE((k) < 256 ? 8 * (k) + 5 : 4096);
        // bPD's next phase is step k+2's, which needs S^T_{k+2} -> this arrival seen
        mbar_arrive(&bPD[s]);
      }
      // ---- epilogue: dV, dK = (main + 2^-11 corr) [scale] (this warp: 16 columns);
      // the next problem's first S^T / dP^T run meanwhile (other TMEM columns),
      // its first gradient MMAs (which overwrite dV / dK) wait for this CTA's
      // bPD arrivals of its first step, issued after these reads ----
      {
        const uint32_t kl = k - 1;  // bM's next phase is step kl + kSt's: needs our bPD
        mbar_wait(&bM[kl % kSt], (kl / kSt) & 1);
        tc_after();
        if (tid == 0) FTRACE(2048 + 4 * pi + 1);
      }
      {
        const int col = qq * 16;
        auto put = [&](const Mat& o, const Mat& ohl, const float* v) {
          if (o.ok()) {
            float* p = o.at(g, b, h) + (long long)key * o.ld + col;
            if ((reinterpret_cast<uintptr_t>(p) & 31) == 0) {  // 256-bit stores
#pragma unroll
              for (int e = 0; e < 16; e += 8)
                st_v8(p + e, __float_as_uint(v[e]), __float_as_uint(v[e + 1]), __float_as_uint(v[e + 2]),
                      __float_as_uint(v[e + 3]), __float_as_uint(v[e + 4]), __float_as_uint(v[e + 5]),
                      __float_as_uint(v[e + 6]), __float_as_uint(v[e + 7]));
            } else {
#pragma unroll
              for (int e = 0; e < 16; e += 4)
                *reinterpret_cast<float4*>(p + e) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
            }
          }
          if (ohl.ok()) {
            char* p = reinterpret_cast<char*>(ohl.at(g, b, h) + (long long)key * ohl.ld);
            uint4 hi[2], lo[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) split8(v + 8 * e, hi[e], lo[e], amax);
            // columns col .. col + 15 (col % 16 == 0): hi at q, q + 16, lo' at q + 64, q + 80
            char* q = p + (col >> 5) * 128 + (col & 31) * 2;
            if ((reinterpret_cast<uintptr_t>(q) & 31) == 0) {
              st_v8(q, hi[0].x, hi[0].y, hi[0].z, hi[0].w, hi[1].x, hi[1].y, hi[1].z, hi[1].w);
              st_v8(q + 64, lo[0].x, lo[0].y, lo[0].z, lo[0].w, lo[1].x, lo[1].y, lo[1].z, lo[1].w);
            } else {
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                *reinterpret_cast<uint4*>(q + 16 * e) = hi[e];
                *reinterpret_cast<uint4*>(q + 64 + 16 * e) = lo[e];
              }
            }
          }
        };
        uint32_t u[16], w[16];
        float v[16];
        tmem_ld16(tmem + kTdV + lanes + col, u);
        tmem_ld16(tmem + kTdVc + lanes + col, w);
        tmem_wait();
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] = fmaf(__uint_as_float(w[e]), kLo2, __uint_as_float(u[e]));
        if (key < skv) put(a.dV, a.dVhl, v);
        tmem_ld16(tmem + kTdK + lanes + col, u);
        tmem_ld16(tmem + kTdKc + lanes + col, w);
        tmem_wait();
#pragma unroll
        for (int e = 0; e < 16; ++e)
          v[e] = fmaf(__uint_as_float(w[e]), kLo2, __uint_as_float(u[e])) * a.scale;
        if (key < skv) put(a.dK, a.dKhl, v);
      }
      if (tid == 0) FTRACE(2048 + 4 * pi + 2);
      tc_before();
    }
  }
  if (amax >= 65520.f && amax <= FLT_MAX && a.range_flag) atomicOr(a.range_flag, 1);
  bar_sync();
  if (warp == 0) tmem_free(tmem, 512);
}

// ---- backward: dQ = sum over key blocks of dS K (per 128-query block) ----------
// A = dS [128 queries x 128 keys] from two stored tile-pair images (MN-major:
// queries contiguous), B = K (MN-major), main + correction accumulators.
constexpr int kQThreads = 192;  // warps 0-3 epilogue, 4 MMA issue, 5 loads
constexpr int kQStage = 65536 + 32768;  // dS (hi q0 | hi q1 | lo q0 | lo q1) + K (hi | lo')
constexpr int kQSmem = 1024 + 2 * kQStage + 64 + 16;

__global__ void __launch_bounds__(kQThreads, 1)
    attn_bwd_q_flash_kernel(const __grid_constant__ AttnTma tm, const AttnArgs a, const int* active) {
  pdl_wait();
  pdl_trigger();
  extern __shared__ uint8_t smem_raw[];
  if (active && *(volatile const int*)active == 0) return;
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  const uint32_t base = smem_u32(smem);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * kQStage);
  uint64_t* bL = &bars[0];  // [2] stage landed
  uint64_t* bF = &bars[2];  // [2] stage consumed (MMA commit)
  uint64_t* bD = &bars[4];  // dQ of the problem done (MMA commit)
  uint64_t* bE = &bars[5];  // the epilogue has read dQ (TMEM free)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 6);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int sq = a.sq, skv = a.skv;
  const int nkb = (skv + 127) >> 7, nqb = (sq + 127) >> 7;
  const int nprob = a.G * a.Bb * a.H * nqb;
  if (tid == 0) {
    for (int k = 0; k < 6; ++k) mbar_init(&bars[k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) tmem_alloc(tslot, 128);
  bar_sync();
  const uint32_t tmem = *tslot;
  float amax = 0.f;
  auto coords = [&](int z, int& g, int& b, int& h, int& qb) {
    int r;
    head_block(z, nqb, r, qb);
    h = r % a.H;
    r /= a.H;
    b = r % a.Bb;
    g = r / a.Bb;
  };
  auto nblocks = [&](int qb) { return a.causal ? min(nkb, qb + 1) : nkb; };
  if (warp == 5) {
    if (lane == 0) {
      uint32_t c = 0;  // stages issued
      for (int z = blockIdx.x; z < nprob; z += gridDim.x) {
        int g, b, h, qb;
        coords(z, g, b, h, qb);
        const int n = nblocks(qb);
        const float* dsg = a.dS.at(g, b, h);
        for (int kb = 0; kb < n; ++kb, ++c) {
          const int s = c & 1;
          if (c >= 2) mbar_wait(&bF[s], ((c - 2) >> 1) & 1);
          const uint32_t st = base + s * kQStage;
          mbar_expect_tx(&bL[s], kQStage);
          for (int hf = 0; hf < 2; ++hf) {
            const char* img = reinterpret_cast<const char*>(
                dsg + ((long long)(2 * qb + hf) * nkb + kb) * 8192);
            bulk_load(st + hf * 16384, img, 16384, &bL[s]);
            bulk_load(st + 32768 + hf * 16384, img + 16384, 16384, &bL[s]);
          }
          tma_box(st + 65536, tm, TK, g, b, h, &bL[s], kb * 128, 0);
          tma_box(st + 65536 + 16384, tm, TK, g, b, h, &bL[s], kb * 128, 32);
        }
      }
    }
    __syncwarp();
  } else if (warp == 4) {
    if (lane == 0) {
      uint32_t c = 0, nd = 0;
      const uint32_t id = idesc(64, true, true);
      for (int z = blockIdx.x; z < nprob; z += gridDim.x) {
        int g, b, h, qb;
        coords(z, g, b, h, qb);
        const int n = nblocks(qb);
        if (nd > 0) mbar_wait(bE, (nd - 1) & 1);  // the epilogue read the previous dQ
        for (int kb = 0; kb < n; ++kb, ++c) {
          const int s = c & 1;
          mbar_wait(&bL[s], (c >> 1) & 1);
          tc_after();
          const uint32_t st = base + s * kQStage;
          const Opnd A{st, st + 32768, 128, true};          // dS: K = keys (rows)
          const Opnd B{st + 65536, st + 65536 + 16384, 128, true};  // K: K = keys (rows)
          for (int k = 0; k < 8; ++k) {
            const uint32_t oa = A.at(k), ob = B.at(k);
            const uint64_t dah = desc_sw128(A.hi + oa, A.lbo()), dal = desc_sw128(A.lo + oa, A.lbo());
            const uint64_t dbh = desc_sw128(B.hi + ob, B.lbo()), dbl = desc_sw128(B.lo + ob, B.lbo());
            const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
            mma_f16<1>(tmem, dah, dbh, id, acc);
            mma_f16<1>(tmem + 64, dal, dbh, id, acc);
            mma_f16<1>(tmem + 64, dah, dbl, id, 1u);
          }
          mma_commit<1>(&bF[s]);
        }
        mma_commit<1>(bD);
        ++nd;
      }
    }
    __syncwarp();
  } else {
    // ================= epilogue warps 0-3: one query row per thread =================
    const uint32_t lanes = (uint32_t)(warp * 32) << 16;
    const int i = warp * 32 + lane;
    uint32_t nd = 0;
    for (int z = blockIdx.x; z < nprob; z += gridDim.x) {
      int g, b, h, qb;
      coords(z, g, b, h, qb);
      mbar_wait(bD, nd & 1);
      ++nd;
      tc_after();
      const long long ldq = a.dQhl.ok() ? a.dQhl.ld : a.dQ.ld;
      const long long oq = (long long)qb * 128 * ldq;
      rows_out_hl(tmem + lanes, tmem + lanes + 64, a.dQ.ok() ? a.dQ.at(g, b, h) + oq : nullptr,
                  a.dQhl.ok() ? a.dQhl.at(g, b, h) + oq : nullptr, ldq, i, sq - qb * 128, 0, 32,
                  a.scale, amax);
      rows_out_hl(tmem + lanes, tmem + lanes + 64, a.dQ.ok() ? a.dQ.at(g, b, h) + oq : nullptr,
                  a.dQhl.ok() ? a.dQhl.at(g, b, h) + oq : nullptr, ldq, i, sq - qb * 128, 32, 32,
                  a.scale, amax);
      tc_before();
      named_sync(1, 128);
      if (tid == 0) mbar_arrive(bE);
    }
  }
  if (amax >= 65520.f && amax <= FLT_MAX && a.range_flag) atomicOr(a.range_flag, 1);
  bar_sync();
  if (warp == 0) tmem_free(tmem, 128);
}

AttnTma flash_maps(const AttnArgs& a, bool backward) {
  AttnTma t{};
  // head-split pre-split operands: [rows][32] fp32-sized boxes (hi, lo'
  // halves) in the tiles' SWIZZLE_128B layout; rows >= s arrive zero-filled.
  // Forward: 128-query Q, 64-key K / V; backward: 64-query Q / dO, 128-key K / V
  auto mk = [&](int which, const Mat& m, int rows, int box_rows) {
    t.m[which] = tc_make_map(m, a.G, a.Bb, a.H, rows, 64, box_rows, 32, true, &t.op[which]);
  };
  mk(TQ, a.Q, a.sq, backward ? kQB : 128);
  mk(TK, a.K, a.skv, backward ? 128 : KB);
  mk(TV, a.V, a.skv, backward ? 128 : KB);
  if (backward) mk(TDO, a.dO, a.sq, kQB);
  return t;
}

int n_sms() {
  static int n = 0;
  if (!n) MGLP_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, 0));
  return n;
}

}  // namespace

bool attn_flash_supported(const AttnArgs& a, bool backward) {
  if (!(a.qkv_hs && a.dh == 64 && a.sq >= 128 && a.skv >= 128 && a.sq <= 512 && a.skv <= 512 &&
        a.P.ok()))
    return false;
  // backward: pre-split dO, fp32 O (t_q) and the dS tile-pair store (a whole
  // [64-query][128-key] block grid per head)
  return !backward || (a.do_hs && a.O.ok() && a.dS.ok());
}

void launch_attn_bwd_flash(const AttnArgs& a, const int* active, cudaStream_t s) {
  if (!attn_flash_supported(a, true)) throw ContractViolation("attn_bwd_flash: unsupported");
  static bool attr = [] {
    MGLP_CUDA(cudaFuncSetAttribute(attn_bwd_kv_flash_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, kKvSmem));
    MGLP_CUDA(cudaFuncSetAttribute(attn_bwd_q_flash_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, kQSmem));
    return true;
  }();
  (void)attr;
  const long long heads = (long long)a.G * a.Bb * a.H;
  if (heads == 0) return;
  const AttnTma t = flash_maps(a, true);
  const long long rows = heads * a.sq;
  launch_k(flash_rowdot_kernel, dim3((unsigned)((rows + 255) / 256)), dim3(256), 0, s, 1, a, active);
  MGLP_CUDA(cudaGetLastError());
  const long long nkv = heads * ((a.skv + 127) / 128), nq = heads * ((a.sq + 127) / 128);
  static const int full = [] {  // diagnostics: 1 = kv kernel one problem per CTA, 2 = q kernel
    const char* e = getenv("MGLP_FLASH_GRID");
    return e ? atoi(e) : 0;
  }();
  launch_k(attn_bwd_kv_flash_kernel, dim3((unsigned)((full & 1) ? nkv : std::min<long long>(nkv, n_sms()))),
           dim3(kKvThreads), kKvSmem, s, 1, t, a, active);
  MGLP_CUDA(cudaGetLastError());
  launch_k(attn_bwd_q_flash_kernel, dim3((unsigned)((full & 2) ? nq : std::min<long long>(nq, n_sms()))),
           dim3(kQThreads), kQSmem, s, 1, t, a, active);
  MGLP_CUDA(cudaGetLastError());
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

#ifdef MGLP_FLASH_TRACE
extern "C" int mglp_debug_flash_trace(long long* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, mglp::g_flash_trace, sizeof(long long) * (n < 4096 ? n : 4096));
}
#endif
