// Device building blocks of the fused tcgen05 attention kernels (attn_tc.cu
// for s <= 128, attn_long.cu for s <= 512): hi/lo' fp16 tiles in natural
// row-major SWIZZLE_128B layout used K-major or MN-major, 3-pass split MMAs,
// TMA boxes per (member, batch, head), TMEM row helpers.
#pragma once

#include <cfloat>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace mglp {
namespace attn {

using namespace tc;

constexpr int TILE64 = 128 * 128;       // one hi (or lo) tile: 128 rows x 64 fp16
constexpr int PAIR64 = 2 * TILE64;      // hi + lo
constexpr int PAIR128 = 2 * PAIR64;     // hi + lo, two 64-column blocks


__device__ __forceinline__ int rup(int x, int m) { return (x + m - 1) / m * m; }

// SWIZZLE_128B UMMA descriptor; lbo only matters for MN-major operands with
// more than one 64-wide MN block
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr, uint32_t lbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFFu);
  d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= 1ull << 46;
  d |= 2ull << 61;
  return d;
}

// kind::f16 instruction descriptor: f32 accumulate, f16 A/B, major bits
__device__ __forceinline__ uint32_t idesc(int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (a_mn ? 1u << 15 : 0u) | (b_mn ? 1u << 16 : 0u) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

// One operand of an MMA: a hi/lo tile pair with `rows` rows, used K-major
// (K = tile columns) or MN-major (K = tile rows).
struct Opnd {
  uint32_t hi, lo;
  int rows;
  bool mn;
  __device__ __forceinline__ uint32_t at(int k16) const {
    return mn ? (uint32_t)(k16 * 2048) : (uint32_t)((k16 >> 2) * rows * 128 + (k16 & 3) * 32);
  }
  __device__ __forceinline__ uint32_t lbo() const { return mn ? (uint32_t)(rows * 128) : 16u; }
};

// D = A . B^T over nk16 K steps with the 3-pass split: main (tm) and
// correction (tcor) accumulators (M = 128)
// (acc_in: the first K step accumulates into D instead of overwriting it)
__device__ __forceinline__ void mma3(uint32_t tm, uint32_t tcor, const Opnd& A, const Opnd& B,
                                     int N, int nk16, bool acc_in = false) {
  const uint32_t id = idesc(N, A.mn, B.mn);
  for (int k = 0; k < nk16; ++k) {
    const uint32_t oa = A.at(k), ob = B.at(k);
    const uint64_t dah = desc_sw128(A.hi + oa, A.lbo()), dal = desc_sw128(A.lo + oa, A.lbo());
    const uint64_t dbh = desc_sw128(B.hi + ob, B.lbo()), dbl = desc_sw128(B.lo + ob, B.lbo());
    const uint32_t acc = (k > 0 || acc_in) ? 1u : 0u;
    mma_f16<1>(tm, dah, dbh, id, acc);
    mma_f16<1>(tcor, dal, dbh, id, acc);
    mma_f16<1>(tcor, dah, dbl, id, 1u);
  }
}

// byte offset of 16-byte chunk c (8 fp16 columns) of row r in a tile with R rows
__device__ __forceinline__ uint32_t chunk_off(int R, int r, int c) {
  return (uint32_t)((c >> 3) * R * 128 + r * 128 + (((c & 7) ^ (r & 7)) << 4));
}

// fp32 staging rows [0, nvalid) x ncols (pitch ncols) -> hi/lo tiles of R
// rows (rows >= nvalid become 0). ncols multiple of 8.
__device__ __forceinline__ void conv_rows(uint32_t stg, int nvalid, int R, int ncols, uint32_t thi,
                                          uint32_t tlo, int tid, int nthr, float& amax) {
  const int cpr = ncols >> 3;
  for (int i = tid; i < R * cpr; i += nthr) {
    const int r = i / cpr, c = i - r * cpr;
    float x[8];
    if (r < nvalid) {
      const uint32_t s = stg + (uint32_t)((r * ncols + c * 8) * 4);
      const float4 u = lds128(s), w = lds128(s + 16);
      x[0] = u.x; x[1] = u.y; x[2] = u.z; x[3] = u.w;
      x[4] = w.x; x[5] = w.y; x[6] = w.z; x[7] = w.w;
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) x[e] = 0.f;
    }
    uint4 hi, lo;
    split8(x, hi, lo, amax);
    const uint32_t off = chunk_off(R, r, c);
    sts128(thi + off, hi);
    sts128(tlo + off, lo);
  }
}

// In-place conversion of a TMA-staged fp32 block [nvalid rows][ncols]
// (pitch ncols, ncols <= 64) at `region` into the hi (region) / lo (region +
// TILE64) tile pair of R rows (rows >= nvalid become 0): every thread loads
// its items first, a CTA barrier, then the stores. R * ncols / 8 <= 4 * nthr.
__device__ __forceinline__ void conv_inplace(uint32_t region, int nvalid, int R, int ncols,
                                             int tid, int nthr, float& amax) {
  const int cpr = ncols >> 3;
  float x[4][8];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i = tid + k * nthr;
    const int r = i / cpr, c = i - r * cpr;
    if (r < nvalid && r < R) {
      const uint32_t s = region + (uint32_t)((r * ncols + c * 8) * 4);
      const float4 u = lds128(s), w = lds128(s + 16);
      x[k][0] = u.x; x[k][1] = u.y; x[k][2] = u.z; x[k][3] = u.w;
      x[k][4] = w.x; x[k][5] = w.y; x[k][6] = w.z; x[k][7] = w.w;
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) x[k][e] = 0.f;
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i = tid + k * nthr;
    const int r = i / cpr, c = i - r * cpr;
    if (r < R) {
      uint4 hi, lo;
      split8(x[k], hi, lo, amax);
      const uint32_t off = (uint32_t)(r * 128 + ((((c & 7) ^ (r & 7))) << 4));
      sts128(region + off, hi);
      sts128(region + TILE64 + off, lo);
    }
  }
}

// exp(x) for x <= 0 as ex2.approx(x log2 e): relative error ~1e-6 over the
// softmax range (the reference's exp is f64; the parity bar is 1e-4) at a
// fraction of expf's instruction count
__device__ __forceinline__ float fast_exp(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x * 1.4426950408889634f));
  return y;
}

// 8 values of row r (chunk c) into a hi/lo tile pair
__device__ __forceinline__ void put8(uint32_t thi, uint32_t tlo, int R, int r, int c,
                                     const float* x, float& amax) {
  uint4 hi, lo;
  split8(x, hi, lo, amax);
  const uint32_t off = chunk_off(R, r, c);
  sts128(thi + off, hi);
  sts128(tlo + off, lo);
}

__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// 16 columns of main + correction -> combined fp32 (one TMEM wait)
__device__ __forceinline__ void tmem_pair16(uint32_t tmain, uint32_t tcor, float* out) {
  uint32_t rm[16], rc[16];
  tmem_ld16(tmain, rm);
  tmem_ld16(tcor, rc);
  tmem_wait();
#pragma unroll
  for (int e = 0; e < 16; ++e) out[e] = fmaf(__uint_as_float(rc[e]), kLoInv, __uint_as_float(rm[e]));
}

// this warp's TMEM lanes -> global rows (row < nvalid), columns [c0, c0 + nc)
// (nc multiple of 16, <= 32), scaled by alpha
__device__ __forceinline__ void rows_out(uint32_t tmain, uint32_t tcor, float* out, long long ld,
                                         int row, int nvalid, int c0, int nc, float alpha) {
#pragma unroll
  for (int c = 0; c < 32; c += 16) {
    if (c < nc) {
      float v[16];
      tmem_pair16(tmain + c0 + c, tcor + c0 + c, v);
      if (row < nvalid) {
        float* o = out + row * ld + c0 + c;
#pragma unroll
        for (int e = 0; e < 16; e += 4)
          *reinterpret_cast<float4*>(o + e) =
              make_float4(alpha * v[e], alpha * v[e + 1], alpha * v[e + 2], alpha * v[e + 3]);
      }
    }
  }
}

// output rows (forward O; backward dQ, dK, dV) scaled by alpha: fp32 (out,
// nullable) and/or pre-split hi|lo' (hl, nullable; the next GEMM's A operand,
// common.cuh). hl follows out's strides; the head's column offset must be a
// multiple of 32 so the fp32 offset of the head equals its packed byte offset.
// one 256-bit global store (sm_100: STG.256), 32-byte aligned
__device__ __forceinline__ void st_v8(void* p, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                      uint32_t a4, uint32_t a5, uint32_t a6, uint32_t a7) {
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a0), "r"(a1), "r"(a2),
               "r"(a3), "r"(a4), "r"(a5), "r"(a6), "r"(a7)
               : "memory");
}

__device__ __forceinline__ void rows_out_hl(uint32_t tmain, uint32_t tcor, float* out, float* hl,
                                            long long ld, int row, int nvalid, int c0, int nc,
                                            float alpha, float& amax) {
#pragma unroll
  for (int c = 0; c < 32; c += 16) {
    if (c < nc) {
      float v[16];
      tmem_pair16(tmain + c0 + c, tcor + c0 + c, v);
      if (alpha != 1.f) {
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] *= alpha;
      }
      if (row < nvalid) {
        if (out) {
          float* o = out + row * ld + c0 + c;
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
        if (hl) {
          // 16 values -> hi at p, p + 16 and lo' at p + 64, p + 80 (c0 + c is
          // a multiple of 16: one 32-byte run each)
          uint4 hi[2], lo[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) split8(v + 8 * e, hi[e], lo[e], amax);
          const int col = c0 + c;
          char* p = reinterpret_cast<char*>(hl + row * ld) + (col >> 5) * 128 + (col & 31) * 2;
          if (((reinterpret_cast<uintptr_t>(p) & 31) == 0) && (col & 15) == 0) {
            st_v8(p, hi[0].x, hi[0].y, hi[0].z, hi[0].w, hi[1].x, hi[1].y, hi[1].z, hi[1].w);
            st_v8(p + 64, lo[0].x, lo[0].y, lo[0].z, lo[0].w, lo[1].x, lo[1].y, lo[1].z, lo[1].w);
          } else {
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int ce = col + 8 * e;
              char* q = reinterpret_cast<char*>(hl + row * ld) + (ce >> 5) * 128 + (ce & 31) * 2;
              *reinterpret_cast<uint4*>(q) = hi[e];
              *reinterpret_cast<uint4*>(q + 64) = lo[e];
            }
          }
        }
      }
    }
  }
}

// 1-D bulk copies (P kept pre-split, AttnArgs::p_hl)
__device__ __forceinline__ void bulk_store(void* gdst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(src),
               "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_store_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_store_wait() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* gsrc, uint32_t bytes,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(gsrc), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void problem_of(const AttnArgs& a, int z, int& g, int& b, int& h) {
  h = z % a.H;
  b = (z / a.H) % a.Bb;
  g = z / (a.H * a.Bb);
}

__device__ __forceinline__ void tmem_alloc(uint32_t* slot, uint32_t cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(slot)),
               "r"(cols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_free(uint32_t base, uint32_t cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(cols));
}

// tensor maps of the operand families (one [rows][cols] box per problem)
struct AttnTma {
  CUtensorMap m[5];
  TcOperand op[5];
  int hs_mask = 0;  // bit `which`: the operand is head-split pre-split (AttnArgs::qkv_hs / do_hs)
};
enum { TQ = 0, TK = 1, TV = 2, TP = 3, TDO = 4 };

__device__ __forceinline__ void tma_box(uint32_t dst, const AttnTma& t, int which, int g, int b,
                                        int h, uint64_t* bar, int row0 = 0, int col = 0) {
  int c[5];
  tma_coords(t.op[which], col, row0, g, b, h, c);
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(&t.m[which])), "r"(smem_u32(bar)), "r"(c[0]), "r"(c[1]),
      "r"(c[2]), "r"(c[3]), "r"(c[4])
      : "memory");
}


// A head-split pre-split operand (AttnArgs::qkv_hs / do_hs): its hi and lo'
// halves ([rows][32] fp32-sized boxes, SWIZZLE_128B) land by TMA directly as
// the tile pair X (no staging, no conversion): 2 x 128 rows x 128 B
__device__ __forceinline__ void tma_pair(const Opnd& X, const AttnTma& t, int which, int g, int b,
                                         int h, uint64_t* bar, int row0 = 0) {
  tma_box(X.hi, t, which, g, b, h, bar, row0, 0);
  tma_box(X.lo, t, which, g, b, h, bar, row0, 32);
}
constexpr uint32_t kHsBytes = 2 * 128 * 128;  // one operand tile pair by TMA

}  // namespace attn
}  // namespace mglp
