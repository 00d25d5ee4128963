// Parity-grade tensor-core GEMM for sm_100a: tcgen05.mma kind::tf32 with a
// 3-pass hi/lo split (A_hi.B_hi + A_hi.B_lo + A_lo.B_hi, fp32 accumulation in
// TMEM), the device counterpart of the reference's f64 matmul/linear
// (tensor.cpp:173-237). Single-pass TF32 misses the 1e-4 parity tolerance at
// depth 64; the split keeps ~21 mantissa bits.
//
// Structure (one 128 x BN output tile per CTA, 8 warps):
//   warp 0      TMA producer: A (raw fp32), B_hi/B_lo (pre-split weights) or
//               B raw, into a STAGES-deep smem ring (SWIZZLE_128B)
//   warp 1      MMA issuer (one elected thread): 3 x (BK/8) tcgen05.mma per stage
//   warp 2      TMEM allocator
//   warps 4-7   split converters (x -> hi = x & ~0x1fff, lo = x - hi, in smem)
//               and then the fused epilogue: tcgen05.ld TMEM -> registers ->
//               epilogue_row (bias / GELU / residual / MGRIT combine / grads)
// Operands are 3-D TMA tensor maps [slot][rows][cols], so a whole family of G
// problems (one per coarse interval or per layer) is one launch; member g
// reads slot slot0 + g*step of each operand.
// K-major operands load one [rows x 32] box per stage; MN-major operands
// (weights read transposed in dgrad, activations in wgrad) load
// [32 K-rows x 32 MN] boxes, matching the UMMA MN-major SWIZZLE_128B canonical
// layout ((8,n),(8,k)):((1,LBO),(8,SBO)) with LBO = 4 KiB, SBO = 1 KiB.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "kernels.cuh"

namespace mglp {

namespace {

constexpr int BM = 128;
constexpr int BK = 32;  // fp32 elements per stage = one 128-byte swizzle span
constexpr int kThreads = 256;

struct TcOperand {
  int slot0, step;  // normalized slot coordinates (member g -> slot0 + g*step)
  int mn;           // 1 = MN-major
  // positions of the (row, head, batch, slot) coordinates in the 5-D tensor
  // map (dimension 0 is always the contiguous 32-wide column box); unused
  // head / batch dimensions have extent 1 and coordinate 0
  int pos_row, pos_h, pos_b, pos_slot;
  int use_h, use_b;
};

struct TcParams {
  int G, M, N, K;
  int Bb, H;
  TcOperand a, b, blo;
  int b_presplit;
  int passes;  // 3 = hi.hi + (lo.hi + hi.lo); 1 = hi.hi only (diagnostics)
  EpiArgs ep;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n\t"
      ".reg .pred P1;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra WAIT_%=;\n\t"
      "}" ::"r"(a),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            const int* c) {
  asm volatile(
      "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c[0]), "r"(c[1]), "r"(c[2]),
      "r"(c[3]), "r"(c[4])
      : "memory");
}

// TMA coordinates of one box of operand `op` for problem (g, b, h)
__device__ __forceinline__ void tma_coords(const TcOperand& op, int col, int row, int g, int b,
                                           int h, int* c) {
  c[0] = col;
  c[op.pos_row] = row;
  c[op.pos_h] = op.use_h ? h : 0;
  c[op.pos_b] = op.use_b ? b : 0;
  c[op.pos_slot] = op.slot0 + g * op.step;
}

// UMMA shared-memory descriptor. K-major operands use SWIZZLE_128B (layout
// type 2); MN-major tf32 operands must use SWIZZLE_128B_BASE32B (type 1,
// 32-byte granules over 4 rows -- the only MN-major layout tf32 supports,
// matched by TMA's CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B).
__device__ __forceinline__ uint64_t smem_desc(const void* p, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
  const uint64_t addr = smem_u32(p);
  uint64_t d = 0;
  d |= (addr >> 4) & 0x3FFFull;
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;  // sm100 descriptor version
  d |= (uint64_t)layout << 61;
  return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t"
      ".reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t"
      "}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// x -> (hi, lo): hi keeps the top 10 explicit mantissa bits (exactly a tf32),
// lo = x - hi exactly; the tensor core then sees hi exactly and lo to ~11 bits.
__device__ __forceinline__ void split_tile(float* raw, float* lo, int nfloat, int tid,
                                           int nthreads) {
  float4* r4 = reinterpret_cast<float4*>(raw);
  float4* l4 = reinterpret_cast<float4*>(lo);
  for (int i = tid; i < nfloat / 4; i += nthreads) {
    float4 x = r4[i];
    float4 h, l;
    h.x = __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
    h.y = __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
    h.z = __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
    h.w = __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
    l.x = x.x - h.x;
    l.y = x.y - h.y;
    l.z = x.z - h.z;
    l.w = x.w - h.w;
    r4[i] = h;
    l4[i] = l;
  }
}

template <int BN, int STAGES>
struct Smem {
  static constexpr int A_BYTES = BM * BK * 4;
  static constexpr int B_BYTES = BN * BK * 4;
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;  // A, A_lo, B_hi, B_lo
  static constexpr int BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap mapA,
                   const __grid_constant__ CUtensorMap mapB,
                   const __grid_constant__ CUtensorMap mapBlo, const TcParams p,
                   const int* active) {
  using S = Smem<BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  if (active && *(volatile const int*)active == 0) return;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * S::STAGE_BYTES);
  uint64_t* conv = full + STAGES;
  uint64_t* empty = conv + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);
  double* red = reinterpret_cast<double*>(tmem_slot + 2);  // 8 doubles

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int zi = blockIdx.z;
  const int hh = zi % p.H, bb = (zi / p.H) % p.Bb, g = zi / (p.H * p.Bb);
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int nk = (p.K + BK - 1) / BK;
  const bool convert_b = !p.b_presplit;

  auto stage_a = [&](int s) { return smem + s * S::STAGE_BYTES; };
  auto stage_alo = [&](int s) { return smem + s * S::STAGE_BYTES + S::A_BYTES; };
  auto stage_b = [&](int s) { return smem + s * S::STAGE_BYTES + 2 * S::A_BYTES; };
  auto stage_blo = [&](int s) {
    return smem + s * S::STAGE_BYTES + 2 * S::A_BYTES + S::B_BYTES;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], 4);  // one elected lane per converter warp
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"((uint32_t)(2 * BN)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;


  if (warp == 0) {
    if (lane == 0) {
      const uint32_t bytes =
          S::A_BYTES + S::B_BYTES + (convert_b ? 0 : S::B_BYTES);
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], bytes);
        const int k0 = kb * BK;
        int c[5];
        if (!p.a.mn) {
          tma_coords(p.a, k0, m0, g, bb, hh, c);
          tma_load_5d(stage_a(s), &mapA, &full[s], c);
        } else {
#pragma unroll
          for (int i = 0; i < BM / 32; ++i) {
            tma_coords(p.a, m0 + 32 * i, k0, g, bb, hh, c);
            tma_load_5d(stage_a(s) + i * 4096, &mapA, &full[s], c);
          }
        }
        if (!p.b.mn) {
          tma_coords(p.b, k0, n0, g, bb, hh, c);
          tma_load_5d(stage_b(s), &mapB, &full[s], c);
          if (!convert_b) {
            tma_coords(p.blo, k0, n0, g, bb, hh, c);
            tma_load_5d(stage_blo(s), &mapBlo, &full[s], c);
          }
        } else {
#pragma unroll
          for (int i = 0; i < BN / 32; ++i) {
            tma_coords(p.b, n0 + 32 * i, k0, g, bb, hh, c);
            tma_load_5d(stage_b(s) + i * 4096, &mapB, &full[s], c);
            if (!convert_b) {
              tma_coords(p.blo, n0 + 32 * i, k0, g, bb, hh, c);
              tma_load_5d(stage_blo(s) + i * 4096, &mapBlo, &full[s], c);
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      // instruction descriptor: D f32, A/B tf32, majors, N, M
      const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)p.a.mn << 15) |
                             ((uint32_t)p.b.mn << 16) | ((uint32_t)(BN >> 3) << 17) |
                             ((uint32_t)(BM >> 4) << 24);
      // MN-major: LBO = stride between 32-element MN blocks (one 32-row TMA
      // box), SBO = stride between 4-row K groups of the BASE32B atom
      const uint32_t a_lbo = p.a.mn ? 4096u : 16u, a_sbo = p.a.mn ? 512u : 1024u;
      const uint32_t b_lbo = p.b.mn ? 4096u : 16u, b_sbo = p.b.mn ? 512u : 1024u;
      const uint32_t a_lay = p.a.mn ? 1u : 2u, b_lay = p.b.mn ? 1u : 2u;
      const uint32_t a_kstep = p.a.mn ? 1024u : 32u;  // bytes per K=8 step
      const uint32_t b_kstep = p.b.mn ? 1024u : 32u;
      for (int kb = 0; kb < nk; ++kb) {
        const int s = kb % STAGES;
        const uint32_t ph = (kb / STAGES) & 1;
        mbar_wait(&conv[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int k = 0; k < BK / 8; ++k) {
          const uint64_t dah = smem_desc(stage_a(s) + k * a_kstep, a_lbo, a_sbo, a_lay);
          const uint64_t dal = smem_desc(stage_alo(s) + k * a_kstep, a_lbo, a_sbo, a_lay);
          const uint64_t dbh = smem_desc(stage_b(s) + k * b_kstep, b_lbo, b_sbo, b_lay);
          const uint64_t dbl = smem_desc(stage_blo(s) + k * b_kstep, b_lbo, b_sbo, b_lay);
          const uint32_t acc0 = (kb > 0 || k > 0) ? 1u : 0u;
          // main product and the two correction products accumulate in
          // separate TMEM accumulators, so the small terms are not rounded
          // against the large running sum
          mma_tf32(tmem_base, dah, dbh, idesc, acc0);
          if (p.passes > 1) {
            mma_tf32(tmem_base + BN, dal, dbh, idesc, acc0);
            mma_tf32(tmem_base + BN, dah, dbl, idesc, 1u);
          }
        }
        mma_commit(&empty[s]);
      }
      mma_commit(tmem_full);
    }
    __syncwarp();
  } else if (warp >= 4) {
    const int ct = threadIdx.x - 128;  // 0..127
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % STAGES;
      const uint32_t ph = (kb / STAGES) & 1;
      mbar_wait(&full[s], ph);
      split_tile(reinterpret_cast<float*>(stage_a(s)), reinterpret_cast<float*>(stage_alo(s)),
                 BM * BK, ct, 128);
      if (convert_b)
        split_tile(reinterpret_cast<float*>(stage_b(s)), reinterpret_cast<float*>(stage_blo(s)),
                   BN * BK, ct, 128);
      // generic-proxy smem writes -> visible to the tensor core (async proxy)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&conv[s]);
    }
  }

  // ---- epilogue: TMEM -> registers -> fused epilogue -> global ----
  double r2 = 0.0;
  if (warp >= 4) {
    mbar_wait(tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int q = warp & 3;
    const int row = m0 + q * 32 + lane;
    const uint32_t lane_addr = tmem_base + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
    for (int c = 0; c < BN; c += 16) {
      float v[16];
      tmem_ld16(lane_addr + c, v);
      if (p.passes > 1) {
        float w[16];
        tmem_ld16(lane_addr + BN + c, w);
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] += w[i];
      }
      const int col0 = n0 + c;
      const int nvalid = min(16, p.N - col0);
      if (row < p.M && nvalid > 0) r2 += epilogue_row(p.ep, g, bb, hh, row, col0, v, nvalid);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"((uint32_t)(2 * BN)));
  if (p.ep.kind == EPI_FINAL && p.ep.cmb.mode == CM_RES0) {
    for (int o = 16; o > 0; o >>= 1) r2 += __shfl_xor_sync(0xffffffffu, r2, o);
    if (lane == 0) red[warp] = r2;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int i = 0; i < kThreads / 32; ++i) t += red[i];
      const int blk = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
      p.ep.cmb.norm_partials[p.ep.cmb.norm_base + blk] = t;
    }
  }
}

// split kernel for weights
__global__ void split_tf32_kernel(float* hi, float* lo, const float* src, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const float x = src[i];
    const float h = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
    hi[i] = h;
    lo[i] = x - h;
  }
}

// ---- host side: tensor maps ---------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess || fn == nullptr)
      throw ContractViolation("cuTensorMapEncodeTiled is unavailable");
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode;
}

// 5-D map over the slots (and per-(batch, head) sub-blocks) a family touches:
// member g -> slot slot0 + g*step. rows x cols is the [rows][cols] matrix of
// one problem (row stride ld). Dimensions are ordered by increasing stride
// (a head slice of a [tokens][3d] qkv buffer has a smaller stride than a
// row); dimension 0 is always the contiguous columns.
CUtensorMap make_map(const Mat& m, int G, int Bb, int H, int rows, int cols, int box_rows,
                     TcOperand* op, bool mn_major) {
  long long lo = m.slot0, hi = m.slot0 + (long long)(G - 1) * m.step;
  if (hi < lo) std::swap(lo, hi);
  const float* base = m.ptr + lo * m.slot_stride;
  long long nslots = hi - lo + 1;
  long long sstride = m.slot_stride;
  if (nslots == 1 || sstride == 0) {
    nslots = 1;
    sstride = 0;
    op->slot0 = 0;
    op->step = 0;
  } else {
    op->slot0 = (int)(m.slot0 - lo);
    op->step = m.step;
  }
  op->use_h = (m.hstride != 0 && H > 1) ? 1 : 0;
  op->use_b = (m.bstride != 0 && Bb > 1) ? 1 : 0;
  struct D {
    long long extent, stride;
    int which, box;
  };
  D dims[4] = {{rows, (long long)m.ld, 0, box_rows},
               {op->use_h ? H : 1, op->use_h ? m.hstride : 0, 1, 1},
               {op->use_b ? Bb : 1, op->use_b ? m.bstride : 0, 2, 1},
               {nslots, sstride, 3, 1}};
  // used dimensions first, by increasing stride; unused (extent 1) last
  std::sort(dims, dims + 4, [](const D& a, const D& b) {
    const bool ua = a.stride != 0 || a.which == 0, ub = b.stride != 0 || b.which == 0;
    if (ua != ub) return ua;
    return a.stride < b.stride;
  });
  long long maxs = 16;
  for (const D& d : dims) maxs = std::max(maxs, d.stride);
  cuuint64_t gdim[5] = {(cuuint64_t)cols, 1, 1, 1, 1};
  cuuint64_t gstr[4];
  cuuint32_t box[5] = {32, 1, 1, 1, 1};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  for (int i = 0; i < 4; ++i) {
    gdim[i + 1] = (cuuint64_t)dims[i].extent;
    gstr[i] = (cuuint64_t)((dims[i].stride != 0 || dims[i].which == 0) ? dims[i].stride : maxs) * 4;
    box[i + 1] = (cuuint32_t)dims[i].box;
    const int pos = i + 1;
    switch (dims[i].which) {
      case 0: op->pos_row = pos; break;
      case 1: op->pos_h = pos; break;
      case 2: op->pos_b = pos; break;
      default: op->pos_slot = pos; break;
    }
  }
  if ((reinterpret_cast<uintptr_t>(base) & 15))
    throw ContractViolation("gemm_tc: operand base is not 16-byte aligned");
  for (int i = 0; i < 4; ++i)
    if (gstr[i] % 16 || gstr[i] == 0)
      throw ContractViolation("gemm_tc: operand strides must be multiples of 16 bytes");
  CUtensorMap map;
  CUresult r = encoder()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, const_cast<float*>(base), gdim,
                         gstr, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                                  : CU_TENSOR_MAP_SWIZZLE_128B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw ContractViolation("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return map;
}

template <int BN, int STAGES>
void launch_cfg(const GemmArgs& a, const int* active, cudaStream_t s) {
  TcParams p;
  p.G = a.G;
  p.M = a.M;
  p.N = a.N;
  p.K = a.K;
  p.ep = a.ep;
  p.b_presplit = a.Blo.ok() ? 1 : 0;
  static const int passes = [] {
    const char* e = getenv("MGLP_DEBUG_TF32_PASSES");
    return e ? atoi(e) : 3;
  }();
  p.passes = passes;
  p.a.mn = a.a_mn;
  p.b.mn = a.b_mn;
  p.blo.mn = a.b_mn;
  // A: [M][K] (K-major) or [K][M] (MN-major); box rows: BM, or 32 K-rows
  p.Bb = a.Bb;
  p.H = a.H;
  CUtensorMap mA = a.a_mn ? make_map(a.A, a.G, a.Bb, a.H, a.K, a.M, BK, &p.a, true)
                          : make_map(a.A, a.G, a.Bb, a.H, a.M, a.K, BM, &p.a, false);
  CUtensorMap mB = a.b_mn ? make_map(a.B, a.G, a.Bb, a.H, a.K, a.N, BK, &p.b, true)
                          : make_map(a.B, a.G, a.Bb, a.H, a.N, a.K, BN, &p.b, false);
  CUtensorMap mBlo = mB;
  if (p.b_presplit)
    mBlo = a.b_mn ? make_map(a.Blo, a.G, a.Bb, a.H, a.K, a.N, BK, &p.blo, true)
                  : make_map(a.Blo, a.G, a.Bb, a.H, a.N, a.K, BN, &p.blo, false);
  else
    p.blo = p.b;
  const int smem = Smem<BN, STAGES>::BYTES;
  MGLP_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<BN, STAGES>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  dim3 grid(ceil_div(a.N, BN), ceil_div(a.M, BM), a.G * a.Bb * a.H);
  gemm_tc_kernel<BN, STAGES><<<grid, kThreads, smem, s>>>(mA, mB, mBlo, p, active);
  MGLP_CUDA(cudaGetLastError());
}

constexpr int kBN = 128;
constexpr int kStages = 3;

}  // namespace

int gemm_tc_blocks(const GemmArgs& a) {
  return ceil_div(a.N, kBN) * ceil_div(a.M, BM) * a.G * a.Bb * a.H;
}

void launch_gemm_tc(const GemmArgs& a, const int* active, cudaStream_t s) {
  if (a.G == 0 || a.M == 0 || a.N == 0) return;
  if (a.K == 0) throw ContractViolation("gemm_tc: K must be positive");
  launch_cfg<kBN, kStages>(a, active, s);
}

void launch_split_tf32(float* hi, float* lo, const float* src, long long n, cudaStream_t s) {
  if (n == 0) return;
  const int blocks = (int)std::min<long long>(148 * 8, (n + 255) / 256);
  split_tf32_kernel<<<blocks, 256, 0, s>>>(hi, lo, src, n);
}

}  // namespace mglp
