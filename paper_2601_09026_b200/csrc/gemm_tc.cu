// Parity-grade tensor-core GEMM for sm_100a: tcgen05.mma kind::f16 over a
// 3-pass fp16 hi/lo split with fp32 accumulation in TMEM, the device
// counterpart of the reference's f64 matmul/linear (tensor.cpp:173-237).
//
// Split ("fp16x3"): every fp32 operand value x becomes
//     hi  = fp16_rn(x)                   (11 significant bits)
//     lo' = fp16_rn((x - hi) * 2^11)     (the next 11 bits, pre-scaled so the
//                                         residual stays a normal fp16)
// and C = A_hi.B_hi + 2^-11 (A_lo'.B_hi + A_hi.B_lo'), the main product and
// the correction products accumulating in separate TMEM accumulators (so the
// small terms are not rounded against the large running sum). Per element the
// representation error is <= 2^-22 |x| (plus 2^-35 absolute below the fp16
// normal range): the same ~22-bit operand precision as a tf32x3 split, at the
// fp16 tensor-core rate (2x tf32). Single-pass tensor-core GEMMs miss the
// 1e-4 parity tolerance at depth 64. Finite values
// |x| >= 65520 do not fit fp16: the converters raise GemmArgs::range_flag and
// the engine reports it (no silent overflow).
//
// Structure (persistent; one CTA, or with cta_group::2 one CTA pair, per SM):
//   warp 0      TMA producer: fp32 operand tiles -> staging ring; or, with
//               A produced pre-split (GemmArgs::Ahl: LayerNorm, attention,
//               GELU / GELU' epilogues, LN VJP, the upstream pack), hi|lo
//               A tiles straight into the MMA ring (no conversion at all)
//   warp 1      MMA issuer (one elected thread): 3 x 2 tcgen05.mma per 32-K stage
//   warp 2      TMEM allocator
//   warp 3      TMA producer for a pre-split B (weights): hi|lo tiles straight
//               into the MMA ring, no conversion
//   warps 4-7   converters: staging (fp32, K- or MN-major) -> hi|lo fp16 tiles
//               (always K-major SWIZZLE_128B: one 128-byte row = 32 hi + 32 lo')
//   warps 8-    epilogue: tcgen05.ld TMEM -> registers -> epilogue_row (bias /
//               GELU / residual / MGRIT combine / grads) -> global
// The staging ring is released as soon as a stage is converted, so the next
// TMA loads overlap both the conversion and the MMAs of earlier stages.
// Operands are 5-D TMA tensor maps [slot][batch][head][rows][cols] (sorted by
// stride), so a whole family of G problems (one per coarse interval or per
// layer, each possibly a grid of per-(batch, head) attention problems) is one
// launch; member g reads slot slot0 + g*step of each operand.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace mglp {

using namespace tc;

namespace {

constexpr int BK = 32;          // K elements per stage (one 128-byte fp32 row span)
constexpr int ROWS = 128;       // operand rows per CTA per stage (A and B)
constexpr int TILE_BYTES = ROWS * BK * 4;  // 16 KiB: fp32 staging tile == hi|lo tile
// 12 tile slots shared by the rings. B converted in smem: 3 staging stages
// (stgA, stgB) + 3 hi|lo stages (hlA, hlB). B pre-split: A staging, hi|lo A
// and the B ring 4 deep each (measured best of the 12-slot splits; the
// mainloop is MMA-bound at the power-capped clock, not load-bound).
constexpr int NSLOTS = 12;
constexpr int MAXR = 8;  // barrier array length
// + barriers (1 KiB) + per-epilogue-warp 32 x 16 fp32 transpose buffers
constexpr int SMEM_BYTES = NSLOTS * TILE_BYTES + 1024 /*align*/ + 1024 + 8 * 2048;
// Drain variant (DR = 1; CTA pair, both operands pre-split): the epilogue
// first copies the whole accumulator (main + 2^-11 correction, combined)
// from TMEM into shared memory -- 32 rows x 128 columns fp32 per epilogue
// warp, 128 KiB per CTA -- and releases TMEM at once, so the next tile's
// MMAs run while the bias / activation / combine math and the global stores
// of this tile proceed from shared memory. The hi|lo rings shrink to 3 + 3
// stages to make room.
constexpr int NSLOTS_DR = 6;
constexpr int DRAIN_WARP_BYTES = 32 * 128 * 4;
constexpr int SMEM_BYTES_DR = NSLOTS_DR * TILE_BYTES + 1024 + 1024 + 8 * DRAIN_WARP_BYTES;
static_assert(SMEM_BYTES_DR <= 232448, "drain variant exceeds 227 KiB of shared memory");
template <int DR>
constexpr int nslots() { return DR ? NSLOTS_DR : NSLOTS; }
template <int DR>
constexpr int smem_bytes() { return DR ? SMEM_BYTES_DR : SMEM_BYTES; }
// 16-byte piece swizzle of the drain buffer (512-byte rows): the drain's
// lane = row stores and the epilogue's 4-lanes-per-row loads are both
// bank-conflict free
__device__ __forceinline__ int drain_swz(int r) { return ((r & 1) << 2) | ((r >> 1) & 3); }


struct TcParams {
  int G, M, N, K;
  int Bb, H;
  TcOperand a, b;
  int a_mn, b_mn;  // staging layout of the converted operands
  int b_hl;        // B's MN-major staging holds pre-split rows (GemmArgs::b_mn_hl)
  int a_hl;        // likewise A (GemmArgs::a_mn_hl)
  int b_direct;    // B comes pre-split (hi|lo tiles TMA'd straight into the MMA ring)
  int a_direct;    // A too (K-major, produced pre-split): no conversion at all
  int passes;      // 3 = hi.hi + (lo.hi + hi.lo); 1 = hi.hi only (diagnostics)
  int ring_a, ring_h, ring_b;  // pre-split B: staging / hi|lo / B ring depths
  int vec_ok;      // every epilogue operand row start is 16-byte aligned
  int* range_flag;
  unsigned long long* prof;  // MGLP_GEMM_PROF: cycles spent per barrier wait kind (diagnostics)
  int debug;  // MGLP_DEBUG_GEMM bits (timing diagnostics only): 1 skip conversion, 2 skip
              // epilogue stores, 4 every unit loads the same (L2-resident) pre-split tiles
  EpiArgs ep;
};


// One 128-row operand tile: fp32 staging -> K-major SW128 hi|lo tile (row r =
// [32 hi | 32 lo'] in 16-byte chunks at r*128 + ((chunk ^ (r & 7)) << 4)).
// Staging is either K-major SWIZZLE_128B ([128 rows][32 K]) or MN-major dense
// ([32 K][128 rows]). Converter warp c (of 4) handles K chunk kc = c (8
// values) of every row, lane = row within a 32-row block: all shared-memory
// accesses are bank-conflict free.
// MN-major staging whose rows are already pre-split (row k: per 32-column
// chunk 32 hi | 32 lo' fp16): regroup the halves of 8 K values of row r
// into the K-major hi|lo tile (no arithmetic; the producer range-checked)
__device__ __forceinline__ void regroup_tile(uint32_t stg, uint32_t hl, int kc, int lane) {
#pragma unroll
  for (int rb = 0; rb < ROWS / 32; ++rb) {
    const int r = rb * 32 + lane;
    uint32_t h[4], l[4];
#pragma unroll
    for (int e = 0; e < 8; e += 2) {
      const uint32_t a0 = stg + (kc * 8 + e) * (ROWS * 4) + (r >> 5) * 128 + (r & 31) * 2;
      const uint32_t a1 = a0 + ROWS * 4;
      uint16_t h0, h1, l0, l1;
      asm volatile("ld.shared.u16 %0, [%1];" : "=h"(h0) : "r"(a0));
      asm volatile("ld.shared.u16 %0, [%1];" : "=h"(h1) : "r"(a1));
      asm volatile("ld.shared.u16 %0, [%1];" : "=h"(l0) : "r"(a0 + 64));
      asm volatile("ld.shared.u16 %0, [%1];" : "=h"(l1) : "r"(a1 + 64));
      h[e >> 1] = (uint32_t)h0 | ((uint32_t)h1 << 16);
      l[e >> 1] = (uint32_t)l0 | ((uint32_t)l1 << 16);
    }
    const uint32_t orow = hl + r * 128;
    sts128(orow + ((kc ^ (r & 7)) << 4), make_uint4(h[0], h[1], h[2], h[3]));
    sts128(orow + (((4 + kc) ^ (r & 7)) << 4), make_uint4(l[0], l[1], l[2], l[3]));
  }
}

// The same regroup from a SWIZZLE_128B staging: the MN-major pre-split rows
// arrive as four [32 K rows][32 M columns] boxes (each 128-byte row = 32 hi |
// 32 lo' fp16; box j = M columns 32 j ..), so every 8 K rows x 8 M values of
// one half are an 8x8 b16 matrix whose 16-byte rows sit in distinct bank
// groups: ldmatrix .trans reads them conflict-free and hands each thread two
// consecutive K values of one M row (4 bytes of the K-major output chunk).
// Converter warp kc: K rows kc*8 .. +7, all 128 M rows, both halves.
__device__ __forceinline__ void regroup_tile_sw(uint32_t stg, uint32_t hl, int kc, int lane) {
  const int krow = kc * 8 + (lane & 7);
#pragma unroll
  for (int c = 0; c < 8; ++c) {  // 8 x 4 matrices = 16 M blocks of 8 x {hi, lo'}
    const int g = 4 * c + (lane >> 3);       // the matrix this lane addresses a row of
    const int mb = g & 15, part = g >> 4;    // M block, half
    const int ch = (mb & 3) + 4 * part;      // 16-byte chunk within the staging row
    const uint32_t addr = stg + (mb >> 2) * 4096 + krow * 128 + ((ch ^ (krow & 7)) << 4);
    uint32_t d[4];
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3])
                 : "r"(addr));
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int gi = 4 * c + i, mbi = gi & 15, pi = gi >> 4;
      const int M = mbi * 8 + (lane >> 2);  // K values 2 (lane & 3), +1 of M row M
      const uint32_t o = hl + M * 128 + (((pi * 4 + kc) ^ (M & 7)) << 4) + (lane & 3) * 4;
      asm volatile("st.shared.b32 [%0], %1;" ::"r"(o), "r"(d[i]) : "memory");
    }
  }
}

__device__ __forceinline__ void convert_tile(uint32_t stg, uint32_t hl, bool mn, int kc,
                                             int lane, float& amax) {
  // all staging loads first (the compiler cannot reorder them across the
  // hi|lo stores, which it cannot prove disjoint): 4 independent rows in flight
  float x[ROWS / 32][8];
#pragma unroll
  for (int rb = 0; rb < ROWS / 32; ++rb) {
    const int r = rb * 32 + lane;
    if (!mn) {
      const uint32_t row = stg + r * 128;
      const float4 u = lds128(row + (((2 * kc) ^ (r & 7)) << 4));
      const float4 v = lds128(row + (((2 * kc + 1) ^ (r & 7)) << 4));
      x[rb][0] = u.x; x[rb][1] = u.y; x[rb][2] = u.z; x[rb][3] = u.w;
      x[rb][4] = v.x; x[rb][5] = v.y; x[rb][6] = v.z; x[rb][7] = v.w;
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) x[rb][e] = lds32(stg + ((kc * 8 + e) * ROWS + r) * 4);
    }
  }
#pragma unroll
  for (int rb = 0; rb < ROWS / 32; ++rb) {
    const int r = rb * 32 + lane;
    uint4 hi, lo;
    split8(x[rb], hi, lo, amax);
    const uint32_t orow = hl + r * 128;
    sts128(orow + ((kc ^ (r & 7)) << 4), hi);
    sts128(orow + (((4 + kc) ^ (r & 7)) << 4), lo);
  }
}

// ---- the kernel -------------------------------------------------------------------
// CG = 1: one CTA computes a 128 x 128 tile; two TMEM accumulator buffers
//         (each main + correction, 256 columns) let the epilogue of tile t
//         overlap the MMAs of tile t+1.
// CG = 2: a CTA pair computes a 256 x 256 tile with cta_group::2 MMAs issued
//         by the leader: each CTA holds its 128 rows of A and 128 of the 256
//         B rows; per SM the B operand traffic through shared memory halves.
//         TMEM (512 columns) holds one main + one correction accumulator.
template <int CG>
struct Cfg {
  static constexpr int TM = 128 * CG;     // tile rows
  static constexpr int TN = 128 * CG;     // tile columns
  static constexpr int NACC = CG == 1 ? 2 : 1;  // TMEM accumulator buffers
  static constexpr int EPI_WARPS = 4 * CG;
  static constexpr int THREADS = 32 * (8 + EPI_WARPS);
};

template <int CG, int DR>
__global__ void __launch_bounds__(Cfg<CG>::THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap mapA,
                   const __grid_constant__ CUtensorMap mapB, const TcParams p,
                   const int* active) {
  pdl_wait();
  pdl_trigger();
  using C = Cfg<CG>;
  constexpr int TN = C::TN, NACC = C::NACC;
  extern __shared__ uint8_t smem_raw[];
  // the early exit is uniform over a cluster (same flag): no CTA is left
  // waiting on its peer
  if (active && *(volatile const int*)active == 0) return;
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  constexpr int NS = nslots<DR>();
  uint64_t* fullA = reinterpret_cast<uint64_t*>(smem + NS * TILE_BYTES);  // [NA]
  uint64_t* fullB = fullA + MAXR;    // [NB]
  uint64_t* emptyB = fullB + MAXR;   // [NB]
  uint64_t* sfree = emptyB + MAXR;   // [NA]
  uint64_t* conv = sfree + MAXR;     // [NH]
  uint64_t* empty = conv + MAXR;     // [NH]
  uint64_t* cdone = empty + MAXR;    // [NH] CG = 2, follower CTA: converters -> signaler
  uint64_t* tfull = cdone + MAXR;    // [NACC]
  uint64_t* tempty = tfull + NACC;    // [NACC]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + NACC);
  double* red = reinterpret_cast<double*>(tmem_slot + 2);  // [NACC][EPI_WARPS]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cr = CG == 2 ? cluster_rank() : 0;
  const bool leader = cr == 0;
  const int unit = CG == 2 ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int nunits = CG == 2 ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  const int nk = (p.K + BK - 1) / BK;
  const int tiles_n = (p.N + TN - 1) / TN, tiles_m = (p.M + C::TM - 1) / C::TM;
  const int tiles_m128 = (p.M + 127) / 128;
  const int per_prob = tiles_n * tiles_m;
  const int total = per_prob * p.G * p.Bb * p.H;

  // ring depths: NA staging stages, NH hi|lo stages, NB pre-split B slots
  const bool direct = p.b_direct != 0, adirect = p.a_direct != 0;
  // both operands pre-split: 6 A + 6 B hi|lo slots, no staging
  const int NA = adirect ? 0 : (direct ? p.ring_a : 3);
  const int NH = adirect ? (DR ? 3 : 6) : (direct ? p.ring_h : 3);
  const int NB = adirect ? (DR ? 3 : 6) : p.ring_b;
  auto slot = [&](int i) { return smem + i * TILE_BYTES; };
  auto stg_a = [&](int s) { return direct ? slot(s) : slot(2 * s); };
  auto stg_b = [&](int s) { return slot(2 * s + 1); };
  auto hl_a = [&](int s) { return direct ? slot(NA + s) : slot(6 + 2 * s); };
  auto hl_b = [&](int s) { return slot(7 + 2 * s); };
  auto b_slot = [&](int j) { return slot(NA + NH + j); };
  struct Tile {
    int z, g, b, h, m0, n0, mt, nt;
  };
  auto tile_of = [&](int t) {
    Tile T;
    T.z = t / per_prob;
    const int r = t % per_prob;
    T.nt = r % tiles_n;
    T.h = T.z % p.H;
    T.b = (T.z / p.H) % p.Bb;
    T.g = T.z / (p.H * p.Bb);
    T.mt = (r / tiles_n) * CG + (int)cr;  // this CTA's 128-row tile
    T.m0 = T.mt * 128;
    T.n0 = T.nt * TN;
    return T;
  };

  if (threadIdx.x == 0) {
    for (int j = 0; j < MAXR; ++j) {
      mbar_init(&fullB[j], 1);
      mbar_init(&emptyB[j], 1);  // MMA commit
      mbar_init(&fullA[j], 1);
      mbar_init(&sfree[j], 4);  // each converter warp, after its staging reads
      // leader: its 4 converter warps (+ the follower's signaler for CG = 2)
      mbar_init(&conv[j], CG == 1 ? 4 : 5);
      mbar_init(&empty[j], 1);  // MMA commit
      mbar_init(&cdone[j], 4);
    }
    for (int a = 0; a < NACC; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], CG);  // one arrive per CTA
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    if constexpr (CG == 1) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(512u));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       smem_u32(tmem_slot)),
                   "r"(512u));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if constexpr (CG == 2) cluster_sync();  // peer barriers initialised before any remote arrive
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;
  // diagnostics: cycles a role spends waiting, per barrier kind
  unsigned long long wt = 0;
  auto wait = [&](uint64_t* bar, uint32_t parity) {
    if (p.prof) {
      const long long t0 = clock64();
      mbar_wait(bar, parity);
      wt += (unsigned long long)(clock64() - t0);
    } else {
      mbar_wait(bar, parity);
    }
  };
  auto flush = [&](int kind) {
    if (p.prof && wt) atomicAdd(&p.prof[kind], wt);
    wt = 0;
  };
  const long long t_start = clock64();

  if (warp == 0) {
    // ===== TMA producer: fp32 operand tiles into the staging ring =====
    if (lane == 0 && adirect) {
      // pre-split A: hi|lo tiles straight into the MMA ring once the MMAs
      // have released the slot
      int kg = 0;
      for (int t = unit; t < total; t += nunits) {
        const Tile T = tile_of(t);
        for (int kb = 0; kb < nk; ++kb, ++kg) {
          const int s = kg % NH;
          wait(&empty[s], ((kg / NH) & 1) ^ 1);
          flush(0);
          mbar_expect_tx(&fullA[s], TILE_BYTES);
          int c[5];
          if (p.debug & 4)  // diagnostics: every unit reads the same (L2-resident) A rows
            tma_coords(p.a, kb * BK, (int)cr * 128, 0, 0, 0, c);
          else
            tma_coords(p.a, kb * BK, T.m0, T.g, T.b, T.h, c);
          tma_load_5d(hl_a(s), &mapA, &fullA[s], c);
        }
      }
    } else if (lane == 0) {
      const uint32_t bytes = TILE_BYTES * (p.b_direct ? 1 : 2);
      int kg = 0;
      for (int t = unit; t < total; t += nunits) {
        const Tile T = tile_of(t);
        const int nb0 = T.n0 + (int)cr * 128;
        for (int kb = 0; kb < nk; ++kb, ++kg) {
          const int s = kg % NA;
          const uint32_t ph = (kg / NA) & 1;
          wait(&sfree[s], ph ^ 1);
          flush(0);
          mbar_expect_tx(&fullA[s], bytes);
          const int k0 = kb * BK;
          int c[5];
          if (p.a_hl) {  // four swizzled [32][32] boxes (regroup_tile_sw)
            for (int j = 0; j < 4; ++j) {
              tma_coords(p.a, T.m0 + 32 * j, k0, T.g, T.b, T.h, c);
              tma_load_5d(stg_a(s) + j * 4096, &mapA, &fullA[s], c);
            }
          } else {
            if (!p.a_mn)
              tma_coords(p.a, k0, T.m0, T.g, T.b, T.h, c);
            else
              tma_coords(p.a, T.m0, k0, T.g, T.b, T.h, c);
            tma_load_5d(stg_a(s), &mapA, &fullA[s], c);
          }
          if (!p.b_direct) {
            if (p.b_hl) {
              for (int j = 0; j < 4; ++j) {
                tma_coords(p.b, nb0 + 32 * j, k0, T.g, T.b, T.h, c);
                tma_load_5d(stg_b(s) + j * 4096, &mapB, &fullA[s], c);
              }
            } else {
              if (!p.b_mn)
                tma_coords(p.b, k0, nb0, T.g, T.b, T.h, c);
              else
                tma_coords(p.b, nb0, k0, T.g, T.b, T.h, c);
              tma_load_5d(stg_b(s), &mapB, &fullA[s], c);
            }
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 3) {
    // ===== TMA producer for a pre-split B: hi|lo tiles into the MMA ring =====
    if (p.b_direct && lane == 0) {
      int kg = 0;
      for (int t = unit; t < total; t += nunits) {
        const Tile T = tile_of(t);
        const int nb0 = T.n0 + (int)cr * 128;
        for (int kb = 0; kb < nk; ++kb, ++kg) {
          const int j = kg % NB;
          wait(&emptyB[j], ((kg / NB) & 1) ^ 1);
          flush(1);
          mbar_expect_tx(&fullB[j], TILE_BYTES);
          int c[5];
          if (p.debug & 4)  // diagnostics: every unit reads the same (L2-resident) B rows
            tma_coords(p.b, kb * BK, (int)cr * 128, 0, 0, 0, c);
          else
            tma_coords(p.b, kb * BK, nb0, T.g, T.b, T.h, c);
          tma_load_5d(b_slot(j), &mapB, &fullB[j], c);
        }
      }
    }
    __syncwarp();
  } else if (warp == 2) {
    // ===== follower CTA of a pair: forward "stage converted" to the leader =====
    if (CG == 2 && !leader && lane == 0) {
      const uint32_t conv_leader0 = map_to_rank(smem_u32(&conv[0]), 0);
      int kg = 0;
      for (int t = unit; t < total; t += nunits)
        for (int kb = 0; kb < nk; ++kb, ++kg) {
          const int s = kg % NH;
          wait(&cdone[s], (kg / NH) & 1);
          flush(2);
          mbar_arrive_cluster(conv_leader0 + s * 8);
        }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===== MMA issuer (one thread; for CG = 2 the leader's drives both SMs) =====
    if (leader && lane == 0) {
      // instruction descriptor: D f32, A/B f16, both K-major, N, M
      const uint32_t idesc = (1u << 4) | ((uint32_t)(TN >> 3) << 17) |
                             ((uint32_t)(C::TM >> 4) << 24);
      int kg = 0, tc = 0;
      for (int t = unit; t < total; t += nunits, ++tc) {
        const int acc = tc % NACC;
        const uint32_t aph = (tc / NACC) & 1;
        wait(&tempty[acc], aph ^ 1);
        flush(3);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t tm = tmem_base + (uint32_t)(acc * 2 * TN);
        for (int kb = 0; kb < nk; ++kb, ++kg) {
          const int s = kg % NH;
          const uint32_t ph = (kg / NH) & 1;
          wait(&conv[s], ph);
          flush(4);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const int j = kg % NB;
          const uint8_t* bt = p.b_direct ? b_slot(j) : hl_b(s);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t dah = smem_desc_sw128(hl_a(s) + k * 32);
            const uint64_t dal = smem_desc_sw128(hl_a(s) + 64 + k * 32);
            const uint64_t dbh = smem_desc_sw128(bt + k * 32);
            const uint64_t dbl = smem_desc_sw128(bt + 64 + k * 32);
            const uint32_t acc0 = (kb > 0 || k > 0) ? 1u : 0u;
            mma_f16<CG>(tm, dah, dbh, idesc, acc0);
            if (p.passes > 1) {
              mma_f16<CG>(tm + TN, dal, dbh, idesc, acc0);
              mma_f16<CG>(tm + TN, dah, dbl, idesc, 1u);
            }
          }
          mma_commit<CG>(&empty[s]);
          if (p.b_direct) mma_commit<CG>(&emptyB[j]);
        }
        mma_commit<CG>(&tfull[acc]);
      }
    }
    __syncwarp();
  } else if (warp >= 4 && warp < 8) {
    // ===== converters: staging -> hi|lo tiles; release the staging stage,
    // then (all four warps done) signal the MMA issuer =====
    const int kc = warp - 4;
    float amax = 0.f;
    int kg = 0;
    for (int t = unit; t < total; t += nunits) {
      for (int kb = 0; kb < nk; ++kb, ++kg) {
        if (adirect) {
          // nothing to convert: relay "A and B landed" to the MMA issuer
          const int s = kg % NH;
          wait(&fullA[s], (kg / NH) & 1);
          wait(&fullB[kg % NB], (kg / NB) & 1);
          __syncwarp();
          if (lane == 0) mbar_arrive(leader ? &conv[s] : &cdone[s]);
          continue;
        }
        const int sa = kg % NA, s = kg % NH;
        wait(&fullA[sa], (kg / NA) & 1);
        if (kc == 0 && lane == 0) flush(5);
        wait(&empty[s], ((kg / NH) & 1) ^ 1);  // hi|lo buffers no longer read by the MMAs
        if (kc == 0 && lane == 0) flush(6);
        if (!(p.debug & 1)) {
          if (p.a_hl)
            regroup_tile_sw(smem_u32(stg_a(sa)), smem_u32(hl_a(s)), kc, lane);
          else
            convert_tile(smem_u32(stg_a(sa)), smem_u32(hl_a(s)), p.a_mn, kc, lane, amax);
          if (!p.b_direct) {
            if (p.b_hl)
              regroup_tile_sw(smem_u32(stg_b(sa)), smem_u32(hl_b(s)), kc, lane);
            else
              convert_tile(smem_u32(stg_b(sa)), smem_u32(hl_b(s)), p.b_mn, kc, lane, amax);
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sfree[sa]);
        if (p.b_direct) wait(&fullB[kg % NB], (kg / NB) & 1);
        if (kc == 0 && lane == 0) flush(7);
        // generic-proxy smem writes -> visible to the tensor core (async proxy)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        // leader: straight to the MMA issuer; follower: to the signaler warp,
        // which forwards one cluster-scope arrive (keeps the release fence of
        // the remote arrive off the converters' critical path)
        if (lane == 0) mbar_arrive(leader ? &conv[s] : &cdone[s]);
      }
    }
    if (amax >= 65520.f && amax <= FLT_MAX && p.range_flag) atomicOr(p.range_flag, 1);
  } else if (warp >= 8) {
    // ===== epilogue: (4 lane quarters) x (CG column halves) =====
    const int ew = warp - 8;
    const int q = warp & 3, half = ew >> 2;
    constexpr int COLS = TN / CG;  // columns per epilogue warp
    const bool res0 = p.ep.kind == EPI_FINAL && p.ep.cmb.mode == CM_RES0;
    const uint32_t tempty_leader = CG == 2 ? map_to_rank(smem_u32(&tempty[0]), 0) : 0u;
    const uint32_t ebuf = smem_u32(smem + NS * TILE_BYTES + 1024) + ew * (DR ? DRAIN_WARP_BYTES : 2048);
    int tc = 0;
    for (int t = unit; t < total; t += nunits, ++tc) {
      if constexpr (DR != 0 && CG == 2) {
        const Tile T = tile_of(t);
        wait(&tfull[0], tc & 1);
        if (ew == 0 && lane == 0) flush(8);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t lane_addr = tmem_base + ((uint32_t)(q * 32) << 16);
        // (1) drain: TMEM (main + correction) -> combined fp32 rows in smem
#pragma unroll 1
        for (int c = 0; c < COLS; c += 16) {
          uint32_t rv[16], rw[16];
          tmem_ld16(lane_addr + half * COLS + c, rv);
          if (p.passes > 1) tmem_ld16(lane_addr + TN + half * COLS + c, rw);
          tmem_wait();
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            uint4 w4;
            float* f = reinterpret_cast<float*>(&w4);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float mv = __uint_as_float(rv[4 * cc + i]);
              f[i] = p.passes > 1 ? fmaf(__uint_as_float(rw[4 * cc + i]), kLoInv, mv) : mv;
            }
            sts128(ebuf + lane * 512 + ((((c >> 2) + cc) ^ drain_swz(lane)) << 4), w4);
          }
        }
        // the accumulator is free for the next tile's MMAs
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        asm volatile("bar.sync 2, %0;" ::"n"(32 * C::EPI_WARPS) : "memory");
        if (ew == 0 && lane == 0) {
          if (leader)
            mbar_arrive(&tempty[0]);
          else
            mbar_arrive_cluster(tempty_leader);
        }
        __syncwarp();
        // (2) the epilogue proper from shared memory, 4 lanes per row
        double r2 = 0.0;
#pragma unroll 1
        for (int c = 0; c < COLS; c += 16) {
          const int col = T.n0 + half * COLS + c + (lane & 3) * 4;
          const int nvalid = min(4, p.N - col);
          float4 w[4];
          int rows[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int r = i * 8 + (lane >> 2);
            w[i] = lds128(ebuf + r * 512 + ((((c >> 2) + (lane & 3)) ^ drain_swz(r)) << 4));
            const int row = T.m0 + q * 32 + r;
            rows[i] = (row < p.M && nvalid > 0) ? row : -1;
          }
          if (!(p.debug & 2)) {
            if (nvalid == 4 && p.vec_ok) {
              r2 += epilogue_4x4(p.ep, T.g, T.b, T.h, rows, col, w);
            } else {
#pragma unroll
              for (int i = 0; i < 4; ++i)
                if (rows[i] >= 0)
                  r2 += epilogue_row(p.ep, T.g, T.b, T.h, rows[i], col, &w[i].x, nvalid);
            }
          }
        }
        __syncwarp();  // this warp's reads of the drain buffer precede the next drain
        if (res0) {
          for (int o = 16; o > 0; o >>= 1) r2 += __shfl_xor_sync(0xffffffffu, r2, o);
          if (lane == 0) red[ew] = r2;
          asm volatile("bar.sync 1, %0;" ::"n"(32 * C::EPI_WARPS) : "memory");
          if (ew == 0 && lane == 0 && T.mt < tiles_m128) {
            double tsum = 0.0;
            for (int i = 0; i < C::EPI_WARPS; ++i) tsum += red[i];
            p.ep.cmb.norm_partials[p.ep.cmb.norm_base + T.z * p.ep.cmb.norm_member_stride +
                                   T.mt * tiles_n + T.nt] = tsum;
          }
          asm volatile("bar.sync 1, %0;" ::"n"(32 * C::EPI_WARPS) : "memory");
        }
        continue;
      }
      const Tile T = tile_of(t);
      const int acc = tc % NACC;
      const uint32_t aph = (tc / NACC) & 1;
      wait(&tfull[acc], aph);
      if (ew == 0 && lane == 0) flush(8);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t lane_addr =
          tmem_base + (uint32_t)(acc * 2 * TN) + ((uint32_t)(q * 32) << 16);
      double r2 = 0.0;
#pragma unroll 1
      for (int c = half * COLS; c < (half + 1) * COLS; c += 16) {
        // main and correction columns in flight together, one wait
        uint32_t rv[16], rw[16];
        tmem_ld16(lane_addr + c, rv);
        if (p.passes > 1) tmem_ld16(lane_addr + TN + c, rw);
        tmem_wait();
        if (c + 16 == (half + 1) * COLS) {
          // last TMEM read of this tile by this warp: once every epilogue
          // warp is here, the accumulator can take the next tile's MMAs
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          asm volatile("bar.sync 2, %0;" ::"n"(32 * C::EPI_WARPS) : "memory");
          if (ew == 0 && lane == 0) {
            if (leader)
              mbar_arrive(&tempty[acc]);
            else
              mbar_arrive_cluster(tempty_leader + acc * 8);
          }
        }
        if constexpr (CG == 1) {
          // small problems (attention, per-layer): lane = row, 16 columns
          float v[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float mv = __uint_as_float(rv[i]);
            v[i] = p.passes > 1 ? fmaf(__uint_as_float(rw[i]), kLoInv, mv) : mv;
          }
          const int row = T.m0 + q * 32 + lane;
          const int col0 = T.n0 + c;
          const int nvalid = min(16, p.N - col0);
          if (row < p.M && nvalid > 0 && !(p.debug & 2))
            r2 += (nvalid == 16 && p.vec_ok)
                      ? epilogue_rowv<16>(p.ep, T.g, T.b, T.h, row, col0, v)
                      : epilogue_row(p.ep, T.g, T.b, T.h, row, col0, v, nvalid);
        } else {
          // lane = row: stage the 32 x 16 chunk in shared memory (16-byte
          // pieces XOR-swizzled by row pair: conflict-free both ways), then
          // read it back with 4 lanes per row so every global access of the
          // epilogue covers 64 contiguous bytes of a row
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            uint4 w4;
            float* f = reinterpret_cast<float*>(&w4);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float mv = __uint_as_float(rv[4 * cc + i]);
              f[i] = p.passes > 1 ? fmaf(__uint_as_float(rw[4 * cc + i]), kLoInv, mv) : mv;
            }
            sts128(ebuf + lane * 64 + ((cc ^ ((lane >> 1) & 3)) << 4), w4);
          }
          __syncwarp();
          const int col = T.n0 + c + (lane & 3) * 4;
          const int nvalid = min(4, p.N - col);
          float4 w[4];
          int rows[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int r = i * 8 + (lane >> 2), cc = lane & 3;
            w[i] = lds128(ebuf + r * 64 + ((cc ^ ((r >> 1) & 3)) << 4));
            const int row = T.m0 + q * 32 + r;
            rows[i] = (row < p.M && nvalid > 0) ? row : -1;
          }
          __syncwarp();
          if (!(p.debug & 2)) {
            if (nvalid == 4 && p.vec_ok) {
              r2 += epilogue_4x4(p.ep, T.g, T.b, T.h, rows, col, w);
            } else {
#pragma unroll
              for (int i = 0; i < 4; ++i)
                if (rows[i] >= 0) r2 += epilogue_row(p.ep, T.g, T.b, T.h, rows[i], col, &w[i].x, nvalid);
            }
          }
        }
      }
      if (res0) {
        // one partial per (128-row, TN-column) tile of this CTA
        for (int o = 16; o > 0; o >>= 1) r2 += __shfl_xor_sync(0xffffffffu, r2, o);
        if (lane == 0) red[acc * C::EPI_WARPS + ew] = r2;
        asm volatile("bar.sync 1, %0;" ::"n"(32 * C::EPI_WARPS) : "memory");
        if (ew == 0 && lane == 0 && T.mt < tiles_m128) {
          double tsum = 0.0;
          for (int i = 0; i < C::EPI_WARPS; ++i) tsum += red[acc * C::EPI_WARPS + i];
          p.ep.cmb.norm_partials[p.ep.cmb.norm_base + T.z * p.ep.cmb.norm_member_stride +
                                 T.mt * tiles_n + T.nt] = tsum;
        }
        if constexpr (NACC == 1)
          asm volatile("bar.sync 1, %0;" ::"n"(32 * C::EPI_WARPS) : "memory");
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (p.prof && threadIdx.x == 0) atomicAdd(&p.prof[9], (unsigned long long)(clock64() - t_start));
  if constexpr (CG == 2) cluster_sync();
  if (warp == 2) {
    if constexpr (CG == 1)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(512u));
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                   "r"(512u));
  }
}

// ---- pre-split operands (weights) --------------------------------------------------
// dst row r of slot g = for each 32-wide K block: 32 hi | 32 lo' fp16 values
// (K zero-padded to a multiple of 32); with `transpose`, B = src^T.
__global__ void pack_hl_kernel(const float* __restrict__ src, long long src_slot, int src_ld,
                               float* __restrict__ dst, long long dst_slot, int dst_ld, int G,
                               int rows, int K, int transpose, int vec, int* range_flag) {
  pdl_wait();
  pdl_trigger();
  const int kblocks = (K + BK - 1) / BK;
  const long long n = (long long)G * rows * kblocks * 4;  // 8-value chunks
  float amax = 0.f;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const int chunk = (int)(i % (kblocks * 4));
    const long long rg = i / (kblocks * 4);
    const int r = (int)(rg % rows);
    const int g = (int)(rg / rows);
    const int k0 = chunk * 8;
    float x[8];
    if (vec) {  // row-major source, 16-byte rows, K % 8 == 0
      const float4* p = reinterpret_cast<const float4*>(src + g * src_slot + (long long)r * src_ld + k0);
      const float4 u = p[0], v = p[1];
      x[0] = u.x; x[1] = u.y; x[2] = u.z; x[3] = u.w;
      x[4] = v.x; x[5] = v.y; x[6] = v.z; x[7] = v.w;
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int k = k0 + e;
        x[e] = k < K ? (transpose ? src[g * src_slot + (long long)k * src_ld + r]
                                  : src[g * src_slot + (long long)r * src_ld + k])
                     : 0.f;
      }
    }
    uint4 hi, lo;
    split8(x, hi, lo, amax);
    uint8_t* row = reinterpret_cast<uint8_t*>(dst + g * dst_slot + (long long)r * dst_ld) +
                   (chunk >> 2) * 128;
    *reinterpret_cast<uint4*>(row + (chunk & 3) * 16) = hi;
    *reinterpret_cast<uint4*>(row + 64 + (chunk & 3) * 16) = lo;
  }
  if (range_flag && amax >= 65520.f && amax <= FLT_MAX) atomicOr(range_flag, 1);
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
// row); dimension 0 is always the contiguous columns. Boxes are
// [box_rows][box_cols]: K-major tiles [128][32] with SWIZZLE_128B, MN-major
// staging tiles [32 K][128] dense.
CUtensorMap make_map(const Mat& m, int G, int Bb, int H, int rows, int cols, int box_rows,
                     int box_cols, bool swizzle, TcOperand* op) {
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
  cuuint32_t box[5] = {(cuuint32_t)box_cols, 1, 1, 1, 1};
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
                         swizzle ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    throw ContractViolation("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return map;
}

// host-side parameter block + tensor maps for one launch
struct Prepared {
  TcParams p;
  CUtensorMap mA, mB;
};

Prepared prepare(const GemmArgs& a) {
  Prepared P;
  TcParams& p = P.p;
  p.G = a.G;
  p.M = a.M;
  p.N = a.N;
  p.K = a.K;
  p.Bb = a.Bb;
  p.H = a.H;
  p.ep = a.ep;
  p.range_flag = a.range_flag;
  static const int passes = [] {
    const char* e = getenv("MGLP_DEBUG_SPLIT_PASSES");
    return e ? atoi(e) : 3;
  }();
  p.passes = passes;
  // ring depths for a pre-split B (12 slots): MGLP_GEMM_RINGS="a,h,b" overrides
  static const int* rings = [] {
    static int r[3] = {4, 4, 4};
    if (const char* e = getenv("MGLP_GEMM_RINGS")) {
      int a = 0, h = 0, b = 0;
      if (sscanf(e, "%d,%d,%d", &a, &h, &b) == 3 && a >= 1 && h >= 1 && b >= 1 && a <= MAXR &&
          h <= MAXR && b <= MAXR && a + h + b <= NSLOTS) {
        r[0] = a;
        r[1] = h;
        r[2] = b;
      }
    }
    return r;
  }();
  p.ring_a = rings[0];
  p.ring_h = rings[1];
  p.ring_b = rings[2];
  static const int debug = [] {
    const char* e = getenv("MGLP_DEBUG_GEMM");
    return e ? atoi(e) : 0;
  }();
  p.debug = debug;
  p.prof = nullptr;
  static unsigned long long* prof_buf = [] {
    unsigned long long* b = nullptr;
    if (getenv("MGLP_GEMM_PROF")) {
      if (cudaMalloc(&b, 16 * sizeof(unsigned long long)) != cudaSuccess) b = nullptr;
    }
    return b;
  }();
  p.prof = prof_buf;
  {
    auto al = [](const Mat& m) {
      return !m.ok() || ((reinterpret_cast<uintptr_t>(m.ptr) & 15) == 0 && m.ld % 4 == 0 &&
                         m.slot_stride % 4 == 0 && m.bstride % 4 == 0 && m.hstride % 4 == 0);
    };
    const EpiArgs& e = a.ep;
    const Combine& c = e.cmb;
    p.vec_ok = al(e.out1) && al(e.out2) && al(e.add1) && al(e.add2) && al(e.aux) && al(e.bias) &&
               al(c.z) && al(c.out) && al(c.base) && al(c.phib) && al(c.rho) && al(c.v) &&
               !e.drop.on();  // dropout sites use the scalar epilogue (common.cuh)
  }
  p.a_mn = a.a_mn;
  p.b_direct = a.Bhl.ok() ? 1 : 0;
  p.b_mn = p.b_direct ? 0 : a.b_mn;
  p.b_hl = (!p.b_direct && a.b_mn && a.b_mn_hl) ? 1 : 0;
  p.a_hl = (a.a_mn && a.a_mn_hl && !a.Ahl.ok()) ? 1 : 0;
  if (a.a_mn_hl && (!a.a_mn || a.M % 32))
    throw ContractViolation("gemm_tc: pre-split MN-major A needs an MN-major, 32-aligned A");
  if (a.b_mn_hl && (p.b_direct || !a.b_mn || a.N % 32))
    throw ContractViolation("gemm_tc: pre-split MN-major B needs an MN-major, 32-aligned B");
  p.a_direct = (a.Ahl.ok() && p.b_direct && !a.a_mn) ? 1 : 0;
  // A: [M][K] (K-major) or [K][M] (MN-major)
  if (p.a_direct) {
    const int kpa = ceil_div(a.K, BK) * BK;  // packed row: hi|lo per 32-wide K block
    P.mA = make_map(a.Ahl, a.G, a.Bb, a.H, a.M, kpa, ROWS, BK, true, &p.a);
  } else {
    P.mA = p.a_hl  ? make_map(a.A, a.G, a.Bb, a.H, a.K, a.M, BK, 32, true, &p.a)
           : a.a_mn ? make_map(a.A, a.G, a.Bb, a.H, a.K, a.M, BK, ROWS, false, &p.a)
                    : make_map(a.A, a.G, a.Bb, a.H, a.M, a.K, ROWS, BK, true, &p.a);
  }
  if (p.b_direct) {
    const int kp = ceil_div(a.K, BK) * BK;  // packed row: kp floats = kp hi + kp lo'
    P.mB = make_map(a.Bhl, a.G, a.Bb, a.H, a.N, kp, ROWS, BK, true, &p.b);
  } else {
    P.mB = p.b_hl  ? make_map(a.B, a.G, a.Bb, a.H, a.K, a.N, BK, 32, true, &p.b)
           : a.b_mn ? make_map(a.B, a.G, a.Bb, a.H, a.K, a.N, BK, ROWS, false, &p.b)
                    : make_map(a.B, a.G, a.Bb, a.H, a.N, a.K, ROWS, BK, true, &p.b);
  }
  return P;
}

int num_sms() {
  static int sms = 0;
  if (!sms) MGLP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  return sms;
}

template <int CG, int DR>
void launch_cg(const GemmArgs& a, const int* active, cudaStream_t s, Prepared& P) {
  using C = Cfg<CG>;
  constexpr int SMEM = smem_bytes<DR>();
  static bool attr = [] {
    MGLP_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<CG, DR>,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
    return true;
  }();
  (void)attr;
  const long long tiles =
      (long long)ceil_div(a.N, C::TN) * ceil_div(a.M, C::TM) * a.G * a.Bb * a.H;
  const int units = (int)std::min<long long>(tiles, num_sms() / CG);
  // CG = 2: one cluster of two CTAs per unit
  launch_k(gemm_tc_kernel<CG, DR>, dim3(CG * units), dim3(C::THREADS), SMEM, s, CG, P.mA, P.mB,
           P.p, active);
  MGLP_CUDA(cudaGetLastError());
  if (P.p.prof) {
    // diagnostics: average cycles per CTA spent in each wait kind
    unsigned long long h[16];
    MGLP_CUDA(cudaDeviceSynchronize());
    MGLP_CUDA(cudaMemcpy(h, P.p.prof, sizeof(h), cudaMemcpyDeviceToHost));
    MGLP_CUDA(cudaMemset(P.p.prof, 0, sizeof(h)));
    const double n = (double)(CG * units);
    static const char* names[10] = {"prodA.sfree", "prodB.emptyB", "signal.cdone", "mma.tempty",
                                    "mma.conv",    "cvt.fullA",    "cvt.empty",    "cvt.fullB",
                                    "epi.tfull",   "total"};
    fprintf(stderr, "[gemm_prof CG=%d M=%d N=%d K=%d G=%d]", CG, a.M, a.N, a.K, a.G);
    for (int i = 0; i < 10; ++i) fprintf(stderr, " %s=%.0f", names[i], h[i] / n);
    fprintf(stderr, "\n");
  }
}

// the CTA-pair kernel needs at least a full 256 x 256 tile to pay off; the
// choice depends only on (M, N), so a given layer GEMM always runs the same
// kernel (bitwise determinism of Phi does not depend on the family size)
bool use_pair(const GemmArgs& a) {
  // MGLP_GEMM_NO_PAIR: bitmask over EpiKind (bit k: epilogue kind k stays on
  // the 1-CTA kernel, whose double-buffered TMEM overlaps the epilogue)
  static const int off = [] {
    const char* e = getenv("MGLP_GEMM_NO_PAIR");
    return e ? (int)strtol(e, nullptr, 0) : 0;
  }();
  return !((off >> a.ep.kind) & 1) && a.M >= 256 && a.N >= 256;
}

}  // namespace

CUtensorMap tc_make_map(const Mat& m, int G, int Bb, int H, int rows, int cols, int box_rows,
                        int box_cols, bool swizzle, TcOperand* op) {
  return make_map(m, G, Bb, H, rows, cols, box_rows, box_cols, swizzle, op);
}

int gemm_tc_blocks(const GemmArgs& a) {
  // residual-norm partial slots: one per (128-row, column-tile) of each problem
  const int tn = use_pair(a) ? Cfg<2>::TN : Cfg<1>::TN;
  return ceil_div(a.N, tn) * ceil_div(a.M, 128) * a.G * a.Bb * a.H;
}

void launch_gemm_tc(const GemmArgs& a, const int* active, cudaStream_t s) {
  if (a.G == 0 || a.M == 0 || a.N == 0) return;
  if (a.K == 0) throw ContractViolation("gemm_tc: K must be positive");
  Prepared P = prepare(a);
  // MGLP_GEMM_DRAIN=0: the pair kernel releases TMEM only after its epilogue;
  // 1: drain converter-free launches with K <= 1024 only; 2: every
  // converter-free launch; 3 (default): K <= 1024, and long K when the
  // epilogue is the MGRIT combine (EPI_FINAL)
  static const int drain = [] {
    const char* e = getenv("MGLP_GEMM_DRAIN");
    return e ? atoi(e) : 3;
  }();
  if (use_pair(a)) {
    // measured (tools/gpu_drain_diag.sh, same box): draining wins where the
    // epilogue is large against the K loop (K = 768: MLP-in, QKV) and for the
    // MGRIT-combine epilogue at K = 3072 (MLP-out family 14.8 -> 13.6 ms per
    // BERT step); the full-depth rings win for the other long-K shapes
    // (MLP-in dgrad K = 3072: 12.4 vs 12.9 ms)
    const bool long_k_ok = drain == 2 || (drain == 3 && a.ep.kind == EPI_FINAL);
    if (drain && P.p.a_direct && (a.K <= 1024 || long_k_ok))
      launch_cg<2, 1>(a, active, s, P);
    else
      launch_cg<2, 0>(a, active, s, P);
  } else {
    launch_cg<1, 0>(a, active, s, P);
  }
}

long long pack_hl_cols(int K) { return (long long)ceil_div(K, BK) * BK; }

void launch_pack_hl(const float* src, long long src_slot, int src_ld, float* dst,
                    long long dst_slot, int dst_ld, int G, int rows, int K, bool transpose,
                    cudaStream_t s, int* range_flag) {
  if (G == 0 || rows == 0 || K == 0) return;
  if (dst_ld < pack_hl_cols(K) || (dst_ld % 4) || (reinterpret_cast<uintptr_t>(dst) & 15))
    throw ContractViolation("pack_hl: destination rows must hold pad32(K) 16-byte aligned floats");
  const long long n = (long long)G * rows * ceil_div(K, BK) * 4;
  const int blocks = (int)std::min<long long>(148 * 16, (n + 255) / 256);
  const bool vec = !transpose && K % 32 == 0 && src_ld % 4 == 0 && src_slot % 4 == 0 &&
                   (reinterpret_cast<uintptr_t>(src) & 15) == 0;
  launch_k(pack_hl_kernel, dim3(blocks), dim3(256), 0, s, 1, src, src_slot, src_ld, dst, dst_slot, dst_ld, G, rows, K,
                                        transpose ? 1 : 0, vec ? 1 : 0, range_flag);
  MGLP_CUDA(cudaGetLastError());
}

}  // namespace mglp
