// Shared device/host types for the MGRIT hot path on sm_100a.
//
// Every kernel works on a *family* of G independent problems launched at once
// (the coarse intervals of one relaxation sweep, the layers of the parameter
// pass, ...). Member g of a family lives at an affine slot index
// slot0 + g * step of a strided buffer (a state array, an activation arena,
// the per-layer parameter slab), which is what `Mat` describes. This is the
// B200 replacement for the reference's per-chunk Executor tasks
// (executor.cpp:75-110, mgrit.hpp:125-187): one launch covers every chunk.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace mglp {

// Error taxonomy of the reference (errors.hpp:25-35): ValidationError is a
// user-input problem (C-ABI status 1), ContractViolation a broken invariant
// (status 2).
struct ValidationError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ContractViolation : std::logic_error {
  using std::logic_error::logic_error;
};

#define MGLP_CUDA(x)                                                            \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess)                                                      \
      throw ::mglp::ContractViolation(std::string("CUDA error: ") +             \
                                      cudaGetErrorString(e_) + " at " +         \
                                      __FILE__ + ":" + std::to_string(__LINE__)); \
  } while (0)

// ---- programmatic dependent launch (PDL) ------------------------------------
// Every kernel of the solver stream starts with pdl_wait() (returns once the
// preceding kernel has completed and its writes are visible; a no-op for a
// normal launch) and is launched by launch_k with the programmatic
// stream-serialisation attribute, so the next kernel's launch overlaps this
// one's execution, also inside the captured graph: the serial layer chain
// (device serial fwd+bwd) runs 4% faster, the MGRIT step is unchanged.
// pdl_trigger() (an early griddepcontrol.launch_dependents, so dependents are
// scheduled while the last wave drains) measured 1-3% slower on the MGRIT
// step and is compiled in only with -DMGLP_PDL_EARLY_TRIGGER.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
#ifdef MGLP_PDL_EARLY_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;");
#endif
}

bool pdl_on();  // MGLP_NO_PDL=1 disables (rowops.cu)

template <typename... KArgs, typename... Args>
inline void launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     int cluster_x, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  unsigned n = 0;
  if (cluster_x > 1) {
    at[n].id = cudaLaunchAttributeClusterDimension;
    at[n].val.clusterDim.x = (unsigned)cluster_x;
    at[n].val.clusterDim.y = 1;
    at[n].val.clusterDim.z = 1;
    ++n;
  }
  if (pdl_on()) {
    at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  cfg.attrs = at;
  cfg.numAttrs = n;
  MGLP_CUDA(cudaLaunchKernelEx(&cfg, k, args...));
}

// A strided family of row-major fp32 matrices. Member g starts at
// ptr + (slot0 + g*step) * slot_stride; rows are ld elements apart.
struct Mat {
  float* ptr = nullptr;
  long long slot_stride = 0;  // elements between consecutive slots
  int ld = 0;                 // row stride (elements)
  int slot0 = 0;
  int step = 1;
  // optional (batch, head) sub-blocks of a slot, for per-(b,h) attention GEMMs
  long long bstride = 0, hstride = 0;
  __host__ __device__ __forceinline__ float* at(int g) const {
    return ptr + (long long)(slot0 + g * step) * slot_stride;
  }
  __host__ __device__ __forceinline__ float* at(int g, int b, int h) const {
    return ptr + (long long)(slot0 + g * step) * slot_stride + b * bstride + h * hstride;
  }
  __host__ __device__ __forceinline__ bool ok() const { return ptr != nullptr; }
  __host__ Mat slot(int s0, int st) const {
    Mat m = *this;
    m.slot0 = s0;
    m.step = st;
    return m;
  }
  __host__ Mat offset(long long elems) const {
    Mat m = *this;
    m.ptr += elems;
    return m;
  }
};

// How the propagated value p = z + dt*F of one evaluation is folded into the
// solver state -- the four update forms of mgrit.hpp:
//   PLAIN : v[j] = p                                   (relax_update, level 0; 273-277)
//   FAS   : v[j] = base[j] + ((p - phib[j]) + rho[j])  (relax_update, level>0; 279-280)
//   RES0  : r[j] = p - v[j], plus sum r^2              (residual_rows, level 0; 177)
//   RESL  : r[j] = ((p - phib[j]) + rho[j]) - (v[j] - base[j])   (179-180)
//   NONE  : value discarded (linearization-only evaluation)
enum CombineMode : int { CM_PLAIN = 0, CM_FAS = 1, CM_RES0 = 2, CM_RESL = 3, CM_NONE = 4 };

struct Combine {
  int mode = CM_NONE;
  float dt = 0.f;
  Mat z;  // the state the step starts from (p = z + dt*F)
  Mat out, base, phib, rho, v;
  double* norm_partials = nullptr;  // RES0: one f64 partial per CTA, fixed order
  int norm_base = 0;                // slot of member 0's first CTA
  int norm_member_stride = 0;       // slots between consecutive members
};

__device__ __forceinline__ float combine_apply(const Combine& c, int g, long long off_out,
                                               long long off_z, float F, double& r2) {
  const float p = c.z.at(g)[off_z] + c.dt * F;
  switch (c.mode) {
    case CM_PLAIN:
      c.out.at(g)[off_out] = p;
      break;
    case CM_FAS: {
      const float corr = (p - c.phib.at(g)[off_out]) + c.rho.at(g)[off_out];
      c.out.at(g)[off_out] = c.base.at(g)[off_out] + corr;
    } break;
    case CM_RES0: {
      const float r = p - c.v.at(g)[off_out];
      c.out.at(g)[off_out] = r;
      r2 += (double)r * (double)r;
    } break;
    case CM_RESL: {
      const float lhs = (p - c.phib.at(g)[off_out]) + c.rho.at(g)[off_out];
      const float r = lhs - (c.v.at(g)[off_out] - c.base.at(g)[off_out]);
      c.out.at(g)[off_out] = r;
    } break;
    default:
      break;
  }
  return p;
}

// combine_apply over 4 consecutive elements (16-byte aligned rows): same
// per-element arithmetic, r^2 accumulated in element order
__device__ __forceinline__ float4 combine_apply4(const Combine& c, int g, long long off_out,
                                                 long long off_z, float4 F, double& r2) {
  const float4 z = *reinterpret_cast<const float4*>(c.z.at(g) + off_z);
  float4 p = make_float4(z.x + c.dt * F.x, z.y + c.dt * F.y, z.z + c.dt * F.z, z.w + c.dt * F.w);
  float4 o = p;
  switch (c.mode) {
    case CM_PLAIN:
      break;
    case CM_FAS: {
      const float4 pb = *reinterpret_cast<const float4*>(c.phib.at(g) + off_out);
      const float4 rh = *reinterpret_cast<const float4*>(c.rho.at(g) + off_out);
      const float4 bs = *reinterpret_cast<const float4*>(c.base.at(g) + off_out);
      o.x = bs.x + ((p.x - pb.x) + rh.x);
      o.y = bs.y + ((p.y - pb.y) + rh.y);
      o.z = bs.z + ((p.z - pb.z) + rh.z);
      o.w = bs.w + ((p.w - pb.w) + rh.w);
    } break;
    case CM_RES0: {
      const float4 v = *reinterpret_cast<const float4*>(c.v.at(g) + off_out);
      o = make_float4(p.x - v.x, p.y - v.y, p.z - v.z, p.w - v.w);
      r2 += (double)o.x * (double)o.x;
      r2 += (double)o.y * (double)o.y;
      r2 += (double)o.z * (double)o.z;
      r2 += (double)o.w * (double)o.w;
    } break;
    case CM_RESL: {
      const float4 pb = *reinterpret_cast<const float4*>(c.phib.at(g) + off_out);
      const float4 rh = *reinterpret_cast<const float4*>(c.rho.at(g) + off_out);
      const float4 bs = *reinterpret_cast<const float4*>(c.base.at(g) + off_out);
      const float4 v = *reinterpret_cast<const float4*>(c.v.at(g) + off_out);
      o.x = ((p.x - pb.x) + rh.x) - (v.x - bs.x);
      o.y = ((p.y - pb.y) + rh.y) - (v.y - bs.y);
      o.z = ((p.z - pb.z) + rh.z) - (v.z - bs.z);
      o.w = ((p.w - pb.w) + rh.w) - (v.w - bs.w);
    } break;
    default:
      return p;
  }
  *reinterpret_cast<float4*>(c.out.at(g) + off_out) = o;
  return p;
}

// GEMM epilogues. acc is the fp32 accumulator of C = A.B^T (row `row`, column
// `col`); everything else is fused here so the activations of one layer are
// written exactly once (tensor.cpp:205-218 linear = x W^T + b, blocks.cpp:246-292).
enum EpiKind : int {
  EPI_STORE = 0,      // out1 = acc (+ bias)
  EPI_BIAS_ADD2 = 1,  // a = acc + bias; o1 = add1 ? add1 + a : a -> out1; out2 = add2 + o1
  EPI_BIAS_GELU = 2,  // h = acc + bias: gelu'(h) -> out1 (for the VJP), gelu(h) -> out2
  EPI_FINAL = 3,      // mo = acc + bias; F = add1 + mo; p = z + dt*F; combine
  EPI_GELU_BWD = 4,   // out1 = acc * aux, aux = gelu'(h)   (tensor.cpp:360-372)
  EPI_GRAD_ACC = 5,   // out1 += gscale * acc               (blocks.cpp:108, 126-129)
};

// ---- activations produced pre-split for the tensor-core GEMM ----------------
// Row layout of a hi|lo' buffer (GemmArgs::Ahl / Bhl, gemm_tc.cu): per 32-wide
// column block 128 bytes = 32 fp16 hi then 32 fp16 lo'. The split is
// bit-identical to the GEMM converters' (split8), so a GEMM reading it gives
// exactly the bits of reading the fp32 values. `row` points at the row start.
__device__ __forceinline__ void st_hl4(float* row, int col, float4 v, float& amax) {
  const __half2 h01 = __floats2half2_rn(v.x, v.y), h23 = __floats2half2_rn(v.z, v.w);
  const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
  const __half2 l01 = __floats2half2_rn((v.x - f01.x) * 2048.f, (v.y - f01.y) * 2048.f);
  const __half2 l23 = __floats2half2_rn((v.z - f23.x) * 2048.f, (v.w - f23.y) * 2048.f);
  amax = fmaxf(amax, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
  char* b = reinterpret_cast<char*>(row) + (col >> 5) * 128 + (col & 31) * 2;
  *reinterpret_cast<uint2*>(b) =
      make_uint2(*reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23));
  *reinterpret_cast<uint2*>(b + 64) =
      make_uint2(*reinterpret_cast<const uint32_t*>(&l01), *reinterpret_cast<const uint32_t*>(&l23));
}
__device__ __forceinline__ void st_hl1(float* row, int col, float v, float& amax) {
  const __half h = __float2half_rn(v);
  const __half l = __float2half_rn((v - __half2float(h)) * 2048.f);
  amax = fmaxf(amax, fabsf(v));
  __half* b = reinterpret_cast<__half*>(reinterpret_cast<char*>(row) + (col >> 5) * 128) + (col & 31);
  b[0] = h;
  b[32] = l;
}
// Head-split pre-split rows (attention operands Q, K, V, dO with dh = 64):
// every 64-column group (one head) is stored as 64 fp16 hi then 64 fp16 lo'
// (256 bytes, the size of its 64 fp32 values), so a [rows][64] box of each
// half lands by TMA directly as the attention kernels' SWIZZLE_128B hi / lo'
// tiles (attn_common.cuh).
__device__ __forceinline__ void st_hs4(float* row, int col, float4 v, float& amax) {
  const __half2 h01 = __floats2half2_rn(v.x, v.y), h23 = __floats2half2_rn(v.z, v.w);
  const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
  const __half2 l01 = __floats2half2_rn((v.x - f01.x) * 2048.f, (v.y - f01.y) * 2048.f);
  const __half2 l23 = __floats2half2_rn((v.z - f23.x) * 2048.f, (v.w - f23.y) * 2048.f);
  amax = fmaxf(amax, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
  char* b = reinterpret_cast<char*>(row) + (col >> 6) * 256 + (col & 63) * 2;
  *reinterpret_cast<uint2*>(b) =
      make_uint2(*reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23));
  *reinterpret_cast<uint2*>(b + 128) =
      make_uint2(*reinterpret_cast<const uint32_t*>(&l01), *reinterpret_cast<const uint32_t*>(&l23));
}
__device__ __forceinline__ void st_hs1(float* row, int col, float v, float& amax) {
  const __half h = __float2half_rn(v);
  const __half l = __float2half_rn((v - __half2float(h)) * 2048.f);
  amax = fmaxf(amax, fabsf(v));
  __half* b = reinterpret_cast<__half*>(reinterpret_cast<char*>(row) + (col >> 6) * 256) + (col & 63);
  b[0] = h;
  b[64] = l;
}
// a finite value beyond the fp16 split range (the GEMM converters' flag)
__device__ __forceinline__ void hl_range_check(float amax, int* flag) {
  if (flag && amax >= 65520.f && amax <= 3.402823466e38f) atomicOr(flag, 1);
}

// Frozen dropout masks (blocks.cpp:576-599) as generated by
// Engine::refresh_dropout: one byte per element (1 = keep) of every (layer,
// site) [B, s, d] tensor, value 1/keep where kept. The member g of a family
// uses block (layer0 + g*step) * 3 + site; element index = row * cols + col.
struct DropMask {
  const unsigned char* m = nullptr;  // [total layers][3][slot]; null = no dropout
  long long slot = 0;                // elements per (layer, site) block
  int layer0 = 0, step = 1, site = 0;
  int cols = 0;
  float scale = 1.f;  // 1 / keep
  __host__ __device__ bool on() const { return m != nullptr; }
  __device__ __forceinline__ const unsigned char* at(int g, long long row) const {
    return m + ((long long)(layer0 + g * step) * 3 + site) * slot + row * cols;
  }
};

__device__ __forceinline__ float drop_val(const DropMask& m, int g, long long row, int col) {
  return m.at(g, row)[col] ? m.scale : 0.f;
}
struct EpiArgs {
  int kind = EPI_STORE;
  Mat out1, out2, add1, add2, aux;
  Mat bias;  // bias vector family (slot = layer); null => no bias
  float gscale = 1.f;
  // EPI_GRAD_ACC, optional: the effective scale is gscale * *gscale_mul (the
  // adjoint's exact 2^-k, LamScale::down, read on the device)
  const float* gscale_mul = nullptr;
  float alpha = 1.f;  // EPI_STORE: out1 = alpha*acc (+ bias)
  // EPI_STORE: out1 is written in the head-split pre-split form (st_hs4; the
  // fused attention's Q, K, V / dO operands), range-checked into range_flag
  int hs = 0;
  Combine cmb;  // EPI_FINAL
  // EPI_BIAS_GELU: gelu(h) also (or only) as a pre-split hi|lo' buffer for
  // the next GEMM's A operand (see st_hl4); range_flag for its split
  Mat hl2;
  int* range_flag = nullptr;
  // EPI_BIAS_ADD2 / EPI_FINAL: the projection output (acc + bias) is a
  // dropout site (attention output phi1 / phi3, MLP output phi2). Applied by
  // the scalar epilogue_row only: a GEMM with an active mask takes that path
  // (gemm_tc.cu clears vec_ok), so the vectorised epilogues keep their
  // register budget.
  DropMask drop;
};

constexpr float kGeluC = 0.7978845608028654f;  // tensor.cpp:345
constexpr float kGeluA = 0.044715f;            // tensor.cpp:346

// tanh-GELU (tensor.cpp:345-372) through the logistic form
//   0.5 (1 + tanh(u)) = s = 1 / (1 + exp(-2u)),   gelu(v) = v s,
//   gelu'(v) = s + 2 v s (1 - s) c (1 + 3 a v^2),  u = c (v + a v^3):
// one exp and one reciprocal per element (few-ulp accurate; exp(-2u) -> inf
// gives s = 0, the exact limit).
__device__ __forceinline__ float gelu_s(float v) {
  const float u = kGeluC * fmaf(kGeluA * v * v, v, v);
  // exp(-2u) = 2^(-2u log2 e) on the SFU (ex2.approx: ~2 ulp, plus the
  // rounding of the scaled argument; s = 1/(1+e) stays within ~1e-6 relative)
  float e;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(u * -2.8853900817779268f));
  return __fdividef(1.f, 1.f + e);  // 1 + e >= 1: the fast reciprocal is exact to 2 ulp
}

__device__ __forceinline__ float gelu_f(float v) { return v * gelu_s(v); }

// gelu'(v) given s = gelu_s(v); the backward multiplies it into the upstream
// (up * gelu'(v), tensor.cpp:360-372), so storing gelu'(v) in the forward
// instead of v gives the bitwise-same VJP
__device__ __forceinline__ float gelu_deriv_s(float v, float s) {
  const float ds = 2.f * s * (1.f - s) * kGeluC * fmaf(3.f * kGeluA * v, v, 1.f);
  return fmaf(v, ds, s);
}
__device__ __forceinline__ float gelu_grad_f(float v, float up) { return up * gelu_deriv_s(v, gelu_s(v)); }

// Applies the epilogue to n consecutive columns [col0, col0+n) of one output
// row. Returns this row-segment's contribution to the residual norm^2.
__device__ __forceinline__ double epilogue_row(const EpiArgs& e, int g, int b, int h, int row,
                                               int col0, const float* acc, int n);

// W (a multiple of 4) full columns: the same epilogue through 128-bit
// loads/stores (W = 4: one float4 per thread, lanes along a row)
template <int W>
__device__ __forceinline__ double epilogue_rowv(const EpiArgs& e, int g, int b, int h, int row,
                                                int col0, const float* acc) {
  double r2 = 0.0;
  const float* bias = e.bias.ok() ? e.bias.at(g) + col0 : nullptr;
  float bv[W];
#pragma unroll
  for (int i = 0; i < W; i += 4) {
    if (bias) {
      const float4 t = *reinterpret_cast<const float4*>(bias + i);
      bv[i] = t.x; bv[i + 1] = t.y; bv[i + 2] = t.z; bv[i + 3] = t.w;
    } else {
      bv[i] = bv[i + 1] = bv[i + 2] = bv[i + 3] = 0.f;
    }
  }
  auto ld4 = [](const float* p, float* v) {
#pragma unroll
    for (int i = 0; i < W; i += 4) {
      const float4 t = *reinterpret_cast<const float4*>(p + i);
      v[i] = t.x; v[i + 1] = t.y; v[i + 2] = t.z; v[i + 3] = t.w;
    }
  };
  auto st4 = [](float* p, const float* v) {
#pragma unroll
    for (int i = 0; i < W; i += 4)
      *reinterpret_cast<float4*>(p + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
  };
  float o[W], t1[W];
  switch (e.kind) {
    case EPI_STORE: {
#pragma unroll
      for (int i = 0; i < W; ++i) o[i] = bias ? e.alpha * acc[i] + bv[i] : e.alpha * acc[i];
      if (e.hs) {
        float amax = 0.f;
        float* hr = e.out1.at(g, b, h) + (long long)row * e.out1.ld;
#pragma unroll
        for (int i = 0; i < W; i += 4)
          st_hs4(hr, col0 + i, make_float4(o[i], o[i + 1], o[i + 2], o[i + 3]), amax);
        hl_range_check(amax, e.range_flag);
      } else {
        st4(e.out1.at(g, b, h) + (long long)row * e.out1.ld + col0, o);
      }
    } break;
    case EPI_BIAS_ADD2: {
      float a2[W];
      ld4(e.add2.at(g) + (long long)row * e.add2.ld + col0, a2);
      if (e.add1.ok()) ld4(e.add1.at(g) + (long long)row * e.add1.ld + col0, t1);
#pragma unroll
      for (int i = 0; i < W; ++i) {
        const float a = acc[i] + bv[i];
        o[i] = e.add1.ok() ? t1[i] + a : a;
        t1[i] = a2[i] + o[i];
      }
      if (e.out1.ok()) st4(e.out1.at(g) + (long long)row * e.out1.ld + col0, o);
      if (e.out2.ok()) st4(e.out2.at(g) + (long long)row * e.out2.ld + col0, t1);
    } break;
    case EPI_BIAS_GELU: {
#pragma unroll
      for (int i = 0; i < W; ++i) {
        const float hv = acc[i] + bv[i], sv = gelu_s(hv);
        t1[i] = hv * sv;
        o[i] = gelu_deriv_s(hv, sv);
      }
      if (e.out1.ok()) st4(e.out1.at(g) + (long long)row * e.out1.ld + col0, o);
      if (e.out2.ok()) st4(e.out2.at(g) + (long long)row * e.out2.ld + col0, t1);
      if (e.hl2.ok()) {
        float amax = 0.f;
        float* hr = e.hl2.at(g) + (long long)row * e.hl2.ld;
#pragma unroll
        for (int i = 0; i < W; i += 4)
          st_hl4(hr, col0 + i, make_float4(t1[i], t1[i + 1], t1[i + 2], t1[i + 3]), amax);
        hl_range_check(amax, e.range_flag);
      }
    } break;
    case EPI_GELU_BWD: {
      ld4(e.aux.at(g) + (long long)row * e.aux.ld + col0, t1);
#pragma unroll
      for (int i = 0; i < W; ++i) o[i] = acc[i] * t1[i];
      if (e.out1.ok()) st4(e.out1.at(g) + (long long)row * e.out1.ld + col0, o);
      if (e.hl2.ok()) {
        float amax = 0.f;
        float* hr = e.hl2.at(g) + (long long)row * e.hl2.ld;
#pragma unroll
        for (int i = 0; i < W; i += 4)
          st_hl4(hr, col0 + i, make_float4(o[i], o[i + 1], o[i + 2], o[i + 3]), amax);
        hl_range_check(amax, e.range_flag);
      }
    } break;
    case EPI_GRAD_ACC: {
      float* p = e.out1.at(g) + (long long)row * e.out1.ld + col0;
      ld4(p, t1);
      const float gs = e.gscale_mul ? e.gscale * *e.gscale_mul : e.gscale;
#pragma unroll
      for (int i = 0; i < W; ++i) o[i] = t1[i] + gs * acc[i];
      st4(p, o);
    } break;
    default:
      return epilogue_row(e, g, b, h, row, col0, acc, W);
  }
  return r2;
}

// Four rows x 4 columns (one float4 per row; rows[i] < 0 = invalid): every
// global operand of the four rows is loaded first, then the math, then the
// stores -- four independent row segments in flight per thread, so a
// latency-bound epilogue (operands read from HBM) overlaps its loads.
// Requires 16-byte aligned rows for every operand (TcParams::vec_ok).
__device__ __forceinline__ float4 ld4g(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4g(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }
__device__ __forceinline__ const float* rowp(const Mat& m, int g, long long row, int col) {
  return m.at(g) + row * m.ld + col;
}

__device__ __forceinline__ double epilogue_4x4(const EpiArgs& e, int g, int b, int h,
                                               const int* rows, int col, const float4* acc) {
  double r2 = 0.0;
  float4 bv = make_float4(0.f, 0.f, 0.f, 0.f);
  if (e.bias.ok()) bv = ld4g(e.bias.at(g) + col);
  auto add = [](float4 a, float4 c) {
    return make_float4(a.x + c.x, a.y + c.y, a.z + c.z, a.w + c.w);
  };
  float4 x1[4], x2[4];
  switch (e.kind) {
    case EPI_STORE: {
      const float al = e.alpha;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (rows[i] < 0) continue;
        const float4 a = acc[i];
        float4 o = make_float4(al * a.x, al * a.y, al * a.z, al * a.w);
        if (e.bias.ok()) o = add(o, bv);
        if (e.hs) {
          float amax = 0.f;
          st_hs4(e.out1.at(g, b, h) + (long long)rows[i] * e.out1.ld, col, o, amax);
          hl_range_check(amax, e.range_flag);
        } else {
          st4g(e.out1.at(g, b, h) + (long long)rows[i] * e.out1.ld + col, o);
        }
      }
    } break;
    case EPI_BIAS_ADD2: {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (rows[i] < 0) continue;
        x2[i] = ld4g(rowp(e.add2, g, rows[i], col));
        if (e.add1.ok()) x1[i] = ld4g(rowp(e.add1, g, rows[i], col));
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (rows[i] < 0) continue;
        const float4 a = add(acc[i], bv);
        const float4 o1 = e.add1.ok() ? add(x1[i], a) : a;
        if (e.out1.ok()) st4g(e.out1.at(g) + (long long)rows[i] * e.out1.ld + col, o1);
        if (e.out2.ok()) st4g(e.out2.at(g) + (long long)rows[i] * e.out2.ld + col, add(x2[i], o1));
      }
    } break;
    case EPI_BIAS_GELU: {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (rows[i] < 0) continue;
        const float4 hv = add(acc[i], bv);
        const float4 sv = make_float4(gelu_s(hv.x), gelu_s(hv.y), gelu_s(hv.z), gelu_s(hv.w));
        if (e.out1.ok())
          st4g(e.out1.at(g) + (long long)rows[i] * e.out1.ld + col,
               make_float4(gelu_deriv_s(hv.x, sv.x), gelu_deriv_s(hv.y, sv.y),
                           gelu_deriv_s(hv.z, sv.z), gelu_deriv_s(hv.w, sv.w)));
        const float4 gv = make_float4(hv.x * sv.x, hv.y * sv.y, hv.z * sv.z, hv.w * sv.w);
        if (e.out2.ok()) st4g(e.out2.at(g) + (long long)rows[i] * e.out2.ld + col, gv);
        if (e.hl2.ok()) {
          float amax = 0.f;
          st_hl4(e.hl2.at(g) + (long long)rows[i] * e.hl2.ld, col, gv, amax);
          hl_range_check(amax, e.range_flag);
        }
      }
    } break;
    case EPI_GELU_BWD: {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (rows[i] >= 0) x1[i] = ld4g(rowp(e.aux, g, rows[i], col));
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (rows[i] < 0) continue;
        const float4 a = acc[i], v = x1[i];
        const float4 dv = make_float4(a.x * v.x, a.y * v.y, a.z * v.z, a.w * v.w);
        if (e.out1.ok()) st4g(e.out1.at(g) + (long long)rows[i] * e.out1.ld + col, dv);
        if (e.hl2.ok()) {
          float amax = 0.f;
          st_hl4(e.hl2.at(g) + (long long)rows[i] * e.hl2.ld, col, dv, amax);
          hl_range_check(amax, e.range_flag);
        }
      }
    } break;
    case EPI_GRAD_ACC: {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (rows[i] >= 0) x1[i] = ld4g(rowp(e.out1, g, rows[i], col));
      const float gs = e.gscale_mul ? e.gscale * *e.gscale_mul : e.gscale;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (rows[i] < 0) continue;
        const float4 a = acc[i], o = x1[i];
        st4g(e.out1.at(g) + (long long)rows[i] * e.out1.ld + col,
             make_float4(o.x + gs * a.x, o.y + gs * a.y, o.z + gs * a.z, o.w + gs * a.w));
      }
    } break;
    case EPI_FINAL: {
      // one row at a time, its (up to five) operands loaded together
      const Combine& c = e.cmb;
      const bool fas = c.mode == CM_FAS, res0 = c.mode == CM_RES0, resl = c.mode == CM_RESL;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if (rows[i] < 0) continue;
        const float4 a1v = ld4g(rowp(e.add1, g, rows[i], col));
        const float4 zv = ld4g(rowp(c.z, g, rows[i], col));
        float4 pb = make_float4(0.f, 0.f, 0.f, 0.f), rh = pb, bs = pb, vv = pb;
        if (fas || resl) {
          pb = ld4g(rowp(c.phib, g, rows[i], col));
          rh = ld4g(rowp(c.rho, g, rows[i], col));
          bs = ld4g(rowp(c.base, g, rows[i], col));
        }
        if (res0 || resl) vv = ld4g(rowp(c.v, g, rows[i], col));
        const float* a = &acc[i].x;
        float o[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float mo = e.bias.ok() ? a[k] + (&bv.x)[k] : a[k];
          const float F = (&a1v.x)[k] + mo;
          const float p = (&zv.x)[k] + c.dt * F;
          if (fas) {
            const float corr = (p - (&pb.x)[k]) + (&rh.x)[k];
            o[k] = (&bs.x)[k] + corr;
          } else if (res0) {
            const float r = p - (&vv.x)[k];
            o[k] = r;
            r2 += (double)r * (double)r;
          } else if (resl) {
            const float lhs = (p - (&pb.x)[k]) + (&rh.x)[k];
            o[k] = lhs - ((&vv.x)[k] - (&bs.x)[k]);
          } else {
            o[k] = p;
          }
        }
        if (c.mode != CM_NONE)
          st4g(c.out.at(g) + (long long)rows[i] * c.out.ld + col,
               make_float4(o[0], o[1], o[2], o[3]));
      }
    } break;
  }
  return r2;
}

__device__ __forceinline__ double epilogue_row(const EpiArgs& e, int g, int b, int h, int row,
                                               int col0, const float* acc, int n) {
  double r2 = 0.0;
  const float* bias = e.bias.ok() ? e.bias.at(g) : nullptr;
  switch (e.kind) {
    case EPI_STORE: {
      const float al = e.alpha;
      if (e.hs) {
        float* hr = e.out1.at(g, b, h) + (long long)row * e.out1.ld;
        float amax = 0.f;
        for (int i = 0; i < n; ++i)
          st_hs1(hr, col0 + i, bias ? al * acc[i] + bias[col0 + i] : al * acc[i], amax);
        hl_range_check(amax, e.range_flag);
        break;
      }
      float* o = e.out1.at(g, b, h) + (long long)row * e.out1.ld + col0;
      for (int i = 0; i < n; ++i) o[i] = bias ? al * acc[i] + bias[col0 + i] : al * acc[i];
    } break;
    case EPI_BIAS_ADD2: {
      float* o1 = e.out1.ok() ? e.out1.at(g) + (long long)row * e.out1.ld + col0 : nullptr;
      float* o2 = e.out2.ok() ? e.out2.at(g) + (long long)row * e.out2.ld + col0 : nullptr;
      const float* a1 = e.add1.ok() ? e.add1.at(g) + (long long)row * e.add1.ld + col0 : nullptr;
      const float* a2 = e.add2.at(g) + (long long)row * e.add2.ld + col0;
      for (int i = 0; i < n; ++i) {
        float a = bias ? acc[i] + bias[col0 + i] : acc[i];
        if (e.drop.on()) a *= drop_val(e.drop, g, row, col0 + i);
        const float v1 = a1 ? a1[i] + a : a;
        if (o1) o1[i] = v1;
        if (o2) o2[i] = a2[i] + v1;
      }
    } break;
    case EPI_BIAS_GELU: {
      float* o1 = e.out1.ok() ? e.out1.at(g) + (long long)row * e.out1.ld + col0 : nullptr;
      float* o2 = e.out2.ok() ? e.out2.at(g) + (long long)row * e.out2.ld + col0 : nullptr;
      float* hr = e.hl2.ok() ? e.hl2.at(g) + (long long)row * e.hl2.ld : nullptr;
      float amax = 0.f;
      for (int i = 0; i < n; ++i) {
        const float hv = bias ? acc[i] + bias[col0 + i] : acc[i];
        const float sv = gelu_s(hv);
        if (o1) o1[i] = gelu_deriv_s(hv, sv);
        if (o2) o2[i] = hv * sv;
        if (hr) st_hl1(hr, col0 + i, hv * sv, amax);
      }
      if (hr) hl_range_check(amax, e.range_flag);
    } break;
    case EPI_FINAL: {
      const float* a1 = e.add1.at(g) + (long long)row * e.add1.ld + col0;
      const long long off_out = (long long)row * e.cmb.out.ld + col0;
      const long long off_z = (long long)row * e.cmb.z.ld + col0;
      for (int i = 0; i < n; ++i) {
        float mo = bias ? acc[i] + bias[col0 + i] : acc[i];
        if (e.drop.on()) mo *= drop_val(e.drop, g, row, col0 + i);
        const float F = a1[i] + mo;
        combine_apply(e.cmb, g, off_out + i, off_z + i, F, r2);
      }
    } break;
    case EPI_GELU_BWD: {
      float* o = e.out1.ok() ? e.out1.at(g) + (long long)row * e.out1.ld + col0 : nullptr;
      float* hr = e.hl2.ok() ? e.hl2.at(g) + (long long)row * e.hl2.ld : nullptr;
      const float* dv = e.aux.at(g) + (long long)row * e.aux.ld + col0;
      float amax = 0.f;
      for (int i = 0; i < n; ++i) {
        const float x = acc[i] * dv[i];
        if (o) o[i] = x;
        if (hr) st_hl1(hr, col0 + i, x, amax);
      }
      if (hr) hl_range_check(amax, e.range_flag);
    } break;
    case EPI_GRAD_ACC: {
      float* o = e.out1.at(g) + (long long)row * e.out1.ld + col0;
      const float gs = e.gscale_mul ? e.gscale * *e.gscale_mul : e.gscale;
      for (int i = 0; i < n; ++i) o[i] = o[i] + gs * acc[i];
    } break;
  }
  return r2;
}

// GEMM problem family: for g < G, C_g[M,N] = A_g . B_g^T with
//   A_g [M,K] row-major ("K-major") or, if a_mn, stored [K,M] ("MN-major");
//   B_g [N,K] row-major, or if b_mn stored [K,N].
// B may come pre-split into fp16 hi/lo' parts (weights); see gemm_tc.cu.
struct GemmArgs {
  int G = 1, M = 0, N = 0, K = 0;
  // each of the G members may itself be a Bb x H grid of per-(batch, head)
  // problems (attention); operands then use Mat::bstride / hstride
  int Bb = 1, H = 1;
  // A, B: fp32 operands, [M][K] / [N][K] (K-major) or [K][M] / [K][N] (MN-major).
  // Bhl (optional): B pre-split by launch_pack_hl into the fp16 hi|lo' form
  // the tensor-core kernel stages (always K-major, [N][pad32(K)] in float
  // units); when set, the tensor-core path reads it instead of B.
  Mat A, B, Bhl;
  // Ahl (optional, K-major A only, with a pre-split B): A produced in the same
  // hi|lo' form by the kernel that wrote it -- the mainloop runs converter-free
  Mat Ahl;
  bool a_mn = false, b_mn = false;
  // b_mn with B's rows already pre-split (hi|lo' rows of the same byte size,
  // e.g. the cached LN / GELU outputs the weight gradients read): the
  // converters only regroup the halves into the K-major tile, no split
  bool b_mn_hl = false;
  bool a_mn_hl = false;  // likewise for an MN-major A (the cached dgrad chain)
  EpiArgs ep;
  // set to 1 when a finite operand value overflows fp16 (|x| >= 65520)
  int* range_flag = nullptr;
};

inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

}  // namespace mglp
