// Row / element kernels of the hot path: LayerNorm forward and VJP
// (tensor.cpp:239-308), parameter column sums (tensor.cpp:232-235, 303-304),
// the MGRIT state algebra (mgrit.hpp:199-223, 273-282) and the per-cycle
// residual-norm bookkeeping (mgrit.hpp:189-193, 248-262).
//
// All are HBM-bound: one warp per row with the row held in registers, grids
// sized in multiples of the 148 SMs, no float atomics (every reduction runs
// in a fixed order, so results never depend on scheduling).
#include <cstdlib>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace mglp {

bool pdl_on() {
  static const bool on = [] {
    const char* e = getenv("MGLP_NO_PDL");
    return !(e && atoi(e) != 0);
  }();
  return on;
}


namespace {

constexpr int kRowsPerBlock = 8;  // 8 warps of 32 lanes

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double block_sum_f64(double v, double* smem) {
  // fixed-order: warp shuffle tree, then warp 0 over the warp partials
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if (l == 0) smem[w] = v;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
    t = l < nw ? smem[l] : 0.0;
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  return t;  // valid in thread 0
}

__device__ __forceinline__ bool stopped(const int* active) {
  return active != nullptr && *(volatile const int*)active == 0;
}

// ---- LayerNorm forward --------------------------------------------------------
template <int V>
__global__ void __launch_bounds__(256) ln_fwd_kernel(LnFwdArgs a, const int* active) {
  pdl_wait();
  pdl_trigger();
  if (stopped(active)) return;
  const int g = blockIdx.y;
  const int row = blockIdx.x * kRowsPerBlock + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= a.rows) return;
  const float* x = a.x.at(g) + (long long)row * a.x.ld;
  float v[V];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int j = lane + 32 * i;
    v[i] = j < a.d ? x[j] : 0.f;
    s += v[i];
  }
  const float inv_d = 1.f / (float)a.d;
  const float mean = warp_sum(s) * inv_d;
  float q = 0.f;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int j = lane + 32 * i;
    const float c = j < a.d ? v[i] - mean : 0.f;
    q += c * c;
  }
  const float var = warp_sum(q) * inv_d;
  const float rstd = 1.f / sqrtf(var + a.eps);
  const float* gain = a.gain.at(g);
  const float* bias = a.bias.at(g);
  float* o = a.out.ok() ? a.out.at(g) + (long long)row * a.out.ld : nullptr;
  float* hl = a.out_hl.ok() ? a.out_hl.at(g) + (long long)row * a.out_hl.ld : nullptr;
  float amax = 0.f;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int j = lane + 32 * i;
    if (j < a.d) {
      const float y = gain[j] * ((v[i] - mean) * rstd) + bias[j];
      if (o) o[j] = y;
      if (hl) st_hl1(hl, j, y, amax);
    }
  }
  if (hl) hl_range_check(amax, a.range_flag);
  if (lane == 0 && a.stats.ok()) {
    float* st = a.stats.at(g) + 2LL * row;
    st[0] = mean;
    st[1] = rstd;
  }
}

// ---- LayerNorm VJP (+ fused sums and solver combine) ----------------------------
template <int V>
__global__ void __launch_bounds__(256) ln_bwd_kernel(LnBwdArgs a, const int* active) {
  pdl_wait();
  pdl_trigger();
  __shared__ double red[32];
  if (stopped(active)) return;
  const int g = blockIdx.y;
  const int row = blockIdx.x * kRowsPerBlock + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  double r2 = 0.0;
  if (row < a.rows) {
    const float* x = a.x.at(g) + (long long)row * a.x.ld;
    const float* up = a.up.at(g) + (long long)row * a.up.ld;
    const float* gain = a.gain.at(g);
    const float mean = a.stats.at(g)[2LL * row];
    const float rstd = a.stats.at(g)[2LL * row + 1];
    float xh[V], dxh[V];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int j = lane + 32 * i;
      if (j < a.d) {
        xh[i] = (x[j] - mean) * rstd;
        dxh[i] = up[j] * gain[j];
      } else {
        xh[i] = 0.f;
        dxh[i] = 0.f;
      }
      s1 += dxh[i];
      s2 += dxh[i] * xh[i];
    }
    const float inv_d = 1.f / (float)a.d;
    const float m1 = warp_sum(s1) * inv_d;
    const float m2 = warp_sum(s2) * inv_d;
    const float* addA = a.addA.ok() ? a.addA.at(g) + (long long)row * a.addA.ld : nullptr;
    const float* addB = a.addB.ok() ? a.addB.at(g) + (long long)row * a.addB.ld : nullptr;
    float* o1 = a.out1.ok() ? a.out1.at(g) + (long long)row * a.out1.ld : nullptr;
    float* o2 = a.out2.ok() ? a.out2.at(g) + (long long)row * a.out2.ld : nullptr;
    float* h2 = a.out2_hl.ok() ? a.out2_hl.at(g) + (long long)row * a.out2_hl.ld : nullptr;
    float amax = 0.f;
    const bool comb = a.cmb.mode != CM_NONE;
    const long long off_out = comb ? (long long)row * a.cmb.out.ld : 0;
    const long long off_z = comb ? (long long)row * a.cmb.z.ld : 0;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int j = lane + 32 * i;
      if (j < a.d) {
        const float L = rstd * (dxh[i] - m1 - xh[i] * m2);
        const float v1 = addA ? addA[j] + L : L;
        if (o1) o1[j] = v1;
        if (o2 || h2) {
          const float w =
              a.drop2.on() ? (addB[j] + L) * drop_val(a.drop2, g, row, j) : addB[j] + L;
          if (o2) o2[j] = w;
          if (h2) st_hl1(h2, j, w, amax);
        }
        if (comb) combine_apply(a.cmb, g, off_out + j, off_z + j, v1, r2);
      }
    }
    if (h2) hl_range_check(amax, a.range_flag);
  }
  if (a.cmb.mode == CM_RES0) {
    const double t = block_sum_f64(r2, red);
    if (threadIdx.x == 0)
      a.cmb.norm_partials[a.cmb.norm_base + blockIdx.y * a.cmb.norm_member_stride + blockIdx.x] = t;
  }
}

// ---- 128-bit vectorised forms (d % 4 == 0, 16-byte aligned rows): lane
// handles float4 q = lane + 32 i; all of a row's loads are issued before any
// arithmetic (the row lives in registers) ----
__device__ __forceinline__ float4 ld4(const float* p) { return *reinterpret_cast<const float4*>(p); }
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }

template <int V4>
__global__ void __launch_bounds__(256) ln_fwd4_kernel(LnFwdArgs a, const int* active) {
  pdl_wait();
  pdl_trigger();
  if (stopped(active)) return;
  const int g = blockIdx.y;
  const int row = blockIdx.x * kRowsPerBlock + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= a.rows) return;
  const float* x = a.x.at(g) + (long long)row * a.x.ld;
  const int d4 = a.d >> 2;
  float4 v[V4];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < V4; ++i) {
    const int q = lane + 32 * i;
    v[i] = q < d4 ? ld4(x + 4 * q) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int i = 0; i < V4; ++i) s += (v[i].x + v[i].y) + (v[i].z + v[i].w);
  const float inv_d = 1.f / (float)a.d;
  const float mean = warp_sum(s) * inv_d;
  float qs = 0.f;
#pragma unroll
  for (int i = 0; i < V4; ++i) {
    if (lane + 32 * i < d4) {
      const float c0 = v[i].x - mean, c1 = v[i].y - mean, c2 = v[i].z - mean, c3 = v[i].w - mean;
      qs += (c0 * c0 + c1 * c1) + (c2 * c2 + c3 * c3);
    }
  }
  const float var = warp_sum(qs) * inv_d;
  const float rstd = 1.f / sqrtf(var + a.eps);
  const float* gain = a.gain.at(g);
  const float* bias = a.bias.at(g);
  float* o = a.out.ok() ? a.out.at(g) + (long long)row * a.out.ld : nullptr;
  float* hl = a.out_hl.ok() ? a.out_hl.at(g) + (long long)row * a.out_hl.ld : nullptr;
  float amax = 0.f;
#pragma unroll
  for (int i = 0; i < V4; ++i) {
    const int q = lane + 32 * i;
    if (q < d4) {
      const float4 gn = ld4(gain + 4 * q), bs = ld4(bias + 4 * q);
      const float4 y = make_float4(gn.x * ((v[i].x - mean) * rstd) + bs.x,
                                   gn.y * ((v[i].y - mean) * rstd) + bs.y,
                                   gn.z * ((v[i].z - mean) * rstd) + bs.z,
                                   gn.w * ((v[i].w - mean) * rstd) + bs.w);
      if (o) st4(o + 4 * q, y);
      if (hl) st_hl4(hl, 4 * q, y, amax);
    }
  }
  if (hl) hl_range_check(amax, a.range_flag);
  if (lane == 0 && a.stats.ok()) {
    float* st = a.stats.at(g) + 2LL * row;
    st[0] = mean;
    st[1] = rstd;
  }
}

// 256-bit form of ln_fwd4 (d % 256 == 0, 32-byte aligned rows): lane l holds
// columns 8 (l + 32 i) .. + 7, one LDG.256 / STG.256 per 8 values (half the
// memory instructions of the float4 form; its own fixed reduction order)
__device__ __forceinline__ void ld8g(const float* p, float* v) {
  asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]),
                 "=f"(v[7])
               : "l"(p));
}
__device__ __forceinline__ void st8g(float* p, const float* v) {
  asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v[0]), "f"(v[1]),
               "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}

template <int V8>
__global__ void __launch_bounds__(256) ln_fwd8_kernel(LnFwdArgs a, const int* active) {
  pdl_wait();
  pdl_trigger();
  if (stopped(active)) return;
  const int g = blockIdx.y;
  const int row = blockIdx.x * kRowsPerBlock + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= a.rows) return;
  const float* x = a.x.at(g) + (long long)row * a.x.ld;
  float v[V8][8];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < V8; ++i) ld8g(x + 8 * (lane + 32 * i), v[i]);
#pragma unroll
  for (int i = 0; i < V8; ++i)
    s += ((v[i][0] + v[i][1]) + (v[i][2] + v[i][3])) + ((v[i][4] + v[i][5]) + (v[i][6] + v[i][7]));
  const float inv_d = 1.f / (float)a.d;
  const float mean = warp_sum(s) * inv_d;
  float qs = 0.f;
#pragma unroll
  for (int i = 0; i < V8; ++i)
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const float c = v[i][e] - mean;
      qs = fmaf(c, c, qs);
    }
  const float var = warp_sum(qs) * inv_d;
  const float rstd = 1.f / sqrtf(var + a.eps);
  const float* gain = a.gain.at(g);
  const float* bias = a.bias.at(g);
  float* o = a.out.ok() ? a.out.at(g) + (long long)row * a.out.ld : nullptr;
  float* hl = a.out_hl.ok() ? a.out_hl.at(g) + (long long)row * a.out_hl.ld : nullptr;
  float amax = 0.f;
#pragma unroll
  for (int i = 0; i < V8; ++i) {
    const int c0 = 8 * (lane + 32 * i);
    float gn[8], bs[8], y[8];
    ld8g(gain + c0, gn);
    ld8g(bias + c0, bs);
#pragma unroll
    for (int e = 0; e < 8; ++e) y[e] = gn[e] * ((v[i][e] - mean) * rstd) + bs[e];
    if (o) st8g(o + c0, y);
    if (hl) {
      uint4 h, l;
      tc::split8(y, h, l, amax);
      char* b = reinterpret_cast<char*>(hl) + (c0 >> 5) * 128 + (c0 & 31) * 2;
      *reinterpret_cast<uint4*>(b) = h;
      *reinterpret_cast<uint4*>(b + 64) = l;
    }
  }
  if (hl) hl_range_check(amax, a.range_flag);
  if (lane == 0 && a.stats.ok()) {
    float* st = a.stats.at(g) + 2LL * row;
    st[0] = mean;
    st[1] = rstd;
  }
}

template <int V4>
__global__ void __launch_bounds__(256) ln_bwd4_kernel(LnBwdArgs a, const int* active) {
  pdl_wait();
  pdl_trigger();
  __shared__ double red[32];
  if (stopped(active)) return;
  const int g = blockIdx.y;
  const int row = blockIdx.x * kRowsPerBlock + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  const int d4 = a.d >> 2;
  double r2 = 0.0;
  if (row < a.rows) {
    const float* x = a.x.at(g) + (long long)row * a.x.ld;
    const float* up = a.up.at(g) + (long long)row * a.up.ld;
    const float* gain = a.gain.at(g);
    const float mean = a.stats.at(g)[2LL * row];
    const float rstd = a.stats.at(g)[2LL * row + 1];
    float4 xh[V4], dxh[V4];
#pragma unroll
    for (int i = 0; i < V4; ++i) {
      const int q = lane + 32 * i;
      if (q < d4) {
        xh[i] = ld4(x + 4 * q);
        dxh[i] = ld4(up + 4 * q);
      }
    }
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < V4; ++i) {
      const int q = lane + 32 * i;
      if (q < d4) {
        const float4 gn = ld4(gain + 4 * q);
        xh[i] = make_float4((xh[i].x - mean) * rstd, (xh[i].y - mean) * rstd,
                            (xh[i].z - mean) * rstd, (xh[i].w - mean) * rstd);
        dxh[i] = make_float4(dxh[i].x * gn.x, dxh[i].y * gn.y, dxh[i].z * gn.z, dxh[i].w * gn.w);
        s1 += (dxh[i].x + dxh[i].y) + (dxh[i].z + dxh[i].w);
        s2 += (dxh[i].x * xh[i].x + dxh[i].y * xh[i].y) + (dxh[i].z * xh[i].z + dxh[i].w * xh[i].w);
      }
    }
    const float inv_d = 1.f / (float)a.d;
    const float m1 = warp_sum(s1) * inv_d;
    const float m2 = warp_sum(s2) * inv_d;
    const float* addA = a.addA.ok() ? a.addA.at(g) + (long long)row * a.addA.ld : nullptr;
    const float* addB = a.addB.ok() ? a.addB.at(g) + (long long)row * a.addB.ld : nullptr;
    float* o1 = a.out1.ok() ? a.out1.at(g) + (long long)row * a.out1.ld : nullptr;
    float* o2 = a.out2.ok() ? a.out2.at(g) + (long long)row * a.out2.ld : nullptr;
    float* h2 = a.out2_hl.ok() ? a.out2_hl.at(g) + (long long)row * a.out2_hl.ld : nullptr;
    float amax = 0.f;
    const bool comb = a.cmb.mode != CM_NONE;
    const long long off_out = comb ? (long long)row * a.cmb.out.ld : 0;
    const long long off_z = comb ? (long long)row * a.cmb.z.ld : 0;
    float4 ad[V4];
#pragma unroll
    for (int i = 0; i < V4; ++i) {
      const int q = lane + 32 * i;
      if (q < d4) {
        if (addA) ad[i] = ld4(addA + 4 * q);
        else if (addB) ad[i] = ld4(addB + 4 * q);
      }
    }
#pragma unroll
    for (int i = 0; i < V4; ++i) {
      const int q = lane + 32 * i;
      if (q < d4) {
        const float4 L = make_float4(rstd * (dxh[i].x - m1 - xh[i].x * m2),
                                     rstd * (dxh[i].y - m1 - xh[i].y * m2),
                                     rstd * (dxh[i].z - m1 - xh[i].z * m2),
                                     rstd * (dxh[i].w - m1 - xh[i].w * m2));
        const float4 v1 = addA ? make_float4(ad[i].x + L.x, ad[i].y + L.y, ad[i].z + L.z, ad[i].w + L.w) : L;
        if (o1) st4(o1 + 4 * q, v1);
        if (o2 || h2) {
          const float4 b = addA ? ld4(addB + 4 * q) : ad[i];
          float4 w = make_float4(b.x + L.x, b.y + L.y, b.z + L.z, b.w + L.w);
          if (a.drop2.on()) {
            w.x *= drop_val(a.drop2, g, row, 4 * q);
            w.y *= drop_val(a.drop2, g, row, 4 * q + 1);
            w.z *= drop_val(a.drop2, g, row, 4 * q + 2);
            w.w *= drop_val(a.drop2, g, row, 4 * q + 3);
          }
          if (o2) st4(o2 + 4 * q, w);
          if (h2) st_hl4(h2, 4 * q, w, amax);
        }
        if (comb) combine_apply4(a.cmb, g, off_out + 4 * q, off_z + 4 * q, v1, r2);
      }
    }
    if (h2) hl_range_check(amax, a.range_flag);
  }
  if (a.cmb.mode == CM_RES0) {
    const double t = block_sum_f64(r2, red);
    if (threadIdx.x == 0)
      a.cmb.norm_partials[a.cmb.norm_base + blockIdx.y * a.cmb.norm_member_stride + blockIdx.x] = t;
  }
}

// combine_apply4 over 8 consecutive values with 256-bit loads / stores
// (elementwise: the same results as two combine_apply4 calls)
__device__ __forceinline__ void combine_apply8(const Combine& c, int g, long long off_out,
                                               long long off_z, const float* F, double& r2) {
  float z[8], o[8];
  ld8g(c.z.at(g) + off_z, z);
#pragma unroll
  for (int e = 0; e < 8; ++e) o[e] = z[e] + c.dt * F[e];
  switch (c.mode) {
    case CM_PLAIN:
      break;
    case CM_FAS: {
      float pb[8], rh[8], bs[8];
      ld8g(c.phib.at(g) + off_out, pb);
      ld8g(c.rho.at(g) + off_out, rh);
      ld8g(c.base.at(g) + off_out, bs);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = bs[e] + ((o[e] - pb[e]) + rh[e]);
    } break;
    case CM_RES0: {
      float v[8];
      ld8g(c.v.at(g) + off_out, v);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        o[e] = o[e] - v[e];
        r2 += (double)o[e] * (double)o[e];
      }
    } break;
    case CM_RESL: {
      float pb[8], rh[8], bs[8], v[8];
      ld8g(c.phib.at(g) + off_out, pb);
      ld8g(c.rho.at(g) + off_out, rh);
      ld8g(c.base.at(g) + off_out, bs);
      ld8g(c.v.at(g) + off_out, v);
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = ((o[e] - pb[e]) + rh[e]) - (v[e] - bs[e]);
    } break;
    default:
      return;
  }
  st8g(c.out.at(g) + off_out, o);
}

// 256-bit form of ln_bwd4 (d % 256 == 0, 32-byte aligned rows): lane l holds
// columns 8 (l + 32 i) .. + 7 (its own fixed reduction order)
template <int V8>
__global__ void __launch_bounds__(256) ln_bwd8_kernel(LnBwdArgs a, const int* active) {
  pdl_wait();
  pdl_trigger();
  __shared__ double red[32];
  if (stopped(active)) return;
  const int g = blockIdx.y;
  const int row = blockIdx.x * kRowsPerBlock + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  double r2 = 0.0;
  if (row < a.rows) {
    const float* x = a.x.at(g) + (long long)row * a.x.ld;
    const float* up = a.up.at(g) + (long long)row * a.up.ld;
    const float* gain = a.gain.at(g);
    const float mean = a.stats.at(g)[2LL * row];
    const float rstd = a.stats.at(g)[2LL * row + 1];
    float xh[V8][8], dxh[V8][8];
#pragma unroll
    for (int i = 0; i < V8; ++i) {
      const int c0 = 8 * (lane + 32 * i);
      ld8g(x + c0, xh[i]);
      ld8g(up + c0, dxh[i]);
    }
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int i = 0; i < V8; ++i) {
      float gn[8];
      ld8g(gain + 8 * (lane + 32 * i), gn);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        xh[i][e] = (xh[i][e] - mean) * rstd;
        dxh[i][e] *= gn[e];
        s1 += dxh[i][e];
        s2 = fmaf(dxh[i][e], xh[i][e], s2);
      }
    }
    const float inv_d = 1.f / (float)a.d;
    const float m1 = warp_sum(s1) * inv_d;
    const float m2 = warp_sum(s2) * inv_d;
    const float* addA = a.addA.ok() ? a.addA.at(g) + (long long)row * a.addA.ld : nullptr;
    const float* addB = a.addB.ok() ? a.addB.at(g) + (long long)row * a.addB.ld : nullptr;
    float* o1 = a.out1.ok() ? a.out1.at(g) + (long long)row * a.out1.ld : nullptr;
    float* o2 = a.out2.ok() ? a.out2.at(g) + (long long)row * a.out2.ld : nullptr;
    float* h2 = a.out2_hl.ok() ? a.out2_hl.at(g) + (long long)row * a.out2_hl.ld : nullptr;
    float amax = 0.f;
    const bool comb = a.cmb.mode != CM_NONE;
    const long long off_out = comb ? (long long)row * a.cmb.out.ld : 0;
    const long long off_z = comb ? (long long)row * a.cmb.z.ld : 0;
#pragma unroll
    for (int i = 0; i < V8; ++i) {
      const int c0 = 8 * (lane + 32 * i);
      float L[8], v1[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) L[e] = rstd * (dxh[i][e] - m1 - xh[i][e] * m2);
      if (addA) {
        float ad[8];
        ld8g(addA + c0, ad);
#pragma unroll
        for (int e = 0; e < 8; ++e) v1[e] = ad[e] + L[e];
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) v1[e] = L[e];
      }
      if (o1) st8g(o1 + c0, v1);
      if (o2 || h2) {
        float bb[8], w[8];
        if (addB) ld8g(addB + c0, bb);
        else
#pragma unroll
          for (int e = 0; e < 8; ++e) bb[e] = 0.f;
#pragma unroll
        for (int e = 0; e < 8; ++e) w[e] = bb[e] + L[e];
        if (a.drop2.on())
#pragma unroll
          for (int e = 0; e < 8; ++e) w[e] *= drop_val(a.drop2, g, row, c0 + e);
        if (o2) st8g(o2 + c0, w);
        if (h2) {
          uint4 h, l;
          tc::split8(w, h, l, amax);
          char* b = reinterpret_cast<char*>(h2) + (c0 >> 5) * 128 + (c0 & 31) * 2;
          *reinterpret_cast<uint4*>(b) = h;
          *reinterpret_cast<uint4*>(b + 64) = l;
        }
      }
      if (comb) combine_apply8(a.cmb, g, off_out + c0, off_z + c0, v1, r2);
    }
    if (h2) hl_range_check(amax, a.range_flag);
  }
  if (a.cmb.mode == CM_RES0) {
    const double t = block_sum_f64(r2, red);
    if (threadIdx.x == 0)
      a.cmb.norm_partials[a.cmb.norm_base + blockIdx.y * a.cmb.norm_member_stride + blockIdx.x] = t;
  }
}

template <int V4>
struct LnFwd4L {
  static void launch(dim3 g, const LnFwdArgs& a, const int* act, cudaStream_t s) {
    launch_k(ln_fwd4_kernel<V4>, dim3(g), dim3(256), 0, s, 1, a, act);
  }
};
template <int V4>
struct LnBwd4L {
  static void launch(dim3 g, const LnBwdArgs& a, const int* act, cudaStream_t s) {
    launch_k(ln_bwd4_kernel<V4>, dim3(g), dim3(256), 0, s, 1, a, act);
  }
};

template <template <int> class K, class Args>
void dispatch_rows4(int d, const Args& a, int G, int rows, const int* active, cudaStream_t s) {
  dim3 grid(ceil_div(rows, kRowsPerBlock), G);
  const int v = (d / 4 + 31) / 32;
  if (v <= 1) K<1>::launch(grid, a, active, s);
  else if (v <= 2) K<2>::launch(grid, a, active, s);
  else if (v <= 4) K<4>::launch(grid, a, active, s);
  else if (v <= 6) K<6>::launch(grid, a, active, s);
  else K<8>::launch(grid, a, active, s);
}

bool vec8_ok(const Mat& m) {
  return !m.ok() || ((reinterpret_cast<uintptr_t>(m.ptr) & 31) == 0 && m.ld % 8 == 0 &&
                     m.slot_stride % 8 == 0);
}

bool vec_ok(const Mat& m) {
  return !m.ok() || ((reinterpret_cast<uintptr_t>(m.ptr) & 15) == 0 && m.ld % 4 == 0 &&
                     m.slot_stride % 4 == 0);
}

// Column sums in two stages: stage 1 = (128-column tile, row chunk, member)
// blocks, float4 rows, f64 partials reduced over the 8 row lanes in fixed
// order; stage 2 = ordered sum over the chunks, scaled into the gradients.
__global__ void __launch_bounds__(256) colred_part_kernel(ColRedArgs a, const int* active) {
  pdl_wait();
  pdl_trigger();
  __shared__ double sb[8][129];
  __shared__ double sg[8][129];
  if (stopped(active)) return;
  const int g = blockIdx.z, chunk = blockIdx.y;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int c = blockIdx.x * 128 + 4 * tx;
  const int rpc = (a.rows + kColRedChunks - 1) / kColRedChunks;
  const int r0 = chunk * rpc, r1 = min(a.rows, r0 + rpc);
  double b[4] = {0.0, 0.0, 0.0, 0.0}, gs[4] = {0.0, 0.0, 0.0, 0.0};
  if (c < a.cols) {
    const float* up = a.up.at(g);
    const float* x = a.x.ok() ? a.x.at(g) : nullptr;
    const float* st = x ? a.stats.at(g) : nullptr;
#pragma unroll 4
    for (int r = r0 + ty; r < r1; r += 8) {
      float4 u;
      if (a.up_hl) {
        const char* row = reinterpret_cast<const char*>(up + (long long)r * a.up.ld);
        const char* hp = row + (c >> 5) * 128 + (c & 31) * 2;
        const uint2 hv = *reinterpret_cast<const uint2*>(hp);
        const uint2 lv = *reinterpret_cast<const uint2*>(hp + 64);
        const float2 h01 = __half22float2(*reinterpret_cast<const __half2*>(&hv.x));
        const float2 h23 = __half22float2(*reinterpret_cast<const __half2*>(&hv.y));
        const float2 l01 = __half22float2(*reinterpret_cast<const __half2*>(&lv.x));
        const float2 l23 = __half22float2(*reinterpret_cast<const __half2*>(&lv.y));
        u = make_float4(fmaf(l01.x, 1.f / 2048.f, h01.x), fmaf(l01.y, 1.f / 2048.f, h01.y),
                        fmaf(l23.x, 1.f / 2048.f, h23.x), fmaf(l23.y, 1.f / 2048.f, h23.y));
      } else {
        u = ld4(up + (long long)r * a.up.ld + c);
      }
      b[0] += (double)u.x;
      b[1] += (double)u.y;
      b[2] += (double)u.z;
      b[3] += (double)u.w;
      if (x) {
        const float4 xv = ld4(x + (long long)r * a.x.ld + c);
        const float m = st[2LL * r], rs = st[2LL * r + 1];
        gs[0] += (double)u.x * (double)((xv.x - m) * rs);
        gs[1] += (double)u.y * (double)((xv.y - m) * rs);
        gs[2] += (double)u.z * (double)((xv.z - m) * rs);
        gs[3] += (double)u.w * (double)((xv.w - m) * rs);
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    sb[ty][4 * tx + e] = b[e];
    sg[ty][4 * tx + e] = gs[e];
  }
  __syncthreads();
  if (threadIdx.x < 128) {
    const int col = blockIdx.x * 128 + threadIdx.x;
    if (col < a.cols) {
      double tb = 0.0, tg = 0.0;
      for (int i = 0; i < 8; ++i) {
        tb += sb[i][threadIdx.x];
        tg += sg[i][threadIdx.x];
      }
      double* p = a.partials + (((long long)g * kColRedChunks + chunk) * a.cols + col) * 2;
      p[0] = tb;
      p[1] = tg;
    }
  }
}

__global__ void __launch_bounds__(256) colred_sum_kernel(ColRedArgs a, const int* active) {
  pdl_wait();
  pdl_trigger();
  if (stopped(active)) return;
  const int g = blockIdx.y;
  const int col = blockIdx.x * 256 + threadIdx.x;
  if (col >= a.cols) return;
  double tb = 0.0, tg = 0.0;
  for (int ch = 0; ch < kColRedChunks; ++ch) {
    const double* p = a.partials + (((long long)g * kColRedChunks + ch) * a.cols + col) * 2;
    tb += p[0];
    tg += p[1];
  }
  if (a.dbias.ok()) {
    float* db = a.dbias.at(g);
    db[col] = db[col] + (a.gscale_mul ? a.gscale * *a.gscale_mul : a.gscale) * (float)tb;
  }
  if (a.x.ok() && a.dgain.ok()) {
    float* dg = a.dgain.at(g);
    dg[col] = dg[col] + (a.gscale_mul ? a.gscale * *a.gscale_mul : a.gscale) * (float)tg;
  }
}

template <template <int> class K, class Args>
void dispatch_rows(int d, const Args& a, int G, int rows, const int* active, cudaStream_t s) {
  dim3 grid(ceil_div(rows, kRowsPerBlock), G);
  const int v = (d + 31) / 32;
  if (v <= 1) K<1>::launch(grid, a, active, s);
  else if (v <= 2) K<2>::launch(grid, a, active, s);
  else if (v <= 4) K<4>::launch(grid, a, active, s);
  else if (v <= 8) K<8>::launch(grid, a, active, s);
  else if (v <= 16) K<16>::launch(grid, a, active, s);
  else if (v <= 24) K<24>::launch(grid, a, active, s);
  else if (v <= 32) K<32>::launch(grid, a, active, s);
  else throw ValidationError("LayerNorm: width > 1024 is not supported");
}

template <int V>
struct LnFwdL {
  static void launch(dim3 g, const LnFwdArgs& a, const int* act, cudaStream_t s) {
    launch_k(ln_fwd_kernel<V>, dim3(g), dim3(256), 0, s, 1, a, act);
  }
};
template <int V>
struct LnBwdL {
  static void launch(dim3 g, const LnBwdArgs& a, const int* act, cudaStream_t s) {
    launch_k(ln_bwd_kernel<V>, dim3(g), dim3(256), 0, s, 1, a, act);
  }
};

// ---- attention softmax and its VJP (tensor.cpp:310-342, blocks.cpp:160-166) ------
// P = softmax_rows(S * scale [+ causal -inf above the diagonal]) in place.
// Masked probabilities are exactly 0, as with the reference's -1e30.
template <int V>
__global__ void __launch_bounds__(256) softmax_kernel(SoftmaxArgs a, const int* active) {
  pdl_wait();
  pdl_trigger();
  if (stopped(active)) return;
  const int g = blockIdx.y;
  const long long row = (long long)blockIdx.x * kRowsPerBlock + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= a.rows) return;
  float* S = a.S.at(g) + row * a.S.ld;
  const int qi = (int)(row % a.sq);
  float v[V];
  float m = -INFINITY;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int j = lane + 32 * i;
    const bool ok = j < a.ncols && !(a.causal && j > qi);
    v[i] = ok ? S[j] * a.scale : -INFINITY;
    m = fmaxf(m, v[i]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    v[i] = v[i] == -INFINITY ? 0.f : expf(v[i] - m);
    sum += v[i];
  }
  sum = warp_sum(sum);
  const float inv = 1.f / sum;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int j = lane + 32 * i;
    if (j < a.ncols) S[j] = v[i] * inv;
  }
}

// dS = P * (dP - sum_j dP_j P_j), in place over dP (vjp_softmax_rows)
template <int V>
__global__ void __launch_bounds__(256) softmax_bwd_kernel(SoftmaxArgs a, const int* active) {
  pdl_wait();
  pdl_trigger();
  if (stopped(active)) return;
  const int g = blockIdx.y;
  const long long row = (long long)blockIdx.x * kRowsPerBlock + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= a.rows) return;
  const float* P = a.S.at(g) + row * a.S.ld;
  float* dP = a.dS.at(g) + row * a.dS.ld;
  float pv[V], dv[V];
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int j = lane + 32 * i;
    pv[i] = j < a.ncols ? P[j] : 0.f;
    dv[i] = j < a.ncols ? dP[j] : 0.f;
    t += dv[i] * pv[i];
  }
  t = warp_sum(t);
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int j = lane + 32 * i;
    if (j < a.ncols) dP[j] = pv[i] * (dv[i] - t);
  }
}

template <int V>
struct SmL {
  static void launch(dim3 g, const SoftmaxArgs& a, const int* act, cudaStream_t s) {
    if (a.dS.ok())
      launch_k(softmax_bwd_kernel<V>, dim3(g), dim3(256), 0, s, 1, a, act);
    else
      launch_k(softmax_kernel<V>, dim3(g), dim3(256), 0, s, 1, a, act);
  }
};

// ---- column sums for parameter gradients -----------------------------------------
__global__ void __launch_bounds__(256) colred_kernel(ColRedArgs a, const int* active) {
  pdl_wait();
  pdl_trigger();
  __shared__ double sb[8][33];
  __shared__ double sg[8][33];
  if (stopped(active)) return;
  const int g = blockIdx.y;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int col = blockIdx.x * 32 + tx;
  double accb = 0.0, accg = 0.0;
  if (col < a.cols) {
    const float* up = a.up.at(g);
    const float* x = a.x.ok() ? a.x.at(g) : nullptr;
    const float* st = a.x.ok() ? a.stats.at(g) : nullptr;
    for (int r = ty; r < a.rows; r += 8) {
      const float u = up[(long long)r * a.up.ld + col];
      accb += (double)u;
      if (x) {
        const float xh = (x[(long long)r * a.x.ld + col] - st[2LL * r]) * st[2LL * r + 1];
        accg += (double)u * (double)xh;
      }
    }
  }
  sb[ty][tx] = accb;
  sg[ty][tx] = accg;
  __syncthreads();
  if (ty == 0 && col < a.cols) {
    double tb = 0.0, tg = 0.0;
    for (int i = 0; i < 8; ++i) {
      tb += sb[i][tx];
      tg += sg[i][tx];
    }
    if (a.dbias.ok()) {
      float* db = a.dbias.at(g);
      db[col] = db[col] + (a.gscale_mul ? a.gscale * *a.gscale_mul : a.gscale) * (float)tb;
    }
    if (a.x.ok() && a.dgain.ok()) {
      float* dg = a.dgain.at(g);
      dg[col] = dg[col] + (a.gscale_mul ? a.gscale * *a.gscale_mul : a.gscale) * (float)tg;
    }
  }
}

// ---- elementwise state algebra ------------------------------------------------------
constexpr int kElemThreads = 256;
constexpr int kElemPerThread = 8;

__global__ void __launch_bounds__(kElemThreads) elem_combine_kernel(ElemCombineArgs a,
                                                                    const int* active) {
  pdl_wait();
  pdl_trigger();
  __shared__ double red[32];
  if (stopped(active)) return;
  const int g = blockIdx.y;
  double r2 = 0.0;
  const long long base = (long long)blockIdx.x * kElemThreads * kElemPerThread + threadIdx.x;
  const float* F = a.F.ok() ? a.F.at(g) : nullptr;
#pragma unroll
  for (int i = 0; i < kElemPerThread; ++i) {
    const long long e = base + (long long)i * kElemThreads;
    if (e < a.n) combine_apply(a.cmb, g, e, e, F ? F[e] : 0.f, r2);
  }
  if (a.cmb.mode == CM_RES0) {
    const double t = block_sum_f64(r2, red);
    if (threadIdx.x == 0)
      a.cmb.norm_partials[a.cmb.norm_base + blockIdx.y * a.cmb.norm_member_stride + blockIdx.x] = t;
  }
}

__global__ void copy_kernel(int G, long long n4, Mat dst, Mat src, const int* active) {
  pdl_wait();
  pdl_trigger();
  if (stopped(active)) return;
  const int g = blockIdx.y;
  float4* d = reinterpret_cast<float4*>(dst.at(g));
  const float4* s = reinterpret_cast<const float4*>(src.at(g));
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  // four independent loads in flight per thread (the stream is latency-bound
  // with one), then the tail
  for (; i + 3 * stride < n4; i += 4 * stride) {
    const float4 v0 = s[i], v1 = s[i + stride], v2 = s[i + 2 * stride], v3 = s[i + 3 * stride];
    d[i] = v0;
    d[i + stride] = v1;
    d[i + 2 * stride] = v2;
    d[i + 3 * stride] = v3;
  }
  for (; i < n4; i += stride) d[i] = s[i];
}

__global__ void correct_kernel(int G, long long n4, Mat dst, Mat a, Mat b, const int* active) {
  pdl_wait();
  pdl_trigger();
  if (stopped(active)) return;
  const int g = blockIdx.y;
  float4* d = reinterpret_cast<float4*>(dst.at(g));
  const float4* pa = reinterpret_cast<const float4*>(a.at(g));
  const float4* pb = reinterpret_cast<const float4*>(b.at(g));
  const long long stride = (long long)gridDim.x * blockDim.x;
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  auto fix = [](float4 x, float4 u, float4 w) {
    return make_float4(x.x + (u.x - w.x), x.y + (u.y - w.y), x.z + (u.z - w.z), x.w + (u.w - w.w));
  };
  for (; i + stride < n4; i += 2 * stride) {  // two rows of loads in flight per thread
    const float4 x0 = d[i], u0 = pa[i], w0 = pb[i];
    const float4 x1 = d[i + stride], u1 = pa[i + stride], w1 = pb[i + stride];
    d[i] = fix(x0, u0, w0);
    d[i + stride] = fix(x1, u1, w1);
  }
  for (; i < n4; i += stride) d[i] = fix(d[i], pa[i], pb[i]);
}

__global__ void zero_kernel(int G, long long n4, Mat dst, const int* active) {
  pdl_wait();
  pdl_trigger();
  if (stopped(active)) return;
  float4* d = reinterpret_cast<float4*>(dst.at(blockIdx.y));
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x)
    d[i] = make_float4(0.f, 0.f, 0.f, 0.f);
}

int stream_grid(long long n4, int G) {
  // ~4 waves of 148 SMs across the whole family
  long long want = (592LL + G - 1) / G;
  long long need = (n4 + 255) / 256;
  return (int)std::max<long long>(1, std::min(want, need));
}

// ---- solve control -------------------------------------------------------------------
__global__ void ctrl_begin_kernel(SolveCtrl* c, int host_cycles, const int* budget_dev) {
  pdl_wait();
  pdl_trigger();
  c->active = 1;
  c->n_trace = 0;
  c->converged = 0;
  c->cycles_run = 0;
  c->pending = 0.0;
  const int want = budget_dev ? *budget_dev : host_cycles;
  c->budget = min(want, host_cycles);
  c->truncated = want > host_cycles ? 1 : 0;
  if (c->budget < 1) c->active = 0;
}

// last_pair_factor (controller.hpp:63-67) of a solve's trace
__device__ double trace_factor(const SolveCtrl* c) {
  const int n = min(c->n_trace, kMaxTrace);
  if (n < 2 || c->trace[n - 2] == 0.0) return 0.0;
  return c->trace[n - 1] / c->trace[n - 2];
}

__global__ void monitor_init_kernel(MonitorDev* m, double thr, int policy_switch, int cap, int fwd,
                                    int bwd) {
  pdl_wait();
  pdl_trigger();
  m->threshold = thr;
  m->policy_switch = policy_switch;
  m->cap = cap;
  m->switched = 0;
  m->n_reports = 0;
  m->budget[0] = fwd;
  m->budget[1] = bwd;
  m->saved[0] = fwd;
  m->saved[1] = bwd;
  m->last_decision = 0;
  m->last_ff = m->last_bf = 0.0;
}

__global__ void monitor_set_budget_kernel(MonitorDev* m, int fwd, int bwd) {
  pdl_wait();
  pdl_trigger();
  m->budget[0] = fwd;
  m->budget[1] = bwd;
}

__global__ void monitor_probe_kernel(MonitorDev* m, int begin) {
  pdl_wait();
  pdl_trigger();
  if (begin) {
    m->saved[0] = m->budget[0];
    m->saved[1] = m->budget[1];
    m->budget[0] *= 2;
    m->budget[1] *= 2;
  } else {
    m->budget[0] = m->saved[0];
    m->budget[1] = m->saved[1];
  }
}

__global__ void monitor_record_kernel(MonitorDev* m, const SolveCtrl* f, const SolveCtrl* b,
                                      long long batch, MonitorSummary* out) {
  pdl_wait();
  pdl_trigger();
  const double ff = trace_factor(f), bf = trace_factor(b);
  if (batch >= 0) {
    // decide (controller.hpp:71-84) with the budgets as they are now
    const double worst = ff > bf ? ff : bf;  // std::max(f, b): NaN-free traces
    int dec = 0;
    if (worst > m->threshold) {
      if (m->policy_switch)
        dec = 2;
      else
        dec = (m->budget[0] < m->cap || m->budget[1] < m->cap) ? 1 : 2;
    }
    if (dec == 1) {
      m->budget[0] = min(2 * m->budget[0], m->cap);
      m->budget[1] = min(2 * m->budget[1], m->cap);
    } else if (dec == 2) {
      m->switched = 1;
    }
    const int i = m->n_reports % kMonReports;
    m->rep_batch[i] = batch;
    m->rep_ff[i] = ff;
    m->rep_bf[i] = bf;
    m->rep_dec[i] = dec;
    m->n_reports += 1;
    m->last_decision = dec;
    m->last_ff = ff;
    m->last_bf = bf;
  }
  out->switched = m->switched;
  out->n_reports = m->n_reports;
  out->last_decision = m->last_decision;
  out->budget[0] = m->budget[0];
  out->budget[1] = m->budget[1];
  out->used[0] = f->budget;
  out->used[1] = b->budget;
  out->last_ff = m->last_ff;
  out->last_bf = m->last_bf;
  out->trace_ff = ff;
  out->trace_bf = bf;
}

// sum of the per-interval partials in interval order (each interval's slots
// by a fixed tree): the trace does not depend on the rank count. With
// `reversed`, rank r's block of `per_rank` intervals holds intervals of time
// position P-1-r (the adjoint solve's partition).
__global__ void trace_record_kernel(SolveCtrl* c, const double* partials, int n_chunks, int S,
                                    int per_rank, int reversed, const LamScale* sc) {
  pdl_wait();
  pdl_trigger();
  __shared__ double red[32];
  if (!c->active) return;
  const int P = n_chunks / per_rank;
  double total = 0.0;
  for (int k = 0; k < n_chunks; ++k) {
    const int pos = reversed ? (P - 1 - k / per_rank) * per_rank + k % per_rank : k;
    const double* q = partials + (size_t)pos * S;
    double s = 0.0;
    for (int i = threadIdx.x; i < S; i += blockDim.x) s += q[i];
    const double t = block_sum_f64(s, red);
    if (threadIdx.x == 0) total += t;
    __syncthreads();
  }
  // the adjoint's norms are of 2^k-scaled rows: * 2^-k is exact
  if (threadIdx.x == 0) c->pending = sc ? sqrt(total) * sc->down_d : sqrt(total);
}

__global__ void lam_amax_kernel(const float* x, long long n, LamScale* sc, int warm) {
  pdl_wait();
  pdl_trigger();
  unsigned int m = 0;
  // warm: the stored states are at 2^k_state; * 2^-k_state is exact (the
  // states are normal floats, k_state in [-100, 100])
  const float f = warm ? ldexpf(1.f, -sc->k_state) : 1.f;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    m = max(m, __float_as_uint(x[i] * f) & 0x7fffffffu);  // NaN bits sort above inf
#pragma unroll
  for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(&sc->amax_bits, m);
}

// k with max|x| * 2^k in [1, 2): k = -(unbiased exponent of max); kept in
// [-100, 100] so 2^k and 2^-k are normal floats; 0 for 0 / inf / NaN
__device__ __forceinline__ int lam_k(unsigned int bits) {
  if (bits == 0u || bits >= 0x7f800000u) return 0;
  const int e = (int)(bits >> 23) - 127;  // subnormal max: e = -127 (k clamps anyway)
  return max(-100, min(100, -e));
}

__global__ void lam_rescale_kernel(long long n4, Mat dst, const LamScale* sc) {
  pdl_wait();
  pdl_trigger();
  const int dk = sc->k - sc->k_state;
  if (dk == 0) return;
  const float f = ldexpf(1.f, dk);
  float4* d = reinterpret_cast<float4*>(dst.at(blockIdx.y));
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    const float4 v = d[i];
    d[i] = make_float4(v.x * f, v.y * f, v.z * f, v.w * f);
  }
}

__global__ void lam_bits_to_f64_kernel(const LamScale* sc, double* out) {
  pdl_wait();
  pdl_trigger();
  out[0] = (double)sc->amax_bits;
}

__global__ void lam_bits_max_kernel(const double* in, int n, LamScale* sc) {
  pdl_wait();
  pdl_trigger();
  unsigned int m = 0;
  for (int r = 0; r < n; ++r) m = max(m, (unsigned int)in[r]);
  sc->amax_bits = m;
}

__global__ void lam_commit_kernel(LamScale* sc) {
  pdl_wait();
  pdl_trigger();
  sc->k_state = sc->k;
}

__global__ void lam_scale_kernel(const float* src, float* dst, long long n4, LamScale* sc,
                                 int dir) {
  pdl_wait();
  pdl_trigger();
  const int k = lam_k(sc->amax_bits);
  const float f = ldexpf(1.f, dir > 0 ? k : -k);
  if (dir > 0 && blockIdx.x == 0 && threadIdx.x == 0) {
    sc->k = k;
    sc->up = ldexpf(1.f, k);
    sc->down = ldexpf(1.f, -k);
    sc->down_d = ldexp(1.0, -k);
  }
  const float4* s4 = reinterpret_cast<const float4*>(src);
  float4* d4 = reinterpret_cast<float4*>(dst);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    const float4 v = s4[i];
    d4[i] = make_float4(v.x * f, v.y * f, v.z * f, v.w * f);
  }
}

__global__ void cycle_end_kernel(SolveCtrl* c, double tol) {
  pdl_wait();
  pdl_trigger();
  if (!c->active) return;
  const double nrm = c->pending;
  if (c->n_trace < kMaxTrace) c->trace[c->n_trace] = nrm;
  c->n_trace += 1;
  c->cycles_run += 1;
  if (!isfinite(nrm)) {
    c->active = 0;
  } else if (nrm <= tol * c->trace[0]) {
    c->converged = 1;
    c->active = 0;
  } else if (c->cycles_run >= c->budget) {
    c->active = 0;  // budget spent (the remaining host-issued cycles are no-ops)
  }
}

}  // namespace

void launch_ln_fwd(const LnFwdArgs& a, const int* active, cudaStream_t s) {
  if (a.rows == 0 || a.G == 0) return;
  static const bool v8 = [] {  // MGLP_LN_V8=0: the float4 form only (A/B)
    const char* e = getenv("MGLP_LN_V8");
    return !(e && atoi(e) == 0);
  }();
  if (v8 && (a.d == 512 || a.d == 768 || a.d == 1024) && vec8_ok(a.x) && vec8_ok(a.out) &&
      vec8_ok(a.out_hl) && vec8_ok(a.gain) && vec8_ok(a.bias)) {
    dim3 grid(ceil_div(a.rows, kRowsPerBlock), a.G);
    if (a.d == 512) launch_k(ln_fwd8_kernel<2>, grid, dim3(256), 0, s, 1, a, active);
    else if (a.d == 768) launch_k(ln_fwd8_kernel<3>, grid, dim3(256), 0, s, 1, a, active);
    else launch_k(ln_fwd8_kernel<4>, grid, dim3(256), 0, s, 1, a, active);
  } else if (a.d % 4 == 0 && vec_ok(a.x) && vec_ok(a.out) && vec_ok(a.out_hl) && vec_ok(a.gain) &&
      vec_ok(a.bias))
    dispatch_rows4<LnFwd4L>(a.d, a, a.G, a.rows, active, s);
  else
    dispatch_rows<LnFwdL>(a.d, a, a.G, a.rows, active, s);
}

int ln_bwd_blocks(int rows) { return ceil_div(rows, kRowsPerBlock); }

void launch_ln_bwd(const LnBwdArgs& a, const int* active, cudaStream_t s) {
  if (a.rows == 0 || a.G == 0) return;
  const Combine& c = a.cmb;
  static const bool v8 = [] {  // MGLP_LN_V8=0: the float4 form only (A/B)
    const char* e = getenv("MGLP_LN_V8");
    return !(e && atoi(e) == 0);
  }();
  if (v8 && (a.d == 512 || a.d == 768 || a.d == 1024) && vec8_ok(a.x) && vec8_ok(a.up) &&
      vec8_ok(a.gain) && vec8_ok(a.addA) && vec8_ok(a.addB) && vec8_ok(a.out1) && vec8_ok(a.out2) &&
      vec8_ok(a.out2_hl) && vec8_ok(c.z) && vec8_ok(c.out) && vec8_ok(c.base) && vec8_ok(c.phib) &&
      vec8_ok(c.rho) && vec8_ok(c.v)) {
    dim3 grid(ceil_div(a.rows, kRowsPerBlock), a.G);
    if (a.d == 512) launch_k(ln_bwd8_kernel<2>, grid, dim3(256), 0, s, 1, a, active);
    else if (a.d == 768) launch_k(ln_bwd8_kernel<3>, grid, dim3(256), 0, s, 1, a, active);
    else launch_k(ln_bwd8_kernel<4>, grid, dim3(256), 0, s, 1, a, active);
  } else if (a.d % 4 == 0 && vec_ok(a.x) && vec_ok(a.up) && vec_ok(a.gain) && vec_ok(a.addA) &&
      vec_ok(a.addB) && vec_ok(a.out1) && vec_ok(a.out2) && vec_ok(a.out2_hl) && vec_ok(c.z) && vec_ok(c.out) &&
      vec_ok(c.base) && vec_ok(c.phib) && vec_ok(c.rho) && vec_ok(c.v))
    dispatch_rows4<LnBwd4L>(a.d, a, a.G, a.rows, active, s);
  else
    dispatch_rows<LnBwdL>(a.d, a, a.G, a.rows, active, s);
}

void launch_softmax(const SoftmaxArgs& a, const int* active, cudaStream_t s) {
  if (a.rows == 0 || a.G == 0) return;
  if (a.rows > (long long)INT32_MAX) throw ContractViolation("softmax: too many rows");
  dispatch_rows<SmL>(a.ncols, a, a.G, (int)a.rows, active, s);
}

void launch_colred(const ColRedArgs& a, const int* active, cudaStream_t s) {
  if (a.rows == 0 || a.G == 0) return;
  const bool two_stage = a.partials && a.cols % 4 == 0 && vec_ok(a.up) && vec_ok(a.x) &&
                         (long long)a.G * kColRedChunks * a.cols * 2 <= a.partials_cap;
  if (a.up_hl && (!two_stage || a.cols % 32))
    throw ContractViolation("colred: pre-split rows need the two-stage form and 32-aligned columns");
  if (two_stage) {
    launch_k(colred_part_kernel, dim3(dim3(ceil_div(a.cols, 128), kColRedChunks, a.G)), dim3(256), 0, s, 1, a, active);
    launch_k(colred_sum_kernel, dim3(dim3(ceil_div(a.cols, 256), a.G)), dim3(256), 0, s, 1, a, active);
    return;
  }
  dim3 grid(ceil_div(a.cols, 32), a.G);
  launch_k(colred_kernel, dim3(grid), dim3(256), 0, s, 1, a, active);
}

int elem_combine_blocks(long long n) {
  return ceil_div(n, (long long)kElemThreads * kElemPerThread);
}

void launch_elem_combine(const ElemCombineArgs& a, const int* active, cudaStream_t s) {
  if (a.n == 0 || a.G == 0) return;
  dim3 grid(elem_combine_blocks(a.n), a.G);
  launch_k(elem_combine_kernel, dim3(grid), dim3(kElemThreads), 0, s, 1, a, active);
}

static void require_vec4(long long n, const char* what) {
  if (n % 4) throw ContractViolation(std::string(what) + ": size must be a multiple of 4");
}

void launch_copy(int G, long long n, Mat dst, Mat src, const int* active, cudaStream_t s) {
  if (G == 0 || n == 0) return;
  require_vec4(n, "copy");
  dim3 grid(stream_grid(n / 4, G), G);
  launch_k(copy_kernel, dim3(grid), dim3(256), 0, s, 1, G, n / 4, dst, src, active);
}

__global__ void __launch_bounds__(256) mask_copy_kernel(int rows, int d, Mat dst, Mat src,
                                                        DropMask m, const int* active) {
  pdl_wait();
  pdl_trigger();
  if (stopped(active)) return;
  const int g = blockIdx.y;
  const long long n = (long long)rows * d;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x) {
    const long long r = k / d;
    const int c = (int)(k - r * d);
    dst.at(g)[r * dst.ld + c] = src.at(g)[r * src.ld + c] * drop_val(m, g, r, c);
  }
}

void launch_mask_copy(int G, int rows, int d, Mat dst, Mat src, const DropMask& m,
                      const int* active, cudaStream_t s) {
  if (G == 0 || rows == 0) return;
  const long long n = (long long)rows * d;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 148 * 8);
  launch_k(mask_copy_kernel, dim3(dim3(blocks, G)), dim3(256), 0, s, 1, rows, d, dst, src, m, active);
  MGLP_CUDA(cudaGetLastError());
}

void launch_correct(int G, long long n, Mat dst, Mat a, Mat b, const int* active,
                    cudaStream_t s) {
  if (G == 0 || n == 0) return;
  require_vec4(n, "correct");
  dim3 grid(stream_grid(n / 4, G), G);
  launch_k(correct_kernel, dim3(grid), dim3(256), 0, s, 1, G, n / 4, dst, a, b, active);
}

void launch_zero(int G, long long n, Mat dst, const int* active, cudaStream_t s) {
  if (G == 0 || n == 0) return;
  require_vec4(n, "zero");
  dim3 grid(stream_grid(n / 4, G), G);
  launch_k(zero_kernel, dim3(grid), dim3(256), 0, s, 1, G, n / 4, dst, active);
}

void launch_ctrl_begin(SolveCtrl* c, int host_cycles, const int* budget_dev, cudaStream_t s) {
  launch_k(ctrl_begin_kernel, dim3(1), dim3(1), 0, s, 1, c, host_cycles, budget_dev);
}

void launch_monitor_init(MonitorDev* m, double threshold, int policy_switch, int cap, int fwd,
                         int bwd, cudaStream_t s) {
  launch_k(monitor_init_kernel, dim3(1), dim3(1), 0, s, 1, m, threshold, policy_switch, cap, fwd,
           bwd);
}

void launch_monitor_set_budget(MonitorDev* m, int fwd, int bwd, cudaStream_t s) {
  launch_k(monitor_set_budget_kernel, dim3(1), dim3(1), 0, s, 1, m, fwd, bwd);
}

void launch_monitor_probe(MonitorDev* m, int begin, cudaStream_t s) {
  launch_k(monitor_probe_kernel, dim3(1), dim3(1), 0, s, 1, m, begin);
}

void launch_monitor_record(MonitorDev* m, const SolveCtrl* f, const SolveCtrl* b,
                           long long batch, MonitorSummary* out, cudaStream_t s) {
  launch_k(monitor_record_kernel, dim3(1), dim3(1), 0, s, 1, m, f, b, batch, out);
}

void launch_trace_record(SolveCtrl* c, const double* partials, int n_chunks, int S, int per_rank,
                         bool reversed, cudaStream_t s, const LamScale* sc) {
  launch_k(trace_record_kernel, dim3(1), dim3(256), 0, s, 1, c, partials, n_chunks, S, per_rank,
           reversed ? 1 : 0, sc);
}

void launch_lam_rescale(int G, long long n, Mat dst, const LamScale* sc, cudaStream_t s) {
  if (G == 0 || n == 0) return;
  require_vec4(n, "lam_rescale");
  dim3 grid(stream_grid(n / 4, G), G);
  launch_k(lam_rescale_kernel, grid, dim3(256), 0, s, 1, n / 4, dst, sc);
}

void launch_lam_bits_to_f64(const LamScale* sc, double* out, cudaStream_t s) {
  launch_k(lam_bits_to_f64_kernel, dim3(1), dim3(1), 0, s, 1, sc, out);
}

void launch_lam_bits_max(const double* in, int n, LamScale* sc, cudaStream_t s) {
  launch_k(lam_bits_max_kernel, dim3(1), dim3(1), 0, s, 1, in, n, sc);
}

void launch_lam_commit(LamScale* sc, cudaStream_t s) {
  launch_k(lam_commit_kernel, dim3(1), dim3(1), 0, s, 1, sc);
}

void launch_lam_amax(const float* x, long long n, LamScale* sc, cudaStream_t s) {
  MGLP_CUDA(cudaMemsetAsync(&sc->amax_bits, 0, sizeof(unsigned int), s));
  if (n == 0) return;
  const int grid = (int)std::max<long long>(1, std::min<long long>(592, (n + 255) / 256));
  launch_k(lam_amax_kernel, dim3(grid), dim3(256), 0, s, 1, x, n, sc, 0);
}

void launch_lam_amax_warm(const float* x, long long n, LamScale* sc, cudaStream_t s) {
  if (n == 0) return;
  const int grid = (int)std::max<long long>(1, std::min<long long>(1184, (n + 255) / 256));
  launch_k(lam_amax_kernel, dim3(grid), dim3(256), 0, s, 1, x, n, sc, 1);
}

void launch_lam_scale(const float* src, float* dst, long long n, LamScale* sc, int dir,
                      cudaStream_t s) {
  require_vec4(n, "lam_scale");
  const int grid = std::max(1, stream_grid(n / 4, 1));
  launch_k(lam_scale_kernel, dim3(grid), dim3(256), 0, s, 1, src, dst, n / 4, sc, dir);
}

void launch_cycle_end(SolveCtrl* c, double tol, cudaStream_t s) {
  launch_k(cycle_end_kernel, dim3(1), dim3(1), 0, s, 1, c, tol);
}

}  // namespace mglp
