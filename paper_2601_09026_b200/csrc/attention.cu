// Multi-head attention forward and VJP (blocks.cpp:142-236), fp32 on CUDA
// cores, flash-style: scores are never materialised in HBM. The forward
// stores the per-row log-sum-exp so the VJP recomputes P = exp(S - lse)
// tile by tile instead of caching s x s probabilities.
//
// Semantics match the reference exactly: S = (q.k^T) * (1/sqrt(dh)); the
// causal mask makes masked probabilities exactly 0 (the reference adds
// -1e30, blocks.cpp:85,161-165, which underflows to an exact zero too);
// dS = P (dP - rowsum(dP P)) with rowsum(dP P) = dO.O (vjp_softmax_rows,
// tensor.cpp:329-342).
//
// Layout: q/k/v/o rows are tokens (b*s + i), head h owns columns
// [h*dh, (h+1)*dh). dh <= 64.
#include "kernels.cuh"

namespace mglp {

namespace {

constexpr int BQ = 32, BKV = 32, MAXDH = 64, NT = 128;
constexpr float kNeg = -1e30f;

__device__ __forceinline__ bool stopped(const int* active) {
  return active != nullptr && *(volatile const int*)active == 0;
}

__device__ __forceinline__ float quad_max(float v) {
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 1));
  return fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 2));
}
__device__ __forceinline__ float quad_sum(float v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v + __shfl_xor_sync(0xffffffffu, v, 2);
}

// load a [rows x dh] head tile (rows r0.., clipped at nrows) into smem [BQ][MAXDH+1]
__device__ __forceinline__ void load_tile(float (*dst)[MAXDH + 1], const float* src, int ld,
                                          int r0, int nrows, int col0, int dh) {
  for (int e = threadIdx.x; e < 32 * dh; e += NT) {
    const int r = e / dh, c = e % dh;
    dst[r][c] = (r0 + r < nrows) ? src[(long long)(r0 + r) * ld + col0 + c] : 0.f;
  }
}

__global__ void __launch_bounds__(NT) attn_fwd_kernel(AttnArgs a, const int* active) {
  __shared__ float Qs[BQ][MAXDH + 1];
  __shared__ float Ks[BKV][MAXDH + 1];
  __shared__ float Vs[BKV][MAXDH + 1];
  __shared__ float Ps[BQ][BKV + 1];
  if (stopped(active)) return;
  const int g = blockIdx.z;
  const int b = blockIdx.y / a.H, h = blockIdx.y % a.H;
  const int q0 = blockIdx.x * BQ;
  const int tq = threadIdx.x >> 2, sub = threadIdx.x & 3;
  const int qi = q0 + tq;
  const int dh = a.dh, col0 = h * dh;
  const float* Q = a.q.at(g) + (long long)b * a.sq * a.q.ld;
  const float* K = a.k.at(g) + (long long)b * a.skv * a.k.ld;
  const float* V = a.v.at(g) + (long long)b * a.skv * a.v.ld;
  load_tile(Qs, Q, a.q.ld, q0, a.sq, col0, dh);
  float o[MAXDH / 4];
#pragma unroll
  for (int u = 0; u < MAXDH / 4; ++u) o[u] = 0.f;
  float m = kNeg, l = 0.f;
  int kv_end = a.skv;
  if (a.causal) kv_end = min(kv_end, q0 + BQ);
  for (int kv0 = 0; kv0 < kv_end; kv0 += BKV) {
    __syncthreads();
    load_tile(Ks, K, a.k.ld, kv0, a.skv, col0, dh);
    load_tile(Vs, V, a.v.ld, kv0, a.skv, col0, dh);
    __syncthreads();
    float s[BKV / 4];
    float tmax = kNeg;
#pragma unroll
    for (int t = 0; t < BKV / 4; ++t) {
      const int j = sub + 4 * t, kj = kv0 + j;
      float acc = 0.f;
      for (int c = 0; c < dh; ++c) acc = fmaf(Qs[tq][c], Ks[j][c], acc);
      acc *= a.scale;
      const bool masked = kj >= a.skv || (a.causal && kj > qi);
      s[t] = masked ? kNeg : acc;
      tmax = fmaxf(tmax, s[t]);
    }
    tmax = quad_max(tmax);
    const float mnew = fmaxf(m, tmax);
    const float alpha = __expf(m - mnew);
    float psum = 0.f;
#pragma unroll
    for (int t = 0; t < BKV / 4; ++t) {
      const float p = s[t] <= kNeg ? 0.f : expf(s[t] - mnew);
      Ps[tq][sub + 4 * t] = p;
      psum += p;
    }
    psum = quad_sum(psum);
    l = l * alpha + psum;
    m = mnew;
    __syncwarp();
    const int ncol = dh / 4;
    for (int u = 0; u < ncol; ++u) {
      const int c = sub + 4 * u;
      float acc = o[u] * alpha;
      for (int j = 0; j < BKV; ++j) acc = fmaf(Ps[tq][j], Vs[j][c], acc);
      o[u] = acc;
    }
  }
  if (qi < a.sq) {
    float* O = a.o.at(g) + (long long)(b * a.sq + qi) * a.o.ld + col0;
    const float inv = 1.f / l;
    for (int u = 0; u < dh / 4; ++u) O[sub + 4 * u] = o[u] * inv;
    if (sub == 0) a.lse.at(g)[((long long)b * a.H + h) * a.sq + qi] = m + logf(l);
  }
}

// D_i = dO_i . O_i per (b, h, i)
__global__ void attn_dd_kernel(AttnArgs a, const int* active) {
  if (stopped(active)) return;
  const int g = blockIdx.y;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)a.B * a.H * a.sq;
  if (idx >= total) return;
  const int i = (int)(idx % a.sq);
  const int h = (int)((idx / a.sq) % a.H);
  const int b = (int)(idx / ((long long)a.sq * a.H));
  const float* dO = a.dout.at(g) + (long long)(b * a.sq + i) * a.dout.ld + h * a.dh;
  const float* O = a.o.at(g) + (long long)(b * a.sq + i) * a.o.ld + h * a.dh;
  float acc = 0.f;
  for (int c = 0; c < a.dh; ++c) acc = fmaf(dO[c], O[c], acc);
  a.dd.at(g)[idx] = acc;
}

// dK, dV for 32 keys of one (b, h); loops over query tiles.
__global__ void __launch_bounds__(NT) attn_dkdv_kernel(AttnArgs a, const int* active) {
  __shared__ float Ks[BKV][MAXDH + 1];
  __shared__ float Vs[BKV][MAXDH + 1];
  __shared__ float Qs[BQ][MAXDH + 1];
  __shared__ float dOs[BQ][MAXDH + 1];
  __shared__ float Ps[BQ][BKV + 1];
  __shared__ float dSs[BQ][BKV + 1];
  __shared__ float lse_s[BQ], dd_s[BQ];
  if (stopped(active)) return;
  const int g = blockIdx.z;
  const int b = blockIdx.y / a.H, h = blockIdx.y % a.H;
  const int kv0 = blockIdx.x * BKV;
  const int tk = threadIdx.x >> 2, sub = threadIdx.x & 3;
  const int kj = kv0 + tk;
  const int dh = a.dh, col0 = h * dh;
  const float* Q = a.q.at(g) + (long long)b * a.sq * a.q.ld;
  const float* K = a.k.at(g) + (long long)b * a.skv * a.k.ld;
  const float* V = a.v.at(g) + (long long)b * a.skv * a.v.ld;
  const float* dO = a.dout.at(g) + (long long)b * a.sq * a.dout.ld;
  const float* lse = a.lse.at(g) + ((long long)b * a.H + h) * a.sq;
  const float* dd = a.dd.at(g) + ((long long)b * a.H + h) * a.sq;
  load_tile(Ks, K, a.k.ld, kv0, a.skv, col0, dh);
  load_tile(Vs, V, a.v.ld, kv0, a.skv, col0, dh);
  float dk[MAXDH / 4], dv[MAXDH / 4];
#pragma unroll
  for (int u = 0; u < MAXDH / 4; ++u) dk[u] = dv[u] = 0.f;
  const int qstart = a.causal ? (kv0 / BQ) * BQ : 0;
  for (int q0 = qstart; q0 < a.sq; q0 += BQ) {
    __syncthreads();
    load_tile(Qs, Q, a.q.ld, q0, a.sq, col0, dh);
    load_tile(dOs, dO, a.dout.ld, q0, a.sq, col0, dh);
    if (threadIdx.x < BQ) {
      const int qi = q0 + threadIdx.x;
      lse_s[threadIdx.x] = qi < a.sq ? lse[qi] : 0.f;
      dd_s[threadIdx.x] = qi < a.sq ? dd[qi] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < BQ / 4; ++t) {
      const int i = sub + 4 * t, qi = q0 + i;
      float sacc = 0.f, dpacc = 0.f;
      for (int c = 0; c < dh; ++c) {
        sacc = fmaf(Qs[i][c], Ks[tk][c], sacc);
        dpacc = fmaf(dOs[i][c], Vs[tk][c], dpacc);
      }
      const bool masked = qi >= a.sq || kj >= a.skv || (a.causal && kj > qi);
      const float p = masked ? 0.f : expf(sacc * a.scale - lse_s[i]);
      Ps[i][tk] = p;
      dSs[i][tk] = p * (dpacc - dd_s[i]);
    }
    __syncthreads();
    const int ncol = dh / 4;
    for (int u = 0; u < ncol; ++u) {
      const int c = sub + 4 * u;
      float av = dv[u], ak = dk[u];
      for (int i = 0; i < BQ; ++i) {
        av = fmaf(Ps[i][tk], dOs[i][c], av);
        ak = fmaf(dSs[i][tk], Qs[i][c], ak);
      }
      dv[u] = av;
      dk[u] = ak;
    }
  }
  if (kj < a.skv) {
    float* DK = a.dk.at(g) + (long long)(b * a.skv + kj) * a.dk.ld + col0;
    float* DV = a.dv.at(g) + (long long)(b * a.skv + kj) * a.dv.ld + col0;
    for (int u = 0; u < dh / 4; ++u) {
      DK[sub + 4 * u] = dk[u] * a.scale;
      DV[sub + 4 * u] = dv[u];
    }
  }
}

// dQ for 32 queries of one (b, h); loops over key tiles.
__global__ void __launch_bounds__(NT) attn_dq_kernel(AttnArgs a, const int* active) {
  __shared__ float Qs[BQ][MAXDH + 1];
  __shared__ float dOs[BQ][MAXDH + 1];
  __shared__ float Ks[BKV][MAXDH + 1];
  __shared__ float Vs[BKV][MAXDH + 1];
  __shared__ float dSs[BQ][BKV + 1];
  if (stopped(active)) return;
  const int g = blockIdx.z;
  const int b = blockIdx.y / a.H, h = blockIdx.y % a.H;
  const int q0 = blockIdx.x * BQ;
  const int tq = threadIdx.x >> 2, sub = threadIdx.x & 3;
  const int qi = q0 + tq;
  const int dh = a.dh, col0 = h * dh;
  const float* Q = a.q.at(g) + (long long)b * a.sq * a.q.ld;
  const float* K = a.k.at(g) + (long long)b * a.skv * a.k.ld;
  const float* V = a.v.at(g) + (long long)b * a.skv * a.v.ld;
  const float* dO = a.dout.at(g) + (long long)b * a.sq * a.dout.ld;
  load_tile(Qs, Q, a.q.ld, q0, a.sq, col0, dh);
  load_tile(dOs, dO, a.dout.ld, q0, a.sq, col0, dh);
  const float lse_i = qi < a.sq ? a.lse.at(g)[((long long)b * a.H + h) * a.sq + qi] : 0.f;
  const float dd_i = qi < a.sq ? a.dd.at(g)[((long long)b * a.H + h) * a.sq + qi] : 0.f;
  float dq[MAXDH / 4];
#pragma unroll
  for (int u = 0; u < MAXDH / 4; ++u) dq[u] = 0.f;
  int kv_end = a.skv;
  if (a.causal) kv_end = min(kv_end, q0 + BQ);
  for (int kv0 = 0; kv0 < kv_end; kv0 += BKV) {
    __syncthreads();
    load_tile(Ks, K, a.k.ld, kv0, a.skv, col0, dh);
    load_tile(Vs, V, a.v.ld, kv0, a.skv, col0, dh);
    __syncthreads();
#pragma unroll
    for (int t = 0; t < BKV / 4; ++t) {
      const int j = sub + 4 * t, kj = kv0 + j;
      float sacc = 0.f, dpacc = 0.f;
      for (int c = 0; c < dh; ++c) {
        sacc = fmaf(Qs[tq][c], Ks[j][c], sacc);
        dpacc = fmaf(dOs[tq][c], Vs[j][c], dpacc);
      }
      const bool masked = qi >= a.sq || kj >= a.skv || (a.causal && kj > qi);
      const float p = masked ? 0.f : expf(sacc * a.scale - lse_i);
      dSs[tq][j] = p * (dpacc - dd_i);
    }
    __syncwarp();
    const int ncol = dh / 4;
    for (int u = 0; u < ncol; ++u) {
      const int c = sub + 4 * u;
      float acc = dq[u];
      for (int j = 0; j < BKV; ++j) acc = fmaf(dSs[tq][j], Ks[j][c], acc);
      dq[u] = acc;
    }
  }
  if (qi < a.sq) {
    float* DQ = a.dq.at(g) + (long long)(b * a.sq + qi) * a.dq.ld + col0;
    for (int u = 0; u < dh / 4; ++u) DQ[sub + 4 * u] = dq[u] * a.scale;
  }
}

void check(const AttnArgs& a) {
  if (a.dh > MAXDH || a.dh % 4 != 0)
    throw ValidationError("attention: head width must be a multiple of 4 and <= 64");
}

}  // namespace

void launch_attn_fwd(const AttnArgs& a, const int* active, cudaStream_t s) {
  if (a.G == 0) return;
  check(a);
  dim3 grid(ceil_div(a.sq, BQ), a.B * a.H, a.G);
  attn_fwd_kernel<<<grid, NT, 0, s>>>(a, active);
}

void launch_attn_bwd(const AttnArgs& a, const int* active, cudaStream_t s) {
  if (a.G == 0) return;
  check(a);
  const long long rows = (long long)a.B * a.H * a.sq;
  attn_dd_kernel<<<dim3(ceil_div(rows, 256), a.G), 256, 0, s>>>(a, active);
  attn_dkdv_kernel<<<dim3(ceil_div(a.skv, BKV), a.B * a.H, a.G), NT, 0, s>>>(a, active);
  attn_dq_kernel<<<dim3(ceil_div(a.sq, BQ), a.B * a.H, a.G), NT, 0, s>>>(a, active);
}

}  // namespace mglp
