// Plain fp32 CUDA-core GEMM with the same operand families and fused
// epilogues as the tensor-core path. It is NOT on the product path: the
// engine always runs gemm_tc.cu; this kernel exists so tests can check the
// tcgen05 kernel (and its epilogues) against an independent fp32 GEMM on the
// device (tests/test_gemm.py).
#include "kernels.cuh"

namespace mglp {

namespace {

constexpr int BM = 64, BN = 64, BK = 16;

__global__ void __launch_bounds__(256) gemm_simt_kernel(GemmArgs a, const int* active) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  __shared__ double red[32];
  if (active && *(volatile const int*)active == 0) return;
  const int z = blockIdx.z;
  const int hh = z % a.H, bb = (z / a.H) % a.Bb, g = z / (a.H * a.Bb);
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const float* A = a.A.at(g, bb, hh);
  const float* B = a.B.at(g, bb, hh);
  float acc[4][4] = {};
  for (int k0 = 0; k0 < a.K; k0 += BK) {
    // 64x16 tiles, 4 elements per thread
    for (int e = threadIdx.x; e < BM * BK; e += 256) {
      int mm, kk;
      if (a.a_mn) { kk = e / BM; mm = e % BM; } else { mm = e / BK; kk = e % BK; }
      const int m = m0 + mm, k = k0 + kk;
      float v = 0.f;
      if (m < a.M && k < a.K) v = a.a_mn ? A[(long long)k * a.A.ld + m] : A[(long long)m * a.A.ld + k];
      As[kk][mm] = v;
    }
    for (int e = threadIdx.x; e < BN * BK; e += 256) {
      int nn, kk;
      if (a.b_mn) { kk = e / BN; nn = e % BN; } else { nn = e / BK; kk = e % BK; }
      const int n = n0 + nn, k = k0 + kk;
      float v = 0.f;
      if (n < a.N && k < a.K) v = a.b_mn ? B[(long long)k * a.B.ld + n] : B[(long long)n * a.B.ld + k];
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
  double r2 = 0.0;
  const int col0 = n0 + tx * 4;
  const int nvalid = min(4, a.N - col0);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + ty * 4 + i;
    if (row < a.M && nvalid > 0) r2 += epilogue_row(a.ep, g, bb, hh, row, col0, acc[i], nvalid);
  }
  if (a.ep.kind == EPI_FINAL && a.ep.cmb.mode == CM_RES0) {
    for (int o = 16; o > 0; o >>= 1) r2 += __shfl_xor_sync(0xffffffffu, r2, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) red[w] = r2;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int i = 0; i < 8; ++i) t += red[i];
      a.ep.cmb.norm_partials[a.ep.cmb.norm_base + blockIdx.z * a.ep.cmb.norm_member_stride +
                             blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
  }
}

}  // namespace

int gemm_simt_blocks(const GemmArgs& a) {
  return ceil_div(a.N, BN) * ceil_div(a.M, BM) * a.G * a.Bb * a.H;
}

void launch_gemm_simt(const GemmArgs& a, const int* active, cudaStream_t s) {
  if (a.G == 0 || a.M == 0 || a.N == 0) return;
  dim3 grid(ceil_div(a.N, BN), ceil_div(a.M, BM), a.G * a.Bb * a.H);
  gemm_simt_kernel<<<grid, 256, 0, s>>>(a, active);
}

}  // namespace mglp
