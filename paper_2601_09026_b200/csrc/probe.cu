// Lipschitz probe of every layer's residual map on the device: the
// reference's estimate_lipschitz / estimate_stack (lipschitz.cpp:53-149).
//
// For layer l and sample i the reference draws a base point
// x_i = input_scale * N(layer_seed, kProbeInput, i, e) and a perturbation
// delta_i = delta_scale * N(layer_seed, kProbeDelta, i, e) over one [1, seq_len,
// d] sequence (e = flat element index), evaluates F(x_i) and F(x_i + delta_i)
// and keeps max_i ||F(x_i + delta_i) - F(x_i)|| / ||delta_i||. Here all samples
// of a layer are one batch (two residual evaluations per layer: base points
// and perturbed points as a family of G = 2 states), the draws come from the
// same counter-based generator on the device (rng.h), and the per-sample norms
// are f64 block reductions in a fixed order. Decoder layers of an
// encoder-decoder stack see a frozen context stream shared by all samples
// (lipschitz.cpp:105-114). The estimate is an fp32 finite difference of fp32
// evaluations: it tracks the f64 reference to ~1e-4 relative for delta ~ 1e-2.
#include <algorithm>
#include <memory>
#include <vector>

#include "engine.h"
#include "rng.h"

namespace mglp {

namespace {

constexpr uint64_t kProbeInput = 4, kProbeDelta = 5;  // rng.hpp:37-38

__device__ __forceinline__ double u01_d(uint64_t bits) { return (double)(bits >> 11) * 0x1.0p-53; }

// rng.hpp:75-83 (Box-Muller with two counters per value)
__device__ __forceinline__ double gaussian_d(uint64_t seed, uint64_t a, uint64_t b, uint64_t c) {
  const uint64_t k1 = derive(seed, a, b, c, 0);
  const uint64_t k2 = splitmix64(k1 ^ 0x452821e638d01377ULL);
  double x1 = u01_d(k1);
  const double x2 = u01_d(k2);
  if (x1 <= 0.0) x1 = 0x1.0p-53;
  return sqrt(-2.0 * log(x1)) * cos(6.283185307179586 * x2);
}

struct FillArgs {
  float* z;            // two states: base points, perturbed points
  long long state_n;   // floats per state
  long long adv_off;   // offset of the advancing stream
  long long ctx_off;   // offset of the context stream (-1: none)
  long long per;       // elements per sample (seq_len * d)
  int samples, i0;     // this chunk: samples [i0, i0 + samples)
  uint64_t seed;
  double input_scale, delta_scale;
};

__global__ void probe_fill_kernel(FillArgs a) {
  const long long n = (long long)a.samples * a.per;
  for (long long k = (long long)blockIdx.x * blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x) {
    const long long i = k / a.per, e = k - i * a.per;
    const uint64_t si = (uint64_t)(a.i0 + i);
    const double x = a.input_scale * gaussian_d(a.seed, kProbeInput, si, (uint64_t)e);
    const double dl = a.delta_scale * gaussian_d(a.seed, kProbeDelta, si, (uint64_t)e);
    a.z[a.adv_off + k] = (float)x;
    a.z[a.state_n + a.adv_off + k] = (float)(x + dl);
    if (a.ctx_off >= 0) {
      // one frozen context for every sample, keyed past the advancing stream
      const float c = (float)gaussian_d(a.seed, kProbeInput, 0, (uint64_t)(a.per + e));
      a.z[a.ctx_off + k] = c;
      a.z[a.state_n + a.ctx_off + k] = c;
    }
  }
}

struct RatioArgs {
  const float* F;  // two states of residuals
  long long state_n, adv_off, per;
  int i0;
  uint64_t seed;
  double delta_scale;
  double* ratios;  // [samples of this chunk]
};

// one block per sample: ||F(x + delta) - F(x)|| / ||delta|| (the denominator
// from the f64 draws, as the reference)
__global__ void __launch_bounds__(256) probe_ratio_kernel(RatioArgs a) {
  __shared__ double sn[256], sd[256];
  const int i = blockIdx.x;
  const uint64_t si = (uint64_t)(a.i0 + i);
  const float* f0 = a.F + a.adv_off + (long long)i * a.per;
  const float* f1 = f0 + a.state_n;
  double num = 0.0, den = 0.0;
  for (long long e = threadIdx.x; e < a.per; e += blockDim.x) {
    const double d = (double)f1[e] - (double)f0[e];
    num += d * d;
    const double dl = a.delta_scale * gaussian_d(a.seed, kProbeDelta, si, (uint64_t)e);
    den += dl * dl;
  }
  sn[threadIdx.x] = num;
  sd[threadIdx.x] = den;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) {
      sn[threadIdx.x] += sn[threadIdx.x + s];
      sd[threadIdx.x] += sd[threadIdx.x + s];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) a.ratios[i] = sd[0] > 0.0 ? sqrt(sn[0]) / sqrt(sd[0]) : 0.0;
}

}  // namespace

void lipschitz_probe(const Engine& src, int samples, double delta_scale, double input_scale,
                     int seq_len, uint64_t seed, const std::vector<int>& layers,
                     std::vector<double>* est) {
  if (samples < 1) throw ValidationError("estimate_lipschitz: need at least one sample");
  if (seq_len < 1) throw ValidationError("estimate_lipschitz: seq_len must be positive");
  const StackDesc& sd = src.stack_desc();
  for (int l : layers)
    if (l < 0 || l >= src.total_layers())
      throw ValidationError("estimate_lipschitz: layer out of range");
  // an eval-only engine with the source's parameters; samples are the batch
  // (chunked to bound the activation scratch)
  Engine pe(sd, src.config(), src.device(), nullptr);
  pe.set_eval_only(true);
  MGLP_CUDA(cudaMemcpy(pe.params_dev(), src.params_dev(), (size_t)src.slab_elems() * sizeof(float),
                       cudaMemcpyDeviceToDevice));
  pe.params_updated();
  const bool encdec = sd.kind == 2;
  const int chunk = std::max(1, std::min(samples, 16384 / seq_len));
  pe.set_shape(chunk, seq_len, encdec ? seq_len : 0);
  const long long sn = pe.state_elems();
  float *z = nullptr, *F = nullptr;
  double* ratios = nullptr;
  MGLP_CUDA(cudaMalloc(&z, (size_t)2 * sn * sizeof(float)));
  MGLP_CUDA(cudaMalloc(&F, (size_t)2 * sn * sizeof(float)));
  MGLP_CUDA(cudaMalloc(&ratios, (size_t)chunk * sizeof(double)));
  std::vector<double> host(chunk);
  cudaStream_t s = pe.stream();
  est->assign(layers.size(), 0.0);
  try {
    for (size_t li = 0; li < layers.size(); ++li) {
      const int layer = layers[li];
      const bool enc_phase = !encdec || layer < pe.n_split();
      const uint64_t layer_seed = derive(seed, kProbeInput, (uint64_t)layer, 0, 1);
      double best = 0.0;  // max over samples (lipschitz.cpp:44-48)
      for (int i0 = 0; i0 < samples; i0 += chunk) {
        const int nb = std::min(chunk, samples - i0);
        MGLP_CUDA(cudaMemsetAsync(z, 0, (size_t)2 * sn * sizeof(float), s));
        FillArgs fa;
        fa.z = z;
        fa.state_n = sn;
        fa.adv_off = enc_phase ? 0 : pe.y_offset();
        fa.ctx_off = (encdec && !enc_phase) ? 0 : -1;
        fa.per = (long long)seq_len * sd.d;
        fa.samples = nb;
        fa.i0 = i0;
        fa.seed = layer_seed;
        fa.input_scale = input_scale;
        fa.delta_scale = delta_scale;
        const long long n = (long long)nb * fa.per;
        probe_fill_kernel<<<(int)std::min<long long>((n + 255) / 256, 148 * 32), 256, 0, s>>>(fa);
        MGLP_CUDA(cudaGetLastError());
        pe.residual_device(layer, z, 2, F);
        RatioArgs ra;
        ra.F = F;
        ra.state_n = sn;
        ra.adv_off = fa.adv_off;
        ra.per = fa.per;
        ra.i0 = i0;
        ra.seed = layer_seed;
        ra.delta_scale = delta_scale;
        ra.ratios = ratios;
        probe_ratio_kernel<<<nb, 256, 0, s>>>(ra);
        MGLP_CUDA(cudaGetLastError());
        MGLP_CUDA(cudaMemcpyAsync(host.data(), ratios, (size_t)nb * sizeof(double),
                                  cudaMemcpyDeviceToHost, s));
        MGLP_CUDA(cudaStreamSynchronize(s));
        for (int i = 0; i < nb; ++i) best = std::max(best, host[i]);
      }
      (*est)[li] = best;
    }
  } catch (...) {
    cudaFree(z);
    cudaFree(F);
    cudaFree(ratios);
    throw;
  }
  cudaFree(z);
  cudaFree(F);
  cudaFree(ratios);
}

}  // namespace mglp
