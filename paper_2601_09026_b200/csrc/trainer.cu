// Device training step: see trainer.h for the map to the reference.
#include "trainer.h"

#include <cstring>
#include <thread>

#include "rng.h"

namespace mglp {

namespace {

inline long long align32(long long n) { return (n + 31) & ~31LL; }

// ---- synthetic batches (tasks.cpp:33-89): integer-exact --------------------------
struct TaskDev {
  int kind, vocab, seq, split_size;
  uint64_t seed;
};

__device__ __forceinline__ int draw_token(const TaskDev& t, int split, long long sample, int pos) {
  const uint64_t bits = derive(t.seed, kRngData, (uint64_t)split, (uint64_t)sample, (uint64_t)pos);
  return 1 + (int)uniform_index(bits, (uint64_t)(t.vocab - 1));
}

__global__ void make_batch_kernel(TaskDev t, int split, long long start, int B, int* src, int* tin,
                                  int* tout) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= B * t.seq) return;
  const int j = i / t.seq, p = i % t.seq;
  const long long sample = (start + j) % t.split_size;
  const int s = draw_token(t, split, sample, p);
  src[i] = s;
  switch (t.kind) {
    case 0:  // copy_sequence
      tout[i] = s;
      break;
    case 1:  // token_classification: (token + left neighbour) mod vocab
      tout[i] = (s + (p > 0 ? draw_token(t, split, sample, p - 1) : 0)) % t.vocab;
      break;
    default: {  // tiny_translation: reversal, decoder input = start marker + shifted labels
      tout[i] = draw_token(t, split, sample, t.seq - 1 - p);
      tin[i] = p == 0 ? 0 : draw_token(t, split, sample, t.seq - p);
    }
  }
}

// ---- embedding (model.cpp:133-164): row r = j*S + t, tok + pos in f64 ---------
__global__ void embed_kernel(const int* toks, const double* tok, const double* pos, float* out,
                             int rows, int S, int d) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)rows * d) return;
  const int r = (int)(i / d), e = (int)(i % d);
  const int t = r % S;
  out[i] = (float)(tok[(long long)toks[r] * d + e] + pos[(long long)t * d + e]);
}

// stable bucketing of the token rows by id, so the embedding gradient sums
// each table row in (j, t) order: one block; thread v walks the tokens in row
// order and appends the rows holding v (tokens staged in shared memory)
__global__ void __launch_bounds__(1024) sort_tokens_kernel(const int* toks, int T, int V,
                                                           int* perm, int* offs) {
  extern __shared__ int sm[];  // [T] tokens + [V + 1] counts (when they fit)
  const bool staged = (T + V + 1) * 4 <= 48 * 1024;
  const int* tk = toks;
  int* cnt = offs;
  if (staged) {
    for (int r = threadIdx.x; r < T; r += blockDim.x) sm[r] = toks[r];
    cnt = sm + T;
    tk = sm;
  }
  for (int v = threadIdx.x; v <= V; v += blockDim.x) cnt[v] = 0;
  __syncthreads();
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    int c = 0;
    for (int r = 0; r < T; ++r) c += tk[r] == v;
    cnt[v + 1] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int v = 0; v < V; ++v) cnt[v + 1] += cnt[v];
    if (staged)
      for (int v = 0; v <= V; ++v) offs[v] = cnt[v];
  }
  __syncthreads();
  for (int v = threadIdx.x; v < V; v += blockDim.x) {
    int o = cnt[v];
    for (int r = 0; r < T; ++r)
      if (tk[r] == v) perm[o++] = r;
  }
}

// embed_backward (model.cpp:250-275): dtok[v] += sum over rows with token v,
// dpos[t] += sum over samples j; f64 running sums in the reference's order
__global__ void embed_bwd_tok_kernel(const int* perm, const int* offs, const float* lam, float* dtok,
                                     int V, int d) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)V * d) return;
  const int v = (int)(i / d), e = (int)(i % d);
  double acc = 0.0;
  for (int k = offs[v]; k < offs[v + 1]; ++k) acc += (double)lam[(long long)perm[k] * d + e];
  dtok[i] = (float)((double)dtok[i] + acc);
}

__global__ void embed_bwd_pos_kernel(const float* lam, float* dpos, int B, int S, int d) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)S * d) return;
  const int t = (int)(i / d), e = (int)(i % d);
  double acc = 0.0;
  for (int j = 0; j < B; ++j) acc += (double)lam[((long long)j * S + t) * d + e];
  dpos[i] = (float)((double)dpos[i] + acc);
}

// ---- cross-entropy (model.cpp:185-217): one warp per row, f64 -----------------
__global__ void cross_entropy_kernel(const float* logits, int ldv, const int* labels, int rows,
                                     int V, float* dl, double* row_loss, int want_dl) {
  const int r = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float* row = logits + (long long)r * ldv;
  double mx = -INFINITY;
  for (int c = lane; c < V; c += 32) mx = fmax(mx, (double)row[c]);
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  double z = 0.0;
  for (int c = lane; c < V; c += 32) z += exp((double)row[c] - mx);
  for (int o = 16; o > 0; o >>= 1) z += __shfl_xor_sync(0xffffffffu, z, o);
  const int label = labels[r];
  const double inv_n = 1.0 / (double)rows;
  if (lane == 0) row_loss[r] = (mx + log(z)) - (double)row[label];
  if (want_dl) {
    float* drow = dl + (long long)r * ldv;
    for (int c = lane; c < V; c += 32) {
      double g = exp((double)row[c] - mx) / z * inv_n;
      if (c == label) g -= inv_n;
      drow[c] = (float)g;
    }
  }
}

// mean over rows, summed in row order (model.cpp:211-216): the rows are
// staged through shared memory, one thread adds them up
__global__ void __launch_bounds__(1024) loss_sum_kernel(const double* row_loss, int rows,
                                                        double* out) {
  __shared__ double buf[1024];
  double s = 0.0;
  for (int base = 0; base < rows; base += 1024) {
    const int n = min(1024, rows - base);
    __syncthreads();
    if ((int)threadIdx.x < n) buf[threadIdx.x] = row_loss[base + threadIdx.x];
    __syncthreads();
    if (threadIdx.x == 0)
      for (int r = 0; r < n; ++r) s += buf[r];
  }
  if (threadIdx.x == 0) *out = s * (1.0 / (double)rows);
}

// accuracy (model.cpp:277-292): first maximum wins
__global__ void accuracy_kernel(const float* logits, int ldv, const int* labels, int rows, int V,
                                int* hits) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const float* row = logits + (long long)r * ldv;
  int best = 0;
  for (int c = 1; c < V; ++c)
    if (row[c] > row[best]) best = c;
  if (best == labels[r]) atomicAdd(hits, 1);
}

// ---- optimizer (optimizer.cpp:43-88), f64 masters; no contraction, like the
// reference's -ffp-contract=off build ----------------------------------------------
struct OptDev {
  int kind;
  double lr, b1, b2, eps, wd, mom, bc1, bc2;
};

__global__ void opt_kernel(OptDev o, long long n, double* p, double* m, double* v, const float* g,
                           float* p32) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const double ge = (double)g[i];
    double pe = p[i];
    if (o.kind == 0) {
      if (o.mom != 0.0) {
        const double me = __dadd_rn(__dmul_rn(o.mom, m[i]), ge);
        m[i] = me;
        pe = __dsub_rn(pe, __dmul_rn(o.lr, me));
      } else {
        pe = __dsub_rn(pe, __dmul_rn(o.lr, ge));
      }
    } else {
      const double me = __dadd_rn(__dmul_rn(o.b1, m[i]), __dmul_rn(1.0 - o.b1, ge));
      const double ve =
          __dadd_rn(__dmul_rn(o.b2, v[i]), __dmul_rn(__dmul_rn(1.0 - o.b2, ge), ge));
      m[i] = me;
      v[i] = ve;
      const double mhat = __ddiv_rn(me, o.bc1);
      const double vhat = __ddiv_rn(ve, o.bc2);
      double upd = __ddiv_rn(mhat, __dadd_rn(__dsqrt_rn(vhat), o.eps));
      if (o.kind == 2) upd = __dadd_rn(upd, __dmul_rn(o.wd, pe));
      pe = __dsub_rn(pe, __dmul_rn(o.lr, upd));
    }
    p[i] = pe;
    p32[i] = (float)pe;
  }
}

__global__ void cast_kernel(const double* src, float* dst, long long n) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    dst[i] = (float)src[i];
}

int blocks_for(long long n, int threads) {
  return (int)std::min<long long>(148LL * 16, (n + threads - 1) / threads);
}

Mat mat(float* p, int ld) {
  Mat m;
  m.ptr = p;
  m.ld = ld;
  return m;
}

// ---- MGLP v1 wire format (checkpoint.cpp:30-80) ----------------------------------
void put_u32(std::string& o, uint32_t v) { o.append(reinterpret_cast<const char*>(&v), 4); }
void put_u64(std::string& o, uint64_t v) { o.append(reinterpret_cast<const char*>(&v), 8); }
struct Reader {
  const std::string& s;
  size_t pos = 0;
  void need(size_t n) {
    if (pos + n > s.size()) throw ValidationError("checkpoint: truncated stream");
  }
  uint32_t u32() {
    need(4);
    uint32_t v;
    std::memcpy(&v, s.data() + pos, 4);
    pos += 4;
    return v;
  }
  uint64_t u64() {
    need(8);
    uint64_t v;
    std::memcpy(&v, s.data() + pos, 8);
    pos += 8;
    return v;
  }
};

}  // namespace

Trainer::Trainer(const StackDesc& sd, const SolveCfg& solve, int vocab, int max_seq,
                 const TaskDesc& task, const OptDesc& opt, int batch_size, uint64_t seed,
                 int device)
    : sd_(sd), task_(task), opt_(opt), seed_(seed) {
  if (vocab < 2) throw ValidationError("Model: vocab must be >= 2");
  if (max_seq < 1) throw ValidationError("Model: max_seq must be >= 1");
  if (task.vocab != vocab) throw ValidationError("train: task and model vocabularies differ");
  if (task.seq_len > max_seq)
    throw ValidationError("train: sequence longer than the position table");
  if ((task.kind == 2) != (sd.kind == 2))
    throw ValidationError(
        "train: translation needs an encoder-decoder model, and only translation feeds one");
  if (batch_size < 1) throw ValidationError("train: batch_size must be >= 1");
  if (opt.lr <= 0.0) throw ValidationError("Optimizer: lr must be positive");
  if (opt.beta1 < 0.0 || opt.beta1 >= 1.0 || opt.beta2 < 0.0 || opt.beta2 >= 1.0)
    throw ValidationError("Optimizer: betas must lie in [0, 1)");
  if (opt.eps <= 0.0) throw ValidationError("Optimizer: eps must be positive");
  V_ = vocab;
  S_ = max_seq;
  B_ = batch_size;
  T_ = batch_size * task.seq_len;
  d_ = sd.d;
  ldv_ = (vocab + 3) & ~3;
  two_stream_ = sd.kind == 2;
  eng_ = std::make_unique<Engine>(sd, solve, device, nullptr);
  s_ = eng_->stream();
  eng_->set_shape(batch_size, task.seq_len, two_stream_ ? task.seq_len : 0);

  // head slab (model.cpp:50-72), every piece 32-aligned
  long long off = 0;
  auto take = [&](long long n) {
    const long long o = off;
    off += align32(n);
    return o;
  };
  hl_.tok = take((long long)V_ * d_);
  hl_.pos = take((long long)S_ * d_);
  hl_.tok_out = two_stream_ ? take((long long)V_ * d_) : -1;
  hl_.pos_out = two_stream_ ? take((long long)S_ * d_) : -1;
  hl_.lnf_g = take(d_);
  hl_.lnf_b = take(d_);
  hl_.w = take((long long)V_ * d_);
  hl_.b = take(V_);
  hl_.size = off;

  // parameter shapes in param_tensors order: stack (visit_params), then head
  const long long d = d_, f = sd.ffn;
  auto lin = [&](long long out, long long in) {
    shapes_.push_back({out, in});
    shapes_.push_back({out});
  };
  auto ln = [&] {
    shapes_.push_back({d});
    shapes_.push_back({d});
  };
  auto attn = [&] {
    for (int q = 0; q < 4; ++q) lin(d, d);
  };
  for (int l = 0; l < eng_->total_layers(); ++l) {
    const bool dec = sd.kind == 2 && l >= sd.n_enc;
    ln();
    attn();
    if (dec) {
      ln();
      attn();
    }
    ln();
    lin(f, d);
    lin(d, f);
  }
  n_stack_flat_ = eng_->num_params();
  shapes_.push_back({V_, d});
  shapes_.push_back({S_, d});
  if (two_stream_) {
    shapes_.push_back({V_, d});
    shapes_.push_back({S_, d});
  }
  shapes_.push_back({d});
  shapes_.push_back({d});
  shapes_.push_back({V_, d});
  shapes_.push_back({V_});
  n_head_flat_ = 2LL * V_ * d + (long long)S_ * d + 2 * d + V_ +
                 (two_stream_ ? (long long)(V_ + S_) * d : 0);
  n_flat_ = n_stack_flat_ + n_head_flat_;

  MGLP_CUDA(cudaSetDevice(device));
  const long long ns = eng_->slab_elems();
  auto alloc = [&](auto** p, size_t n) {
    MGLP_CUDA(cudaMalloc(p, n * sizeof(**p)));
    MGLP_CUDA(cudaMemsetAsync(*p, 0, n * sizeof(**p), s_));
  };
  alloc(&H32_, hl_.size);
  alloc(&HG_, hl_.size);
  alloc(&Whl_, (size_t)V_ * pack_hl_cols(d_) + (size_t)d_ * pack_hl_cols(V_));
  alloc(&P64_, ns);
  alloc(&H64_, hl_.size);
  alloc(&Pm_, ns);
  alloc(&Pv_, ns);
  alloc(&Hm_, hl_.size);
  alloc(&Hv_, hl_.size);
  alloc(&src_, T_);
  alloc(&tin_, T_);
  alloc(&tout_, T_);
  alloc(&perm_, T_);
  alloc(&offs_, V_ + 1);
  alloc(&hits_, 1);
  const long long sn = eng_->state_elems();
  alloc(&z0_, sn);
  alloc(&lamN_, sn);
  alloc(&lam0_, sn);
  alloc(&n_, (size_t)T_ * d_);
  alloc(&stats_, (size_t)T_ * 2);
  alloc(&logits_, (size_t)T_ * ldv_);
  alloc(&dl_, (size_t)T_ * ldv_);
  alloc(&dn_, (size_t)T_ * d_);
  alloc(&row_loss_, T_);
  alloc(&loss_, 1);

  // Model(mcfg, seed): the stack init (blocks.cpp:432-449) and the head tables
  std::vector<double> flat((size_t)n_flat_);
  std::vector<double> stack_flat;
  eng_->init_params(seed, &stack_flat);
  std::copy(stack_flat.begin(), stack_flat.end(), flat.begin());
  std::vector<double> head_flat;
  init_head(seed, &head_flat);
  std::copy(head_flat.begin(), head_flat.end(), flat.begin() + n_stack_flat_);
  set_params(flat.data());
}

Trainer::~Trainer() {
  cudaStreamSynchronize(s_);
  for (void* p : {(void*)H32_, (void*)HG_, (void*)Whl_, (void*)P64_, (void*)H64_, (void*)Pm_,
                  (void*)Pv_, (void*)Hm_, (void*)Hv_, (void*)src_, (void*)tin_, (void*)tout_,
                  (void*)perm_, (void*)offs_, (void*)hits_, (void*)z0_, (void*)lamN_,
                  (void*)lam0_, (void*)n_, (void*)stats_, (void*)logits_, (void*)dl_,
                  (void*)dn_, (void*)row_loss_, (void*)loss_})
    if (p) cudaFree(p);
}

// init_table (model.cpp:40-45): truncated N(0, std^2) keyed by the tensor name
void Trainer::init_head(uint64_t seed, std::vector<double>* flat) {
  flat->assign((size_t)n_head_flat_, 0.0);
  constexpr uint64_t kHeadSlot = 1000000007ULL;
  const double sd = sd_.init_std;
  struct Table {
    const char* name;
    long long n;
    bool gain;
    bool zero;
  };
  std::vector<Table> tabs = {{"head.tok_embed", (long long)V_ * d_, false, false},
                             {"head.pos_embed", (long long)S_ * d_, false, false}};
  if (two_stream_) {
    tabs.push_back({"head.tok_embed_out", (long long)V_ * d_, false, false});
    tabs.push_back({"head.pos_embed_out", (long long)S_ * d_, false, false});
  }
  tabs.push_back({"ln_f.gain", d_, true, false});
  tabs.push_back({"ln_f.bias", d_, false, true});
  tabs.push_back({"head.out", (long long)V_ * d_, false, false});
  tabs.push_back({"head.b", V_, false, true});
  double* o = flat->data();
  for (const Table& t : tabs) {
    if (t.gain) {
      for (long long i = 0; i < t.n; ++i) o[i] = 1.0;
    } else if (!t.zero) {
      const uint64_t site = kHeadSlot * 1000003u + fnv1a(t.name);
      const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
      std::vector<std::thread> th;
      for (unsigned w = 0; w < nt; ++w)
        th.emplace_back([&, w] {
          for (long long i = w; i < t.n; i += nt)
            o[i] = truncated_gaussian(sd, seed, kRngInit, site, (uint64_t)i);
        });
      for (auto& x : th) x.join();
    }
    o += t.n;
  }
}

void Trainer::flat_to_head(const double* flat, double* slab) const {
  std::fill(slab, slab + hl_.size, 0.0);
  const long long vd = (long long)V_ * d_, sdd = (long long)S_ * d_;
  long long fo = 0;
  auto put = [&](long long off, long long n) {
    std::memcpy(slab + off, flat + fo, n * sizeof(double));
    fo += n;
  };
  put(hl_.tok, vd);
  put(hl_.pos, sdd);
  if (two_stream_) {
    put(hl_.tok_out, vd);
    put(hl_.pos_out, sdd);
  }
  put(hl_.lnf_g, d_);
  put(hl_.lnf_b, d_);
  put(hl_.w, vd);
  put(hl_.b, V_);
}

void Trainer::head_to_flat(const double* slab, double* flat) const {
  const long long vd = (long long)V_ * d_, sdd = (long long)S_ * d_;
  long long fo = 0;
  auto get = [&](long long off, long long n) {
    std::memcpy(flat + fo, slab + off, n * sizeof(double));
    fo += n;
  };
  get(hl_.tok, vd);
  get(hl_.pos, sdd);
  if (two_stream_) {
    get(hl_.tok_out, vd);
    get(hl_.pos_out, sdd);
  }
  get(hl_.lnf_g, d_);
  get(hl_.lnf_b, d_);
  get(hl_.w, vd);
  get(hl_.b, V_);
}

void Trainer::set_params(const double* flat) {
  std::vector<double> slab((size_t)eng_->slab_elems());
  eng_->flat_to_slab(flat, slab.data());
  MGLP_CUDA(cudaMemcpyAsync(P64_, slab.data(), slab.size() * sizeof(double),
                            cudaMemcpyHostToDevice, s_));
  std::vector<double> head((size_t)hl_.size);
  flat_to_head(flat + n_stack_flat_, head.data());
  MGLP_CUDA(cudaMemcpyAsync(H64_, head.data(), head.size() * sizeof(double),
                            cudaMemcpyHostToDevice, s_));
  sync_fp32();
  MGLP_CUDA(cudaStreamSynchronize(s_));
}

void Trainer::get_params(double* flat) const {
  std::vector<double> slab((size_t)eng_->slab_elems());
  MGLP_CUDA(cudaMemcpyAsync(slab.data(), P64_, slab.size() * sizeof(double),
                            cudaMemcpyDeviceToHost, s_));
  std::vector<double> head((size_t)hl_.size);
  MGLP_CUDA(cudaMemcpyAsync(head.data(), H64_, head.size() * sizeof(double),
                            cudaMemcpyDeviceToHost, s_));
  MGLP_CUDA(cudaStreamSynchronize(s_));
  eng_->slab_to_flat(slab.data(), flat);
  head_to_flat(head.data(), flat + n_stack_flat_);
}

void Trainer::get_grads(double* flat) const {
  std::vector<float> g32((size_t)eng_->slab_elems());
  MGLP_CUDA(cudaMemcpyAsync(g32.data(), eng_->grads_dev(), g32.size() * sizeof(float),
                            cudaMemcpyDeviceToHost, s_));
  std::vector<float> h32((size_t)hl_.size);
  MGLP_CUDA(cudaMemcpyAsync(h32.data(), HG_, h32.size() * sizeof(float), cudaMemcpyDeviceToHost,
                            s_));
  MGLP_CUDA(cudaStreamSynchronize(s_));
  std::vector<double> a(g32.begin(), g32.end()), b(h32.begin(), h32.end());
  eng_->slab_to_flat(a.data(), flat);
  head_to_flat(b.data(), flat + n_stack_flat_);
}

void Trainer::sync_fp32() {
  const long long ns = eng_->slab_elems();
  cast_kernel<<<blocks_for(ns, 256), 256, 0, s_>>>(P64_, eng_->params_dev(), ns);
  cast_kernel<<<blocks_for(hl_.size, 256), 256, 0, s_>>>(H64_, H32_, hl_.size);
  MGLP_CUDA(cudaGetLastError());
  eng_->params_updated();
  // head.w pre-split: logits (B = W, K = d) and dn = dlogits . W (B = W^T, K = V)
  const long long kd = pack_hl_cols(d_), kv = pack_hl_cols(V_);
  launch_pack_hl(H32_ + hl_.w, 0, d_, Whl_, 0, (int)kd, 1, V_, d_, false, s_,
                 eng_->range_flag());
  launch_pack_hl(H32_ + hl_.w, 0, d_, Whl_ + (long long)V_ * kd, 0, (int)kv, 1, d_, V_, true, s_,
                 eng_->range_flag());
}

void Trainer::make_batch(int split, long long start) {
  TaskDev t{task_.kind, task_.vocab, task_.seq_len,
            split == 0 ? task_.train_size : task_.val_size, task_.seed};
  if (t.split_size < 1) throw ValidationError("make_batch: empty split");
  make_batch_kernel<<<(T_ + 255) / 256, 256, 0, s_>>>(t, split, start, B_, src_, tin_, tout_);
  MGLP_CUDA(cudaGetLastError());
}

void Trainer::embed() {
  const long long n = (long long)T_ * d_;
  MGLP_CUDA(cudaMemsetAsync(z0_, 0, eng_->state_elems() * sizeof(float), s_));
  embed_kernel<<<(int)((n + 255) / 256), 256, 0, s_>>>(src_, H64_ + hl_.tok, H64_ + hl_.pos, z0_,
                                                        T_, task_.seq_len, d_);
  if (two_stream_)
    embed_kernel<<<(int)((n + 255) / 256), 256, 0, s_>>>(
        tin_, H64_ + hl_.tok_out, H64_ + hl_.pos_out, z0_ + eng_->y_offset(), T_, task_.seq_len, d_);
  MGLP_CUDA(cudaGetLastError());
}

// logits = LN_f(stream) . W^T + b (model.cpp:166-183); loss (and dlogits)
double Trainer::head_forward_loss(const float* zfin, bool want_dl) {
  const float* stream = zfin + (two_stream_ ? eng_->y_offset() : 0);
  LnFwdArgs ln;
  ln.rows = T_;
  ln.d = d_;
  ln.eps = (float)sd_.ln_eps;
  ln.x = mat(const_cast<float*>(stream), d_);
  ln.out = mat(n_, d_);
  ln.stats = mat(stats_, 2);
  ln.gain = mat(H32_ + hl_.lnf_g, 0);
  ln.bias = mat(H32_ + hl_.lnf_b, 0);
  launch_ln_fwd(ln, nullptr, s_);
  GemmArgs g;
  g.M = T_;
  g.N = V_;
  g.K = d_;
  g.A = mat(n_, d_);
  g.B = mat(H32_ + hl_.w, d_);
  g.Bhl = mat(Whl_, (int)pack_hl_cols(d_));
  g.ep.kind = EPI_STORE;
  g.ep.out1 = mat(logits_, ldv_);
  g.ep.bias = mat(H32_ + hl_.b, 0);
  g.range_flag = eng_->range_flag();
  launch_gemm_tc(g, nullptr, s_);
  cross_entropy_kernel<<<(T_ + 7) / 8, 256, 0, s_>>>(logits_, ldv_, tout_, T_, V_, dl_, row_loss_,
                                                      want_dl ? 1 : 0);
  loss_sum_kernel<<<1, 1024, 0, s_>>>(row_loss_, T_, loss_);
  MGLP_CUDA(cudaGetLastError());
  double loss = 0.0;
  MGLP_CUDA(cudaMemcpyAsync(&loss, loss_, sizeof(double), cudaMemcpyDeviceToHost, s_));
  MGLP_CUDA(cudaStreamSynchronize(s_));
  return loss;
}

// head_backward (model.cpp:219-248): head grads and lambda_N
void Trainer::head_backward(const float* zfin) {
  const float* stream = zfin + (two_stream_ ? eng_->y_offset() : 0);
  // db += colsum(dlogits); dW += dlogits^T . n
  ColRedArgs cb;
  cb.rows = T_;
  cb.cols = V_;
  cb.up = mat(dl_, ldv_);
  cb.dbias = mat(HG_ + hl_.b, 0);
  launch_colred(cb, nullptr, s_);
  GemmArgs w;
  w.M = V_;
  w.N = d_;
  w.K = T_;
  w.A = mat(dl_, ldv_);
  w.a_mn = true;
  w.B = mat(n_, d_);
  w.b_mn = true;
  w.ep.kind = EPI_GRAD_ACC;
  w.ep.out1 = mat(HG_ + hl_.w, d_);
  w.ep.gscale = 1.f;
  w.range_flag = eng_->range_flag();
  launch_gemm_tc(w, nullptr, s_);
  // dn = dlogits . W
  GemmArgs g;
  g.M = T_;
  g.N = d_;
  g.K = V_;
  g.A = mat(dl_, ldv_);
  g.B = mat(H32_ + hl_.w, d_);
  g.b_mn = true;
  g.Bhl = mat(Whl_ + (long long)V_ * pack_hl_cols(d_), (int)pack_hl_cols(V_));
  g.ep.kind = EPI_STORE;
  g.ep.out1 = mat(dn_, d_);
  g.range_flag = eng_->range_flag();
  launch_gemm_tc(g, nullptr, s_);
  // lambda on the advancing stream = LN_f^T dn; the other stream is zero
  MGLP_CUDA(cudaMemsetAsync(lamN_, 0, eng_->state_elems() * sizeof(float), s_));
  LnBwdArgs lb;
  lb.rows = T_;
  lb.d = d_;
  lb.x = mat(const_cast<float*>(stream), d_);
  lb.stats = mat(stats_, 2);
  lb.up = mat(dn_, d_);
  lb.gain = mat(H32_ + hl_.lnf_g, 0);
  lb.out1 = mat(lamN_ + (two_stream_ ? eng_->y_offset() : 0), d_);
  launch_ln_bwd(lb, nullptr, s_);
  ColRedArgs cg;
  cg.rows = T_;
  cg.cols = d_;
  cg.up = mat(dn_, d_);
  cg.x = mat(const_cast<float*>(stream), d_);
  cg.stats = mat(stats_, 2);
  cg.dgain = mat(HG_ + hl_.lnf_g, 0);
  cg.dbias = mat(HG_ + hl_.lnf_b, 0);
  launch_colred(cg, nullptr, s_);
}

void Trainer::embed_backward(const float* lam0) {
  auto scatter = [&](const int* toks, const float* lam, long long tok_off, long long pos_off) {
    const int shm = (T_ + V_ + 1) * 4 <= 48 * 1024 ? (T_ + V_ + 1) * 4 : 0;
    sort_tokens_kernel<<<1, 1024, shm, s_>>>(toks, T_, V_, perm_, offs_);
    const long long nv = (long long)V_ * d_, np = (long long)task_.seq_len * d_;
    embed_bwd_tok_kernel<<<(int)((nv + 255) / 256), 256, 0, s_>>>(perm_, offs_, lam, HG_ + tok_off,
                                                                  V_, d_);
    embed_bwd_pos_kernel<<<(int)((np + 255) / 256), 256, 0, s_>>>(lam, HG_ + pos_off, B_,
                                                                  task_.seq_len, d_);
    MGLP_CUDA(cudaGetLastError());
  };
  scatter(src_, lam0, hl_.tok, hl_.pos);
  if (two_stream_) scatter(tin_, lam0 + eng_->y_offset(), hl_.tok_out, hl_.pos_out);
}

void Trainer::optimizer_step() {
  ++t_;
  OptDev o;
  o.kind = opt_.kind;
  o.lr = opt_.lr;
  o.b1 = opt_.beta1;
  o.b2 = opt_.beta2;
  o.eps = opt_.eps;
  o.wd = opt_.weight_decay;
  o.mom = opt_.momentum;
  o.bc1 = 1.0 - std::pow(opt_.beta1, (double)t_);
  o.bc2 = 1.0 - std::pow(opt_.beta2, (double)t_);
  const long long ns = eng_->slab_elems();
  opt_kernel<<<blocks_for(ns, 256), 256, 0, s_>>>(o, ns, P64_, Pm_, Pv_, eng_->grads_dev(),
                                                  eng_->params_dev());
  opt_kernel<<<blocks_for(hl_.size, 256), 256, 0, s_>>>(o, hl_.size, H64_, Hm_, Hv_, HG_, H32_);
  MGLP_CUDA(cudaGetLastError());
  eng_->params_updated();
  const long long kd = pack_hl_cols(d_), kv = pack_hl_cols(V_);
  launch_pack_hl(H32_ + hl_.w, 0, d_, Whl_, 0, (int)kd, 1, V_, d_, false, s_,
                 eng_->range_flag());
  launch_pack_hl(H32_ + hl_.w, 0, d_, Whl_ + (long long)V_ * kd, 0, (int)kv, 1, d_, V_, true, s_,
                 eng_->range_flag());
}

double Trainer::update(long long k, bool parallel, bool apply) {
  MGLP_CUDA(cudaSetDevice(eng_->device()));
  make_batch(0, k * B_);
  // frozen masks of batch k (training.cpp:209-210); no-op without dropout
  eng_->refresh_dropout(seed_, (uint64_t)k);
  embed();
  Engine& e = *eng_;
  if (parallel)
    e.forward_device(z0_);
  else
    e.serial_forward_device(z0_);
  const float* zfin = e.traj_dev() + (long long)e.total_layers() * e.state_elems();
  e.zero_grads();
  MGLP_CUDA(cudaMemsetAsync(HG_, 0, hl_.size * sizeof(float), s_));
  const double loss = head_forward_loss(zfin, true);
  head_backward(zfin);
  if (parallel)
    e.backward_device(lamN_, lam0_, true, true);
  else
    e.serial_adjoint_device(lamN_, lam0_, true);
  embed_backward(lam0_);
  if (apply) optimizer_step();
  // the factors of this update's traces into the monitor's summary (device)
  if (parallel && e.monitor_on()) e.monitor_record(-1);
  MGLP_CUDA(cudaStreamSynchronize(s_));
  eng_->check_range();
  return loss;
}

ProbeOutcome Trainer::update_probe(long long k, bool use_probe_gradient) {
  Engine& e = *eng_;
  if (!e.monitor_on()) throw ValidationError("update_probe: attach the monitor first");
  ProbeOutcome o;
  if (use_probe_gradient) {
    e.monitor_probe(true);
    o.loss = update(k, true, true);
    e.monitor_probe(false);
    e.monitor_record(k);
    const MonitorSummary& m = e.monitor_read();
    o.fwd_iters = m.used[0];  // the doubled budget the update ran with
    o.bwd_iters = m.used[1];
    o.fwd_factor = m.last_ff;
    o.bwd_factor = m.last_bf;
    o.decision = m.last_decision;
    o.switched = m.switched;
    return o;
  }
  const long long snap = e.snapshot();
  e.monitor_probe(true);
  update(k, true, false);
  e.monitor_probe(false);
  e.restore(snap);
  e.monitor_record(k);
  const MonitorSummary& m = e.monitor_read();
  o.fwd_factor = m.last_ff;
  o.bwd_factor = m.last_bf;
  o.decision = m.last_decision;
  o.switched = m.switched;
  o.fwd_iters = m.budget[0];
  o.bwd_iters = m.budget[1];
  o.loss = update(k, true, true);
  return o;
}

int Trainer::correct_predictions() {
  MGLP_CUDA(cudaMemsetAsync(hits_, 0, sizeof(int), s_));
  accuracy_kernel<<<(T_ + 255) / 256, 256, 0, s_>>>(logits_, ldv_, tout_, T_, V_, hits_);
  int h = 0;
  MGLP_CUDA(cudaMemcpyAsync(&h, hits_, sizeof(int), cudaMemcpyDeviceToHost, s_));
  MGLP_CUDA(cudaStreamSynchronize(s_));
  return h;
}

double Trainer::evaluate() {
  MGLP_CUDA(cudaSetDevice(eng_->device()));
  eng_->clear_dropout();  // the exact map (training.cpp:296-300)
  const int vb = task_.val_size / B_;
  double acc = 0.0;
  Engine& e = *eng_;
  for (int i = 0; i < vb; ++i) {
    make_batch(1, (long long)i * B_);
    embed();
    e.serial_forward_device(z0_);
    const float* zfin = e.traj_dev() + (long long)e.total_layers() * e.state_elems();
    head_forward_loss(zfin, false);
    acc += (double)correct_predictions() / (double)T_;
  }
  eng_->check_range();
  return acc / vb;
}

void Trainer::read_batch(int split, long long start, int* src, int* tin, int* tout) {
  make_batch(split, start);
  MGLP_CUDA(cudaMemcpyAsync(src, src_, T_ * sizeof(int), cudaMemcpyDeviceToHost, s_));
  if (tin) MGLP_CUDA(cudaMemcpyAsync(tin, tin_, T_ * sizeof(int), cudaMemcpyDeviceToHost, s_));
  MGLP_CUDA(cudaMemcpyAsync(tout, tout_, T_ * sizeof(int), cudaMemcpyDeviceToHost, s_));
  MGLP_CUDA(cudaStreamSynchronize(s_));
}

void Trainer::read_logits(float* out) const {
  MGLP_CUDA(cudaMemcpy2DAsync(out, V_ * sizeof(float), logits_, ldv_ * sizeof(float),
                              V_ * sizeof(float), T_, cudaMemcpyDeviceToHost, s_));
  MGLP_CUDA(cudaStreamSynchronize(s_));
}

// ---- checkpoint (checkpoint.cpp:88-180) ---------------------------------------------
std::string Trainer::save_checkpoint(long long batch, const std::string& echo) const {
  std::vector<double> p((size_t)n_flat_), m, v;
  get_params(p.data());
  const bool adam = opt_.kind != 0;
  const bool momentum = opt_.kind == 0 && opt_.momentum != 0.0;
  auto bank = [&](const double* slab, const double* head, std::vector<double>* out) {
    std::vector<double> a((size_t)eng_->slab_elems()), b((size_t)hl_.size);
    MGLP_CUDA(cudaMemcpyAsync(a.data(), slab, a.size() * sizeof(double), cudaMemcpyDeviceToHost, s_));
    MGLP_CUDA(cudaMemcpyAsync(b.data(), head, b.size() * sizeof(double), cudaMemcpyDeviceToHost, s_));
    MGLP_CUDA(cudaStreamSynchronize(s_));
    out->assign((size_t)n_flat_, 0.0);
    eng_->slab_to_flat(a.data(), out->data());
    head_to_flat(b.data(), out->data() + n_stack_flat_);
  };
  if (adam || momentum) bank(Pm_, Hm_, &m);
  if (adam) bank(Pv_, Hv_, &v);
  std::string o;
  o.append("MGLP", 4);
  put_u32(o, 1);
  put_u64(o, echo.size());
  o.append(echo);
  put_u64(o, (uint64_t)batch);
  auto tensors = [&](const std::vector<double>& flat) {
    put_u32(o, (uint32_t)shapes_.size());
    long long fo = 0;
    for (const auto& sh : shapes_) {
      put_u32(o, (uint32_t)sh.size());
      long long n = 1;
      for (long long dd : sh) {
        put_u64(o, (uint64_t)dd);
        n *= dd;
      }
      o.append(reinterpret_cast<const char*>(flat.data() + fo), (size_t)n * sizeof(double));
      fo += n;
    }
  };
  tensors(p);
  o.push_back((char)1);  // has optimizer
  put_u64(o, (uint64_t)t_);
  if (adam || momentum)
    tensors(m);
  else
    put_u32(o, 0);
  if (adam)
    tensors(v);
  else
    put_u32(o, 0);
  return o;
}

CheckpointMeta Trainer::load_checkpoint(const std::string& blob) {
  Reader r{blob};
  r.need(4);
  if (std::memcmp(blob.data(), "MGLP", 4) != 0) throw ValidationError("checkpoint: bad magic");
  r.pos = 4;
  CheckpointMeta meta;
  meta.version = r.u32();
  if (meta.version != 1) throw ValidationError("checkpoint: unsupported version");
  const uint64_t elen = r.u64();
  r.need(elen);
  meta.config_echo.assign(blob.data() + r.pos, elen);
  r.pos += elen;
  meta.batch = (long long)r.u64();
  auto tensors = [&](std::vector<double>* flat, const char* what) {
    flat->assign((size_t)n_flat_, 0.0);
    long long fo = 0;
    for (const auto& sh : shapes_) {
      const uint32_t rank = r.u32();
      if (rank != sh.size())
        throw ValidationError(std::string("checkpoint: rank mismatch for ") + what);
      long long n = 1;
      for (long long dd : sh) {
        if (r.u64() != (uint64_t)dd)
          throw ValidationError(std::string("checkpoint: shape mismatch for ") + what);
        n *= dd;
      }
      r.need((size_t)n * 8);
      std::memcpy(flat->data() + fo, blob.data() + r.pos, (size_t)n * 8);
      r.pos += (size_t)n * 8;
      fo += n;
    }
  };
  if (r.u32() != shapes_.size()) throw ValidationError("checkpoint: parameter count mismatch");
  std::vector<double> p;
  tensors(&p, "parameter");
  r.need(1);
  meta.has_optimizer = blob[r.pos++] != 0;
  set_params(p.data());
  if (!meta.has_optimizer) return meta;
  const uint64_t steps = r.u64();
  const bool adam = opt_.kind != 0;
  const bool momentum = opt_.kind == 0 && opt_.momentum != 0.0;
  auto bank = [&](bool present, double* slab, double* head, const char* name) {
    const uint32_t stored = r.u32();
    if (stored != (present ? shapes_.size() : 0u))
      throw ValidationError(std::string("checkpoint: optimizer ") + name +
                            " bank size mismatch (wrong optimizer kind for this file?)");
    if (!present) return;
    std::vector<double> flat;
    auto get_one = [&] {
      flat.assign((size_t)n_flat_, 0.0);
      long long fo = 0;
      for (const auto& sh : shapes_) {
        if (r.u32() != sh.size()) throw ValidationError(std::string("checkpoint: rank mismatch for ") + name);
        long long n = 1;
        for (long long dd : sh) {
          if (r.u64() != (uint64_t)dd)
            throw ValidationError(std::string("checkpoint: shape mismatch for ") + name);
          n *= dd;
        }
        r.need((size_t)n * 8);
        std::memcpy(flat.data() + fo, blob.data() + r.pos, (size_t)n * 8);
        r.pos += (size_t)n * 8;
        fo += n;
      }
    };
    get_one();
    std::vector<double> a((size_t)eng_->slab_elems()), b((size_t)hl_.size);
    eng_->flat_to_slab(flat.data(), a.data());
    flat_to_head(flat.data() + n_stack_flat_, b.data());
    MGLP_CUDA(cudaMemcpyAsync(slab, a.data(), a.size() * sizeof(double), cudaMemcpyHostToDevice, s_));
    MGLP_CUDA(cudaMemcpyAsync(head, b.data(), b.size() * sizeof(double), cudaMemcpyHostToDevice, s_));
    MGLP_CUDA(cudaStreamSynchronize(s_));
  };
  // attach() semantics: moments reset, then overwritten by the stored banks
  MGLP_CUDA(cudaMemsetAsync(Pm_, 0, eng_->slab_elems() * sizeof(double), s_));
  MGLP_CUDA(cudaMemsetAsync(Pv_, 0, eng_->slab_elems() * sizeof(double), s_));
  MGLP_CUDA(cudaMemsetAsync(Hm_, 0, hl_.size * sizeof(double), s_));
  MGLP_CUDA(cudaMemsetAsync(Hv_, 0, hl_.size * sizeof(double), s_));
  bank(adam || momentum, Pm_, Hm_, "first-moment");
  bank(adam, Pv_, Hv_, "second-moment");
  t_ = (long long)steps;
  return meta;
}

}  // namespace mglp
