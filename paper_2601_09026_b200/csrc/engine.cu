// Host orchestration of the device-resident MGRIT forward solve and adjoint
// MGRIT backpropagation. See engine.h for the map to the reference.
#include "engine.h"
#include "rng.h"
#include "vmm.h"

#include <algorithm>
#include <atomic>
#include <climits>
#include <map>
#include <mutex>
#include <cmath>
#include <cstring>
#include <thread>

namespace mglp {

namespace {

inline long long align32(long long n) { return (n + 31) & ~31LL; }

bool depth_scaled_component(const std::string& c) {  // blocks.cpp:368-372
  return c == "attn.v.w" || c == "attn.o.w" || c == "self.v.w" || c == "self.o.w" ||
         c == "cross.v.w" || c == "cross.o.w" || c == "mlp.in.w" || c == "mlp.out.w";
}

Mat state_mat(float* base, long long n, int d, int slot0, int step) {
  Mat m;
  m.ptr = base;
  m.slot_stride = n;
  m.ld = d;
  m.slot0 = slot0;
  m.step = step;
  return m;
}

Mat shift(Mat m, int g0) {
  m.slot0 += g0 * m.step;
  return m;
}

}  // namespace

void rng_gaussian_fill(uint64_t seed, uint64_t a, uint64_t b, double scale, double* out,
                       long long n) {
  const unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t)
    th.emplace_back([=] {
      for (long long i = t; i < n; i += nt) out[i] = scale * gaussian(seed, a, b, (uint64_t)i, 0);
    });
  for (auto& x : th) x.join();
}

// =============================================================================
// construction, parameters
// =============================================================================

Engine::Engine(const StackDesc& sd, const SolveCfg& cfg, int device,
               std::shared_ptr<Transport> tr)
    : sd_(sd), cfg_(cfg), device_(device), tr_(std::move(tr)) {
  if (sd_.d <= 0 || sd_.heads <= 0 || sd_.ffn <= 0)
    throw ValidationError("LayerStack: width, heads, ffn must be positive");
  if (sd_.d % sd_.heads != 0) throw ValidationError("LayerStack: head count must divide width");
  if (sd_.d % 4 != 0 || sd_.ffn % 4 != 0)
    throw ValidationError("device stack: width and ffn must be multiples of 4");
  if ((sd_.d / sd_.heads) % 4 != 0 || sd_.d / sd_.heads > 64)
    throw ValidationError("device stack: head width must be a multiple of 4 and <= 64");
  switch (sd_.kind) {
    case 0:
      if (sd_.n_enc <= 0) throw ValidationError("LayerStack: n_enc must be positive");
      total_ = n_split_ = sd_.n_enc;
      break;
    case 1:
      if (sd_.n_dec <= 0) throw ValidationError("LayerStack: n_dec must be positive");
      total_ = n_split_ = sd_.n_dec;
      causal_ = true;
      break;
    case 2:
      if (sd_.n_enc <= 0 || sd_.n_dec <= 0)
        throw ValidationError("LayerStack: encoder-decoder needs both n_enc and n_dec");
      total_ = sd_.n_enc + sd_.n_dec;
      n_split_ = sd_.n_enc;
      break;
    default:
      throw ValidationError("LayerStack: unknown model kind");
  }
  if (sd_.buffer_open < 0 || sd_.buffer_close < 0 ||
      sd_.buffer_open + sd_.buffer_close >= total_)
    throw ValidationError("LayerStack: buffer layers must leave a non-empty interior");
  ib_ = sd_.buffer_open;
  ie_ = total_ - sd_.buffer_close;
  N_ = ie_ - ib_;
  h_.assign(total_, sd_.base_h);  // blocks.cpp:421-430
  if (sd_.buffer_open + sd_.buffer_close > 0)
    for (int i = 0; i < total_; ++i)
      h_[i] = (i < ib_ || i >= ie_) ? 1.0 : 1.0 / static_cast<double>(N_);
  // MgritSolver construction checks (mgrit.hpp:68-95)
  if (cfg_.coarsen < 2) throw ValidationError("MgritSolver: coarsening factor must be >= 2");
  if (cfg_.levels < 1) throw ValidationError("MgritSolver: need at least one level");
  long long stride = 1;
  for (int l = 0; l < std::max(cfg_.levels - 1, 1); ++l) {
    stride *= cfg_.coarsen;
    if (stride > N_)
      throw ValidationError("MgritSolver: too many levels, the coarsest would hold no full step");
  }
  if (N_ % stride != 0)
    throw ValidationError("MgritSolver: step count must be divisible by coarsen^(levels-1)");
  if (tr_) {
    rank_ = tr_->rank();
    world_ = tr_->size();
  }
  if (world_ > 1) {
    // every level's intervals must split evenly over the ranks
    long long n = N_;
    for (int l = 0; l + 1 < std::max(cfg_.levels, 2); ++l) {
      if ((n / cfg_.coarsen) % world_ != 0)
        throw ValidationError("layer partition: the " + std::to_string(n / cfg_.coarsen) +
                              " coarse intervals of level " + std::to_string(l) +
                              " do not split over " + std::to_string(world_) + " ranks");
      n /= cfg_.coarsen;
      if (l + 2 >= cfg_.levels) break;
    }
  }

  MGLP_CUDA(cudaSetDevice(device_));
  MGLP_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  build_layouts();
  build_ranges();
  P_ = dalloc(layer_stride_, total_, lay_r_);
  Gr_ = dalloc(layer_stride_, total_, lay_r_);
  Whl_ = dalloc(hl_stride_, total_, lay_r_);
  MGLP_CUDA(cudaMalloc(&range_flag_, sizeof(int)));
  MGLP_CUDA(cudaMalloc(&lam_sc_, sizeof(LamScale)));
  MGLP_CUDA(cudaMemsetAsync(lam_sc_, 0, sizeof(LamScale), stream_));
  if (world_ > 1) MGLP_CUDA(cudaMalloc(&lam_gather_, 2 * world_ * sizeof(double)));
  dmemset(P_, layer_stride_, lay_r_);
  dmemset(Whl_, hl_stride_, lay_r_);
  MGLP_CUDA(cudaMemsetAsync(range_flag_, 0, sizeof(int), stream_));
  dmemset(Gr_, layer_stride_, lay_r_);
  // the largest launch family: this rank's coarse intervals
  Gmax_ = std::max(1, N_ / cfg_.coarsen / world_);
  cache_valid_.assign(total_, 0);
}

Engine::~Engine() {
  cudaSetDevice(device_);
  if (stream_) cudaStreamSynchronize(stream_);
  free_solver(fwd_);
  free_solver(bwd_);
  if (range_flag_) cudaFree(range_flag_);
  if (lam_sc_) cudaFree(lam_sc_);
  if (snap_sc_) cudaFree(snap_sc_);
  if (lam_gather_) cudaFree(lam_gather_);
  if (mon_) cudaFree(mon_);
  if (mon_sum_) cudaFree(mon_sum_);
  if (mon_host_) cudaFreeHost(mon_host_);
  if (grad_pin_) cudaFreeHost(grad_pin_);
  for (float** p : {&P_, &Whl_, &Gr_, &scratch_, &hlscr_, &cache_, &bscratch_, &bcache_, &traj_,
                    &lam_all_, &zero_state_, &snap_fwd_, &snap_bwd_, &fwd_stash_})
    dfree(*p);
  if (colred_part_) cudaFree(colred_part_);
  if (drop_masks_) cudaFree(drop_masks_);
  drop_graph();
  for (cudaEvent_t ev : ev_pool_) cudaEventDestroy(ev);
  if (stream_) cudaStreamDestroy(stream_);
}

// ---- per-rank memory ------------------------------------------------------------
Engine::Ranges Engine::clip(const Ranges& r, long long lo, long long hi) {
  Ranges o;
  for (const auto& x : r) {
    const long long a = std::max(x.first, lo), b = std::min(x.second, hi);
    if (a < b) o.push_back({a, b});
  }
  return o;
}

// What rank r of P touches (engine.cu forward_device / backward_device,
// SURVEY 8(e)): the opening buffer layers (every rank runs them for the
// broadcast guess), its interior block [ib + lo, ib + hi) and, on the last
// rank, the closing buffers; time points likewise plus the ghost point
// ib + lo; coarse level l its points (p_lo, p_hi] plus the ghost p_lo and
// point 0 (the guess source). The adjoint windows use the reversed partition.
void Engine::build_ranges() {
  const int P = world_, r = rank_;
  const long long per = N_ / P, lo = (long long)r * per, hi = lo + per;
  const bool last = r == P - 1;
  auto add = [](Ranges& v, long long a, long long b) {
    if (a < b) v.push_back({a, b});
  };
  lay_r_.clear();
  traj_r_.clear();
  lam_r_.clear();
  win_r_.clear();
  bwd0_r_.clear();
  if (P == 1) {
    add(lay_r_, 0, total_);
    add(traj_r_, 0, total_ + 1);
    add(lam_r_, 0, total_ + 1);
    add(win_r_, 0, N_ + 1);
    add(bwd0_r_, 0, N_ + 1);
  } else {
    add(lay_r_, 0, ib_);
    add(lay_r_, ib_ + lo, ib_ + hi);
    if (last) add(lay_r_, ie_, total_);
    add(traj_r_, 0, ib_ + 1);
    add(traj_r_, ib_ + lo, ib_ + hi + 1);
    if (last) add(traj_r_, ie_, total_ + 1);
    if (r == 0) add(lam_r_, 0, ib_ + 1);
    if (last) add(lam_r_, ie_, total_ + 1);
    add(win_r_, 0, 1);
    add(win_r_, lo, hi + 1);
    const long long tp = P - 1 - r;
    add(bwd0_r_, 0, 1);
    add(bwd0_r_, tp * per, tp * per + per + 1);
  }
  // sorted, disjoint, merged (the pieces overlap at the ghosts and point 0)
  auto norm = [](Ranges& v) {
    std::sort(v.begin(), v.end());
    Ranges o;
    for (const auto& x : v) {
      if (!o.empty() && x.first <= o.back().second)
        o.back().second = std::max(o.back().second, x.second);
      else
        o.push_back(x);
    }
    v = o;
  };
  for (Ranges* v : {&lay_r_, &traj_r_, &lam_r_, &win_r_, &bwd0_r_}) norm(*v);
  for (int adj = 0; adj < 2; ++adj) {
    lvl_r_[adj].assign(std::max(cfg_.levels, 2), Ranges{});
    long long n = N_;
    for (size_t l = 1; l < lvl_r_[adj].size(); ++l) {
      n /= cfg_.coarsen;
      Ranges& v = lvl_r_[adj][l];
      if (P == 1) {
        add(v, 0, n + 1);
      } else {
        const long long pl = n / P, tp = adj ? P - 1 - r : r;
        add(v, 0, 1);
        add(v, tp * pl, tp * pl + pl + 1);
      }
      norm(v);
    }
  }
}

bool Engine::holds_points(int first, int count) const {
  long long covered = 0;
  for (const auto& x : clip(traj_r_, first, (long long)first + count)) covered += x.second - x.first;
  return covered == count;
}

bool Engine::owns_layer_slot(int l) const {
  for (const auto& x : lay_r_)
    if (l >= x.first && l < x.second) return true;
  return false;
}

namespace {
std::mutex g_alloc_mu;
std::map<void*, size_t> g_alloc_bytes;  // device bytes held per engine buffer
}  // namespace

float* Engine::dalloc(long long slot_elems, long long nslots, const Ranges& r) {
  const size_t slot_bytes = (size_t)slot_elems * sizeof(float);
  const size_t bytes = slot_bytes * (size_t)std::max(nslots, 1LL);
  long long covered = 0;
  for (const auto& x : r) covered += x.second - x.first;
  void* p = nullptr;
  size_t held = bytes;
  if (world_ == 1 || covered >= nslots) {
    MGLP_CUDA(cudaMalloc(&p, bytes));
  } else {
    std::vector<std::pair<size_t, size_t>> br;
    for (const auto& x : r) br.push_back({(size_t)x.first * slot_bytes, (size_t)x.second * slot_bytes});
    p = partial_alloc(device_, bytes, br, &held);
  }
  {
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    g_alloc_bytes[p] = held;
  }
  hbm_bytes_ += held;
  return static_cast<float*>(p);
}

void Engine::dfree(float*& p) {
  if (!p) return;
  size_t held = 0;
  {
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    auto it = g_alloc_bytes.find(p);
    if (it != g_alloc_bytes.end()) {
      held = it->second;
      g_alloc_bytes.erase(it);
    }
  }
  hbm_bytes_ -= std::min(hbm_bytes_, held);
  if (!partial_free(p)) cudaFree(p);
  p = nullptr;
}

void Engine::dmemset(float* p, long long slot_elems, const Ranges& r) {
  for (const auto& x : r)
    MGLP_CUDA(cudaMemsetAsync(p + x.first * slot_elems, 0,
                              (size_t)(x.second - x.first) * slot_elems * sizeof(float), stream_));
}

void Engine::dcopy(float* dst, const float* src, long long slot_elems, const Ranges& r,
                   long long first) {
  for (const auto& x : clip(r, first, LLONG_MAX))
    MGLP_CUDA(cudaMemcpyAsync(dst + x.first * slot_elems, src + x.first * slot_elems,
                              (size_t)(x.second - x.first) * slot_elems * sizeof(float),
                              cudaMemcpyDeviceToDevice, stream_));
}

void Engine::build_layouts() {
  const long long d = sd_.d, f = sd_.ffn;
  lay_.resize(2);
  for (int kind = 0; kind < 2; ++kind) {
    LayerLayout& L = lay_[kind];
    L.decoder = kind == 1;
    long long off = 0;
    auto take = [&](long long n) {
      const long long o = off;
      off += align32(n);
      return o;
    };
    L.ln1_g = take(d);
    L.ln1_b = take(d);
    L.w_qkv = take(3 * d * d);
    L.b_qkv = take(3 * d);
    L.w_o = take(d * d);
    L.b_o = take(d);
    if (L.decoder) {
      L.ln3_g = take(d);
      L.ln3_b = take(d);
      L.w_cq = take(d * d);
      L.b_cq = take(d);
      L.w_ckv = take(2 * d * d);
      L.b_ckv = take(2 * d);
      L.w_co = take(d * d);
      L.b_co = take(d);
    }
    L.ln2_g = take(d);
    L.ln2_b = take(d);
    L.w_in = take(f * d);
    L.b_in = take(f);
    L.w_out = take(d * f);
    L.b_out = take(d);
    L.size = off;
    // visit_params order (blocks.cpp:627-646)
    long long fo = 0;
    auto piece = [&](long long dev, long long n) {
      L.pieces.push_back(Piece{fo, dev, n});
      fo += n;
    };
    piece(L.ln1_g, d);
    piece(L.ln1_b, d);
    for (int q = 0; q < 3; ++q) {  // q, k, v
      piece(L.w_qkv + q * d * d, d * d);
      piece(L.b_qkv + q * d, d);
    }
    piece(L.w_o, d * d);
    piece(L.b_o, d);
    if (L.decoder) {
      piece(L.ln3_g, d);
      piece(L.ln3_b, d);
      piece(L.w_cq, d * d);
      piece(L.b_cq, d);
      piece(L.w_ckv, d * d);
      piece(L.b_ckv, d);
      piece(L.w_ckv + d * d, d * d);
      piece(L.b_ckv + d, d);
      piece(L.w_co, d * d);
      piece(L.b_co, d);
    }
    piece(L.ln2_g, d);
    piece(L.ln2_b, d);
    piece(L.w_in, f * d);
    piece(L.b_in, f);
    piece(L.w_out, d * f);
    piece(L.b_out, d);
    L.flat_size = fo;
    // pre-split copies of every weight matrix: [rows][pad32(cols)] and the
    // transpose [cols][pad32(rows)]
    long long ho = 0;
    auto pack = [&](long long p_off, long long rows, long long cols) {
      LayerLayout::WPack w;
      w.p_off = p_off;
      w.rows = (int)rows;
      w.cols = (int)cols;
      w.n_off = ho;
      ho += rows * pack_hl_cols((int)cols);
      w.t_off = ho;
      ho += cols * pack_hl_cols((int)rows);
      L.wpack.push_back(w);
    };
    pack(L.w_qkv, 3 * d, d);
    pack(L.w_o, d, d);
    if (L.decoder) {
      pack(L.w_cq, d, d);
      pack(L.w_ckv, 2 * d, d);
      pack(L.w_co, d, d);
    }
    pack(L.w_in, f, d);
    pack(L.w_out, d, f);
    L.hl_size = ho;
  }
  layer_stride_ = std::max(lay_[0].size, sd_.kind == 2 ? lay_[1].size : 0LL);
  hl_stride_ = std::max(lay_[0].hl_size, sd_.kind == 2 ? lay_[1].hl_size : 0LL);
  n_params_flat_ = 0;
  for (int l = 0; l < total_; ++l)
    n_params_flat_ += lay_[(sd_.kind == 2 && l >= n_split_) ? 1 : 0].flat_size;
}

// LayerStack constructor initialisation (blocks.cpp:432-449), bit-identical
// f64 values; runs on the host threads.
void Engine::init_params(uint64_t seed, std::vector<double>* flat_out) {
  static const char* enc_names[] = {"ln1.gain", "ln1.bias", "attn.q.w", "attn.q.b", "attn.k.w",
                                    "attn.k.b", "attn.v.w", "attn.v.b", "attn.o.w", "attn.o.b",
                                    "ln2.gain", "ln2.bias", "mlp.in.w", "mlp.in.b", "mlp.out.w",
                                    "mlp.out.b"};
  static const char* dec_names[] = {
      "ln1.gain",  "ln1.bias",  "self.q.w",  "self.q.b",  "self.k.w",  "self.k.b",  "self.v.w",
      "self.v.b",  "self.o.w",  "self.o.b",  "ln3.gain",  "ln3.bias",  "cross.q.w", "cross.q.b",
      "cross.k.w", "cross.k.b", "cross.v.w", "cross.v.b", "cross.o.w", "cross.o.b", "ln2.gain",
      "ln2.bias",  "mlp.in.w",  "mlp.in.b",  "mlp.out.w", "mlp.out.b"};
  std::vector<double>& flat = *flat_out;
  flat.assign(n_params_flat_, 0.0);
  std::vector<long long> layer_flat(total_ + 1, 0);
  for (int l = 0; l < total_; ++l)
    layer_flat[l + 1] = layer_flat[l] + lay_[(sd_.kind == 2 && l >= n_split_) ? 1 : 0].flat_size;
  const double depth_factor =
      sd_.depth_scaled_init ? std::sqrt(std::log(2.0 * static_cast<double>(total_))) : 1.0;
  // work items: (layer, piece) -- weights dominate, split them across threads
  struct Item {
    int layer, piece;
  };
  std::vector<Item> items;
  for (int l = 0; l < total_; ++l) {
    const int k = (sd_.kind == 2 && l >= n_split_) ? 1 : 0;
    for (int p = 0; p < (int)lay_[k].pieces.size(); ++p) items.push_back({l, p});
  }
  unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  std::atomic<size_t> next{0};
  for (unsigned t = 0; t < nt; ++t)
    th.emplace_back([&] {
      for (;;) {
        const size_t i = next.fetch_add(1);
        if (i >= items.size()) return;
        const int l = items[i].layer;
        const int k = (sd_.kind == 2 && l >= n_split_) ? 1 : 0;
        const Piece& pc = lay_[k].pieces[items[i].piece];
        const std::string comp = k ? dec_names[items[i].piece] : enc_names[items[i].piece];
        double* t = flat.data() + layer_flat[l] + pc.flat_off;
        if (comp.size() >= 4 && comp.compare(comp.size() - 4, 4, "gain") == 0) {
          for (long long e = 0; e < pc.n; ++e) t[e] = 1.0;
        } else if (comp.back() == 'w') {
          double sd = sd_.init_std;
          if (depth_scaled_component(comp)) sd *= depth_factor;
          const uint64_t site = fnv1a(comp);
          for (long long e = 0; e < pc.n; ++e)
            t[e] = truncated_gaussian(sd, seed, 1 /*kInit*/,
                                      (uint64_t)l * 1000003u + site, (uint64_t)e);
        } else {
          for (long long e = 0; e < pc.n; ++e) t[e] = 0.0;
        }
      }
    });
  for (auto& t : th) t.join();
}

void Engine::flat_to_slab(const double* flat, double* slab) const {
  std::fill(slab, slab + slab_elems(), 0.0);
  long long fo = 0;
  for (int l = 0; l < total_; ++l) {
    const LayerLayout& L = lay_[(sd_.kind == 2 && l >= n_split_) ? 1 : 0];
    double* dst = slab + (size_t)l * layer_stride_;
    for (const Piece& p : L.pieces)
      for (long long e = 0; e < p.n; ++e) dst[p.dev_off + e] = flat[fo + p.flat_off + e];
    fo += L.flat_size;
  }
}

void Engine::slab_to_flat(const double* slab, double* flat) const {
  long long fo = 0;
  for (int l = 0; l < total_; ++l) {
    const LayerLayout& L = lay_[(sd_.kind == 2 && l >= n_split_) ? 1 : 0];
    const double* src = slab + (size_t)l * layer_stride_;
    for (const Piece& p : L.pieces)
      for (long long e = 0; e < p.n; ++e) flat[fo + p.flat_off + e] = src[p.dev_off + e];
    fo += L.flat_size;
  }
}

void Engine::params_updated() {
  MGLP_CUDA(cudaSetDevice(device_));
  repack_weights();
  invalidate_linearization();
}

void Engine::set_params(const double* flat) {
  std::vector<float> host((size_t)total_ * layer_stride_, 0.f);
  long long fo = 0;
  for (int l = 0; l < total_; ++l) {
    const LayerLayout& L = lay_[(sd_.kind == 2 && l >= n_split_) ? 1 : 0];
    float* dst = host.data() + (size_t)l * layer_stride_;
    for (const Piece& p : L.pieces)
      for (long long e = 0; e < p.n; ++e) dst[p.dev_off + e] = (float)flat[fo + p.flat_off + e];
    fo += L.flat_size;
  }
  MGLP_CUDA(cudaSetDevice(device_));
  for (const auto& x : lay_r_)  // this rank's layers only (the others are unmapped)
    MGLP_CUDA(cudaMemcpyAsync(P_ + x.first * layer_stride_, host.data() + x.first * layer_stride_,
                              (size_t)(x.second - x.first) * layer_stride_ * sizeof(float),
                              cudaMemcpyHostToDevice, stream_));
  repack_weights();
  // cached activations were computed with the old parameters
  invalidate_linearization();
  MGLP_CUDA(cudaStreamSynchronize(stream_));
}

void Engine::get_params(double* flat) const {
  // a P-rank engine holds its own layers' parameters (the others read 0)
  std::vector<float> host((size_t)total_ * layer_stride_, 0.f);
  MGLP_CUDA(cudaStreamSynchronize(stream_));
  for (const auto& x : lay_r_)
    MGLP_CUDA(cudaMemcpy(host.data() + x.first * layer_stride_, P_ + x.first * layer_stride_,
                         (size_t)(x.second - x.first) * layer_stride_ * sizeof(float),
                         cudaMemcpyDeviceToHost));
  long long fo = 0;
  for (int l = 0; l < total_; ++l) {
    const LayerLayout& L = lay_[(sd_.kind == 2 && l >= n_split_) ? 1 : 0];
    const float* src = host.data() + (size_t)l * layer_stride_;
    for (const Piece& p : L.pieces)
      for (long long e = 0; e < p.n; ++e) flat[fo + p.flat_off + e] = src[p.dev_off + e];
    fo += L.flat_size;
  }
}

void Engine::get_grads(double* flat) const { get_grads_range(0, total_, flat); }

long long Engine::flat_offset(int layer) const {
  long long fo = 0;
  for (int l = 0; l < layer; ++l) fo += lay_[(sd_.kind == 2 && l >= n_split_) ? 1 : 0].flat_size;
  return fo;
}

// Gradients -> host f64 accumulation (+=), the reference's BlockParams
// contract: owned layers only (a P-rank engine's other layers add 0), in
// chunks of layers through two pinned staging buffers -- the DMA of chunk k+1
// overlaps the multithreaded scatter-add of chunk k (layers are disjoint flat
// ranges, so threads split them without synchronisation).
void Engine::get_grads_range(int lo, int hi, double* flat) const {
  if (lo < 0 || hi > total_ || lo > hi) throw ValidationError("get_grads: bad layer range");
  MGLP_CUDA(cudaSetDevice(device_));
  MGLP_CUDA(cudaStreamSynchronize(stream_));
  constexpr long long kChunk = 4;  // layers per staging buffer
  if (!grad_pin_) {
    MGLP_CUDA(cudaMallocHost(&grad_pin_, (size_t)(2 * kChunk * layer_stride_) * sizeof(float)));
    grad_pin_layers_ = kChunk;
  }
  // flat offset of every layer of [lo, hi)
  std::vector<long long> fo((size_t)(hi - lo + 1), 0);
  for (int l = lo; l < hi; ++l)
    fo[l - lo + 1] = fo[l - lo] + lay_[(sd_.kind == 2 && l >= n_split_) ? 1 : 0].flat_size;
  // owned layers of [lo, hi) in chunks
  std::vector<std::pair<int, int>> chunks;
  for (const auto& x : clip(lay_r_, lo, hi))
    for (long long c = x.first; c < x.second; c += kChunk)
      chunks.emplace_back((int)c, (int)std::min<long long>(x.second, c + kChunk));
  if (chunks.empty()) return;
  cudaEvent_t ev[2];
  for (auto& e : ev) MGLP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  auto issue = [&](size_t k) {
    float* dst = grad_pin_ + (k & 1) * kChunk * layer_stride_;
    const int a = chunks[k].first, b = chunks[k].second;
    MGLP_CUDA(cudaMemcpyAsync(dst, Gr_ + (long long)a * layer_stride_,
                              (size_t)(b - a) * layer_stride_ * sizeof(float),
                              cudaMemcpyDeviceToHost, stream_));
    MGLP_CUDA(cudaEventRecord(ev[k & 1], stream_));
  };
  const int nth = (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
  issue(0);
  for (size_t k = 0; k < chunks.size(); ++k) {
    MGLP_CUDA(cudaEventSynchronize(ev[k & 1]));
    if (k + 1 < chunks.size()) issue(k + 1);  // the other buffer: consumed in step k-1
    const float* buf = grad_pin_ + (k & 1) * kChunk * layer_stride_;
    const int a = chunks[k].first, b = chunks[k].second;
    auto work = [&](int t) {
      for (int l = a; l < b; ++l) {
        const LayerLayout& L = lay_[(sd_.kind == 2 && l >= n_split_) ? 1 : 0];
        const float* src = buf + (size_t)(l - a) * layer_stride_;
        double* dst = flat + fo[l - lo];
        for (const Piece& p : L.pieces) {
          // piece split evenly over the threads
          const long long per = (p.n + nth - 1) / nth, e0 = t * per,
                          e1 = std::min<long long>(p.n, e0 + per);
          for (long long e = e0; e < e1; ++e) dst[p.flat_off + e] += src[p.dev_off + e];
        }
      }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < nth; ++t) th.emplace_back(work, t);
    work(0);
    for (auto& x : th) x.join();
  }
  for (auto& e : ev) cudaEventDestroy(e);
}

void Engine::zero_grads() { dmemset(Gr_, layer_stride_, lay_r_); }

// =============================================================================
// shape-dependent buffers
// =============================================================================

void Engine::set_shape(int batch, int s_x, int s_y) {
  if (batch == B_ && s_x == sx_ && s_y == sy_ && traj_) return;
  if (batch <= 0 || s_x <= 0) throw ValidationError("shape: batch and s_x must be positive");
  if ((sd_.kind == 2) != (s_y > 0))
    throw ValidationError("shape: s_y > 0 exactly for encoder-decoder stacks");
  MGLP_CUDA(cudaSetDevice(device_));
  MGLP_CUDA(cudaStreamSynchronize(stream_));
  drop_graph();
  drop_on_ = false;  // masks are per shape: refresh_dropout again
  free_solver(fwd_);
  free_solver(bwd_);
  if (colred_part_) cudaFree(colred_part_);
  colred_part_ = nullptr;
  for (float** p : {&scratch_, &hlscr_, &cache_, &bscratch_, &bcache_, &traj_, &lam_all_, &zero_state_,
                    &snap_fwd_, &snap_bwd_, &fwd_stash_})
    dfree(*p);
  B_ = batch;
  sx_ = s_x;
  sy_ = s_y;
  Tx_ = B_ * sx_;
  Ty_ = B_ * sy_;
  const long long d = sd_.d, f = sd_.ffn, H = sd_.heads;
  x_off_ = 0;
  y_off_ = (long long)Tx_ * d;
  state_n_ = align32((long long)(Tx_ + Ty_) * d);
  const long long R = std::max(Tx_, sd_.kind == 2 ? Ty_ : 0);
  const long long smax = std::max(sx_, sy_);
  long long off = 0;
  auto take = [&](long long n) {
    const long long o = off;
    off += align32(std::max(n, 1LL));
    return o;
  };
  ActLayout& a = al_;
  a.n1 = take(R * d);
  a.qkv = take(R * 3 * d);
  a.ctx = take(R * d);
  a.P = take((long long)B_ * H * smax * ((smax + 3) & ~3));
  a.a1 = take(R * d);
  a.u = take(R * d);
  a.n2 = take(R * d);
  a.h = take(R * f);
  a.g = take(R * f);
  a.st1 = take(2 * R);
  a.st2 = take(2 * R);
  if (sd_.kind == 2) {
    a.n3 = take(Ty_ * d);
    a.u3 = take(Ty_ * d);
    a.cq = take(Ty_ * d);
    a.ckv = take((long long)Tx_ * 2 * d);
    a.cctx = take(Ty_ * d);
    a.cP = take((long long)B_ * H * sy_ * ((sx_ + 3) & ~3));
    a.ybar = take(Ty_ * d);
    a.st3 = take(2LL * Ty_);
  }
  a.size = off;
  off = 0;
  BwdLayout& b = bl_;
  b.dh = take(R * f);
  b.dn2 = take(R * d);
  b.du = take(R * d);
  b.da1 = take(R * d);
  b.dctx = take(R * d);
  b.dqkv = take(R * 3 * d);
  b.dn1 = take(R * d);
  {
    // the long backward's dS tiles (128 x 128 pre-split per block pair) live
    // here too: pad ragged lengths (ViT 197) to whole blocks
    const long long blk = (smax + 127) / 128;
    const long long tiles = smax > 128 ? blk * blk * 128 * 128 : 0;
    b.dP = take((long long)B_ * H * std::max((long long)smax * ((smax + 3) & ~3), tiles));
  }
  // dropout: the upstream of the MLP branch and of the cross-attention output
  // with their masks applied (the operands of those branches' dgrad / wgrad)
  b.upm = take(sd_.dropout > 0.0 ? R * d : 0);
  b.dcpre = take(sd_.dropout > 0.0 && sd_.kind == 2 ? Ty_ * d : 0);
  if (sd_.kind == 2) {
    b.dybar = take(Ty_ * d);
    b.dy = take(Ty_ * d);
    b.dcctx = take(Ty_ * d);
    b.dcq = take(Ty_ * d);
    b.dckv = take((long long)Tx_ * 2 * d);
    b.dn3 = take(Ty_ * d);
    b.dxe = take((long long)Tx_ * d);
    b.dP2 = take((long long)B_ * H * sy_ * ((sx_ + 3) & ~3));
  }
  b.size = off;
  const long long cache_slots = eval_only_ ? 1 : total_;
  const Ranges all1 = {{0, 1}};
  scratch_ = dalloc(al_.size, Gmax_, Ranges{{0, Gmax_}});
  {
    // pre-split A operands: the forward GEMMs of 32-aligned widths skip the
    // fp32 -> hi|lo' conversion (MGLP_NO_PRESPLIT_A=1 disables)
    static const bool off = [] {
      const char* e = getenv("MGLP_NO_PRESPLIT_A");
      return e && atoi(e) != 0;
    }();
    hl_cap_ = 0;
    hl_slot_ = 0;
    const int dh = sd_.d / sd_.heads;
    if (!off && sd_.d % 32 == 0 && sd_.ffn % 32 == 0 && dh % 32 == 0) {
      // buffer 0: LN outputs / da1 / the upstream ([rows][d]); buffer 1:
      // attention O, GELU output, dh, dqkv ([rows][max(ffn, 3d)])
      hl_w1_ = std::max(sd_.ffn, 3 * sd_.d);
      hl_slot_ = (long long)std::max(Tx_, Ty_) * (sd_.d + hl_w1_);
      hlscr_ = dalloc(hl_slot_, Gmax_, Ranges{{0, Gmax_}});
      hl_cap_ = Gmax_;
    }
  }
  const Ranges& cache_r = eval_only_ ? all1 : lay_r_;
  cache_ = dalloc(al_.size, cache_slots, cache_r);
  bscratch_ = dalloc(bl_.size, Gmax_, Ranges{{0, Gmax_}});
  bcache_ = dalloc(bl_.size, cache_slots, cache_r);
  colred_cap_ = (long long)std::max(total_, Gmax_) * kColRedChunks *
                std::max(std::max(3 * sd_.d, sd_.ffn), 2 * sd_.d) * 2;
  MGLP_CUDA(cudaMalloc(&colred_part_, (size_t)colred_cap_ * sizeof(double)));
  bcache_valid_.assign(total_, 0);
  const long long traj_slots = eval_only_ ? 1 : total_ + 1;
  const Ranges& tr_r = eval_only_ ? all1 : traj_r_;
  const Ranges& lam_r = eval_only_ ? all1 : lam_r_;
  traj_ = dalloc(state_n_, traj_slots, tr_r);
  lam_all_ = dalloc(state_n_, traj_slots, lam_r);
  zero_state_ = dalloc(state_n_, 1, all1);
  dmemset(traj_, state_n_, tr_r);
  dmemset(lam_all_, state_n_, lam_r);
  MGLP_CUDA(cudaMemsetAsync(zero_state_, 0, (size_t)state_n_ * sizeof(float), stream_));
  {
    GemmArgs probe;
    probe.G = 1;
    probe.M = std::max(Tx_, Ty_);
    probe.N = sd_.d;
    part_off_ln_ = gemm_blocks(probe);
    part_off_elem_ = part_off_ln_ + ln_bwd_blocks(std::max(Tx_, Ty_));
  }
  if (!eval_only_) {
    alloc_solver(fwd_, false);
    alloc_solver(bwd_, true);
  }
  std::fill(cache_valid_.begin(), cache_valid_.end(), 0);
  first_fwd_ = first_bwd_ = true;
  fwd_displaced_ = false;
  if (!snap_empty_) snap_id_ = 0;  // the slot's states were freed with the old shape
  MGLP_CUDA(cudaStreamSynchronize(stream_));
}

void Engine::alloc_solver(Solver& s, bool adjoint) {
  s.adjoint = adjoint;
  const int L = cfg_.levels;
  s.lv.assign(std::max(L, 2), Level{});
  int n = N_;
  for (int l = 0; l < (int)s.lv.size(); ++l) {
    s.lv[l].n = n;
    if (l + 1 < (int)s.lv.size()) n /= cfg_.coarsen;
  }
  // level 0 of the forward solver is the trajectory window traj[ib..ie]
  if (adjoint) {
    s.lv[0].v = dalloc(state_n_, N_ + 1, bwd0_r_);
    dmemset(s.lv[0].v, state_n_, bwd0_r_);
  } else {
    s.lv[0].v = traj_ + (size_t)ib_ * state_n_;
  }
  for (int l = 1; l < (int)s.lv.size(); ++l) {
    const Ranges& r = lvl_r_[adjoint ? 1 : 0][l];
    for (float** b : {&s.lv[l].v, &s.lv[l].rho, &s.lv[l].phib}) {
      *b = dalloc(state_n_, s.lv[l].n + 1, r);
      dmemset(*b, state_n_, r);  // rho[0] stays 0
    }
  }
  MGLP_CUDA(cudaMalloc(&s.ctrl, sizeof(SolveCtrl)));
  MGLP_CUDA(cudaMemsetAsync(s.ctrl, 0, sizeof(SolveCtrl), stream_));
  // owned points of every level: time position tpos owns (tpos*n_l/P, (tpos+1)*n_l/P]
  s.tpos = adjoint ? world_ - 1 - rank_ : rank_;
  s.p_lo.resize(s.lv.size());
  s.p_hi.resize(s.lv.size());
  for (size_t l = 0; l < s.lv.size(); ++l) {
    const int per = s.lv[l].n / world_;
    s.p_lo[l] = s.tpos * per;
    s.p_hi[l] = (s.tpos + 1) * per;
  }
  // residual-norm partial slots per coarse interval: GEMM tiles | LN rows | elementwise
  s.n_chunks = N_ / cfg_.coarsen;
  s.slots_per_chunk = part_off_elem_ + elem_combine_blocks((long long)std::max(Tx_, Ty_) * sd_.d);
  const size_t np = (size_t)s.n_chunks * s.slots_per_chunk;
  MGLP_CUDA(cudaMalloc(&s.partials, np * sizeof(double)));
  MGLP_CUDA(cudaMemsetAsync(s.partials, 0, np * sizeof(double), stream_));
  if (world_ > 1) MGLP_CUDA(cudaMalloc(&s.gathered, np * sizeof(double)));
}

void Engine::free_solver(Solver& s) {
  if (s.lv.empty()) return;
  if (s.adjoint) dfree(s.lv[0].v);
  for (size_t l = 1; l < s.lv.size(); ++l) {
    dfree(s.lv[l].v);
    dfree(s.lv[l].rho);
    dfree(s.lv[l].phib);
  }
  if (s.ctrl) cudaFree(s.ctrl);
  if (s.partials) cudaFree(s.partials);
  if (s.gathered) cudaFree(s.gathered);
  s = Solver{};
}

// =============================================================================
// operand helpers
// =============================================================================

Mat Engine::act_mat(const ActRef& r, long long off, int ld) const {
  Mat m;
  m.ptr = r.base + off;
  m.slot_stride = r.stride;
  m.ld = ld;
  m.slot0 = r.slot0;
  m.step = r.step;
  return m;
}
Mat Engine::bwd_mat(const EvalSpec& e, long long off, int ld) const {
  if (e.bact.base) return act_mat(e.bact, off, ld);
  Mat m;
  m.ptr = bscratch_ + off;
  m.slot_stride = bl_.size;
  m.ld = ld;
  return m;
}
Mat Engine::par(long long off, int ld, int layer0, int step) const {
  Mat m;
  m.ptr = P_ + off;
  m.slot_stride = layer_stride_;
  m.ld = ld;
  m.slot0 = layer0;
  m.step = step;
  return m;
}
Mat Engine::par_hl(const LayerLayout& L, long long off, int layer0, int step,
                   bool transposed) const {
  for (const LayerLayout::WPack& w : L.wpack) {
    if (w.p_off != off) continue;
    Mat m;
    m.ptr = Whl_ + (transposed ? w.t_off : w.n_off);
    m.slot_stride = hl_stride_;
    m.ld = (int)pack_hl_cols(transposed ? w.rows : w.cols);
    m.slot0 = layer0;
    m.step = step;
    return m;
  }
  throw ContractViolation("par_hl: no pre-split copy of the weight at this offset");
}

// Re-derive the pre-split weights from P_ (after every parameter change).
void Engine::repack_weights() {
  for (int kind = 0; kind < (sd_.kind == 2 ? 2 : 1); ++kind) {
    const LayerLayout& L = lay_[kind];
    // layers of this layout: [0, n_split_) encoders, [n_split_, total_) decoders
    int l0 = 0, nl = total_;
    if (sd_.kind == 2) {
      l0 = kind == 0 ? 0 : n_split_;
      nl = kind == 0 ? n_split_ : total_ - n_split_;
    }
    if (nl == 0) continue;
    for (const auto& x : clip(lay_r_, l0, l0 + nl)) {  // this rank's layers
      const long long a = x.first, cnt = x.second - x.first;
      for (const LayerLayout::WPack& w : L.wpack) {
        const float* src = P_ + a * layer_stride_ + w.p_off;
        float* dn = Whl_ + a * hl_stride_ + w.n_off;
        float* dt = Whl_ + a * hl_stride_ + w.t_off;
        launch_pack_hl(src, layer_stride_, w.cols, dn, hl_stride_, (int)pack_hl_cols(w.cols),
                       (int)cnt, w.rows, w.cols, false, stream_, range_flag_);
        launch_pack_hl(src, layer_stride_, w.cols, dt, hl_stride_, (int)pack_hl_cols(w.rows),
                       (int)cnt, w.cols, w.rows, true, stream_, range_flag_);
      }
    }
  }
}
Mat Engine::grad(long long off, int ld, int layer0, int step) const {
  Mat m = par(off, ld, layer0, step);
  m.ptr = Gr_ + off;
  return m;
}

void Engine::gemm(GemmArgs g) {
  ++launches_;
  const double flops = 2.0 * g.G * g.Bb * g.H * (double)g.M * g.N * g.K;
  // variant (diagnostics): epilogue kind | 16 A pre-split | 32 B pre-split | 64 A MN | 128 B MN
  prof_shape_ = {g.M, g.N, g.K, g.G * g.Bb * g.H,
                 g.ep.kind + (g.Ahl.ok() ? 16 : 0) + (g.Bhl.ok() ? 32 : 0) + (g.a_mn ? 64 : 0) +
                     (g.b_mn ? 128 : 0)};
  g.range_flag = range_flag_;
  timed(PROF_GEMM, flops, 0.0, [&] {
#ifdef MGLP_GEMM_SIMT
    launch_gemm_simt(g, active_, stream_);
#else
    launch_gemm_tc(g, active_, stream_);
#endif
  });
}

// The fused tcgen05 attention (attn_tc.cu) covers sq, skv <= 128; longer
// sequences run as tensor-core GEMMs + softmax row kernels. The choice depends
// only on the shape, so a given layer always takes the same path (Phi stays
// deterministic across families). MGLP_NO_FUSED_ATTN=1 forces the unfused path.
static bool use_fused_attn() {
#ifdef MGLP_GEMM_SIMT
  return false;
#else
  static const bool on = [] {
    const char* e = getenv("MGLP_NO_FUSED_ATTN");
    return !(e && atoi(e) != 0);
  }();
  return on;
#endif
}

// Sequences of 128 < s <= 512 use the streamed kernels (attn_long.cu);
// MGLP_LONG_ATTN=0 falls back to tensor-core GEMMs + softmax row kernels
// (S and P round-trip through HBM).
static bool use_long_attn() {
#ifdef MGLP_GEMM_SIMT
  return false;
#else
  static const bool on = [] {
    const char* e = getenv("MGLP_LONG_ATTN");
    return !(e && atoi(e) == 0);
  }();
  return on;
#endif
}

Mat Engine::hl_mat(int G, int which, int cols) const {
  Mat m;
#ifdef MGLP_GEMM_SIMT
  (void)G;
  (void)which;
  (void)cols;
  return m;  // the SIMT GEMMs read fp32 operands only
#else
  if (!hlscr_ || G > hl_cap_ || cols % 32 || cols > (which ? hl_w1_ : sd_.d)) return m;
  m.ptr = hlscr_ + (which ? (long long)std::max(Tx_, Ty_) * sd_.d : 0);
  m.slot_stride = hl_slot_;
  m.ld = cols;
  return m;
#endif
}

// s = 128: the fused kernels keep P in its pre-split form (AttnArgs::p_hl):
// one 64 KiB hi|lo' tile set per (member, batch, head), exactly the fp32
// P slot. A function of the shape only, so forward and backward agree.
bool Engine::p_hl_ok(int sq, int skv, const Mat& P) const {
  static const bool off = [] {
    const char* e = getenv("MGLP_ATTN_P_FP32");
    return e && atoi(e) != 0;
  }();
  return !off && sq == 128 && skv == 128 && P.ld == 128 && use_fused_attn();
}

// The adjoint's upstream state (lambda, or its dropout-masked copy) as the
// first dgrad GEMM's pre-split A operand: one streaming pack (HBM-bound, ~1/3
// of the converters' cost inside the MMA-bound GEMM) into hl buffer 0.
Mat Engine::pack_upstream(int G, int rows, const Mat& up) {
  Mat h = dgrad_hl(G, 0, sd_.d);
  if (!h.ok()) return h;
  ++launches_;
  prof_shape_ = {8, sd_.d, 0, G};
  timed(PROF_ROW, 0.0, 8.0 * G * (double)rows * sd_.d, [&] {
    launch_pack_hl(up.at(0), up.step * up.slot_stride, up.ld, h.ptr, h.slot_stride, h.ld, G, rows,
                   sd_.d, false, stream_, range_flag_);
  });
  return h;
}

bool Engine::cache_hl_off() {
  static const bool off = [] {
    const char* e = getenv("MGLP_NO_CACHE_HL");
    return e && atoi(e) != 0;
  }();
  return off;
}

// the adjoint's pre-split dgrad operands (MGLP_NO_PRESPLIT_DGRAD=1 disables)
Mat Engine::dgrad_hl(int G, int which, int cols) const {
  static const bool off = [] {
    const char* e = getenv("MGLP_NO_PRESPLIT_DGRAD");
    return e && atoi(e) != 0;
  }();
  return off ? Mat{} : hl_mat(G, which, cols);
}

// MGLP_FLASH128=1 (A/B): s = 128 self-attention through the single-pass
// kernels (attn_flash.cu) instead of the on-chip fused ones (attn_tc.cu)
static bool flash128() {
  static const bool on = [] {
    const char* e = getenv("MGLP_FLASH128");
    return e && atoi(e) != 0;
  }();
  return on;
}

bool Engine::attn_hs(int sq, int skv, bool grad) const {
  static const bool off = [] {
    const char* e = getenv("MGLP_NO_ATTN_HS");
    return e && atoi(e) != 0;
  }();
  if (off || !use_fused_attn() || sd_.d != 64 * sd_.heads) return false;
  if (sq <= 128 && skv <= 128) return sq % 8 == 0 && skv % 8 == 0;  // attn_tc.cu
  // 128 < s <= 512 (attn_flash.cu): Q, K, V for the single-pass forward; dO for
  // the single-pass backward, which stores its dS tiles in the dP slot (self-
  // attention, whole blocks per head: allocated so); MGLP_FLASH_BWD=0 keeps
  // the long backward (fp32 dO)
  static const bool flash_bwd = [] {
    const char* e = getenv("MGLP_FLASH_BWD");
    return !(e && atoi(e) == 0);
  }();
  if (!use_long_attn() || sq <= 128 || skv <= 128 || sq > 512 || skv > 512) return false;
  return !grad || (flash_bwd && sq == skv);
}

bool Engine::attention_fwd(int G, Mat Q, Mat K, Mat V, Mat O, Mat P, int sq, int skv,
                           bool causal, bool keep_p, Mat Ohl, bool qkv_hs) {
  const int H = sd_.heads, dh = sd_.d / H;
  auto heads = [&](Mat m, int s) {
    m.bstride = (long long)s * m.ld;
    m.hstride = dh;
    return m;
  };
  Q = heads(Q, sq);
  K = heads(K, skv);
  V = heads(V, skv);
  O = heads(O, sq);
  const int ldp = (skv + 3) & ~3;  // 16-byte rows for TMA
  P.ld = ldp;
  P.hstride = (long long)sq * ldp;
  P.bstride = (long long)H * sq * ldp;
  if (use_fused_attn()) {
    AttnArgs at;
    at.G = G;
    at.Bb = B_;
    at.H = H;
    at.sq = sq;
    at.skv = skv;
    at.dh = dh;
    at.causal = causal ? 1 : 0;
    at.scale = (float)(1.0 / std::sqrt((double)dh));
    at.Q = Q;
    at.K = K;
    at.V = V;
    at.O = O;
    at.P = P;
    at.range_flag = range_flag_;
    at.p_hl = p_hl_ok(sq, skv, P) ? 1 : 0;
    at.qkv_hs = qkv_hs ? 1 : 0;
    const double fl = 4.0 * G * B_ * H * (double)sq * skv * dh * (causal ? 0.5 : 1.0);
    // O pre-split for the O-projection; fp32 O only where the backward reads it
    auto with_hl = [&] {
      if (!Ohl.ok() || dh % 32) return false;
      at.Ohl = heads(Ohl, sq);
      if (!keep_p) at.O = Mat{};
      return true;
    };
    const bool f128 = flash128() && qkv_hs && sq == 128 && skv == 128 && dh == 64;
    if (!f128 && attn_tc_supported(at, false)) {
      // P is only an intermediate of the backward: not stored for scratch evaluations
      if (!keep_p) at.P = Mat{};
      const bool hl = with_hl();
      ++launches_;
      prof_shape_ = {sq, skv, dh, G * B_ * H};
      timed(PROF_ATTN, fl, 0.0, [&] { launch_attn_fwd(at, active_, stream_); });
      return hl;
    }

    if (use_long_attn() && attn_long_supported(at, false)) {
      // longer sequences: P is recomputed by the backward from per-row
      // statistics stored in the P slot (attn_long.cu)
      const bool hl = with_hl();
      ++launches_;
      prof_shape_ = {sq, skv, dh, G * B_ * H};
      timed(PROF_ATTN, fl, 0.0, [&] { launch_attn_fwd_long(at, active_, stream_); });
      return hl;
    }
  }
  if (qkv_hs) throw ContractViolation("attention: pre-split Q/K/V need a fused kernel");
  GemmArgs g;
  g.G = G;
  g.Bb = B_;
  g.H = H;
  g.M = sq;
  g.N = skv;
  g.K = dh;
  g.A = Q;
  g.B = K;
  g.ep.kind = EPI_STORE;
  g.ep.out1 = P;
  gemm(g);
  SoftmaxArgs sm;
  sm.G = G;
  sm.rows = (long long)B_ * H * sq;
  sm.ncols = skv;
  sm.sq = sq;
  sm.causal = causal;
  sm.scale = (float)(1.0 / std::sqrt((double)dh));
  sm.S = P;
  ++launches_;
  prof_shape_ = {1, sm.ncols, 0, G};
  timed(PROF_ROW, 0.0, 8.0 * G * (double)sm.rows * skv, [&] { launch_softmax(sm, active_, stream_); });
  g = GemmArgs{};
  g.G = G;
  g.Bb = B_;
  g.H = H;
  g.M = sq;
  g.N = dh;
  g.K = skv;
  g.A = P;
  g.B = V;
  g.b_mn = true;
  g.ep.kind = EPI_STORE;
  g.ep.out1 = O;
  gemm(g);
  return false;
}

bool Engine::attention_bwd(int G, Mat Q, Mat K, Mat V, Mat P, Mat O, Mat dO, Mat dP, Mat dQ, Mat dK,
                           Mat dV, int sq, int skv, bool causal, Mat dQhl, Mat dKhl, Mat dVhl,
                           bool keep32, bool qkv_hs, bool do_hs) {
  const int H = sd_.heads, dh = sd_.d / H;
  const float scale = (float)(1.0 / std::sqrt((double)dh));
  auto heads = [&](Mat m, int s) {
    m.bstride = (long long)s * m.ld;
    m.hstride = dh;
    return m;
  };
  Q = heads(Q, sq);
  K = heads(K, skv);
  V = heads(V, skv);
  O = heads(O, sq);  // the long backward forms t_i = dO_i . O_i per (batch, head)
  dO = heads(dO, sq);
  dQ = heads(dQ, sq);
  dK = heads(dK, skv);
  dV = heads(dV, skv);
  const int ldp = (skv + 3) & ~3;
  for (Mat* m : {&P, &dP}) {
    m->ld = ldp;
    m->hstride = (long long)sq * ldp;
    m->bstride = (long long)H * sq * ldp;
  }
  if (use_fused_attn()) {
    AttnArgs at;
    at.G = G;
    at.Bb = B_;
    at.H = H;
    at.sq = sq;
    at.skv = skv;
    at.dh = dh;
    at.scale = scale;
    at.Q = Q;
    at.K = K;
    at.V = V;
    at.P = P;
    at.O = O;
    at.causal = causal ? 1 : 0;
    at.dO = dO;
    at.dQ = dQ;
    at.dK = dK;
    at.dV = dV;
    at.range_flag = range_flag_;
    at.p_hl = p_hl_ok(sq, skv, P) ? 1 : 0;  // as the forward stored it
    at.qkv_hs = qkv_hs ? 1 : 0;
    at.do_hs = do_hs ? 1 : 0;
    // algorithmic: causal problems count the lower triangle only (as the forward)
    const double fl = 8.0 * G * B_ * H * (double)sq * skv * dh * (causal ? 0.5 : 1.0);
    // pre-split gradients for the QKV dgrad; fp32 only where a weight
    // gradient reads them
    auto with_hl = [&] {
      if (!dQhl.ok() || !dKhl.ok() || !dVhl.ok() || dh % 32) return false;
      at.dQhl = heads(dQhl, sq);
      at.dKhl = heads(dKhl, skv);
      at.dVhl = heads(dVhl, skv);
      if (!keep32) at.dQ = at.dK = at.dV = Mat{};
      return true;
    };
    const bool f128 = flash128() && do_hs && sq == 128 && skv == 128 && dh == 64;
    if (!f128 && attn_tc_supported(at, true)) {
      const bool hl = with_hl();
      ++launches_;
      prof_shape_ = {-sq, skv, dh, G * B_ * H};
      timed(PROF_ATTN, fl, 0.0, [&] { launch_attn_bwd(at, active_, stream_); });
      return hl;
    }

    // whole 128-blocks: the long dK/dV kernel stores its dS tiles (pre-split)
    // in the dP slot and dQ reads them (MGLP_LONG_DS=0 recomputes S, P, dP
    // instead); the single-pass backward (pre-split dO) always does
    static const bool ds_on = [] {
      const char* e = getenv("MGLP_LONG_DS");
      return !(e && atoi(e) == 0);
    }();
    // self-attention: the dP slot holds whole-block tiles per head (padded
    // at allocation); cross-attention only when the blocks tile it exactly
    if (do_hs || (ds_on && (sq == skv || (sq % 128 == 0 && skv % 128 == 0 && dP.ld == skv)))) {
      const long long per_head = (long long)((sq + 127) / 128) * ((skv + 127) / 128) * 128 * 128;
      Mat ds = dP;
      ds.hstride = per_head;
      ds.bstride = (long long)H * per_head;
      at.dS = ds;
    }
    if (use_long_attn() && attn_long_supported(at, true)) {
      const bool hl = with_hl();
      ++launches_;
      prof_shape_ = {-sq, skv, dh, G * B_ * H};
      timed(PROF_ATTN, fl, 0.0, [&] { launch_attn_bwd_long(at, active_, stream_); });
      return hl;
    }
  }
  if (qkv_hs || do_hs) throw ContractViolation("attention: pre-split operands need a fused kernel");
  auto mk = [&](int M, int N, int K_, Mat A, bool amn, Mat B, bool bmn, Mat out, float alpha) {
    GemmArgs g;
    g.G = G;
    g.Bb = B_;
    g.H = H;
    g.M = M;
    g.N = N;
    g.K = K_;
    g.A = A;
    g.a_mn = amn;
    g.B = B;
    g.b_mn = bmn;
    g.ep.kind = EPI_STORE;
    g.ep.out1 = out;
    g.ep.alpha = alpha;
    gemm(g);
  };
  mk(sq, skv, dh, dO, false, V, false, dP, 1.f);   // dP = dO . V^T
  SoftmaxArgs sm;
  sm.G = G;
  sm.rows = (long long)B_ * H * sq;
  sm.ncols = skv;
  sm.sq = sq;
  sm.S = P;
  sm.dS = dP;
  ++launches_;
  prof_shape_ = {2, sm.ncols, 0, G};
  timed(PROF_ROW, 0.0, 12.0 * G * (double)sm.rows * skv, [&] { launch_softmax(sm, active_, stream_); });
  mk(skv, dh, sq, P, true, dO, true, dV, 1.f);     // dV = P^T . dO
  mk(sq, dh, skv, dP, false, K, true, dQ, scale);  // dQ = dS . K / sqrt(dh)
  mk(skv, dh, sq, dP, true, Q, true, dK, scale);   // dK = dS^T . Q / sqrt(dh)
  return false;
}

cudaEvent_t Engine::prof_event() {
  if (ev_used_ == ev_pool_.size()) {
    cudaEvent_t e;
    MGLP_CUDA(cudaEventCreate(&e));
    ev_pool_.push_back(e);
  }
  return ev_pool_[ev_used_++];
}

void Engine::set_profiling(bool on) {
  profiling_ = on;
  prof_.clear();
  ev_used_ = 0;
}

int Engine::dump_profile(double* out, int max_rows) {
  MGLP_CUDA(cudaStreamSynchronize(stream_));
  int n = 0;
  for (const ProfRec& r : prof_) {
    if (n >= max_rows) break;
    float t = 0.f;
    MGLP_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    double* o = out + 8 * n;
    o[0] = r.cls;
    o[1] = r.shape[0];
    o[2] = r.shape[1];
    o[3] = r.shape[2];
    o[4] = r.shape[3];
    o[5] = r.cls == PROF_ROW ? r.bytes : r.flops;  // row kernels: HBM bytes
    o[6] = t;
    o[7] = r.shape.size() > 4 ? r.shape[4] : -1;
    ++n;
  }
  return n;
}

void Engine::read_profile(double* ms, double* flops, double* bytes, long long* launches) {
  MGLP_CUDA(cudaStreamSynchronize(stream_));
  for (int c = 0; c < PROF_NCLASS; ++c) {
    ms[c] = flops[c] = bytes[c] = 0.0;
    launches[c] = 0;
  }
  for (const ProfRec& r : prof_) {
    float t = 0.f;
    MGLP_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    ms[r.cls] += t;
    flops[r.cls] += r.flops;
    bytes[r.cls] += r.bytes;
    launches[r.cls] += 1;
  }
}

int Engine::gemm_blocks(const GemmArgs& g) const {
#ifdef MGLP_GEMM_SIMT
  return gemm_simt_blocks(g);
#else
  return gemm_tc_blocks(g);
#endif
}


// =============================================================================
// Phi: one layer step z + dt*F(z) for a family of G layers (blocks.cpp:466-514)
// =============================================================================

// Write-ownership contract of a launch family (the reference Executor
// rejects overlapping task write ranges before running them,
// executor.cpp:75-110): member g writes [at(g), at(g) + extent) of every
// output family, so the members' ranges must be pairwise disjoint --
// equally strided families are iff |step * slot_stride| >= extent -- and no
// member may write a state it (or another member) reads as its input.
void Engine::check_family_writes(const EvalSpec& e, bool adjoint) const {
  if (e.G <= 1) return;
  auto disjoint = [&](const Mat& m, long long extent, const char* what) {
    if (!m.ok()) return;
    const long long stride = std::llabs((long long)m.step * m.slot_stride);
    if (stride < extent)
      throw ContractViolation(std::string("launch family: members' write ranges overlap (") +
                              what + ")");
  };
  const long long sn = state_n_;
  disjoint(e.cmb.out, sn, "solver state");
  if (e.act.base != nullptr && e.act.step == 0)
    throw ContractViolation("launch family: members share one activation slot");
  if (e.bact.base != nullptr && e.bact.step == 0 && !e.wgrad_only)
    throw ContractViolation("launch family: members share one backward slot");
  // in-place families (out = in) are fine member by member; a member's output
  // must not be another member's input
  const Mat& in = adjoint ? e.lam : e.in;
  if (e.cmb.out.ok() && in.ok() && e.cmb.out.ptr == in.ptr && e.cmb.out.slot_stride == in.slot_stride) {
    for (int g = 1; g < e.G && g < 4; ++g) {
      const long long o = (long long)e.cmb.out.slot0 + (long long)g * e.cmb.out.step;
      for (int h = 0; h < e.G; ++h)
        if (h != g && (long long)in.slot0 + (long long)h * in.step == o)
          throw ContractViolation("launch family: a member writes another member's input");
    }
  }
}

void Engine::eval_forward(const EvalSpec& e0) {
  check_family_writes(e0, false);
  // split families that straddle the encoder/decoder boundary
  if (sd_.kind == 2) {
    const int first = e0.layer0, last = e0.layer0 + (e0.G - 1) * e0.layer_step;
    const bool fdec = first >= n_split_, ldec = last >= n_split_;
    if (fdec != ldec) {
      int gsplit = 0;
      while (gsplit < e0.G && ((e0.layer0 + gsplit * e0.layer_step >= n_split_) == fdec)) ++gsplit;
      auto part = [&](int g0, int G) {
        EvalSpec e = e0;
        e.G = G;
        e.layer0 = e0.layer0 + g0 * e0.layer_step;
        e.in = shift(e0.in, g0);
        e.lam = shift(e0.lam, g0);
        e.act.slot0 += g0 * e0.act.step;
        e.bact.slot0 += g0 * e0.bact.step;
        Combine& c = e.cmb;
        c.z = shift(c.z, g0);
        c.out = shift(c.out, g0);
        c.base = shift(c.base, g0);
        c.phib = shift(c.phib, g0);
        c.rho = shift(c.rho, g0);
        c.v = shift(c.v, g0);
        c.norm_base = e0.cmb.norm_base + g0 * e0.cmb.norm_member_stride;
        return e;
      };
      eval_forward(part(0, gsplit));
      eval_forward(part(gsplit, e0.G - gsplit));
      return;
    }
  }
  EvalSpec e = e0;
  e.cmb.z = e.in;
  if (e.residual_only) e.cmb.z = state_mat(zero_state_, 0, sd_.d, 0, 0);  // p = 0 + dt F
  e.cmb.dt = e.dt;
  const int d = sd_.d;
  if (sd_.kind == 2 && e.layer0 >= n_split_) {
    decoder_forward(e);
  } else {
    Mat yp;
    if (sd_.kind == 2) yp = e.in.offset(y_off_);
    encoder_forward(e, Tx_, causal_, e.in.offset(x_off_), yp);
  }
  (void)d;
}

void Engine::encoder_forward(const EvalSpec& e, int R, bool causal, Mat X, Mat Ypass) {
  const int d = sd_.d, f = sd_.ffn, G = e.G;
  const LayerLayout& L = lay_[0];
  const int l0 = e.layer0, ls = e.layer_step;
  X.ld = d;
  Mat n1 = act_mat(e.act, al_.n1, d), qkv = act_mat(e.act, al_.qkv, 3 * d);
  Mat ctx = act_mat(e.act, al_.ctx, d), Pm = act_mat(e.act, al_.P, 0);
  Mat a1 = act_mat(e.act, al_.a1, d), u = act_mat(e.act, al_.u, d);
  Mat n2 = act_mat(e.act, al_.n2, d), hh = act_mat(e.act, al_.h, f), gg = act_mat(e.act, al_.g, f);
  Mat st1 = act_mat(e.act, al_.st1, 2), st2 = act_mat(e.act, al_.st2, 2);

  // pre-split A operands (hl_mat): the LN outputs, attention O and GELU
  // output are written as hi|lo' rows for the next GEMM; their fp32 forms only
  // where the backward reads them (keep_lin)
  const bool keep = keep_lin(e);
  auto pre = [&](int which, int cols, long long w) {
    Mat m = hl_mat(G, which, cols);
    return (m.ok() && par_hl(L, w, l0, ls, false).ok()) ? m : Mat{};
  };
  // a kept linearisation stores its LN / GELU outputs pre-split only: the
  // weight gradients read them as pre-split MN-major B (GemmArgs::b_mn_hl)
  const bool ch = keep && cache_hl();
  const Mat h_n1 = ch ? n1 : pre(0, d, L.w_qkv), h_ctx = pre(1, d, L.w_o),
            h_n2 = ch ? n2 : pre(0, d, L.w_in), h_g = ch ? gg : pre(1, f, L.w_out);

  LnFwdArgs ln;
  ln.G = G;
  ln.rows = R;
  ln.d = d;
  ln.eps = (float)sd_.ln_eps;
  ln.x = X;
  ln.out = ((keep && !ch) || !h_n1.ok()) ? n1 : Mat{};
  ln.out_hl = h_n1;
  ln.range_flag = range_flag_;
  ln.stats = st1;
  ln.gain = par(L.ln1_g, 0, l0, ls);
  ln.bias = par(L.ln1_b, 0, l0, ls);
  ++launches_;
  prof_shape_ = {3, ln.d, 0, ln.G};
  timed(PROF_ROW, 0.0, 8.0 * ln.G * (double)ln.rows * ln.d,
        [&] { launch_ln_fwd(ln, active_, stream_); });

  GemmArgs g;
  g.G = G;
  g.M = R;
  g.N = 3 * d;
  g.K = d;
  g.A = n1;
  g.Ahl = h_n1;
  g.B = par(L.w_qkv, d, l0, ls);
  g.Bhl = par_hl(L, L.w_qkv, l0, ls, false);
  g.ep.kind = EPI_STORE;
  g.ep.out1 = qkv;
  g.ep.bias = par(L.b_qkv, 0, l0, ls);
  const bool hs = attn_hs(R / B_, R / B_);
  g.ep.hs = hs ? 1 : 0;
  g.ep.range_flag = range_flag_;
  gemm(g);

  const bool ctx_hl = attention_fwd(G, qkv, qkv.offset(d), qkv.offset(2 * d), ctx, Pm, R / B_,
                                    R / B_, causal, keep, h_ctx, hs);

  g = GemmArgs{};
  g.G = G;
  g.M = R;
  g.N = d;
  g.K = d;
  g.A = ctx;
  if (ctx_hl) g.Ahl = h_ctx;
  g.B = par(L.w_o, d, l0, ls);
  g.Bhl = par_hl(L, L.w_o, l0, ls, false);
  g.ep.kind = EPI_BIAS_ADD2;
  g.ep.drop = dmask(0, l0, ls);  // attention output phi1
  g.ep.out1 = a1;
  g.ep.out2 = u;
  g.ep.add2 = X;
  g.ep.bias = par(L.b_o, 0, l0, ls);
  gemm(g);

  ln.x = u;
  ln.out = ((keep && !ch) || !h_n2.ok()) ? n2 : Mat{};
  ln.out_hl = h_n2;
  ln.stats = st2;
  ln.gain = par(L.ln2_g, 0, l0, ls);
  ln.bias = par(L.ln2_b, 0, l0, ls);
  ++launches_;
  prof_shape_ = {3, ln.d, 0, ln.G};
  timed(PROF_ROW, 0.0, 8.0 * ln.G * (double)ln.rows * ln.d,
        [&] { launch_ln_fwd(ln, active_, stream_); });

  g = GemmArgs{};
  g.G = G;
  g.M = R;
  g.N = f;
  g.K = d;
  g.A = n2;
  g.Ahl = h_n2;
  g.B = par(L.w_in, d, l0, ls);
  g.Bhl = par_hl(L, L.w_in, l0, ls, false);
  g.ep.kind = EPI_BIAS_GELU;
  if (keep) g.ep.out1 = hh;  // gelu'(h): only the backward reads it
  if ((keep && !ch) || !h_g.ok()) g.ep.out2 = gg;
  g.ep.hl2 = h_g;
  g.ep.range_flag = range_flag_;
  g.ep.bias = par(L.b_in, 0, l0, ls);
  gemm(g);

  g = GemmArgs{};
  g.G = G;
  g.M = R;
  g.N = d;
  g.K = f;
  g.A = gg;
  g.Ahl = h_g;
  g.B = par(L.w_out, f, l0, ls);
  g.Bhl = par_hl(L, L.w_out, l0, ls, false);
  g.ep.kind = EPI_FINAL;
  g.ep.drop = dmask(1, l0, ls);  // MLP output phi2
  g.ep.add1 = a1;
  g.ep.bias = par(L.b_out, 0, l0, ls);
  Combine c = e.cmb;
  const long long xo = (Ypass.ok() || sd_.kind == 2) ? x_off_ : 0;
  auto off = [&](Mat m) { return m.ok() ? m.offset(xo) : m; };
  c.z = off(c.z);
  c.out = off(c.out);
  c.base = off(c.base);
  c.phib = off(c.phib);
  c.rho = off(c.rho);
  c.v = off(c.v);
  for (Mat* m : {&c.z, &c.out, &c.base, &c.phib, &c.rho, &c.v}) m->ld = d;
  if (c.mode == CM_RES0) c.norm_base = e.cmb.norm_base;  // GEMM tiles first
  g.ep.cmb = c;
  gemm(g);
  if (Ypass.ok() && e.cmb.mode != CM_NONE) {
    ElemCombineArgs ec;
    ec.G = G;
    ec.n = (long long)Ty_ * d;
    Combine cy = e.cmb;
    for (Mat* m : {&cy.z, &cy.out, &cy.base, &cy.phib, &cy.rho, &cy.v})
      if (m->ok()) *m = m->offset(y_off_);
    if (cy.mode == CM_RES0) cy.norm_base = e.cmb.norm_base + part_off_elem_;
    ec.cmb = cy;
    ++launches_;
    prof_shape_ = {6, 0, 0, ec.G};
    timed(PROF_ROW, 0.0, 12.0 * ec.G * (double)ec.n,
          [&] { launch_elem_combine(ec, active_, stream_); });
  }
}

void Engine::decoder_forward(const EvalSpec& e) {
  const int d = sd_.d, f = sd_.ffn, G = e.G;
  const LayerLayout& L = lay_[1];
  const int l0 = e.layer0, ls = e.layer_step;
  const int R = Ty_;
  Mat Y = e.in.offset(y_off_), X = e.in.offset(x_off_);
  Y.ld = X.ld = d;
  Mat n1 = act_mat(e.act, al_.n1, d), qkv = act_mat(e.act, al_.qkv, 3 * d);
  Mat ctx = act_mat(e.act, al_.ctx, d), Pm = act_mat(e.act, al_.P, 0);
  Mat a1 = act_mat(e.act, al_.a1, d), u2 = act_mat(e.act, al_.u, d);
  Mat n2 = act_mat(e.act, al_.n2, d), hh = act_mat(e.act, al_.h, f), gg = act_mat(e.act, al_.g, f);
  Mat st1 = act_mat(e.act, al_.st1, 2), st2 = act_mat(e.act, al_.st2, 2);
  Mat n3 = act_mat(e.act, al_.n3, d), u3 = act_mat(e.act, al_.u3, d);
  Mat cq = act_mat(e.act, al_.cq, d), ckv = act_mat(e.act, al_.ckv, 2 * d);
  Mat cctx = act_mat(e.act, al_.cctx, d), cP = act_mat(e.act, al_.cP, 0);
  Mat ybar = act_mat(e.act, al_.ybar, d), st3 = act_mat(e.act, al_.st3, 2);

  // pre-split A operands as in encoder_forward
  const bool keep = keep_lin(e);
  auto pre = [&](int which, int cols, long long w) {
    Mat m = hl_mat(G, which, cols);
    return (m.ok() && par_hl(L, w, l0, ls, false).ok()) ? m : Mat{};
  };
  const bool ch = keep && cache_hl();  // as in encoder_forward
  const Mat h_n1 = ch ? n1 : pre(0, d, L.w_qkv), h_ctx = pre(1, d, L.w_o),
            h_n3 = ch ? n3 : pre(0, d, L.w_cq), h_cctx = pre(1, d, L.w_co),
            h_n2 = ch ? n2 : pre(0, d, L.w_in), h_g = ch ? gg : pre(1, f, L.w_out);

  LnFwdArgs ln;
  ln.G = G;
  ln.rows = R;
  ln.d = d;
  ln.eps = (float)sd_.ln_eps;
  ln.x = Y;
  ln.out = ((keep && !ch) || !h_n1.ok()) ? n1 : Mat{};
  ln.out_hl = h_n1;
  ln.range_flag = range_flag_;
  ln.stats = st1;
  ln.gain = par(L.ln1_g, 0, l0, ls);
  ln.bias = par(L.ln1_b, 0, l0, ls);
  ++launches_;
  prof_shape_ = {3, ln.d, 0, ln.G};
  timed(PROF_ROW, 0.0, 8.0 * ln.G * (double)ln.rows * ln.d,
        [&] { launch_ln_fwd(ln, active_, stream_); });

  auto mk = [&](int M, int N, int K, Mat A, long long w, int ldw) {
    GemmArgs g;
    g.G = G;
    g.M = M;
    g.N = N;
    g.K = K;
    g.A = A;
    g.B = par(w, ldw, l0, ls);
    g.Bhl = par_hl(L, w, l0, ls, false);
    return g;
  };
  GemmArgs g = mk(R, 3 * d, d, n1, L.w_qkv, d);
  g.Ahl = h_n1;
  g.ep.kind = EPI_STORE;
  g.ep.out1 = qkv;
  g.ep.bias = par(L.b_qkv, 0, l0, ls);
  const bool hs = attn_hs(sy_, sy_);
  g.ep.hs = hs ? 1 : 0;
  g.ep.range_flag = range_flag_;
  gemm(g);

  const bool ctx_hl = attention_fwd(G, qkv, qkv.offset(d), qkv.offset(2 * d), ctx, Pm, sy_, sy_,
                                    true, keep, h_ctx, hs);

  g = mk(R, d, d, ctx, L.w_o, d);
  if (ctx_hl) g.Ahl = h_ctx;
  g.ep.kind = EPI_BIAS_ADD2;
  g.ep.drop = dmask(0, l0, ls);  // self-attention output phi1
  g.ep.out1 = a1;
  g.ep.out2 = u3;
  g.ep.add2 = Y;
  g.ep.bias = par(L.b_o, 0, l0, ls);
  gemm(g);

  ln.x = u3;
  ln.out = ((keep && !ch) || !h_n3.ok()) ? n3 : Mat{};
  ln.out_hl = h_n3;
  ln.stats = st3;
  ln.gain = par(L.ln3_g, 0, l0, ls);
  ln.bias = par(L.ln3_b, 0, l0, ls);
  ++launches_;
  prof_shape_ = {3, ln.d, 0, ln.G};
  timed(PROF_ROW, 0.0, 8.0 * ln.G * (double)ln.rows * ln.d,
        [&] { launch_ln_fwd(ln, active_, stream_); });

  const bool chs = attn_hs(sy_, sx_);
  g = mk(R, d, d, n3, L.w_cq, d);
  g.Ahl = h_n3;
  g.ep.kind = EPI_STORE;
  g.ep.out1 = cq;
  g.ep.bias = par(L.b_cq, 0, l0, ls);
  g.ep.hs = chs ? 1 : 0;
  g.ep.range_flag = range_flag_;
  gemm(g);

  g = mk(Tx_, 2 * d, d, X, L.w_ckv, d);
  g.ep.kind = EPI_STORE;
  g.ep.out1 = ckv;
  g.ep.bias = par(L.b_ckv, 0, l0, ls);
  g.ep.hs = chs ? 1 : 0;
  g.ep.range_flag = range_flag_;
  gemm(g);

  const bool cctx_hl =
      attention_fwd(G, cq, ckv, ckv.offset(d), cctx, cP, sy_, sx_, false, keep, h_cctx, chs);

  g = mk(R, d, d, cctx, L.w_co, d);
  if (cctx_hl) g.Ahl = h_cctx;
  g.ep.kind = EPI_BIAS_ADD2;
  g.ep.drop = dmask(2, l0, ls);  // cross-attention output phi3
  g.ep.out1 = ybar;
  g.ep.add1 = a1;
  g.ep.out2 = u2;
  g.ep.add2 = Y;
  g.ep.bias = par(L.b_co, 0, l0, ls);
  gemm(g);

  ln.x = u2;
  ln.out = ((keep && !ch) || !h_n2.ok()) ? n2 : Mat{};
  ln.out_hl = h_n2;
  ln.stats = st2;
  ln.gain = par(L.ln2_g, 0, l0, ls);
  ln.bias = par(L.ln2_b, 0, l0, ls);
  ++launches_;
  prof_shape_ = {3, ln.d, 0, ln.G};
  timed(PROF_ROW, 0.0, 8.0 * ln.G * (double)ln.rows * ln.d,
        [&] { launch_ln_fwd(ln, active_, stream_); });

  g = mk(R, f, d, n2, L.w_in, d);
  g.Ahl = h_n2;
  g.ep.kind = EPI_BIAS_GELU;
  if (keep) g.ep.out1 = hh;  // gelu'(h): only the backward reads it
  if ((keep && !ch) || !h_g.ok()) g.ep.out2 = gg;
  g.ep.hl2 = h_g;
  g.ep.range_flag = range_flag_;
  g.ep.bias = par(L.b_in, 0, l0, ls);
  gemm(g);

  g = mk(R, d, f, gg, L.w_out, f);
  g.Ahl = h_g;
  g.ep.kind = EPI_FINAL;
  g.ep.drop = dmask(1, l0, ls);  // MLP output phi2
  g.ep.add1 = ybar;
  g.ep.bias = par(L.b_out, 0, l0, ls);
  Combine c = e.cmb;
  for (Mat* m : {&c.z, &c.out, &c.base, &c.phib, &c.rho, &c.v})
    if (m->ok()) {
      *m = m->offset(y_off_);
      m->ld = d;
    }
  if (c.mode == CM_RES0) c.norm_base = e.cmb.norm_base;  // GEMM tiles first
  g.ep.cmb = c;
  gemm(g);
  if (e.cmb.mode != CM_NONE) {
    ElemCombineArgs ec;
    ec.G = G;
    ec.n = (long long)Tx_ * d;
    Combine cx = e.cmb;  // x part sits at offset 0
    if (cx.mode == CM_RES0) cx.norm_base = e.cmb.norm_base + part_off_elem_;
    ec.cmb = cx;
    ++launches_;
    prof_shape_ = {6, 0, 0, ec.G};
    timed(PROF_ROW, 0.0, 12.0 * ec.G * (double)ec.n,
          [&] { launch_elem_combine(ec, active_, stream_); });
  }
}

// =============================================================================
// Phi^T: lambda + dt*(dF/dz)^T lambda (+ parameter grads), blocks.cpp:516-574
// =============================================================================

void Engine::eval_adjoint(const EvalSpec& e0) {
  check_family_writes(e0, true);
  if (sd_.kind == 2) {
    const int first = e0.layer0, last = e0.layer0 + (e0.G - 1) * e0.layer_step;
    const bool fdec = first >= n_split_, ldec = last >= n_split_;
    if (fdec != ldec) {
      int gsplit = 0;
      while (gsplit < e0.G && ((e0.layer0 + gsplit * e0.layer_step >= n_split_) == fdec)) ++gsplit;
      auto part = [&](int g0, int G) {
        EvalSpec e = e0;
        e.G = G;
        e.layer0 = e0.layer0 + g0 * e0.layer_step;
        e.in = shift(e0.in, g0);
        e.lam = shift(e0.lam, g0);
        e.act.slot0 += g0 * e0.act.step;
        e.bact.slot0 += g0 * e0.bact.step;
        Combine& c = e.cmb;
        c.z = shift(c.z, g0);
        c.out = shift(c.out, g0);
        c.base = shift(c.base, g0);
        c.phib = shift(c.phib, g0);
        c.rho = shift(c.rho, g0);
        c.v = shift(c.v, g0);
        c.norm_base = e0.cmb.norm_base + g0 * e0.cmb.norm_member_stride;
        return e;
      };
      eval_adjoint(part(0, gsplit));
      eval_adjoint(part(gsplit, e0.G - gsplit));
      return;
    }
  }
  EvalSpec e = e0;
  e.cmb.z = e.lam;
  e.cmb.dt = e.dt;
  if (sd_.kind == 2 && e.layer0 >= n_split_)
    decoder_adjoint(e);
  else
    encoder_adjoint(e, causal_);
}

void Engine::encoder_adjoint(const EvalSpec& e, bool causal) {
  const int d = sd_.d, f = sd_.ffn, G = e.G;
  const LayerLayout& L = lay_[0];
  const int l0 = e.layer0, ls = e.layer_step;
  const int R = Tx_;
  if (G > Gmax_) throw ContractViolation("adjoint family larger than scratch");
  Mat UP = e.lam.offset(x_off_), X = e.in.offset(x_off_);
  UP.ld = X.ld = d;
  Mat qkv = act_mat(e.act, al_.qkv, 3 * d), ctx = act_mat(e.act, al_.ctx, d);
  Mat Pm = act_mat(e.act, al_.P, 0), u = act_mat(e.act, al_.u, d);
  Mat hh = act_mat(e.act, al_.h, f), gg = act_mat(e.act, al_.g, f);
  Mat n1 = act_mat(e.act, al_.n1, d), n2 = act_mat(e.act, al_.n2, d);
  Mat st1 = act_mat(e.act, al_.st1, 2), st2 = act_mat(e.act, al_.st2, 2);
  Mat dh = bwd_mat(e, bl_.dh, f), dn2 = bwd_mat(e, bl_.dn2, d), du = bwd_mat(e, bl_.du, d);
  Mat da1 = bwd_mat(e, bl_.da1, d), dctx = bwd_mat(e, bl_.dctx, d), dqkv = bwd_mat(e, bl_.dqkv, 3 * d);
  Mat dn1 = bwd_mat(e, bl_.dn1, d), dPm = bwd_mat(e, bl_.dP, 0);
  // dropout (blocks.cpp:259-271): the MLP branch sees UP * phi2, the
  // attention branch (UP + du) * phi1
  const bool drop = drop_on_;
  const Mat UPm = drop ? bwd_mat(e, bl_.upm, d) : UP;

  auto mk = [&](int M, int N, int K, Mat A, long long w, int ldw) {
    GemmArgs g;
    g.G = G;
    g.M = M;
    g.N = N;
    g.K = K;
    g.A = A;
    g.B = par(w, ldw, l0, ls);
    g.Bhl = par_hl(L, w, l0, ls, true);
    g.b_mn = true;  // dX = U . W: W [out,in] read as [K,N]
    return g;
  };
  if (!e.wgrad_only) {  // dgrad chain (skipped when the backward cache holds it)
    if (drop) {
      ++launches_;
      prof_shape_ = {7, d, 0, G};
      timed(PROF_ROW, 0.0, 8.0 * G * (double)R * d,
            [&] { launch_mask_copy(G, R, d, UPm, UP, dmask(1, l0, ls), active_, stream_); });
    }
    // pre-split dgrad A operands (dh, da1; hl_mat); their fp32 forms only
    // where a weight gradient reads them (this call, or the captured chain)
    // with cache_hl() the dh / da1 slots hold their pre-split rows only (the
    // weight gradients and the bias column sums read them so)
    const bool keep32 = e.want_grads || e.bact.base != nullptr;  // fp32 dqkv for the wgrad
    const bool keepb = keep32 && !cache_hl();
    const Mat h_dh = cache_hl() ? dh : dgrad_hl(G, 1, f),
              h_da1 = cache_hl() ? da1 : dgrad_hl(G, 0, d);
    GemmArgs g = mk(R, f, d, UPm, L.w_out, f);
    g.Ahl = pack_upstream(G, R, UPm);
    g.ep.kind = EPI_GELU_BWD;
    if (keepb || !h_dh.ok()) g.ep.out1 = dh;
    g.ep.hl2 = h_dh;
    g.ep.range_flag = range_flag_;
    g.ep.aux = hh;
    gemm(g);

    g = mk(R, d, f, dh, L.w_in, d);
    g.Ahl = h_dh;
    g.ep.kind = EPI_STORE;
    g.ep.out1 = dn2;
    gemm(g);

    LnBwdArgs lb;
    lb.G = G;
    lb.rows = R;
    lb.d = d;
    lb.x = u;
    lb.stats = st2;
    lb.up = dn2;
    lb.gain = par(L.ln2_g, 0, l0, ls);
    lb.out1 = du;
    if (keepb || !h_da1.ok()) lb.out2 = da1;
    lb.out2_hl = h_da1;
    lb.range_flag = range_flag_;
    lb.addB = UP;
    lb.drop2 = dmask(0, l0, ls);
    ++launches_;
    prof_shape_ = {4, lb.d, 0, lb.G};
    timed(PROF_ROW, 0.0, 20.0 * lb.G * (double)lb.rows * lb.d,
          [&] { launch_ln_bwd(lb, active_, stream_); });

    const bool hs = attn_hs(R / B_, R / B_), dhs = attn_hs(R / B_, R / B_, true);
    g = mk(R, d, d, da1, L.w_o, d);
    g.Ahl = h_da1;
    g.ep.kind = EPI_STORE;
    g.ep.out1 = dctx;
    g.ep.hs = dhs ? 1 : 0;
    g.ep.range_flag = range_flag_;
    gemm(g);

    const Mat h_dqkv = dgrad_hl(G, 1, 3 * d);
    const bool dqkv_hl =
        attention_bwd(G, qkv, qkv.offset(d), qkv.offset(2 * d), Pm, ctx, dctx, dPm, dqkv,
                      dqkv.offset(d), dqkv.offset(2 * d), R / B_, R / B_, causal, h_dqkv,
                      h_dqkv.offset(d), h_dqkv.offset(2 * d), keep32, hs, dhs);

    g = mk(R, d, 3 * d, dqkv, L.w_qkv, d);
    if (dqkv_hl) g.Ahl = h_dqkv;
    g.ep.kind = EPI_STORE;
    g.ep.out1 = dn1;
    gemm(g);

    if (e.cmb.mode != CM_NONE) {
      LnBwdArgs l1;
      l1.G = G;
      l1.rows = R;
      l1.d = d;
      l1.x = X;
      l1.stats = st1;
      l1.up = dn1;
      l1.gain = par(L.ln1_g, 0, l0, ls);
      l1.addA = du;
      Combine c = e.cmb;
      for (Mat* m : {&c.z, &c.out, &c.base, &c.phib, &c.rho, &c.v})
        if (m->ok()) {
          *m = m->offset(x_off_);
          m->ld = d;
        }
      if (c.mode == CM_RES0) c.norm_base = e.cmb.norm_base + part_off_ln_;
      l1.cmb = c;
      ++launches_;
      prof_shape_ = {4, l1.d, 0, l1.G};
      timed(PROF_ROW, 0.0, 20.0 * l1.G * (double)l1.rows * l1.d,
            [&] { launch_ln_bwd(l1, active_, stream_); });
      if (sd_.kind == 2) {
        ElemCombineArgs ec;
        ec.G = G;
        ec.n = (long long)Ty_ * d;
        Combine cy = e.cmb;
        for (Mat* m : {&cy.z, &cy.out, &cy.base, &cy.phib, &cy.rho, &cy.v})
          if (m->ok()) *m = m->offset(y_off_);
        if (cy.mode == CM_RES0) cy.norm_base = e.cmb.norm_base + part_off_elem_;
        ec.cmb = cy;
        ++launches_;
        prof_shape_ = {6, 0, 0, ec.G};
        timed(PROF_ROW, 0.0, 12.0 * ec.G * (double)ec.n,
              [&] { launch_elem_combine(ec, active_, stream_); });
      }
    }
  }

  if (e.want_grads) {
    const float gs = e.gscale;
    // B pre-split (bhl): a cached LN / GELU output (cache_hl)
    auto wg = [&](int M, int N, Mat A, Mat Bm, long long w, int ldw, bool bhl = false,
                  bool ahl = false) {
      GemmArgs w_;
      w_.G = G;
      w_.M = M;
      w_.N = N;
      w_.K = R;
      w_.A = A;
      w_.B = Bm;
      w_.a_mn = true;
      w_.b_mn = true;
      w_.b_mn_hl = bhl && cache_hl();
      w_.a_mn_hl = ahl && cache_hl();
      w_.ep.kind = EPI_GRAD_ACC;
      w_.ep.out1 = grad(w, ldw, l0, ls);
      w_.ep.gscale = gs;
      w_.ep.gscale_mul = e.gscale_mul;
      gemm(w_);
    };
    auto cr = [&](Mat up, int cols, long long b, Mat x, Mat st, long long gn, bool uhl = false) {
      ColRedArgs c;
      c.up_hl = uhl && cache_hl();
      c.G = G;
      c.rows = R;
      c.cols = cols;
      c.up = up;
      c.x = x;
      c.stats = st;
      c.dbias = grad(b, 0, l0, ls);
      if (x.ok()) c.dgain = grad(gn, 0, l0, ls);
      c.gscale = gs;
      c.gscale_mul = e.gscale_mul;
      c.partials = colred_part_;
      c.partials_cap = colred_cap_;
      ++launches_;
      prof_shape_ = {5, c.cols, 0, c.G};
      timed(PROF_ROW, 0.0, (x.ok() ? 8.0 : 4.0) * c.G * (double)c.rows * c.cols,
            [&] { launch_colred(c, active_, stream_); });
    };
    wg(d, f, UPm, gg, L.w_out, f, true);
    cr(UPm, d, L.b_out, Mat{}, Mat{}, 0);
    wg(f, d, dh, n2, L.w_in, d, true, true);
    cr(dh, f, L.b_in, Mat{}, Mat{}, 0, true);
    cr(dn2, d, L.ln2_b, u, st2, L.ln2_g);
    wg(d, d, da1, ctx, L.w_o, d, false, true);
    cr(da1, d, L.b_o, Mat{}, Mat{}, 0, true);
    wg(3 * d, d, dqkv, n1, L.w_qkv, d, true);
    cr(dqkv, 3 * d, L.b_qkv, Mat{}, Mat{}, 0);
    cr(dn1, d, L.ln1_b, X, st1, L.ln1_g);
  }
}

void Engine::decoder_adjoint(const EvalSpec& e) {
  const int d = sd_.d, f = sd_.ffn, G = e.G;
  const LayerLayout& L = lay_[1];
  const int l0 = e.layer0, ls = e.layer_step;
  const int R = Ty_;
  if (G > Gmax_) throw ContractViolation("adjoint family larger than scratch");
  Mat UPy = e.lam.offset(y_off_), Y = e.in.offset(y_off_), X = e.in.offset(x_off_);
  UPy.ld = Y.ld = X.ld = d;
  Mat qkv = act_mat(e.act, al_.qkv, 3 * d), ctx = act_mat(e.act, al_.ctx, d);
  Mat Pm = act_mat(e.act, al_.P, 0), u2 = act_mat(e.act, al_.u, d);
  Mat hh = act_mat(e.act, al_.h, f), gg = act_mat(e.act, al_.g, f);
  Mat n1 = act_mat(e.act, al_.n1, d), n2 = act_mat(e.act, al_.n2, d);
  Mat st1 = act_mat(e.act, al_.st1, 2), st2 = act_mat(e.act, al_.st2, 2);
  Mat n3 = act_mat(e.act, al_.n3, d), u3 = act_mat(e.act, al_.u3, d);
  Mat cq = act_mat(e.act, al_.cq, d), ckv = act_mat(e.act, al_.ckv, 2 * d);
  Mat cctx = act_mat(e.act, al_.cctx, d), cP = act_mat(e.act, al_.cP, 0);
  Mat st3 = act_mat(e.act, al_.st3, 2);
  Mat dh = bwd_mat(e, bl_.dh, f), dn2 = bwd_mat(e, bl_.dn2, d), dy = bwd_mat(e, bl_.dy, d);
  Mat dybar = bwd_mat(e, bl_.dybar, d), dcctx = bwd_mat(e, bl_.dcctx, d), dcq = bwd_mat(e, bl_.dcq, d);
  Mat dckv = bwd_mat(e, bl_.dckv, 2 * d), dn3 = bwd_mat(e, bl_.dn3, d), dxe = bwd_mat(e, bl_.dxe, d);
  Mat da1 = bwd_mat(e, bl_.da1, d), dctx = bwd_mat(e, bl_.dctx, d), dqkv = bwd_mat(e, bl_.dqkv, 3 * d);
  Mat dn1 = bwd_mat(e, bl_.dn1, d), dPm = bwd_mat(e, bl_.dP, 0), dP2 = bwd_mat(e, bl_.dP2, 0);
  // dropout (blocks.cpp:312-324): MLP branch UP * phi2, cross-attention
  // output dybar * phi3, self-attention output (dybar + du3) * phi1
  const bool drop = drop_on_;
  const Mat UPm = drop ? bwd_mat(e, bl_.upm, d) : UPy;
  const Mat dcp = drop ? bwd_mat(e, bl_.dcpre, d) : dybar;

  auto mk = [&](int M, int N, int K, Mat A, long long w, int ldw) {
    GemmArgs g;
    g.G = G;
    g.M = M;
    g.N = N;
    g.K = K;
    g.A = A;
    g.B = par(w, ldw, l0, ls);
    g.Bhl = par_hl(L, w, l0, ls, true);
    g.b_mn = true;
    return g;
  };
  if (!e.wgrad_only) {  // dgrad chain (skipped when the backward cache holds it)
    if (drop) {
      ++launches_;
      prof_shape_ = {7, d, 0, G};
      timed(PROF_ROW, 0.0, 8.0 * G * (double)R * d,
            [&] { launch_mask_copy(G, R, d, UPm, UPy, dmask(1, l0, ls), active_, stream_); });
    }
    // pre-split dgrad A operands as in encoder_adjoint
    // with cache_hl() the dh / da1 slots hold their pre-split rows only (the
    // weight gradients and the bias column sums read them so)
    const bool keep32 = e.want_grads || e.bact.base != nullptr;  // fp32 dqkv for the wgrad
    const bool keepb = keep32 && !cache_hl();
    const Mat h_dh = cache_hl() ? dh : dgrad_hl(G, 1, f),
              h_da1 = cache_hl() ? da1 : dgrad_hl(G, 0, d);
    GemmArgs g = mk(R, f, d, UPm, L.w_out, f);
    g.Ahl = pack_upstream(G, R, UPm);
    g.ep.kind = EPI_GELU_BWD;
    if (keepb || !h_dh.ok()) g.ep.out1 = dh;
    g.ep.hl2 = h_dh;
    g.ep.range_flag = range_flag_;
    g.ep.aux = hh;
    gemm(g);

    g = mk(R, d, f, dh, L.w_in, d);
    g.Ahl = h_dh;
    g.ep.kind = EPI_STORE;
    g.ep.out1 = dn2;
    gemm(g);

    LnBwdArgs lb;
    lb.G = G;
    lb.rows = R;
    lb.d = d;
    lb.x = u2;
    lb.stats = st2;
    lb.up = dn2;
    lb.gain = par(L.ln2_g, 0, l0, ls);
    lb.out1 = dy;      // du2
    lb.out2 = dybar;   // up + du2
    lb.addB = UPy;
    ++launches_;
    prof_shape_ = {4, lb.d, 0, lb.G};
    timed(PROF_ROW, 0.0, 20.0 * lb.G * (double)lb.rows * lb.d,
          [&] { launch_ln_bwd(lb, active_, stream_); });

    if (drop) {
      ++launches_;
      prof_shape_ = {7, d, 0, G};
      timed(PROF_ROW, 0.0, 8.0 * G * (double)R * d,
            [&] { launch_mask_copy(G, R, d, dcp, dybar, dmask(2, l0, ls), active_, stream_); });
    }
    const bool chs = attn_hs(sy_, sx_), cdhs = attn_hs(sy_, sx_, true);
    g = mk(R, d, d, dcp, L.w_co, d);
    g.ep.kind = EPI_STORE;
    g.ep.out1 = dcctx;
    g.ep.hs = cdhs ? 1 : 0;
    g.ep.range_flag = range_flag_;
    gemm(g);

    attention_bwd(G, cq, ckv, ckv.offset(d), cP, cctx, dcctx, dP2, dcq, dckv, dckv.offset(d), sy_,
                  sx_, false, Mat{}, Mat{}, Mat{}, true, chs, cdhs);

    g = mk(R, d, d, dcq, L.w_cq, d);
    g.ep.kind = EPI_STORE;
    g.ep.out1 = dn3;
    gemm(g);

    g = mk(Tx_, d, 2 * d, dckv, L.w_ckv, d);
    g.ep.kind = EPI_STORE;
    g.ep.out1 = dxe;
    gemm(g);

    lb.x = u3;
    lb.stats = st3;
    lb.up = dn3;
    lb.gain = par(L.ln3_g, 0, l0, ls);
    lb.addA = dy;
    lb.out1 = dy;     // du2 + du3
    lb.addB = dybar;
    lb.out2 = (keepb || !h_da1.ok()) ? da1 : Mat{};  // dybar + du3
    lb.out2_hl = h_da1;
    lb.range_flag = range_flag_;
    lb.drop2 = dmask(0, l0, ls);
    ++launches_;
    prof_shape_ = {4, lb.d, 0, lb.G};
    timed(PROF_ROW, 0.0, 20.0 * lb.G * (double)lb.rows * lb.d,
          [&] { launch_ln_bwd(lb, active_, stream_); });

    const bool hs = attn_hs(sy_, sy_), dhs = attn_hs(sy_, sy_, true);
    g = mk(R, d, d, da1, L.w_o, d);
    g.Ahl = h_da1;
    g.ep.kind = EPI_STORE;
    g.ep.out1 = dctx;
    g.ep.hs = dhs ? 1 : 0;
    g.ep.range_flag = range_flag_;
    gemm(g);

    const Mat h_dqkv = dgrad_hl(G, 1, 3 * d);
    const bool dqkv_hl =
        attention_bwd(G, qkv, qkv.offset(d), qkv.offset(2 * d), Pm, ctx, dctx, dPm, dqkv,
                      dqkv.offset(d), dqkv.offset(2 * d), sy_, sy_, true, h_dqkv, h_dqkv.offset(d),
                      h_dqkv.offset(2 * d), keep32, hs, dhs);

    g = mk(R, d, 3 * d, dqkv, L.w_qkv, d);
    if (dqkv_hl) g.Ahl = h_dqkv;
    g.ep.kind = EPI_STORE;
    g.ep.out1 = dn1;
    gemm(g);

    if (e.cmb.mode != CM_NONE) {
      LnBwdArgs l1;
      l1.G = G;
      l1.rows = R;
      l1.d = d;
      l1.x = Y;
      l1.stats = st1;
      l1.up = dn1;
      l1.gain = par(L.ln1_g, 0, l0, ls);
      l1.addA = dy;
      Combine c = e.cmb;
      for (Mat* m : {&c.z, &c.out, &c.base, &c.phib, &c.rho, &c.v})
        if (m->ok()) {
          *m = m->offset(y_off_);
          m->ld = d;
        }
      if (c.mode == CM_RES0) c.norm_base = e.cmb.norm_base + part_off_ln_;
      l1.cmb = c;
      ++launches_;
      prof_shape_ = {4, l1.d, 0, l1.G};
      timed(PROF_ROW, 0.0, 20.0 * l1.G * (double)l1.rows * l1.d,
            [&] { launch_ln_bwd(l1, active_, stream_); });
      ElemCombineArgs ec;
      ec.G = G;
      ec.n = (long long)Tx_ * d;
      ec.F = dxe;
      Combine cx = e.cmb;
      if (cx.mode == CM_RES0) cx.norm_base = e.cmb.norm_base + part_off_elem_;
      ec.cmb = cx;
      ++launches_;
      prof_shape_ = {6, 0, 0, ec.G};
      timed(PROF_ROW, 0.0, 12.0 * ec.G * (double)ec.n,
            [&] { launch_elem_combine(ec, active_, stream_); });
    }
  }

  if (e.want_grads) {
    const float gs = e.gscale;
    auto wg = [&](int M, int N, int K, Mat A, Mat Bm, long long w, int ldw, bool bhl = false,
                  bool ahl = false) {
      GemmArgs w_;
      w_.G = G;
      w_.M = M;
      w_.N = N;
      w_.K = K;
      w_.A = A;
      w_.B = Bm;
      w_.a_mn = true;
      w_.b_mn = true;
      w_.b_mn_hl = bhl && cache_hl();
      w_.a_mn_hl = ahl && cache_hl();
      w_.ep.kind = EPI_GRAD_ACC;
      w_.ep.out1 = grad(w, ldw, l0, ls);
      w_.ep.gscale = gs;
      w_.ep.gscale_mul = e.gscale_mul;
      gemm(w_);
    };
    auto cr = [&](int rows, Mat up, int cols, long long b, Mat x, Mat st, long long gn,
                  bool uhl = false) {
      ColRedArgs c;
      c.up_hl = uhl && cache_hl();
      c.G = G;
      c.rows = rows;
      c.cols = cols;
      c.up = up;
      c.x = x;
      c.stats = st;
      c.dbias = grad(b, 0, l0, ls);
      if (x.ok()) c.dgain = grad(gn, 0, l0, ls);
      c.gscale = gs;
      c.gscale_mul = e.gscale_mul;
      c.partials = colred_part_;
      c.partials_cap = colred_cap_;
      ++launches_;
      prof_shape_ = {5, c.cols, 0, c.G};
      timed(PROF_ROW, 0.0, (x.ok() ? 8.0 : 4.0) * c.G * (double)c.rows * c.cols,
            [&] { launch_colred(c, active_, stream_); });
    };
    wg(d, f, R, UPm, gg, L.w_out, f, true);
    cr(R, UPm, d, L.b_out, Mat{}, Mat{}, 0);
    wg(f, d, R, dh, n2, L.w_in, d, true, true);
    cr(R, dh, f, L.b_in, Mat{}, Mat{}, 0, true);
    cr(R, dn2, d, L.ln2_b, u2, st2, L.ln2_g);
    wg(d, d, R, dcp, cctx, L.w_co, d);
    cr(R, dcp, d, L.b_co, Mat{}, Mat{}, 0);
    wg(d, d, R, dcq, n3, L.w_cq, d, true);
    cr(R, dcq, d, L.b_cq, Mat{}, Mat{}, 0);
    wg(2 * d, d, Tx_, dckv, X, L.w_ckv, d);
    cr(Tx_, dckv, 2 * d, L.b_ckv, Mat{}, Mat{}, 0);
    cr(R, dn3, d, L.ln3_b, u3, st3, L.ln3_g);
    wg(d, d, R, da1, ctx, L.w_o, d, false, true);
    cr(R, da1, d, L.b_o, Mat{}, Mat{}, 0, true);
    wg(3 * d, d, R, dqkv, n1, L.w_qkv, d, true);
    cr(R, dqkv, 3 * d, L.b_qkv, Mat{}, Mat{}, 0);
    cr(R, dn1, d, L.ln1_b, Y, st1, L.ln1_g);
  }
}

// =============================================================================
// MGRIT (mgrit.hpp:58-303) on device-resident levels, block-partitioned over
// ranks. Rank r owns the points (p_lo, p_hi] of every level (its contiguous
// block of coarse intervals); the adjoint system runs the same
// partition reversed in time. Point p_lo itself is a ghost copy of the
// previous rank's last point.
// =============================================================================

Mat Engine::lv_v(const Solver& s, int l, int slot0, int step) const {
  return state_mat(s.lv[l].v, state_n_, sd_.d, slot0, step);
}
Mat Engine::lv_base(const Solver& s, int l, int slot0, int step) const {
  // base of level l is the level l-1 iterate at the coarse-aligned points
  return state_mat(s.lv[l - 1].v, state_n_, sd_.d, slot0 * cfg_.coarsen, step * cfg_.coarsen);
}
Mat Engine::lv_rho(const Solver& s, int l, int slot0, int step) const {
  return state_mat(s.lv[l].rho, state_n_, sd_.d, slot0, step);
}
Mat Engine::lv_phib(const Solver& s, int l, int slot0, int step) const {
  return state_mat(s.lv[l].phib, state_n_, sd_.d, slot0, step);
}

int Engine::rank_at(const Solver& s, int tpos) const {
  return s.adjoint ? world_ - 1 - tpos : tpos;
}

// ghost exchange of one state: the last local point goes to the next rank in
// time, the previous rank's last point lands in our ghost slot
void Engine::exchange_ghost(Solver& s, int level) {
  if (world_ == 1) return;
  const size_t n = (size_t)state_n_;
  tr_->group_start();
  if (s.tpos + 1 < world_)
    tr_->send(s.lv[level].v + (size_t)s.p_hi[level] * n, n, rank_at(s, s.tpos + 1), stream_);
  if (s.tpos > 0)
    tr_->recv(s.lv[level].v + (size_t)s.p_lo[level] * n, n, rank_at(s, s.tpos - 1), stream_);
  tr_->group_end();
}

// Steps k = k0 + g*kstep (g < G) of level `level` of system s, applied to the
// states `in`; results folded by `cmb`.
void Engine::sys_eval(Solver& s, int level, int k0, int kstep, int G, Mat in, Combine cmb,
                      bool capture) {
  if (G <= 0) return;
  long long stride = 1;
  for (int l = 0; l < level; ++l) stride *= cfg_.coarsen;
  const float dt = (float)((double)stride * h_[ib_]);
  for (int g0 = 0; g0 < G; g0 += Gmax_) {
    const int Gc = std::min(Gmax_, G - g0);
    EvalSpec e;
    e.G = Gc;
    e.dt = dt;
    Combine c = cmb;
    c.out = shift(c.out, g0);
    c.base = shift(c.base, g0);
    c.phib = shift(c.phib, g0);
    c.rho = shift(c.rho, g0);
    c.v = shift(c.v, g0);
    c.norm_base = cmb.norm_base + g0 * cmb.norm_member_stride;
    e.cmb = c;
    const int kk0 = k0 + g0 * kstep;
    if (!s.adjoint) {
      e.layer0 = ib_ + (int)(kk0 * stride);
      e.layer_step = (int)(kstep * stride);
      e.in = shift(in, g0);
      if (capture)
        e.act = ActRef{cache_, al_.size, e.layer0, e.layer_step};
      else
        e.act = ActRef{scratch_, al_.size, 0, 1};
      eval_forward(e);
    } else {
      // adjoint step k applies layer n = N-1-k*stride at traj[ib+n] (adjoint.hpp:45-54)
      e.layer0 = ib_ + (N_ - 1 - (int)(kk0 * stride));
      e.layer_step = -(int)(kstep * stride);
      e.lam = shift(in, g0);
      e.in = state_mat(traj_, state_n_, sd_.d, e.layer0, e.layer_step);
      e.act = ActRef{cache_, al_.size, e.layer0, e.layer_step};
      // level-0 relaxation steps keep their dgrad intermediates per layer:
      // the parameter pass then only forms dW, db for those layers
      if (capture) e.bact = ActRef{bcache_, bl_.size, e.layer0, e.layer_step};
      eval_adjoint(e);
    }
  }
}

// v[j] = relax(Phi(v[j-1])) for j = j0 + g*jstep (mgrit.hpp:273-282)
void Engine::relax_family(Solver& s, int level, int j0, int jstep, int G, bool capture) {
  Combine c;
  c.out = lv_v(s, level, j0, jstep);
  if (level == 0) {
    c.mode = CM_PLAIN;
  } else {
    c.mode = CM_FAS;
    c.base = lv_base(s, level, j0, jstep);
    c.phib = lv_phib(s, level, j0, jstep);
    c.rho = lv_rho(s, level, j0, jstep);
  }
  sys_eval(s, level, j0 - 1, jstep, G, lv_v(s, level, j0 - 1, jstep), c, capture);
}

void Engine::f_relax(Solver& s, int level, bool capture) {  // mgrit.hpp:125-137
  const int cf = cfg_.coarsen;
  const int lo = s.p_lo[level], nc = (s.p_hi[level] - lo) / cf;
  for (int i = 1; i < cf; ++i) relax_family(s, level, lo + i, cf, nc, capture);
}

void Engine::c_relax(Solver& s, int level) {  // mgrit.hpp:139-149
  const int cf = cfg_.coarsen;
  const int lo = s.p_lo[level], nc = (s.p_hi[level] - lo) / cf;
  relax_family(s, level, lo + cf, cf, nc, false);
  exchange_ghost(s, level);
}

// Residual rows at the coarse-aligned points j = k*c_f (mgrit.hpp:159-187).
// After F-relaxation every F-point row is exactly zero at level 0 (v[j] was
// just set to Phi(v[j-1]) by the same deterministic kernels), and at coarser
// levels F-point rows are never read (injection keeps only k*c_f rows), so
// only the C-point rows are evaluated; they are written straight into the
// next level's rho (injection, mgrit.hpp:204).
void Engine::residual_c_rows(Solver& s, int level, bool capture) {
  const int cf = cfg_.coarsen;
  const int lo = s.p_lo[level], nc = (s.p_hi[level] - lo) / cf;
  Combine c;
  c.out = lv_rho(s, level + 1, lo / cf + 1, 1);
  c.v = lv_v(s, level, lo + cf, cf);
  if (level == 0) {
    // per-interval partial slots [chunk][S]: the trace is summed in interval
    // order, independent of the rank count and of how families are launched
    c.mode = CM_RES0;
    c.norm_partials = s.partials;
    c.norm_base = (lo / cf) * s.slots_per_chunk;
    c.norm_member_stride = s.slots_per_chunk;
    const size_t total = (size_t)s.n_chunks * s.slots_per_chunk;
    MGLP_CUDA(cudaMemsetAsync(s.partials, 0, total * sizeof(double), stream_));
    sys_eval(s, level, lo + cf - 1, cf, nc, lv_v(s, level, lo + cf - 1, cf), c, capture);
    const double* summed = s.partials;
    if (world_ > 1) {
      const size_t blk = (size_t)nc * s.slots_per_chunk;
      tr_->allgather(s.partials + (size_t)(lo / cf) * s.slots_per_chunk, s.gathered, blk, stream_);
      summed = s.gathered;
    }
    launch_trace_record(s.ctrl, summed, s.n_chunks, s.slots_per_chunk,
                        world_ > 1 ? s.n_chunks / world_ : s.n_chunks, s.adjoint && world_ > 1,
                        stream_, s.adjoint ? lam_sc_ : nullptr);
    ++launches_;
  } else {
    c.mode = CM_RESL;
    c.base = lv_base(s, level, lo + cf, cf);
    c.phib = lv_phib(s, level, lo + cf, cf);
    c.rho = lv_rho(s, level, lo + cf, cf);
    sys_eval(s, level, lo + cf - 1, cf, nc, lv_v(s, level, lo + cf - 1, cf), c, false);
  }
}

void Engine::restrict_to(Solver& s, int level) {  // mgrit.hpp:199-211
  const bool coarsest = level == cfg_.levels - 1;
  const int lo = s.p_lo[level], hi = s.p_hi[level];
  // v = base on our points and the ghost (the coarsest level only needs its
  // initial condition: exact_solve overwrites every other point)
  prof_shape_ = {7, 0, 0, coarsest ? 1 : hi - lo + 1};
  timed(PROF_ROW, 0.0, 8.0 * (coarsest ? 1 : hi - lo + 1) * (double)state_n_, [&] {
    launch_copy(coarsest ? 1 : hi - lo + 1, state_n_, lv_v(s, level, lo, 1),
                lv_base(s, level, lo, 1), active_, stream_);
  });
  ++launches_;
  Combine cm;
  cm.mode = CM_PLAIN;
  cm.out = lv_phib(s, level, lo + 1, 1);
  sys_eval(s, level, lo, 1, hi - lo, lv_base(s, level, lo, 1), cm, false);
}

void Engine::correct_from(Solver& s, int level) {  // mgrit.hpp:214-223
  // our coarse points and the ghost (its coarse value arrived with the
  // coarse chain / ghost exchange, so the correction is bitwise the owner's)
  const int k0 = std::max(s.p_lo[level], 1), hi = s.p_hi[level];
  prof_shape_ = {8, 0, 0, hi - k0 + 1};
  timed(PROF_ROW, 0.0, 16.0 * (hi - k0 + 1) * (double)state_n_, [&] {
    launch_correct(hi - k0 + 1, state_n_, lv_v(s, level - 1, k0 * cfg_.coarsen, cfg_.coarsen),
                   lv_v(s, level, k0, 1), lv_base(s, level, k0, 1), active_, stream_);
  });
  ++launches_;
}

void Engine::exact_solve(Solver& s, int level) {  // mgrit.hpp:227-231
  // the serial coarse chain, pipelined across ranks
  const size_t n = (size_t)state_n_;
  if (world_ > 1 && s.tpos > 0)
    tr_->recv(s.lv[level].v + (size_t)s.p_lo[level] * n, n, rank_at(s, s.tpos - 1), stream_);
  for (int j = s.p_lo[level] + 1; j <= s.p_hi[level]; ++j) relax_family(s, level, j, 1, 1, false);
  if (world_ > 1 && s.tpos + 1 < world_)
    tr_->send(s.lv[level].v + (size_t)s.p_hi[level] * n, n, rank_at(s, s.tpos + 1), stream_);
}

void Engine::descend(Solver& s, int level) {  // mgrit.hpp:285-296
  if (level == cfg_.levels - 1) {
    exact_solve(s, level);
    return;
  }
  f_relax(s, level, false);
  c_relax(s, level);
  f_relax(s, level, false);
  residual_c_rows(s, level, false);
  restrict_to(s, level + 1);
  descend(s, level + 1);
  correct_from(s, level + 1);
  f_relax(s, level, false);
}

void Engine::v_cycle(Solver& s, double tol, bool first) {  // mgrit.hpp:235-246
  const bool cap = true;  // forward: linearisation cache; adjoint: dgrad cache
  const bool one_level = cfg_.levels == 1;
  // Every cycle ends with the F-points equal to Phi of the current C-points
  // (final F-relaxation, or F + residual with one level), so the opening
  // F-relaxation of the next cycle of the same solve would recompute the same
  // bits: only the first cycle runs it.
  if (first) f_relax(s, 0, cap && one_level);
  c_relax(s, 0);
  f_relax(s, 0, cap);
  residual_c_rows(s, 0, cap && one_level);
  if (!one_level) {
    restrict_to(s, 1);
    descend(s, 1);
    correct_from(s, 1);
    f_relax(s, 0, cap);
  }
  launch_cycle_end(s.ctrl, tol, stream_);
  ++launches_;
}

int Engine::host_cycles(int which) const {
  if (!mon_) return which == 0 ? cfg_.fwd_iters : cfg_.bwd_iters;
  return capture_cycles_ > 0 ? capture_cycles_ : bound_[which];
}

void Engine::monitor_attach(double threshold, int policy_switch, int cap) {
  if (threshold <= 0.0) throw ValidationError("InexactnessMonitor: threshold must be positive");
  if (cap < 1) throw ValidationError("InexactnessMonitor: max_iter_cap must be >= 1");
  MGLP_CUDA(cudaSetDevice(device_));
  if (!mon_) {
    MGLP_CUDA(cudaMalloc(&mon_, sizeof(MonitorDev)));
    MGLP_CUDA(cudaMalloc(&mon_sum_, sizeof(MonitorSummary)));
    MGLP_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&mon_host_), sizeof(MonitorSummary),
                            cudaHostAllocDefault));
  }
  launch_monitor_init(mon_, threshold, policy_switch, cap, cfg_.fwd_iters, cfg_.bwd_iters, stream_);
  MGLP_CUDA(cudaMemsetAsync(mon_sum_, 0, sizeof(MonitorSummary), stream_));
  MGLP_CUDA(cudaMemsetAsync(mon_host_, 0, sizeof(MonitorSummary), stream_));
  bound_[0] = cfg_.fwd_iters;
  bound_[1] = cfg_.bwd_iters;
  mon_cap_ = cap;
  drop_graph();
}

void Engine::monitor_probe(bool begin) {
  if (!mon_) throw ValidationError("monitor: not attached");
  launch_monitor_probe(mon_, begin ? 1 : 0, stream_);
  ++launches_;
  if (begin) {
    bound_saved_[0] = bound_[0];
    bound_saved_[1] = bound_[1];
    bound_[0] *= 2;
    bound_[1] *= 2;
  } else {
    bound_[0] = bound_saved_[0];
    bound_[1] = bound_saved_[1];
  }
}

void Engine::monitor_record(long long batch) {
  if (!mon_) throw ValidationError("monitor: not attached");
  if (!fwd_.ctrl || !bwd_.ctrl) throw ValidationError("monitor: record before any solve");
  launch_monitor_record(mon_, fwd_.ctrl, bwd_.ctrl, batch, mon_sum_, stream_);
  MGLP_CUDA(cudaMemcpyAsync(mon_host_, mon_sum_, sizeof(MonitorSummary), cudaMemcpyDeviceToHost,
                            stream_));
  ++launches_;
  if (batch >= 0) {  // the decision may double both budgets (capped)
    bound_[0] = std::max(bound_[0], std::min(2 * bound_[0], mon_cap_));
    bound_[1] = std::max(bound_[1], std::min(2 * bound_[1], mon_cap_));
  }
}

const MonitorSummary& Engine::monitor_read() {
  if (!mon_) throw ValidationError("monitor: not attached");
  MGLP_CUDA(cudaStreamSynchronize(stream_));
  cfg_.fwd_iters = bound_[0] = mon_host_->budget[0];
  cfg_.bwd_iters = bound_[1] = mon_host_->budget[1];
  return *mon_host_;
}

int Engine::monitor_reports(long long* batch, double* ff, double* bf, int* dec, int cap) {
  if (!mon_) throw ValidationError("monitor: not attached");
  MonitorDev* h = nullptr;
  MGLP_CUDA(cudaMallocHost(reinterpret_cast<void**>(&h), sizeof(MonitorDev)));
  MGLP_CUDA(cudaMemcpyAsync(h, mon_, sizeof(MonitorDev), cudaMemcpyDeviceToHost, stream_));
  MGLP_CUDA(cudaStreamSynchronize(stream_));
  const int n = std::min(h->n_reports, kMonReports);
  const int first = h->n_reports - n;  // oldest kept report
  int k = 0;
  for (; k < n && k < cap; ++k) {
    const int i = (first + k) % kMonReports;
    if (batch) batch[k] = h->rep_batch[i];
    if (ff) ff[k] = h->rep_ff[i];
    if (bf) bf[k] = h->rep_bf[i];
    if (dec) dec[k] = h->rep_dec[i];
  }
  cudaFreeHost(h);
  return n;
}

void Engine::set_budget(int fwd_iters, int bwd_iters) {
  cfg_.fwd_iters = fwd_iters;
  cfg_.bwd_iters = bwd_iters;
  if (mon_) {
    launch_monitor_set_budget(mon_, fwd_iters, bwd_iters, stream_);
    bound_[0] = fwd_iters;
    bound_[1] = bwd_iters;
  }
}

void Engine::solve(Solver& s, int iters, double tol) {  // mgrit.hpp:248-262
  if (iters < 1) throw ValidationError("solve_forward: need at least one iteration");
  launch_ctrl_begin(s.ctrl, iters, mon_ ? &mon_->budget[s.adjoint ? 1 : 0] : nullptr, stream_);
  active_ = &s.ctrl->active;
  for (int it = 0; it < iters; ++it) v_cycle(s, tol, it == 0);
  active_ = nullptr;
}

// =============================================================================
// LayerParallelEngine (adjoint.hpp:113-206)
// =============================================================================

bool Engine::owns_layer(int l) const {
  if (l < ib_) return rank_ == 0;
  if (l >= ie_) return rank_ == world_ - 1;
  const int i = l - ib_;
  return i >= fwd_.p_lo[0] && i < fwd_.p_hi[0];
}

void Engine::forward_device(const float* z0_dev) {
  MGLP_CUDA(cudaSetDevice(device_));
  if (!traj_) throw ValidationError("forward: set_shape first");
  std::fill(cache_valid_.begin(), cache_valid_.end(), 0);
  MGLP_CUDA(cudaMemcpyAsync(traj_, z0_dev, state_n_ * sizeof(float), cudaMemcpyDeviceToDevice,
                            stream_));
  auto serial_step = [&](int l) {
    EvalSpec e;
    e.G = 1;
    e.layer0 = l;
    e.dt = (float)h_[l];
    e.in = state_mat(traj_, state_n_, sd_.d, l, 1);
    e.act = ActRef{cache_, al_.size, l, 1};
    e.cmb.mode = CM_PLAIN;
    e.cmb.out = state_mat(traj_, state_n_, sd_.d, l + 1, 1);
    eval_forward(e);
    cache_valid_[l] = 1;
  };
  // opening buffers run on every rank (each needs the initial condition for
  // the broadcast guess); only rank 0 keeps their linearisation
  for (int l = 0; l < ib_; ++l) serial_step(l);
  const int guess = (first_fwd_ || !cfg_.warm_start) ? cfg_.cold_guess : 2;
  first_fwd_ = false;
  if (fwd_displaced_) {
    // the warm window was displaced by another trajectory: bring it back
    // (points 1..N; point 0 is the initial condition just set)
    if (guess == 2) dcopy(fwd_.lv[0].v, fwd_stash_, state_n_, win_r_, 1);
    fwd_displaced_ = false;
  }
  Mat v0 = lv_v(fwd_, 0, 0, 0);
  // the guess covers this rank's points and its ghost: (max(1, p_lo), p_hi]
  const int g0 = std::max(1, fwd_.p_lo[0]), gn = fwd_.p_hi[0] - g0 + 1;
  if (guess == 0) {
    launch_copy(gn, state_n_, lv_v(fwd_, 0, g0, 1), v0, nullptr, stream_);
  } else if (guess == 1) {
    launch_zero(gn, state_n_, lv_v(fwd_, 0, g0, 1), nullptr, stream_);
  }
  solve(fwd_, host_cycles(0), cfg_.fwd_tol);
  // the level-0 F-relaxations captured the linearization of every layer
  // whose input is final: all but the last layer of each coarse interval
  // (with one level the C-point residual evaluations capture those too)
  const int cf = cfg_.coarsen;
  for (int i = fwd_.p_lo[0]; i < fwd_.p_hi[0]; ++i)
    if (cfg_.levels == 1 || (i % cf) != cf - 1) cache_valid_[ib_ + i] = 1;
  if (rank_ == world_ - 1)
    for (int l = ie_; l < total_; ++l) serial_step(l);
}

// Linearization pass for the owned layers whose activations were not captured.
void Engine::ensure_linearization() {
  std::vector<int> miss;
  for (int l = 0; l < total_; ++l)
    if (!cache_valid_[l] && owns_layer(l)) miss.push_back(l);
  size_t i = 0;
  while (i < miss.size()) {
    // affine run
    size_t j = i + 1;
    const int step = (j < miss.size()) ? miss[j] - miss[i] : 1;
    while (j < miss.size() && miss[j] - miss[j - 1] == step && (int)(j - i) < Gmax_) ++j;
    EvalSpec e;
    e.G = (int)(j - i);
    e.layer0 = miss[i];
    e.layer_step = step;
    e.dt = 0.f;
    e.in = state_mat(traj_, state_n_, sd_.d, miss[i], step);
    e.act = ActRef{cache_, al_.size, miss[i], step};
    e.cmb.mode = CM_NONE;
    eval_forward(e);
    for (size_t k = i; k < j; ++k) cache_valid_[miss[k]] = 1;
    i = j;
  }
}

void Engine::backward_device(const float* lamN_dev, float* lam0_dev, bool want_grads,
                             bool traj_is_current) {
  MGLP_CUDA(cudaSetDevice(device_));
  if (!traj_) throw ValidationError("backward: set_shape first");
  if (!traj_is_current) std::fill(cache_valid_.begin(), cache_valid_.end(), 0);
  ensure_linearization();
  const Mat LAM = state_mat(lam_all_, state_n_, sd_.d, 0, 1);
  const int guess = (first_bwd_ || !cfg_.warm_start) ? cfg_.cold_guess : 2;
  first_bwd_ = false;
  // lambda_N -> 2^k lambda_N (LamScale): the last rank's lambda_N (and, for a
  // warm guess, every rank's stored adjoint states in their true scale)
  // decides k; every rank uses the same factor
  if (rank_ == world_ - 1) launch_lam_amax(lamN_dev, state_n_, lam_sc_, stream_);
  else MGLP_CUDA(cudaMemsetAsync(&lam_sc_->amax_bits, 0, sizeof(unsigned), stream_));
  if (guess == 2) {
    // this rank's owned adjoint points (the ghost is another rank's)
    const int a = bwd_.p_lo[0] + 1, b = bwd_.p_hi[0];
    launch_lam_amax_warm(bwd_.lv[0].v + (size_t)a * state_n_, (long long)(b - a + 1) * state_n_,
                         lam_sc_, stream_);
    ++launches_;
    if (world_ > 1) {
      // max over ranks: all-gather the per-rank maxima (as doubles), then max
      double* mx = lam_gather_;
      launch_lam_bits_to_f64(lam_sc_, mx + world_, stream_);
      tr_->allgather(mx + world_, mx, 1, stream_);
      launch_lam_bits_max(mx, world_, lam_sc_, stream_);
      launches_ += 2;
    }
  } else if (world_ > 1) {
    tr_->bcast(reinterpret_cast<float*>(lam_sc_), 1, world_ - 1, stream_);
  }
  if (rank_ == world_ - 1) {
    launch_lam_scale(lamN_dev, lam_all_ + (size_t)total_ * state_n_, state_n_, lam_sc_, +1,
                     stream_);
  } else {
    // no lambda_N here (its slot is another rank's): publish the factor only
    launch_lam_scale(nullptr, nullptr, 0, lam_sc_, +1, stream_);
  }
  launches_ += 2;
  const float* gmul = &lam_sc_->down;
  auto serial_adj = [&](int l) {
    EvalSpec e;
    e.G = 1;
    e.layer0 = l;
    e.dt = (float)h_[l];
    e.lam = shift(LAM, l + 1);
    e.in = state_mat(traj_, state_n_, sd_.d, l, 1);
    e.act = ActRef{cache_, al_.size, l, 1};
    e.cmb.mode = CM_PLAIN;
    e.cmb.out = shift(LAM, l);
    e.want_grads = want_grads;
    e.gscale = (float)h_[l];
    e.gscale_mul = gmul;
    eval_adjoint(e);
  };
  // closing buffers on the last rank, then mu[0] = lambda at the interior end
  if (rank_ == world_ - 1) {
    for (int l = total_ - 1; l >= ie_; --l) serial_adj(l);
    MGLP_CUDA(cudaMemcpyAsync(bwd_.lv[0].v, lam_all_ + (size_t)ie_ * state_n_,
                              state_n_ * sizeof(float), cudaMemcpyDeviceToDevice, stream_));
  }
  if (world_ > 1) tr_->bcast(bwd_.lv[0].v, (size_t)state_n_, world_ - 1, stream_);
  const int b0 = std::max(1, bwd_.p_lo[0]), bn = bwd_.p_hi[0] - b0 + 1;
  if (guess == 0)
    launch_copy(bn, state_n_, lv_v(bwd_, 0, b0, 1), lv_v(bwd_, 0, 0, 0), nullptr, stream_);
  else if (guess == 1)
    launch_zero(bn, state_n_, lv_v(bwd_, 0, b0, 1), nullptr, stream_);
  else {
    // warm states were stored at the previous solve's 2^k
    launch_lam_rescale(bn, state_n_, lv_v(bwd_, 0, b0, 1), lam_sc_, stream_);
    ++launches_;
  }
  launch_lam_commit(lam_sc_, stream_);
  ++launches_;
  solve(bwd_, host_cycles(1), cfg_.bwd_tol);
  // parameter pass over the owned layers (adjoint.hpp:165-175): layer ib+i at
  // traj[ib+i] with upstream mu[N-1-i], gscale = h. The final level-0
  // relaxation evaluated exactly these (layer, upstream) pairs for every
  // adjoint step k = N-1-i that is not the last of its interval, and kept
  // their dgrad intermediates: those layers only need dW, db.
  if (want_grads) {
    const int cf = cfg_.coarsen;
    const int i_lo = fwd_.p_lo[0], i_hi = fwd_.p_hi[0];
    auto family = [&](int i0, int G, int step, bool cached) {
      EvalSpec e;
      e.G = G;
      e.layer0 = ib_ + i0;
      e.layer_step = step;
      e.dt = 0.f;
      e.lam = lv_v(bwd_, 0, N_ - 1 - i0, -step);
      e.in = state_mat(traj_, state_n_, sd_.d, ib_ + i0, step);
      e.act = ActRef{cache_, al_.size, ib_ + i0, step};
      if (cached) e.bact = ActRef{bcache_, bl_.size, ib_ + i0, step};
      e.cmb.mode = CM_NONE;
      e.want_grads = true;
      e.wgrad_only = cached;
      e.gscale = (float)h_[ib_];
      e.gscale_mul = gmul;
      eval_adjoint(e);
    };
    auto cached = [&](int i) { return cfg_.levels == 1 || ((N_ - 1 - i) % cf) != cf - 1; };
    // families with an affine layer index: the uncached layers share one
    // residue mod c_f, the cached ones split into the other c_f-1 residues
    std::vector<std::vector<int>> groups(cf + 1);
    for (int i = i_lo; i < i_hi; ++i) groups[cached(i) ? i % cf : cf].push_back(i);
    for (int gi = 0; gi <= cf; ++gi) {
      const std::vector<int>& v = groups[gi];
      const bool is_cached = gi < cf;
      for (size_t a = 0; a < v.size();) {
        size_t b = a + 1;
        const int step = (b < v.size()) ? v[b] - v[a] : 1;
        while (b < v.size() && v[b] - v[b - 1] == step && (int)(b - a) < Gmax_) ++b;
        family(v[a], (int)(b - a), step, is_cached);
        a = b;
      }
    }
  }
  // lambda at the interior start lives on rank 0 (the last adjoint block)
  if (rank_ == 0) {
    MGLP_CUDA(cudaMemcpyAsync(lam_all_ + (size_t)ib_ * state_n_,
                              bwd_.lv[0].v + (size_t)N_ * state_n_, state_n_ * sizeof(float),
                              cudaMemcpyDeviceToDevice, stream_));
    for (int l = ib_ - 1; l >= 0; --l) serial_adj(l);
    if (lam0_dev) {
      launch_lam_scale(lam_all_, lam0_dev, state_n_, lam_sc_, -1, stream_);
      ++launches_;
    }
  }
}

void Engine::capture_step(const float* z0_dev, const float* lamN_dev, float* lam0_dev,
                          bool want_grads) {
  MGLP_CUDA(cudaSetDevice(device_));
  drop_graph();
  if (profiling_) throw ValidationError("capture_step: disable profiling first");
  // run once uncaptured so lazily created state (TMA encoder, kernel
  // attributes) exists and the cache bookkeeping reaches its steady state
  forward_device(z0_dev);
  backward_device(lamN_dev, lam0_dev, want_grads, true);
  MGLP_CUDA(cudaStreamSynchronize(stream_));
  const long long before = launches_;
  cudaGraph_t g = nullptr;
  MGLP_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
  try {
    forward_device(z0_dev);
    backward_device(lamN_dev, lam0_dev, want_grads, true);
  } catch (...) {
    cudaStreamEndCapture(stream_, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  MGLP_CUDA(cudaStreamEndCapture(stream_, &g));
  graph_launches_ = launches_ - before;
  MGLP_CUDA(cudaGraphInstantiate(&graph_exec_, g, 0));
  MGLP_CUDA(cudaGraphDestroy(g));
}

void Engine::replay_step() {
  if (!graph_exec_) throw ValidationError("replay_step: no captured step");
  MGLP_CUDA(cudaGraphLaunch(graph_exec_, stream_));
  launches_ += graph_launches_;
}

void Engine::drop_graph() {
  if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
  graph_exec_ = nullptr;
  graph_launches_ = 0;
}

void Engine::read_trace(bool fwd, std::vector<double>* trace, bool* converged) {
  SolveCtrl c;
  MGLP_CUDA(cudaMemcpyAsync(&c, fwd ? fwd_.ctrl : bwd_.ctrl, sizeof(SolveCtrl),
                            cudaMemcpyDeviceToHost, stream_));
  check_range();
  if (c.truncated)
    throw ContractViolation("the device iteration budget exceeds the cycles this (captured) solve "
                            "issues: recapture with more cycles (set_capture_cycles)");
  trace->assign(c.trace, c.trace + std::min(c.n_trace, kMaxTrace));
  *converged = c.converged != 0;
}

long long Engine::snapshot() {  // adjoint.hpp:187-194
  if (!traj_ || fwd_.lv.empty()) {
    // nothing solved yet (no shape): the snapshot is the first-call flags
    snap_first_fwd_ = first_fwd_;
    snap_first_bwd_ = first_bwd_;
    snap_empty_ = true;
    snap_id_ = ++snap_seq_;
    return snap_id_;
  }
  snap_empty_ = false;
  if (!snap_fwd_) snap_fwd_ = dalloc(state_n_, N_ + 1, win_r_);
  if (!snap_bwd_) snap_bwd_ = dalloc(state_n_, N_ + 1, bwd0_r_);
  // the forward solver's warm states: the trajectory window, or its stash
  // while another trajectory occupies traj_
  const float* fv = fwd_displaced_ ? fwd_stash_ : fwd_.lv[0].v;
  dcopy(snap_fwd_, fv, state_n_, win_r_);
  dcopy(snap_bwd_, bwd_.lv[0].v, state_n_, bwd0_r_);
  // ... and the 2^k those adjoint states are stored at
  if (!snap_sc_) MGLP_CUDA(cudaMalloc(&snap_sc_, sizeof(LamScale)));
  MGLP_CUDA(cudaMemcpyAsync(snap_sc_, lam_sc_, sizeof(LamScale), cudaMemcpyDeviceToDevice, stream_));
  snap_first_fwd_ = first_fwd_;
  snap_first_bwd_ = first_bwd_;
  snap_id_ = ++snap_seq_;
  return snap_id_;
}

void Engine::restore(long long id) {  // adjoint.hpp:196-201
  if (snap_id_ == 0) throw ValidationError("restore: no snapshot taken");
  if (id >= 0 && id != snap_id_)
    throw ValidationError("restore: that snapshot was overwritten by a later snapshot or a shape "
                          "change (the engine keeps one snapshot slot)");
  if (snap_empty_) {  // taken before any solve: only the first-call flags
    first_fwd_ = snap_first_fwd_;
    first_bwd_ = snap_first_bwd_;
    return;
  }
  // restore the forward warm states into the stash: traj_ keeps the current
  // trajectory (a following backward may linearise at it); the next forward
  // solve moves the stash back into its window
  if (!fwd_stash_) fwd_stash_ = dalloc(state_n_, N_ + 1, win_r_);
  dcopy(fwd_stash_, snap_fwd_, state_n_, win_r_);
  fwd_displaced_ = true;
  dcopy(bwd_.lv[0].v, snap_bwd_, state_n_, bwd0_r_);
  MGLP_CUDA(cudaMemcpyAsync(&lam_sc_->k_state, &snap_sc_->k_state, sizeof(int),
                            cudaMemcpyDeviceToDevice, stream_));
  first_fwd_ = snap_first_fwd_;
  first_bwd_ = snap_first_bwd_;
}

double Engine::lam_unscale() const {
  LamScale h;
  MGLP_CUDA(cudaMemcpyAsync(&h, lam_sc_, sizeof(LamScale), cudaMemcpyDeviceToHost, stream_));
  MGLP_CUDA(cudaStreamSynchronize(stream_));
  return h.down_d;
}

void Engine::displace_forward_window() {
  if (fwd_displaced_ || eval_only_ || !traj_ || fwd_.lv.empty()) return;
  if (!fwd_stash_) fwd_stash_ = dalloc(state_n_, N_ + 1, win_r_);
  dcopy(fwd_stash_, fwd_.lv[0].v, state_n_, win_r_);
  fwd_displaced_ = true;
}

void Engine::seed_forward_from_traj() {
  if (eval_only_ || !traj_ || fwd_.lv.empty()) throw ValidationError("seed: set_shape first");
  fwd_displaced_ = false;
  displace_forward_window();  // stash := the window as it is now
}

void Engine::check_range() {
  int range = 0;
  MGLP_CUDA(cudaMemcpyAsync(&range, range_flag_, sizeof(int), cudaMemcpyDeviceToHost, stream_));
  MGLP_CUDA(cudaStreamSynchronize(stream_));
  if (range) {
    MGLP_CUDA(cudaMemsetAsync(range_flag_, 0, sizeof(int), stream_));
    MGLP_CUDA(cudaStreamSynchronize(stream_));
    throw ContractViolation(
        "a GEMM operand exceeded the fp16 range of the split tensor-core path (|x| >= 65520)");
  }
}

// ---- serial sweeps (blocks.cpp:659-682) ----
void Engine::serial_forward_device(const float* z0_dev) {
  if (world_ > 1)
    throw ValidationError("serial sweeps run on a single-rank engine (each rank holds its block)");
  MGLP_CUDA(cudaSetDevice(device_));
  displace_forward_window();
  MGLP_CUDA(cudaMemcpyAsync(traj_, z0_dev, state_n_ * sizeof(float), cudaMemcpyDeviceToDevice,
                            stream_));
  for (int l = 0; l < total_; ++l) {
    EvalSpec e;
    e.G = 1;
    e.layer0 = l;
    e.dt = (float)h_[l];
    e.in = state_mat(traj_, state_n_, sd_.d, l, 1);
    e.act = ActRef{cache_, al_.size, l, 1};
    e.cmb.mode = CM_PLAIN;
    e.cmb.out = state_mat(traj_, state_n_, sd_.d, l + 1, 1);
    eval_forward(e);
    cache_valid_[l] = 1;
  }
}

void Engine::serial_adjoint_device(const float* lamN_dev, float* lam0_dev, bool want_grads) {
  if (world_ > 1)
    throw ValidationError("serial sweeps run on a single-rank engine (each rank holds its block)");
  MGLP_CUDA(cudaSetDevice(device_));
  ensure_linearization();
  const Mat LAM = state_mat(lam_all_, state_n_, sd_.d, 0, 1);
  launch_lam_amax(lamN_dev, state_n_, lam_sc_, stream_);
  launch_lam_scale(lamN_dev, lam_all_ + (size_t)total_ * state_n_, state_n_, lam_sc_, +1,
                   stream_);
  launches_ += 2;
  for (int l = total_ - 1; l >= 0; --l) {
    EvalSpec e;
    e.G = 1;
    e.layer0 = l;
    e.dt = (float)h_[l];
    e.lam = shift(LAM, l + 1);
    e.in = state_mat(traj_, state_n_, sd_.d, l, 1);
    e.act = ActRef{cache_, al_.size, l, 1};
    e.cmb.mode = CM_PLAIN;
    e.cmb.out = shift(LAM, l);
    e.want_grads = want_grads;
    e.gscale = (float)h_[l];
    e.gscale_mul = &lam_sc_->down;
    eval_adjoint(e);
  }
  if (lam0_dev) {
    launch_lam_scale(lam_all_, lam0_dev, state_n_, lam_sc_, -1, stream_);
    ++launches_;
  }
}

// ---- single-step hooks ----
namespace {
// byte masks of every (layer, site) block: element i keeps iff
// u01(splitmix64(key ^ i)) < keep (blocks.cpp:583-589; rng.hpp derive/u01),
// key = the first four derive rounds, precomputed per block on the host
__global__ void dropout_gen_kernel(unsigned char* m, const unsigned long long* keys,
                                   const int* rows, long long slot, int d, int nblocks,
                                   double keep_thr) {
  const int blk = blockIdx.y;
  if (blk >= nblocks) return;
  const long long n = (long long)rows[blk] * d;
  unsigned char* out = m + (long long)blk * slot;
  const unsigned long long key = keys[blk];
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = (double)(splitmix64(key ^ (unsigned long long)i) >> 11) < keep_thr ? 1 : 0;
}
}  // namespace

void Engine::clear_dropout() {
  if (!drop_on_) return;
  drop_on_ = false;
  // cached activations / a captured step used the masks
  invalidate_linearization();
  drop_graph();
}

void Engine::refresh_dropout(uint64_t seed, uint64_t batch_index) {
  const bool was_on = drop_on_;
  drop_on_ = false;
  if (sd_.dropout <= 0.0) return;
  invalidate_linearization();  // the cached activations used the old masks
  if (!was_on) drop_graph();   // a captured step ran without masks
  if (!traj_) throw ValidationError("refresh_dropout: set the shape first");
  const long long slot = (long long)std::max(Tx_, Ty_) * sd_.d;
  const int nblk = total_ * 3;
  MGLP_CUDA(cudaSetDevice(device_));
  if (drop_slot_ != slot) {
    if (drop_masks_) cudaFree(drop_masks_);
    drop_masks_ = nullptr;
    MGLP_CUDA(cudaMalloc(&drop_masks_, (size_t)nblk * slot));
    drop_slot_ = slot;
  }
  // rng::derive(seed, kDropout, batch_index, layer*8 + site, i): the first
  // four splitmix rounds per (layer, site) here, the last (^ i) on the device
  std::vector<unsigned long long> keys((size_t)nblk);
  std::vector<int> rows((size_t)nblk);
  for (int l = 0; l < total_; ++l) {
    const bool dec = sd_.kind == 2 && l >= n_split_;
    for (int site = 0; site < 3; ++site) {
      uint64_t k = splitmix64(seed ^ 0x243f6a8885a308d3ULL);
      k = splitmix64(k ^ (uint64_t)kRngDropout);
      k = splitmix64(k ^ batch_index);
      k = splitmix64(k ^ ((uint64_t)l * 8 + (uint64_t)site));
      keys[(size_t)l * 3 + site] = k;
      // phi1, phi2 on every layer; phi3 (cross-attention) on decoder layers
      rows[(size_t)l * 3 + site] = (site < 2 || dec) ? (dec ? Ty_ : Tx_) : 0;
    }
  }
  unsigned long long* dkeys = nullptr;
  int* drows = nullptr;
  MGLP_CUDA(cudaMalloc(&dkeys, keys.size() * sizeof(unsigned long long)));
  MGLP_CUDA(cudaMalloc(&drows, rows.size() * sizeof(int)));
  MGLP_CUDA(cudaMemcpyAsync(dkeys, keys.data(), keys.size() * sizeof(unsigned long long),
                            cudaMemcpyHostToDevice, stream_));
  MGLP_CUDA(cudaMemcpyAsync(drows, rows.data(), rows.size() * sizeof(int), cudaMemcpyHostToDevice,
                            stream_));
  const double keep = 1.0 - sd_.dropout;
  const int gx = (int)std::min<long long>((slot + 255) / 256, 256);
  dropout_gen_kernel<<<dim3(gx, nblk), 256, 0, stream_>>>(drop_masks_, dkeys, drows, slot, sd_.d,
                                                          nblk, keep * 0x1.0p53);
  MGLP_CUDA(cudaGetLastError());
  MGLP_CUDA(cudaStreamSynchronize(stream_));
  cudaFree(dkeys);
  cudaFree(drows);
  drop_on_ = true;
}

void Engine::set_dropout_masks(const unsigned char* keep_host) {
  const bool was_on = drop_on_;
  drop_on_ = false;
  if (sd_.dropout <= 0.0) return;
  invalidate_linearization();
  if (!was_on) drop_graph();
  if (!traj_) throw ValidationError("set_dropout_masks: set the shape first");
  const long long slot = (long long)std::max(Tx_, Ty_) * sd_.d;
  MGLP_CUDA(cudaSetDevice(device_));
  if (drop_slot_ != slot) {
    if (drop_masks_) cudaFree(drop_masks_);
    drop_masks_ = nullptr;
    MGLP_CUDA(cudaMalloc(&drop_masks_, (size_t)total_ * 3 * slot));
    drop_slot_ = slot;
  }
  MGLP_CUDA(cudaMemcpyAsync(drop_masks_, keep_host, (size_t)total_ * 3 * slot,
                            cudaMemcpyHostToDevice, stream_));
  MGLP_CUDA(cudaStreamSynchronize(stream_));
  drop_on_ = true;
}

DropMask Engine::dmask(int site, int layer0, int layer_step) const {
  DropMask m;
  if (!drop_on_) return m;
  m.m = drop_masks_;
  m.slot = drop_slot_;
  m.layer0 = layer0;
  m.step = layer_step;
  m.site = site;
  m.cols = sd_.d;
  m.scale = (float)(1.0 / (1.0 - sd_.dropout));
  return m;
}

void Engine::residual_device(int layer, const float* z, int G, float* F) {
  if (layer < 0 || layer >= total_) throw ValidationError("residual: layer out of range");
  for (int g0 = 0; g0 < G; g0 += Gmax_) {
    EvalSpec e;
    e.G = std::min(Gmax_, G - g0);
    e.layer0 = layer;
    e.layer_step = 0;
    e.dt = 1.f;
    e.in = state_mat(const_cast<float*>(z) + (long long)g0 * state_n_, state_n_, sd_.d, 0, 1);
    e.act = ActRef{scratch_, al_.size, 0, 1};
    e.residual_only = true;
    e.cmb.mode = CM_PLAIN;
    e.cmb.out = state_mat(F + (long long)g0 * state_n_, state_n_, sd_.d, 0, 1);
    eval_forward(e);
  }
}

void Engine::step_device(int layer, double dt, const float* z, float* out) {
  if (layer < 0 || layer >= total_) throw ValidationError("step: layer out of range");
  EvalSpec e;
  e.G = 1;
  e.layer0 = layer;
  e.dt = (float)dt;
  e.in = state_mat(const_cast<float*>(z), state_n_, sd_.d, 0, 1);
  e.act = ActRef{scratch_, al_.size, 0, 1};
  e.cmb.mode = CM_PLAIN;
  e.cmb.out = state_mat(out, state_n_, sd_.d, 0, 1);
  eval_forward(e);
}

void Engine::adjoint_step_device(int layer, double dt, const float* z, const float* lam,
                                 float* out, bool want_grads, double gscale) {
  if (layer < 0 || layer >= total_) throw ValidationError("adjoint_step: layer out of range");
  EvalSpec f;
  f.G = 1;
  f.layer0 = layer;
  f.in = state_mat(const_cast<float*>(z), state_n_, sd_.d, 0, 1);
  f.act = ActRef{scratch_, al_.size, 0, 1};
  f.keep_act = true;
  f.cmb.mode = CM_NONE;
  eval_forward(f);
  EvalSpec e = f;
  e.dt = (float)dt;
  e.lam = state_mat(const_cast<float*>(lam), state_n_, sd_.d, 0, 1);
  e.cmb.mode = CM_PLAIN;
  e.cmb.out = state_mat(out, state_n_, sd_.d, 0, 1);
  e.want_grads = want_grads;
  e.gscale = (float)gscale;
  eval_adjoint(e);
}

}  // namespace mglp
