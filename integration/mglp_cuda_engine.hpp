// mglp_cuda_engine.hpp -- the reference-side drop-in: CudaLayerParallelEngine
// has LayerParallelEngine's constructor and member functions
// (proj/include/mglp/adjoint.hpp:99-219) and runs them through the C-ABI of
// include/mglp_cuda.h on a B200, so Trainer (proj/src/training.cpp:83-84,
// 123-124, 215, 229, 250-274) swaps engines with no other change.
//
// Header-only; include it with the reference's include/ and this repo's
// include/ on the path and link libmglp_cuda.so. integration/swap_engine.hpp
// shows the one-line swap (Trainer's std::optional<LayerParallelEngine>
// becomes std::optional<CudaLayerParallelEngine>), and
// tests/test_integration.py runs the UNMODIFIED reference training.cpp with it
// against the stock engine.
//
// Ownership and data flow follow the reference contract:
//   * parameters belong to the LayerStack (the Trainer's optimizer updates
//     them in place between steps): every forward() uploads the current
//     values in visit_params order (mglp_engine_set_params);
//   * the frozen dropout masks belong to the LayerStack too: forward()
//     uploads masks() (mglp_engine_set_dropout_masks) or clears them;
//   * config() is the live SolveConfig (ProbeScope / InexactnessMonitor
//     change its budgets in place): pushed before every solve;
//   * backward() ACCUMULATES into the caller's grads (+=, scaled by h), like
//     the reference; the trajectory of the last forward() stays on the device
//     and is reused when backward() gets that same trajectory;
//   * snapshot()/restore() keep the warm states on the device (one slot; a
//     restore of an overwritten snapshot throws ValidationError);
//   * ValidationError / ContractViolation map from status 1 / 2.
#ifndef MGLP_CUDA_ENGINE_HPP_
#define MGLP_CUDA_ENGINE_HPP_

#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "mglp/adjoint.hpp"
#include "mglp/blocks.hpp"
#include "mglp/errors.hpp"
#include "mglp/executor.hpp"
#include "mglp_cuda.h"

namespace mglp {

class CudaLayerParallelEngine {
 public:
  // LayerParallelEngine::WarmSnapshot (adjoint.hpp:187-206): the states stay
  // on the device; this is the handle of the engine's snapshot slot
  struct WarmSnapshot {
    long long id = 0;
  };

  CudaLayerParallelEngine(const LayerStack& stack, Executor& /*ex: not used on the device*/,
                          SolveConfig cfg, int device = 0)
      : stack_(stack), cfg_(cfg) {
    const StackConfig& s = stack.config();
    mglp_stack_desc d{};
    d.kind = static_cast<int>(s.kind);
    d.d = s.d;
    d.heads = s.heads;
    d.ffn = s.ffn;
    d.n_enc = s.n_enc;
    d.n_dec = s.n_dec;
    d.buffer_open = s.buffer_open;
    d.buffer_close = s.buffer_close;
    d.ln_eps = s.ln_eps;
    d.base_h = s.base_h;
    d.dropout = s.dropout;
    d.init_std = s.init_std;
    d.depth_scaled_init = s.depth_scaled_init ? 1 : 0;
    const mglp_solve_config c = desc();
    check(mglp_engine_create(&d, &c, device, &e_));
  }
  ~CudaLayerParallelEngine() {
    if (e_) mglp_engine_destroy(e_);
  }
  CudaLayerParallelEngine(const CudaLayerParallelEngine&) = delete;
  CudaLayerParallelEngine& operator=(const CudaLayerParallelEngine&) = delete;

  SolveConfig& config() { return cfg_; }
  const SolveConfig& config() const { return cfg_; }

  ForwardOutcome forward(const State& z0) {
    sync_params();
    shape_of(z0);
    sync_masks();
    push_config();
    const std::vector<double> in = flatten(z0);
    const int total = stack_.total_layers();
    std::vector<double> traj(static_cast<std::size_t>(total + 1) * in.size());
    double tr[256];
    int n = 0, conv = 0;
    check(mglp_engine_forward(e_, b_, sx_, sy_, in.data(), traj.data(), tr, 256, &n, &conv));
    ForwardOutcome out;
    out.traj.resize(total + 1);
    for (int t = 0; t <= total; ++t) out.traj[t] = unflatten(traj.data() + t * in.size(), z0);
    out.phase.trace.assign(tr, tr + std::min(n, 256));
    out.phase.converged = conv != 0;
    last_first_ = out.traj.front().x.data();
    last_last_ = out.traj.back().x.data();
    return out;
  }

  BackwardOutcome backward(const std::vector<State>& traj, const State& lambda_terminal,
                           std::vector<BlockParams>* grads) {
    push_config();
    const std::vector<double> lam = flatten(lambda_terminal);
    // the device still holds the trajectory of the last forward() unless the
    // caller hands in another one
    const bool same = !traj.empty() && traj.front().x.data() == last_first_ &&
                      traj.back().x.data() == last_last_;
    std::vector<double> tin;
    if (!same) {
      for (const State& s : traj) {
        const std::vector<double> f = flatten(s);
        tin.insert(tin.end(), f.begin(), f.end());
      }
    }
    std::vector<double> g;
    if (grads) g = flatten_params(*grads);
    std::vector<double> lam0(lam.size());
    double tr[256];
    int n = 0, conv = 0;
    check(mglp_engine_backward(e_, b_, sx_, sy_, same ? nullptr : tin.data(), lam.data(),
                               lam0.data(), grads ? g.data() : nullptr, tr, 256, &n, &conv));
    if (grads) unflatten_params(g, *grads);
    BackwardOutcome out;
    out.lambda0 = unflatten(lam0.data(), lambda_terminal);
    out.phase.trace.assign(tr, tr + std::min(n, 256));
    out.phase.converged = conv != 0;
    return out;
  }

  WarmSnapshot snapshot() const {
    WarmSnapshot s;
    check(mglp_engine_snapshot_id(e_, &s.id));
    return s;
  }
  void restore(const WarmSnapshot& s) { check(mglp_engine_restore_id(e_, s.id)); }
  void reset() { check(mglp_engine_reset(e_)); }

  mglp_engine* handle() const { return e_; }

 private:
  static void check(mglp_status st) {
    if (st == MGLP_OK) return;
    const std::string msg = mglp_last_error();
    if (st == MGLP_VALIDATION_ERROR) throw ValidationError(msg);
    throw ContractViolation(msg);
  }

  mglp_solve_config desc() const {
    mglp_solve_config c{};
    c.coarsen = cfg_.coarsen;
    c.levels = cfg_.levels;
    c.fwd_iters = cfg_.fwd_iters;
    c.bwd_iters = cfg_.bwd_iters;
    c.fwd_tol = cfg_.fwd_tol;
    c.bwd_tol = cfg_.bwd_tol;
    c.cold_guess = static_cast<int>(cfg_.cold_guess);
    c.warm_start = cfg_.warm_start ? 1 : 0;
    return c;
  }
  void push_config() {
    const mglp_solve_config c = desc();
    check(mglp_engine_set_config(e_, &c));
  }

  void sync_params() {
    std::vector<double> flat;
    visit_params(stack_.params(), [&](int, const std::string&, const Tensor& t) {
      flat.insert(flat.end(), t.data(), t.data() + t.size());
    });
    check(mglp_engine_set_params(e_, flat.data(), static_cast<long long>(flat.size())));
  }

  void shape_of(const State& z) {
    b_ = static_cast<int>(z.x.dim(0));
    sx_ = static_cast<int>(z.x.dim(1));
    sy_ = z.y.size() ? static_cast<int>(z.y.dim(1)) : 0;
  }

  // LayerStack::masks() (blocks.cpp:576-599) -> keep bytes per (layer, site)
  void sync_masks() {
    const std::vector<BlockMasks>& m = stack_.masks();
    if (stack_.config().dropout <= 0.0) return;
    if (m.empty()) {
      check(mglp_engine_clear_dropout(e_));
      return;
    }
    const int total = stack_.total_layers();
    const long long slot =
        static_cast<long long>(b_) * std::max(sx_, sy_) * stack_.config().d;
    std::vector<unsigned char> keep(static_cast<std::size_t>(total) * 3 * slot, 0);
    for (int l = 0; l < total; ++l) {
      const Tensor* site[3] = {&m[l].phi1, &m[l].phi2, &m[l].phi3};
      for (int s = 0; s < 3; ++s) {
        unsigned char* dst = keep.data() + (static_cast<std::size_t>(l) * 3 + s) * slot;
        for (std::size_t i = 0; i < site[s]->size(); ++i)
          dst[i] = site[s]->data()[i] != 0.0 ? 1 : 0;
      }
    }
    check(mglp_engine_set_dropout_masks(e_, b_, sx_, sy_, keep.data()));
  }

  static std::vector<double> flatten(const State& s) {
    std::vector<double> v(s.x.data(), s.x.data() + s.x.size());
    v.insert(v.end(), s.y.data(), s.y.data() + s.y.size());
    return v;
  }
  static State unflatten(const double* p, const State& like) {
    State s = like;  // same shapes (an unused stream stays empty: size 0)
    std::memcpy(s.x.data(), p, s.x.size() * sizeof(double));
    if (s.y.size()) std::memcpy(s.y.data(), p + s.x.size(), s.y.size() * sizeof(double));
    return s;
  }
  static std::vector<double> flatten_params(const std::vector<BlockParams>& g) {
    std::vector<double> flat;
    visit_params(g, [&](int, const std::string&, const Tensor& t) {
      flat.insert(flat.end(), t.data(), t.data() + t.size());
    });
    return flat;
  }
  static void unflatten_params(const std::vector<double>& flat, std::vector<BlockParams>& g) {
    std::size_t o = 0;
    visit_params(g, [&](int, const std::string&, Tensor& t) {
      std::memcpy(t.data(), flat.data() + o, t.size() * sizeof(double));
      o += t.size();
    });
  }

  const LayerStack& stack_;
  SolveConfig cfg_;
  mglp_engine* e_ = nullptr;
  int b_ = 0, sx_ = 0, sy_ = 0;
  const double* last_first_ = nullptr;  // tensor buffers of the last forward's trajectory
  const double* last_last_ = nullptr;
};

}  // namespace mglp

#endif  // MGLP_CUDA_ENGINE_HPP_
