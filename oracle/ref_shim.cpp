// TEST INFRASTRUCTURE ONLY -- never linked into the product library.
//
// A thin extern "C" veneer over the UNMODIFIED reference library (mglp,
// /root/reference/proj/src/{tensor,blocks,executor}.cpp, compiled in place by
// oracle/Makefile into oracle/_ref/libmglp_ref.so). The parity tests, the
// golden-fixture generator and bench.py's reference arm call the reference
// through it; nothing under paper_2601_09026_b200/ may.
//
// Every entry point mirrors one reference API:
//   ref_stack_*          LayerStack ctor / visit_params / step / adjoint_step
//                        (blocks.hpp:120-175, blocks.cpp:385-574, 627-655)
//   ref_serial_*         serial_forward / serial_adjoint (blocks.cpp:659-682)
//   ref_engine_*         LayerParallelEngine (adjoint.hpp:99-219)
//   ref_scalar_*         MgritSolver<ScalarLinearSystem> (mgrit.hpp, systems.hpp:30-71)
//   ref_decide           controller.hpp:71-84
// State buffers are flat f64: x [B,s_x,d] followed by y [B,s_y,d] (y absent
// when s_y == 0), exactly the State{x,y} of blocks.hpp:70-73.
// Status: 0 ok, 1 ValidationError, 2 ContractViolation / other (errors.hpp:25-35).
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "mglp/adjoint.hpp"
#include "mglp/blocks.hpp"
#include "mglp/controller.hpp"
#include "mglp/executor.hpp"
#include "mglp/mgrit.hpp"
#include "mglp/rng.hpp"
#include "mglp/systems.hpp"

using namespace mglp;

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const ValidationError& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

struct Shape {
  int b, sx, sy, d;
  std::size_t nx() const { return (std::size_t)b * sx * d; }
  std::size_t ny() const { return (std::size_t)b * sy * d; }
  std::size_t n() const { return nx() + ny(); }
};

State make_state(const Shape& s, const double* src) {
  State z;
  if (s.sx > 0) {
    z.x = Tensor({(std::size_t)s.b, (std::size_t)s.sx, (std::size_t)s.d});
    if (src) std::memcpy(z.x.data(), src, s.nx() * sizeof(double));
  }
  if (s.sy > 0) {
    z.y = Tensor({(std::size_t)s.b, (std::size_t)s.sy, (std::size_t)s.d});
    if (src) std::memcpy(z.y.data(), src + s.nx(), s.ny() * sizeof(double));
  }
  return z;
}

void put_state(const Shape& s, const State& z, double* dst) {
  if (s.sx > 0) {
    if (z.x.size() != s.nx()) throw ContractViolation("shim: x size mismatch");
    std::memcpy(dst, z.x.data(), s.nx() * sizeof(double));
  }
  if (s.sy > 0) {
    if (z.y.size() != s.ny()) throw ContractViolation("shim: y size mismatch");
    std::memcpy(dst + s.nx(), z.y.data(), s.ny() * sizeof(double));
  }
}

struct RefStack {
  std::unique_ptr<LayerStack> stack;
};

struct RefEngine {
  RefStack* st;
  std::unique_ptr<Executor> ex;
  std::unique_ptr<LayerParallelEngine> eng;
  LayerParallelEngine::WarmSnapshot snap;
};

Shape shape_of(RefStack* s, int b, int sx, int sy) {
  return Shape{b, sx, sy, s->stack->config().d};
}

std::size_t count_params(const std::vector<BlockParams>& p) {
  std::size_t n = 0;
  visit_params(p, [&](int, const std::string&, const Tensor& t) { n += t.size(); });
  return n;
}

void flatten(const std::vector<BlockParams>& p, double* out) {
  std::size_t o = 0;
  visit_params(p, [&](int, const std::string&, const Tensor& t) {
    std::memcpy(out + o, t.data(), t.size() * sizeof(double));
    o += t.size();
  });
}

void unflatten(std::vector<BlockParams>& p, const double* in) {
  std::size_t o = 0;
  visit_params(p, [&](int, const std::string&, Tensor& t) {
    std::memcpy(t.data(), in + o, t.size() * sizeof(double));
    o += t.size();
  });
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---- LayerStack -------------------------------------------------------------

int ref_stack_create(int kind, int d, int heads, int ffn, int n_enc, int n_dec,
                     int buffer_open, int buffer_close, double base_h,
                     double init_std, int depth_scaled, double dropout,
                     unsigned long long seed, void** out) {
  return guard([&] {
    StackConfig cfg;
    cfg.kind = static_cast<ModelKind>(kind);
    cfg.d = d;
    cfg.heads = heads;
    cfg.ffn = ffn;
    cfg.n_enc = n_enc;
    cfg.n_dec = n_dec;
    cfg.buffer_open = buffer_open;
    cfg.buffer_close = buffer_close;
    cfg.base_h = base_h;
    cfg.init_std = init_std;
    cfg.depth_scaled_init = depth_scaled != 0;
    cfg.dropout = dropout;
    auto* s = new RefStack;
    s->stack = std::make_unique<LayerStack>(cfg, seed);
    *out = s;
  });
}

void ref_stack_destroy(void* h) { delete static_cast<RefStack*>(h); }

long long ref_stack_num_params(void* h) {
  return (long long)count_params(static_cast<RefStack*>(h)->stack->params());
}

int ref_stack_get_params(void* h, double* out) {
  return guard([&] { flatten(static_cast<RefStack*>(h)->stack->params(), out); });
}

int ref_stack_set_params(void* h, const double* in) {
  return guard([&] { unflatten(static_cast<RefStack*>(h)->stack->params(), in); });
}

int ref_stack_info(void* h, int* total, int* ib, int* ie, int* n_split_hint) {
  auto* s = static_cast<RefStack*>(h);
  *total = s->stack->total_layers();
  *ib = s->stack->interior_begin();
  *ie = s->stack->interior_end();
  *n_split_hint = s->stack->encoder_layers();
  return 0;
}

double ref_stack_step_size(void* h, int layer) {
  return static_cast<RefStack*>(h)->stack->step_size(layer);
}

int ref_stack_refresh_dropout(void* h, unsigned long long seed,
                              unsigned long long batch_index, int b, int sx,
                              int sy) {
  return guard([&] {
    static_cast<RefStack*>(h)->stack->refresh_dropout(seed, batch_index, b, sx, sy);
  });
}

int ref_stack_step(void* h, int layer, double dt, int b, int sx, int sy,
                   const double* z, double* out) {
  return guard([&] {
    auto* s = static_cast<RefStack*>(h);
    Shape sh = shape_of(s, b, sx, sy);
    put_state(sh, s->stack->step(layer, dt, make_state(sh, z)), out);
  });
}

int ref_stack_residual(void* h, int layer, int b, int sx, int sy,
                       const double* z, double* out) {
  return guard([&] {
    auto* s = static_cast<RefStack*>(h);
    Shape sh = shape_of(s, b, sx, sy);
    put_state(sh, s->stack->residual(layer, make_state(sh, z)), out);
  });
}

// grads_inout (nullable): flat visit_params-ordered gradient bank, accumulated.
int ref_stack_adjoint_step(void* h, int layer, double dt, int b, int sx, int sy,
                           const double* z, const double* lam,
                           double* grads_inout, double gscale, double* out) {
  return guard([&] {
    auto* s = static_cast<RefStack*>(h);
    Shape sh = shape_of(s, b, sx, sy);
    std::vector<BlockParams> g;
    if (grads_inout) {
      g = s->stack->zero_grads();
      unflatten(g, grads_inout);
    }
    State r = s->stack->adjoint_step(layer, dt, make_state(sh, z),
                                     make_state(sh, lam),
                                     grads_inout ? &g : nullptr, gscale);
    put_state(sh, r, out);
    if (grads_inout) flatten(g, grads_inout);
  });
}

// ---- serial sweeps ------------------------------------------------------------

int ref_serial_forward(void* h, int b, int sx, int sy, const double* z0,
                       double* traj_out) {
  return guard([&] {
    auto* s = static_cast<RefStack*>(h);
    Shape sh = shape_of(s, b, sx, sy);
    std::vector<State> traj = serial_forward(*s->stack, make_state(sh, z0));
    for (std::size_t i = 0; i < traj.size(); ++i)
      put_state(sh, traj[i], traj_out + i * sh.n());
  });
}

int ref_serial_adjoint(void* h, int b, int sx, int sy, const double* traj_in,
                       const double* lam_n, double* lam_out,
                       double* grads_inout) {
  return guard([&] {
    auto* s = static_cast<RefStack*>(h);
    Shape sh = shape_of(s, b, sx, sy);
    const int total = s->stack->total_layers();
    std::vector<State> traj;
    for (int i = 0; i <= total; ++i)
      traj.push_back(make_state(sh, traj_in + (std::size_t)i * sh.n()));
    std::vector<BlockParams> g;
    if (grads_inout) {
      g = s->stack->zero_grads();
      unflatten(g, grads_inout);
    }
    std::vector<State> lam = serial_adjoint(*s->stack, traj, make_state(sh, lam_n),
                                            grads_inout ? &g : nullptr);
    for (std::size_t i = 0; i < lam.size(); ++i)
      put_state(sh, lam[i], lam_out + i * sh.n());
    if (grads_inout) flatten(g, grads_inout);
  });
}

// ---- LayerParallelEngine -----------------------------------------------------

int ref_engine_create(void* stack, int coarsen, int levels, int fwd_iters,
                      int bwd_iters, double fwd_tol, double bwd_tol,
                      int cold_guess, int warm_start, int workers, void** out) {
  return guard([&] {
    auto* e = new RefEngine;
    e->st = static_cast<RefStack*>(stack);
    e->ex = std::make_unique<Executor>(workers);
    SolveConfig cfg;
    cfg.coarsen = coarsen;
    cfg.levels = levels;
    cfg.fwd_iters = fwd_iters;
    cfg.bwd_iters = bwd_iters;
    cfg.fwd_tol = fwd_tol;
    cfg.bwd_tol = bwd_tol;
    cfg.cold_guess = static_cast<InitialGuess>(cold_guess);
    cfg.warm_start = warm_start != 0;
    try {
      e->eng = std::make_unique<LayerParallelEngine>(*e->st->stack, *e->ex, cfg);
    } catch (...) {
      delete e;
      throw;
    }
    *out = e;
  });
}

void ref_engine_destroy(void* h) { delete static_cast<RefEngine*>(h); }

int ref_engine_set_iters(void* h, int fwd_iters, int bwd_iters, double fwd_tol,
                         double bwd_tol) {
  auto* e = static_cast<RefEngine*>(h);
  e->eng->config().fwd_iters = fwd_iters;
  e->eng->config().bwd_iters = bwd_iters;
  e->eng->config().fwd_tol = fwd_tol;
  e->eng->config().bwd_tol = bwd_tol;
  return 0;
}

int ref_engine_forward(void* h, int b, int sx, int sy, const double* z0,
                       double* traj_out, double* trace_out, int max_trace,
                       int* n_trace, int* converged) {
  return guard([&] {
    auto* e = static_cast<RefEngine*>(h);
    Shape sh = shape_of(e->st, b, sx, sy);
    ForwardOutcome o = e->eng->forward(make_state(sh, z0));
    for (std::size_t i = 0; i < o.traj.size(); ++i)
      put_state(sh, o.traj[i], traj_out + i * sh.n());
    *n_trace = (int)o.phase.trace.size();
    for (int i = 0; i < *n_trace && i < max_trace; ++i) trace_out[i] = o.phase.trace[i];
    *converged = o.phase.converged ? 1 : 0;
  });
}

int ref_engine_backward(void* h, int b, int sx, int sy, const double* traj_in,
                        const double* lam_n, double* lam0_out,
                        double* grads_inout, double* trace_out, int max_trace,
                        int* n_trace, int* converged) {
  return guard([&] {
    auto* e = static_cast<RefEngine*>(h);
    Shape sh = shape_of(e->st, b, sx, sy);
    const int total = e->st->stack->total_layers();
    std::vector<State> traj;
    for (int i = 0; i <= total; ++i)
      traj.push_back(make_state(sh, traj_in + (std::size_t)i * sh.n()));
    std::vector<BlockParams> g;
    if (grads_inout) {
      g = e->st->stack->zero_grads();
      unflatten(g, grads_inout);
    }
    BackwardOutcome o = e->eng->backward(traj, make_state(sh, lam_n),
                                         grads_inout ? &g : nullptr);
    put_state(sh, o.lambda0, lam0_out);
    if (grads_inout) flatten(g, grads_inout);
    *n_trace = (int)o.phase.trace.size();
    for (int i = 0; i < *n_trace && i < max_trace; ++i) trace_out[i] = o.phase.trace[i];
    *converged = o.phase.converged ? 1 : 0;
  });
}

int ref_engine_snapshot(void* h) {
  auto* e = static_cast<RefEngine*>(h);
  e->snap = e->eng->snapshot();
  return 0;
}

int ref_engine_restore(void* h) {
  auto* e = static_cast<RefEngine*>(h);
  e->eng->restore(e->snap);
  return 0;
}

int ref_engine_reset(void* h) {
  static_cast<RefEngine*>(h)->eng->reset();
  return 0;
}

// ---- scalar MGRIT (the solver's known-answer system) --------------------------

// Runs `cycles` V-cycles (or solve_forward when tol >= 0 and cycles > 0) on
// ScalarLinearSystem(rates, h, cf) from a broadcast guess; writes the fine
// states and the trace.
int ref_scalar_solve(const double* rates, int n, double h, int cf, int levels,
                     double z0, int iters, double tol, int workers,
                     double* states_out, double* trace_out, int* n_trace,
                     int* converged) {
  return guard([&] {
    ScalarLinearSystem sys(std::vector<double>(rates, rates + n), h, cf);
    Executor ex(workers);
    MgritSolver<ScalarLinearSystem> solver(sys, n, cf, levels, ex);
    solver.set_initial_condition(z0);
    solver.apply_initial_guess(InitialGuess::kBroadcast);
    auto res = solver.solve_forward(iters, tol);
    for (int j = 0; j <= n; ++j) states_out[j] = solver.states(0)[j];
    *n_trace = (int)res.trace.size();
    for (int i = 0; i < *n_trace; ++i) trace_out[i] = res.trace[i];
    *converged = res.converged ? 1 : 0;
  });
}

// ---- controller ----------------------------------------------------------------

int ref_decide(double f_fwd, double f_bwd, double threshold, int policy,
               int cap, int fwd_iters, int bwd_iters, int* decision) {
  return guard([&] {
    IndicatorConfig c;
    c.threshold = threshold;
    c.policy = static_cast<IndicatorPolicy>(policy);
    c.max_iter_cap = cap;
    *decision = (int)decide(f_fwd, f_bwd, c, fwd_iters, bwd_iters);
  });
}

double ref_last_pair_factor(const double* trace, int n) {
  return last_pair_factor(std::vector<double>(trace, trace + n));
}

// ---- rng (for fixture generation) ----------------------------------------------

void ref_gaussian_fill(unsigned long long seed, unsigned long long a,
                       unsigned long long b, double scale, double* out,
                       long long n) {
  for (long long i = 0; i < n; ++i)
    out[i] = scale * rng::gaussian(seed, a, b, (std::uint64_t)i);
}

// testutil::random_tensor's draw (tests/test_util.hpp:89-95): gaussian(seed, a, i).
void ref_gaussian_fill_flat(unsigned long long seed, unsigned long long a,
                            double scale, double* out, long long n) {
  for (long long i = 0; i < n; ++i)
    out[i] = scale * rng::gaussian(seed, a, (std::uint64_t)i);
}

}  // extern "C"
