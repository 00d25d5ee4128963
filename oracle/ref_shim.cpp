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
//   ref_make_batch       make_batch (tasks.cpp:45-89)
//   ref_model_*          Model ctor / param_tensors (model.cpp:50-100)
//   ref_lipschitz_*      estimate_lipschitz / select_buffer_layers /
//                        recommend_buffers (lipschitz.cpp:53-239)
//   ref_run_training     run_training -> metrics CSV + final MGLP v1
//                        checkpoint (training.cpp:92-135, 315-352;
//                        checkpoint.cpp:88-112)
// State buffers are flat f64: x [B,s_x,d] followed by y [B,s_y,d] (y absent
// when s_y == 0), exactly the State{x,y} of blocks.hpp:70-73.
// Status: 0 ok, 1 ValidationError, 2 ContractViolation / other (errors.hpp:25-35).
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "mglp/lipschitz.hpp"
#include "mglp/adjoint.hpp"
#include "mglp/blocks.hpp"
#include "mglp/controller.hpp"
#include "mglp/executor.hpp"
#include "mglp/mgrit.hpp"
#include "mglp/rng.hpp"
#include "mglp/systems.hpp"
#include "mglp/checkpoint.hpp"
#include "mglp/model.hpp"
#include "mglp/optimizer.hpp"
#include "mglp/tasks.hpp"
#include "mglp/training.hpp"

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

// ---- training edge ----------------------------------------------

int ref_make_batch(int kind, int vocab, int seq, int train_size, int val_size,
                   unsigned long long seed, int split, long long start, int batch,
                   int* src, int* tgt_in, int* tgt_out) {
  return guard([&] {
    TaskSpec t;
    t.kind = static_cast<TaskKind>(kind);
    t.vocab = vocab;
    t.seq_len = seq;
    t.train_size = train_size;
    t.val_size = val_size;
    t.seed = seed;
    const TokenBatch b = make_batch(t, split, start, batch);
    std::memcpy(src, b.src.data(), b.src.size() * sizeof(int));
    std::memcpy(tgt_out, b.tgt_out.data(), b.tgt_out.size() * sizeof(int));
    if (tgt_in && !b.tgt_in.empty())
      std::memcpy(tgt_in, b.tgt_in.data(), b.tgt_in.size() * sizeof(int));
  });
}

struct RefRun {
  TaskSpec task;
  ModelConfig model;
  TrainConfig train;
};

// cfg arrays (all f64 so the ctypes side stays one signature):
//  task  [kind, vocab, seq, train_size, val_size, seed]
//  model [kind, d, heads, ffn, n_enc, n_dec, open, close, base_h, init_std,
//         depth_scaled, dropout, vocab, max_seq]
//  train [mode, opt_kind, lr, beta1, beta2, eps, wd, momentum, coarsen,
//         levels, fwd_iters, bwd_iters, fwd_tol, bwd_tol, cold_guess,
//         warm_start, probe_period, threshold, policy, cap, use_probe_grad,
//         batch, epochs, seed, manual_switch, val_every]
static RefRun make_run(const double* t, const double* m, const double* r) {
  RefRun o;
  o.task.kind = static_cast<TaskKind>((int)t[0]);
  o.task.vocab = (int)t[1];
  o.task.seq_len = (int)t[2];
  o.task.train_size = (int)t[3];
  o.task.val_size = (int)t[4];
  o.task.seed = (std::uint64_t)t[5];
  StackConfig& c = o.model.stack;
  c.kind = static_cast<ModelKind>((int)m[0]);
  c.d = (int)m[1];
  c.heads = (int)m[2];
  c.ffn = (int)m[3];
  c.n_enc = (int)m[4];
  c.n_dec = (int)m[5];
  c.buffer_open = (int)m[6];
  c.buffer_close = (int)m[7];
  c.base_h = m[8];
  c.init_std = m[9];
  c.depth_scaled_init = m[10] != 0.0;
  c.dropout = m[11];
  o.model.vocab = (int)m[12];
  o.model.max_seq = (int)m[13];
  TrainConfig& tc = o.train;
  tc.mode = static_cast<TrainMode>((int)r[0]);
  tc.opt.kind = static_cast<OptKind>((int)r[1]);
  tc.opt.lr = r[2];
  tc.opt.beta1 = r[3];
  tc.opt.beta2 = r[4];
  tc.opt.eps = r[5];
  tc.opt.weight_decay = r[6];
  tc.opt.momentum = r[7];
  tc.solve.coarsen = (int)r[8];
  tc.solve.levels = (int)r[9];
  tc.solve.fwd_iters = (int)r[10];
  tc.solve.bwd_iters = (int)r[11];
  tc.solve.fwd_tol = r[12];
  tc.solve.bwd_tol = r[13];
  tc.solve.cold_guess = static_cast<InitialGuess>((int)r[14]);
  tc.solve.warm_start = r[15] != 0.0;
  tc.indicator.probe_period = (int)r[16];
  tc.indicator.threshold = r[17];
  tc.indicator.policy = static_cast<IndicatorPolicy>((int)r[18]);
  tc.indicator.max_iter_cap = (int)r[19];
  tc.indicator.use_probe_gradient = r[20] != 0.0;
  tc.batch_size = (int)r[21];
  tc.epochs = (int)r[22];
  tc.seed = (std::uint64_t)r[23];
  tc.manual_switch_batch = (long long)r[24];
  tc.val_every = (int)r[25];
  return o;
}

// metrics CSV and the final checkpoint (and the handover one, if any); the
// size outputs are always written, the buffers only when large enough
int ref_run_training(const double* task, const double* model, const double* train,
                     const char* start_state, long long start_len, char* csv,
                     long long csv_cap, long long* csv_len, char* final_state,
                     long long state_cap, long long* state_len, char* switch_state,
                     long long* switch_len, long long* switch_batch) {
  return guard([&] {
    const RefRun r = make_run(task, model, train);
    const std::string start =
        start_state ? std::string(start_state, (std::size_t)start_len) : std::string();
    const TrainResult res = run_training(r.task, r.model, r.train, start);
    *csv_len = (long long)res.csv.size();
    if (csv && (long long)res.csv.size() <= csv_cap)
      std::memcpy(csv, res.csv.data(), res.csv.size());
    *state_len = (long long)res.final_state.size();
    if (final_state && (long long)res.final_state.size() <= state_cap)
      std::memcpy(final_state, res.final_state.data(), res.final_state.size());
    *switch_len = (long long)res.switch_state.size();
    *switch_batch = res.switch_batch;
    if (switch_state && (long long)res.switch_state.size() <= state_cap)
      std::memcpy(switch_state, res.switch_state.data(), res.switch_state.size());
  });
}

// config_echo (training.cpp:329-346)
int ref_config_echo(const double* task, const double* model, const double* train, char* out,
                    long long cap, long long* len) {
  return guard([&] {
    const RefRun r = make_run(task, model, train);
    const std::string e = config_echo(r.task, r.model, r.train);
    *len = (long long)e.size();
    if (out && (long long)e.size() <= cap) std::memcpy(out, e.data(), e.size());
  });
}

// Model(cfg, seed) parameters in param_tensors order (model.cpp:74-92) and
// their shapes (rank-prefixed dims, one tensor after another)
int ref_model_params(const double* model, unsigned long long seed, double* flat,
                     long long* n_flat, long long* shapes, long long* n_shapes) {
  return guard([&] {
    RefRun r = make_run(std::vector<double>(6, 1.0).data(), model,
                        std::vector<double>(26, 0.0).data());
    Model mdl(r.model, seed);
    long long n = 0, k = 0;
    for (Tensor* t : mdl.param_tensors()) {
      if (flat) std::memcpy(flat + n, t->data(), t->size() * sizeof(double));
      n += (long long)t->size();
      if (shapes) shapes[k] = (long long)t->rank();
      ++k;
      for (std::size_t a = 0; a < t->rank(); ++a) {
        if (shapes) shapes[k] = (long long)t->dim(a);
        ++k;
      }
    }
    *n_flat = n;
    *n_shapes = k;
  });
}

// ---- Lipschitz probe (lipschitz.cpp) -----------------------------------------

int ref_lipschitz_estimate(void* h, int layer, int samples, double delta_scale,
                           double input_scale, int seq_len, unsigned long long seed,
                           double* out) {
  return guard([&] {
    ProbeConfig cfg;
    cfg.samples = samples;
    cfg.delta_scale = delta_scale;
    cfg.input_scale = input_scale;
    cfg.seq_len = seq_len;
    *out = estimate_lipschitz(*static_cast<RefStack*>(h)->stack, layer, cfg, seed).estimate;
  });
}

int ref_lipschitz_select(const double* est, int n, int k_open, int k_close, int* buffered,
                         int* n_buffered, int* spike) {
  return guard([&] {
    std::vector<LipschitzEstimate> es(n);
    for (int i = 0; i < n; ++i) {
      es[i].layer = i;
      es[i].estimate = est[i];
    }
    const BufferPlan plan = select_buffer_layers(es, k_open, k_close);
    *n_buffered = (int)plan.buffered.size();
    for (size_t i = 0; i < plan.buffered.size(); ++i) buffered[i] = plan.buffered[i];
    *spike = plan.interior_spike ? 1 : 0;
  });
}

int ref_lipschitz_recommend(const double* amps, int n, double threshold, int* k_open,
                            int* k_close) {
  return guard([&] {
    const BufferRecommendation rec =
        recommend_buffers(std::vector<double>(amps, amps + n), threshold);
    *k_open = rec.k_open;
    *k_close = rec.k_close;
  });
}

}  // extern "C"
