// extern "C" boundary (include/mglp_cuda.h) over the C++ engine. Exceptions
// never cross it: ValidationError -> 1, everything else -> 2 (errors.hpp:25-35).
#include <algorithm>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/mglp_cuda.h"
#include "engine.h"
#include "trainer.h"
#include "transport.h"

#include <thread>

using namespace mglp;

struct mglp_engine {
  std::unique_ptr<Engine> eng;
  // host staging for the f64 <-> fp32 boundary
  float* dz = nullptr;
  float* dl = nullptr;
  float* dl0 = nullptr;
  long long cap = 0;
  // pinned host staging of one state (fp32): the f64 <-> fp32 conversion runs
  // multithreaded into it and the copies are DMA from pinned memory
  float* pin = nullptr;
  long long pin_cap = 0;
  int B = 0, sx = 0, sy = 0;
};

namespace {

thread_local std::string g_err;

template <class F>
mglp_status guard(F&& f) {
  try {
    f();
    return MGLP_OK;
  } catch (const ValidationError& e) {
    g_err = e.what();
    return MGLP_VALIDATION_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MGLP_CONTRACT_VIOLATION;
  } catch (...) {
    g_err = "unknown error";
    return MGLP_CONTRACT_VIOLATION;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw ValidationError(std::string(what) + " must not be null");
}

struct Shape {
  long long n_logical;  // B*(sx+sy)*d
  long long n_dev;      // padded device state size
};

Shape ensure_shape(mglp_engine* e, int batch, int s_x, int s_y, int d) {
  e->eng->set_shape(batch, s_x, s_y);
  const long long nd = e->eng->state_elems();
  if (nd > e->cap) {
    for (float* p : {e->dz, e->dl, e->dl0})
      if (p) cudaFree(p);
    MGLP_CUDA(cudaMalloc(&e->dz, nd * sizeof(float)));
    MGLP_CUDA(cudaMalloc(&e->dl, nd * sizeof(float)));
    MGLP_CUDA(cudaMalloc(&e->dl0, nd * sizeof(float)));
    e->cap = nd;
  }
  e->B = batch;
  e->sx = s_x;
  e->sy = s_y;
  return Shape{(long long)batch * (s_x + s_y) * d, nd};
}

// f(i) for i in [0, n) on up to 8 host threads (chunks of >= 256K elements)
template <class F>
void host_parallel(long long n, F&& f) {
  const long long chunk = 1LL << 18;
  const int nt = (int)std::min<long long>(8, std::max<long long>(1, n / chunk));
  if (nt <= 1) {
    for (long long i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> th;
  for (int t = 0; t < nt; ++t)
    th.emplace_back([&, t] {
      const long long a = n * t / nt, b = n * (t + 1) / nt;
      for (long long i = a; i < b; ++i) f(i);
    });
  for (auto& x : th) x.join();
}

float* pinned(mglp_engine* e, long long n) {
  if (n > e->pin_cap) {
    if (e->pin) cudaFreeHost(e->pin);
    e->pin = nullptr;
    MGLP_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&e->pin), n * sizeof(float),
                            cudaHostAllocDefault));
    e->pin_cap = n;
  }
  return e->pin;
}

void upload(mglp_engine* e, float* dst, const double* src, const Shape& sh) {
  float* h = pinned(e, sh.n_dev);
  host_parallel(sh.n_dev, [&](long long i) { h[i] = i < sh.n_logical ? (float)src[i] : 0.f; });
  MGLP_CUDA(cudaMemcpyAsync(dst, h, sh.n_dev * sizeof(float), cudaMemcpyHostToDevice,
                            e->eng->stream()));
  MGLP_CUDA(cudaStreamSynchronize(e->eng->stream()));
}

// one state (device fp32) -> host f64 through the pinned staging buffer
void download_state(mglp_engine* e, double* dst, const float* src, const Shape& sh) {
  float* h = pinned(e, sh.n_dev);
  MGLP_CUDA(cudaMemcpyAsync(h, src, sh.n_dev * sizeof(float), cudaMemcpyDeviceToHost,
                            e->eng->stream()));
  MGLP_CUDA(cudaStreamSynchronize(e->eng->stream()));
  host_parallel(sh.n_logical, [&](long long i) { dst[i] = h[i]; });
}

void download(mglp_engine* e, double* dst, const float* src, const Shape& sh, long long count) {
  std::vector<float> h(sh.n_dev * count);
  MGLP_CUDA(cudaMemcpyAsync(h.data(), src, h.size() * sizeof(float), cudaMemcpyDeviceToHost,
                            e->eng->stream()));
  MGLP_CUDA(cudaStreamSynchronize(e->eng->stream()));
  for (long long s = 0; s < count; ++s)
    for (long long i = 0; i < sh.n_logical; ++i) dst[s * sh.n_logical + i] = h[s * sh.n_dev + i];
}

void upload_traj(mglp_engine* e, const double* traj, const Shape& sh) {
  const long long T = e->eng->total_layers() + 1;
  // traj_ also holds the forward solver's warm window: keep it apart
  e->eng->displace_forward_window();
  std::vector<float> h(sh.n_dev * T, 0.f);
  for (long long s = 0; s < T; ++s)
    for (long long i = 0; i < sh.n_logical; ++i) h[s * sh.n_dev + i] = (float)traj[s * sh.n_logical + i];
  MGLP_CUDA(cudaMemcpyAsync(e->eng->traj_dev(), h.data(), h.size() * sizeof(float),
                            cudaMemcpyHostToDevice, e->eng->stream()));
  MGLP_CUDA(cudaStreamSynchronize(e->eng->stream()));
}

void put_trace(mglp_engine* e, bool fwd, double* out, int max_trace, int* n, int* conv) {
  std::vector<double> t;
  bool c = false;
  e->eng->read_trace(fwd, &t, &c);
  if (out)
    for (int i = 0; i < (int)t.size() && i < max_trace; ++i) out[i] = t[i];
  if (n) *n = (int)t.size();
  if (conv) *conv = c ? 1 : 0;
}


}  // namespace

namespace {

StackDesc to_stack(const mglp_stack_desc* stack) {
    StackDesc sd;
    sd.kind = stack->kind;
    sd.d = stack->d;
    sd.heads = stack->heads;
    sd.ffn = stack->ffn;
    sd.n_enc = stack->n_enc;
    sd.n_dec = stack->n_dec;
    sd.buffer_open = stack->buffer_open;
    sd.buffer_close = stack->buffer_close;
    sd.ln_eps = stack->ln_eps;
    sd.base_h = stack->base_h;
    sd.dropout = stack->dropout;
    sd.init_std = stack->init_std;
    sd.depth_scaled_init = stack->depth_scaled_init;
    return sd;
}

SolveCfg to_solve(const mglp_solve_config* solve) {
    SolveCfg c;
    c.coarsen = solve->coarsen;
    c.levels = solve->levels;
    c.fwd_iters = solve->fwd_iters;
    c.bwd_iters = solve->bwd_iters;
    c.fwd_tol = solve->fwd_tol;
    c.bwd_tol = solve->bwd_tol;
    c.cold_guess = solve->cold_guess;
    c.warm_start = solve->warm_start;
    return c;
}

void check_device(int device) {
  int ndev = 0;
  MGLP_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) throw ValidationError("device index out of range");
}

mglp_engine* wrap(std::unique_ptr<Engine> eng) {
  auto* h = new mglp_engine;
  h->eng = std::move(eng);
  return h;
}

}  // namespace

extern "C" {

const char* mglp_last_error(void) { return g_err.c_str(); }

const char* mglp_version(void) {
  return "mglp-b200 sm_100a tcgen05 kind::f16 3-pass hi/lo split (fp32 accumulate)";
}

mglp_status mglp_engine_create(const mglp_stack_desc* stack, const mglp_solve_config* solve,
                               int device, mglp_engine** out) {
  return guard([&] {
    need(stack, "stack");
    need(solve, "solve");
    need(out, "out");
    check_device(device);
    *out = wrap(std::make_unique<Engine>(to_stack(stack), to_solve(solve), device, nullptr));
  });
}

mglp_status mglp_nccl_unique_id(void* id128) {
  return guard([&] {
    need(id128, "id128");
    NcclUniqueId id;
    nccl_unique_id(&id);
    std::memcpy(id128, &id, sizeof id);
  });
}

mglp_status mglp_engine_create_dist(const mglp_stack_desc* stack, const mglp_solve_config* solve,
                                    int device, int rank, int world, const void* id128,
                                    mglp_engine** out) {
  return guard([&] {
    need(stack, "stack");
    need(solve, "solve");
    need(out, "out");
    if (world < 1 || rank < 0 || rank >= world) throw ValidationError("bad rank / world");
    check_device(device);
    std::shared_ptr<Transport> tr;
    if (world > 1) {
      need(id128, "id128");
      NcclUniqueId id;
      std::memcpy(&id, id128, sizeof id);
      tr = make_nccl_transport(rank, world, id, device);
    }
    *out = wrap(std::make_unique<Engine>(to_stack(stack), to_solve(solve), device, tr));
  });
}

mglp_status mglp_engine_rank_info(mglp_engine* e, int* rank, int* world, int* lo, int* hi) {
  return guard([&] {
    need(e, "engine");
    if (rank) *rank = e->eng->rank();
    if (world) *world = e->eng->world();
    int a = 0, b = 0;
    e->eng->owned_layers(&a, &b);
    if (lo) *lo = a;
    if (hi) *hi = b;
  });
}

mglp_status mglp_engine_set_dropout_masks(mglp_engine* e, int batch, int s_x, int s_y,
                                          const unsigned char* keep) {
  return guard([&] {
    need(e, "engine");
    need(keep, "keep");
    ensure_shape(e, batch, s_x, s_y, e->eng->width());
    e->eng->set_dropout_masks(keep);
  });
}

mglp_status mglp_engine_memory(mglp_engine* e, long long* bytes) {
  return guard([&] {
    need(e, "engine");
    need(bytes, "bytes");
    *bytes = (long long)e->eng->hbm_bytes();
  });
}

mglp_status mglp_engine_comm_info(mglp_engine* e, int* backend, int* nranks) {
  return guard([&] {
    need(e, "engine");
    Transport* t = e->eng->transport();
    if (backend) *backend = t ? t->backend() : 0;
    if (nranks) *nranks = t ? t->backend_nranks() : 1;
  });
}

mglp_status mglp_loopback_create(const mglp_stack_desc* stack, const mglp_solve_config* solve,
                                 int device, int world, mglp_engine** engines) {
  return guard([&] {
    need(stack, "stack");
    need(solve, "solve");
    need(engines, "engines");
    if (world < 1) throw ValidationError("world must be >= 1");
    check_device(device);
    auto hub = make_loopback_hub(world);
    std::vector<std::unique_ptr<Engine>> made;
    for (int r = 0; r < world; ++r)
      made.push_back(std::make_unique<Engine>(to_stack(stack), to_solve(solve), device,
                                              world > 1 ? make_loopback_transport(hub, r)
                                                        : nullptr));
    for (int r = 0; r < world; ++r) engines[r] = wrap(std::move(made[r]));
  });
}

mglp_status mglp_loopback_run_fwd_bwd(mglp_engine** engines, int world, const float* z0_dev,
                                      const float* lam_n_dev, float* lam0_dev, int want_grads) {
  return guard([&] {
    need(engines, "engines");
    need(z0_dev, "z0_dev");
    need(lam_n_dev, "lam_n_dev");
    std::vector<std::thread> th;
    std::vector<std::string> errs(world);
    for (int r = 0; r < world; ++r)
      th.emplace_back([&, r] {
        try {
          Engine& E = *engines[r]->eng;
          MGLP_CUDA(cudaSetDevice(E.device()));
          E.forward_device(z0_dev);
          E.backward_device(lam_n_dev, r == 0 ? lam0_dev : nullptr, want_grads != 0, true);
          MGLP_CUDA(cudaStreamSynchronize(E.stream()));
        } catch (const std::exception& ex) {
          errs[r] = ex.what();
        }
      });
    for (auto& t : th) t.join();
    for (int r = 0; r < world; ++r)
      if (!errs[r].empty()) throw ContractViolation("rank " + std::to_string(r) + ": " + errs[r]);
  });
}

mglp_status mglp_engine_destroy(mglp_engine* e) {
  return guard([&] {
    if (!e) return;
    cudaSetDevice(e->eng->device());
    for (float* p : {e->dz, e->dl, e->dl0})
      if (p) cudaFree(p);
    if (e->pin) cudaFreeHost(e->pin);
    delete e;
  });
}

mglp_status mglp_engine_info(mglp_engine* e, int* total, int* ib, int* ie, long long* np) {
  return guard([&] {
    need(e, "engine");
    if (total) *total = e->eng->total_layers();
    if (ib) *ib = e->eng->interior_begin();
    if (ie) *ie = e->eng->interior_end();
    if (np) *np = e->eng->num_params();
  });
}

mglp_status mglp_engine_step_size(mglp_engine* e, int layer, double* h) {
  return guard([&] {
    need(e, "engine");
    if (layer < 0 || layer >= e->eng->total_layers()) throw ValidationError("layer out of range");
    *h = e->eng->step_size(layer);
  });
}

mglp_status mglp_engine_refresh_dropout(mglp_engine* e, unsigned long long seed,
                                        unsigned long long batch_index, int batch, int s_x,
                                        int s_y) {
  return guard([&] {
    need(e, "engine");
    e->eng->set_shape(batch, s_x, s_y);
    e->eng->refresh_dropout(seed, batch_index);
  });
}

mglp_status mglp_engine_clear_dropout(mglp_engine* e) {
  return guard([&] {
    need(e, "engine");
    e->eng->clear_dropout();
  });
}

mglp_status mglp_engine_lipschitz(mglp_engine* e, int samples, double delta_scale,
                                  double input_scale, int seq_len, unsigned long long seed,
                                  const int* layers, int n_layers, double* estimates) {
  return guard([&] {
    need(e, "engine");
    need(estimates, "estimates");
    std::vector<int> ls;
    if (layers) {
      ls.assign(layers, layers + n_layers);
    } else {
      for (int l = 0; l < e->eng->total_layers(); ++l) ls.push_back(l);
    }
    std::vector<double> est;
    lipschitz_probe(*e->eng, samples, delta_scale, input_scale, seq_len, seed, ls, &est);
    std::copy(est.begin(), est.end(), estimates);
  });
}

mglp_status mglp_engine_init_params(mglp_engine* e, unsigned long long seed, double* flat_out) {
  return guard([&] {
    need(e, "engine");
    std::vector<double> flat;
    e->eng->init_params(seed, &flat);
    e->eng->set_params(flat.data());
    if (flat_out) std::memcpy(flat_out, flat.data(), flat.size() * sizeof(double));
  });
}

mglp_status mglp_engine_set_params(mglp_engine* e, const double* flat, long long n) {
  return guard([&] {
    need(e, "engine");
    need(flat, "flat");
    if (n != e->eng->num_params()) throw ValidationError("set_params: parameter count mismatch");
    e->eng->set_params(flat);
  });
}

mglp_status mglp_engine_get_params(mglp_engine* e, double* flat, long long n) {
  return guard([&] {
    need(e, "engine");
    need(flat, "flat");
    if (n != e->eng->num_params()) throw ValidationError("get_params: parameter count mismatch");
    e->eng->get_params(flat);
  });
}

mglp_status mglp_engine_get_config(mglp_engine* e, mglp_solve_config* cfg) {
  return guard([&] {
    need(e, "engine");
    need(cfg, "cfg");
    const SolveCfg& c = e->eng->config();
    cfg->coarsen = c.coarsen;
    cfg->levels = c.levels;
    cfg->fwd_iters = c.fwd_iters;
    cfg->bwd_iters = c.bwd_iters;
    cfg->fwd_tol = c.fwd_tol;
    cfg->bwd_tol = c.bwd_tol;
    cfg->cold_guess = c.cold_guess;
    cfg->warm_start = c.warm_start;
  });
}

mglp_status mglp_engine_set_config(mglp_engine* e, const mglp_solve_config* cfg) {
  return guard([&] {
    need(e, "engine");
    need(cfg, "cfg");
    SolveCfg& c = e->eng->config();
    if (cfg->coarsen != c.coarsen || cfg->levels != c.levels)
      throw ValidationError("set_config: the hierarchy (coarsen, levels) is fixed at creation");
    // the iteration budgets, tolerances and guess policy are baked into a
    // captured step: a change drops it (replay then refuses until recapture)
    // With a device monitor attached the budgets live on the device and gate
    // the captured cycles: a budget change alone keeps the graph.
    if (cfg->fwd_iters < 1 || cfg->bwd_iters < 1)
      throw ValidationError("set_config: iteration budgets must be >= 1");
    const bool iters = cfg->fwd_iters != c.fwd_iters || cfg->bwd_iters != c.bwd_iters;
    if ((iters && !e->eng->monitor_on()) || cfg->fwd_tol != c.fwd_tol ||
        cfg->bwd_tol != c.bwd_tol || cfg->cold_guess != c.cold_guess ||
        cfg->warm_start != c.warm_start)
      e->eng->drop_graph();
    if (iters) e->eng->set_budget(cfg->fwd_iters, cfg->bwd_iters);
    c.fwd_tol = cfg->fwd_tol;
    c.bwd_tol = cfg->bwd_tol;
    c.cold_guess = cfg->cold_guess;
    c.warm_start = cfg->warm_start;
  });
}

mglp_status mglp_engine_forward(mglp_engine* e, int batch, int s_x, int s_y, const double* z0,
                                double* traj_out, double* trace_out, int max_trace, int* n_trace,
                                int* converged) {
  return guard([&] {
    need(e, "engine");
    need(z0, "z0");
    const Shape sh = ensure_shape(e, batch, s_x, s_y, e->eng->width());
    if (traj_out && e->eng->world() > 1)
      throw ValidationError("forward: a rank of a multi-GPU engine holds only its own block of the "
                            "trajectory; pass traj_out = NULL and read it per rank");
    upload(e, e->dz, z0, sh);
    e->eng->forward_device(e->dz);
    if (traj_out) download(e, traj_out, e->eng->traj_dev(), sh, e->eng->total_layers() + 1);
    put_trace(e, true, trace_out, max_trace, n_trace, converged);
  });
}

mglp_status mglp_engine_backward(mglp_engine* e, int batch, int s_x, int s_y,
                                 const double* traj_in, const double* lam_n, double* lam0_out,
                                 double* grads_accum, double* trace_out, int max_trace,
                                 int* n_trace, int* converged) {
  return guard([&] {
    need(e, "engine");
    need(lam_n, "lam_n");
    if (!traj_in && (batch != e->B || s_x != e->sx || s_y != e->sy))
      throw ValidationError("backward: no device trajectory for this shape; pass traj_in");
    const Shape sh = ensure_shape(e, batch, s_x, s_y, e->eng->width());
    if (traj_in) upload_traj(e, traj_in, sh);
    upload(e, e->dl, lam_n, sh);
    if (grads_accum) e->eng->zero_grads();
    e->eng->backward_device(e->dl, e->dl0, grads_accum != nullptr, traj_in == nullptr);
    if (lam0_out) download_state(e, lam0_out, e->dl0, sh);
    if (grads_accum) e->eng->get_grads(grads_accum);
    put_trace(e, false, trace_out, max_trace, n_trace, converged);
  });
}

mglp_status mglp_engine_backward_keep_grads(mglp_engine* e, int batch, int s_x, int s_y,
                                            const double* traj_in, const double* lam_n,
                                            double* lam0_out, double* trace_out, int max_trace,
                                            int* n_trace, int* converged) {
  return guard([&] {
    need(e, "engine");
    need(lam_n, "lam_n");
    if (!traj_in && (batch != e->B || s_x != e->sx || s_y != e->sy))
      throw ValidationError("backward: no device trajectory for this shape; pass traj_in");
    const Shape sh = ensure_shape(e, batch, s_x, s_y, e->eng->width());
    if (traj_in) upload_traj(e, traj_in, sh);
    upload(e, e->dl, lam_n, sh);
    e->eng->zero_grads();
    e->eng->backward_device(e->dl, e->dl0, true, traj_in == nullptr);
    if (lam0_out) download_state(e, lam0_out, e->dl0, sh);
    put_trace(e, false, trace_out, max_trace, n_trace, converged);
  });
}

mglp_status mglp_engine_snapshot(mglp_engine* e) {
  return guard([&] {
    need(e, "engine");
    e->eng->snapshot();
  });
}

mglp_status mglp_engine_restore(mglp_engine* e) {
  return guard([&] {
    need(e, "engine");
    e->eng->restore();
  });
}

mglp_status mglp_engine_snapshot_id(mglp_engine* e, long long* id) {
  return guard([&] {
    need(e, "engine");
    need(id, "id");
    *id = e->eng->snapshot();
  });
}

mglp_status mglp_engine_restore_id(mglp_engine* e, long long id) {
  return guard([&] {
    need(e, "engine");
    if (id <= 0) throw ValidationError("restore: invalid snapshot id");
    e->eng->restore(id);
  });
}

mglp_status mglp_engine_seed_forward_from_traj(mglp_engine* e) {
  return guard([&] {
    need(e, "engine");
    e->eng->seed_forward_from_traj();
  });
}

mglp_status mglp_engine_reset(mglp_engine* e) {
  return guard([&] {
    need(e, "engine");
    e->eng->reset();
  });
}

mglp_status mglp_serial_forward(mglp_engine* e, int batch, int s_x, int s_y, const double* z0,
                                double* traj_out) {
  return guard([&] {
    need(e, "engine");
    need(z0, "z0");
    const Shape sh = ensure_shape(e, batch, s_x, s_y, e->eng->width());
    upload(e, e->dz, z0, sh);
    e->eng->serial_forward_device(e->dz);
    e->eng->check_range();
    if (traj_out) download(e, traj_out, e->eng->traj_dev(), sh, e->eng->total_layers() + 1);
  });
}

mglp_status mglp_serial_adjoint(mglp_engine* e, int batch, int s_x, int s_y,
                                const double* traj_in, const double* lam_n, double* lam_all_out,
                                double* grads_accum) {
  return guard([&] {
    need(e, "engine");
    need(lam_n, "lam_n");
    if (!traj_in && (batch != e->B || s_x != e->sx || s_y != e->sy))
      throw ValidationError("serial_adjoint: no device trajectory for this shape; pass traj_in");
    const Shape sh = ensure_shape(e, batch, s_x, s_y, e->eng->width());
    if (traj_in) {
      upload_traj(e, traj_in, sh);
      e->eng->invalidate_linearization();
    }
    upload(e, e->dl, lam_n, sh);
    if (grads_accum) e->eng->zero_grads();
    e->eng->serial_adjoint_device(e->dl, e->dl0, grads_accum != nullptr);
    e->eng->check_range();
    if (lam_all_out) {
      // lam_all_ holds the adjoint at 2^k lambda_N: undo the exact factor
      download(e, lam_all_out, e->eng->lam_all_dev(), sh, e->eng->total_layers() + 1);
      const double down = e->eng->lam_unscale();
      const long long n = sh.n_logical * (e->eng->total_layers() + 1);
      for (long long i = 0; i < n; ++i) lam_all_out[i] *= down;
    }
    if (grads_accum) e->eng->get_grads(grads_accum);
    MGLP_CUDA(cudaStreamSynchronize(e->eng->stream()));
  });
}

mglp_status mglp_stack_step(mglp_engine* e, int layer, double dt, int batch, int s_x, int s_y,
                            const double* z, double* out) {
  return guard([&] {
    need(e, "engine");
    need(z, "z");
    need(out, "out");
    const Shape sh = ensure_shape(e, batch, s_x, s_y, e->eng->width());
    upload(e, e->dz, z, sh);
    e->eng->step_device(layer, dt, e->dz, e->dl0);
    e->eng->check_range();
    download(e, out, e->dl0, sh, 1);
  });
}

mglp_status mglp_stack_adjoint_step(mglp_engine* e, int layer, double dt, int batch, int s_x,
                                    int s_y, const double* z, const double* lam,
                                    double* grads_accum, double gscale, double* out) {
  return guard([&] {
    need(e, "engine");
    need(z, "z");
    need(lam, "lam");
    need(out, "out");
    const Shape sh = ensure_shape(e, batch, s_x, s_y, e->eng->width());
    upload(e, e->dz, z, sh);
    upload(e, e->dl, lam, sh);
    if (grads_accum) e->eng->zero_grads();
    e->eng->adjoint_step_device(layer, dt, e->dz, e->dl, e->dl0, grads_accum != nullptr, gscale);
    e->eng->check_range();
    download(e, out, e->dl0, sh, 1);
    if (grads_accum) e->eng->get_grads(grads_accum);
  });
}

mglp_status mglp_engine_set_shape(mglp_engine* e, int batch, int s_x, int s_y,
                                  long long* state_elems) {
  return guard([&] {
    need(e, "engine");
    const Shape sh = ensure_shape(e, batch, s_x, s_y, e->eng->width());
    if (state_elems) *state_elems = sh.n_dev;
  });
}

mglp_status mglp_engine_stream(mglp_engine* e, void** s) {
  return guard([&] {
    need(e, "engine");
    need(s, "stream");
    *s = (void*)e->eng->stream();
  });
}

mglp_status mglp_engine_forward_device(mglp_engine* e, const float* z0_dev) {
  return guard([&] {
    need(e, "engine");
    need(z0_dev, "z0_dev");
    e->eng->forward_device(z0_dev);
  });
}

mglp_status mglp_engine_backward_device(mglp_engine* e, const float* lam_n_dev, float* lam0_dev,
                                        int want_grads) {
  return guard([&] {
    need(e, "engine");
    need(lam_n_dev, "lam_n_dev");
    e->eng->backward_device(lam_n_dev, lam0_dev, want_grads != 0, true);
  });
}

mglp_status mglp_serial_forward_device(mglp_engine* e, const float* z0_dev) {
  return guard([&] {
    need(e, "engine");
    need(z0_dev, "z0_dev");
    e->eng->serial_forward_device(z0_dev);
  });
}

mglp_status mglp_serial_adjoint_device(mglp_engine* e, const float* lam_n_dev, float* lam0_dev,
                                       int want_grads) {
  return guard([&] {
    need(e, "engine");
    need(lam_n_dev, "lam_n_dev");
    e->eng->serial_adjoint_device(lam_n_dev, lam0_dev, want_grads != 0);
  });
}

mglp_status mglp_engine_zero_grads(mglp_engine* e) {
  return guard([&] {
    need(e, "engine");
    e->eng->zero_grads();
  });
}

mglp_status mglp_engine_get_grads(mglp_engine* e, double* flat, long long n) {
  return guard([&] {
    need(e, "engine");
    need(flat, "flat");
    if (n != e->eng->num_params()) throw ValidationError("get_grads: parameter count mismatch");
    e->eng->get_grads(flat);
  });
}

mglp_status mglp_engine_get_grads_layers(mglp_engine* e, int layer_lo, int layer_hi,
                                        double* flat, long long n) {
  return guard([&] {
    need(e, "engine");
    need(flat, "flat");
    if (layer_lo < 0 || layer_hi > e->eng->total_layers() || layer_lo >= layer_hi)
      throw ValidationError("get_grads_layers: bad layer range");
    const long long want = e->eng->flat_offset(layer_hi) - e->eng->flat_offset(layer_lo);
    if (n != want) throw ValidationError("get_grads_layers: parameter count mismatch");
    e->eng->get_grads_range(layer_lo, layer_hi, flat);
  });
}

mglp_status mglp_engine_read_traj(mglp_engine* e, int first, int count, float* dst) {
  return guard([&] {
    need(e, "engine");
    need(dst, "dst");
    const int T = e->eng->total_layers() + 1;
    if (first < 0 || count < 0 || first + count > T)
      throw ValidationError("read_traj: time points out of range");
    if (!e->eng->holds_points(first, count))
      throw ValidationError("read_traj: a rank of a multi-GPU engine holds only its own block of "
                            "time points (mglp_engine_rank_info)");
    const size_t n = (size_t)e->eng->state_elems();
    MGLP_CUDA(cudaMemcpyAsync(dst, e->eng->traj_dev() + (size_t)first * n,
                              (size_t)count * n * sizeof(float), cudaMemcpyDefault,
                              e->eng->stream()));
    MGLP_CUDA(cudaStreamSynchronize(e->eng->stream()));
  });
}

mglp_status mglp_engine_trace(mglp_engine* e, int which, double* trace_out, int max_trace,
                              int* n_trace, int* converged) {
  return guard([&] {
    need(e, "engine");
    put_trace(e, which == 0, trace_out, max_trace, n_trace, converged);
  });
}

mglp_status mglp_engine_traj_device(mglp_engine* e, float** traj) {
  return guard([&] {
    need(e, "engine");
    need(traj, "traj");
    *traj = e->eng->traj_dev();
  });
}

mglp_status mglp_engine_sync(mglp_engine* e) {
  return guard([&] {
    need(e, "engine");
    MGLP_CUDA(cudaStreamSynchronize(e->eng->stream()));
    MGLP_CUDA(cudaGetLastError());
  });
}

mglp_status mglp_engine_take_launch_count(mglp_engine* e, long long* n) {
  return guard([&] {
    need(e, "engine");
    need(n, "n");
    *n = e->eng->launch_count();
    e->eng->reset_launch_count();
  });
}

mglp_status mglp_rng_gaussian_fill(unsigned long long seed, unsigned long long a,
                                   unsigned long long b, double scale, double* out, long long n) {
  return guard([&] {
    need(out, "out");
    rng_gaussian_fill(seed, a, b, scale, out, n);
  });
}

mglp_status mglp_engine_graph_capture(mglp_engine* e, const float* z0_dev, const float* lam_n_dev,
                                      float* lam0_dev, int want_grads) {
  return guard([&] {
    need(e, "engine");
    need(z0_dev, "z0_dev");
    need(lam_n_dev, "lam_n_dev");
    e->eng->capture_step(z0_dev, lam_n_dev, lam0_dev, want_grads != 0);
  });
}

mglp_status mglp_engine_graph_replay(mglp_engine* e) {
  return guard([&] {
    need(e, "engine");
    e->eng->replay_step();
  });
}

mglp_status mglp_engine_profile(mglp_engine* e, int enable) {
  return guard([&] {
    need(e, "engine");
    e->eng->set_profiling(enable != 0);
  });
}

mglp_status mglp_engine_profile_read(mglp_engine* e, double* ms, double* flops, double* bytes,
                                     long long* launches) {
  return guard([&] {
    need(e, "engine");
    need(ms, "ms");
    need(flops, "flops");
    need(bytes, "bytes");
    need(launches, "launches");
    e->eng->read_profile(ms, flops, bytes, launches);
  });
}

mglp_status mglp_engine_profile_dump(mglp_engine* e, double* rows, int max_rows, int* n) {
  return guard([&] {
    need(e, "engine");
    need(rows, "rows");
    *n = e->eng->dump_profile(rows, max_rows);
  });
}

mglp_status mglp_engine_monitor_attach(mglp_engine* e, double threshold, int policy_switch,
                                      int max_iter_cap) {
  return guard([&] {
    need(e, "engine");
    e->eng->monitor_attach(threshold, policy_switch, max_iter_cap);
  });
}

mglp_status mglp_engine_monitor_probe(mglp_engine* e, int begin) {
  return guard([&] {
    need(e, "engine");
    e->eng->monitor_probe(begin != 0);
  });
}

mglp_status mglp_monitor_record(mglp_engine* e, long long batch, int* decision) {
  return guard([&] {
    need(e, "engine");
    e->eng->monitor_record(batch);
    if (decision) *decision = e->eng->monitor_read().last_decision;
  });
}

mglp_status mglp_engine_monitor_read(mglp_engine* e, int* switched, int* decision,
                                    double* fwd_factor, double* bwd_factor, int* fwd_iters,
                                    int* bwd_iters, int* used_fwd, int* used_bwd) {
  return guard([&] {
    need(e, "engine");
    const MonitorSummary& m = e->eng->monitor_read();
    if (switched) *switched = m.switched;
    if (decision) *decision = m.last_decision;
    if (fwd_factor) *fwd_factor = m.last_ff;
    if (bwd_factor) *bwd_factor = m.last_bf;
    if (fwd_iters) *fwd_iters = m.budget[0];
    if (bwd_iters) *bwd_iters = m.budget[1];
    if (used_fwd) *used_fwd = m.used[0];
    if (used_bwd) *used_bwd = m.used[1];
  });
}

mglp_status mglp_engine_monitor_reports(mglp_engine* e, long long* batch, double* fwd_factor,
                                       double* bwd_factor, int* decision, int cap, int* n) {
  return guard([&] {
    need(e, "engine");
    const int k = e->eng->monitor_reports(batch, fwd_factor, bwd_factor, decision, cap);
    if (n) *n = k;
  });
}

mglp_status mglp_engine_capture_cycles(mglp_engine* e, int cycles) {
  return guard([&] {
    need(e, "engine");
    if (cycles < 0) throw ValidationError("capture cycles must be >= 0");
    e->eng->set_capture_cycles(cycles);
    e->eng->drop_graph();
  });
}

mglp_status mglp_test_gemm(int G, int M, int N, int K, const float* A, long long a_slot, int lda,
                           int a_mn, const float* B, long long b_slot, int ldb, int b_mn,
                           int b_presplit, const float* bias, float* Cp, long long c_slot, int ldc,
                           int engine, int* range_flag) {
  return guard([&] {
    need(A, "A");
    need(B, "B");
    need(Cp, "C");
    GemmArgs g;
    g.G = G;
    g.M = M;
    g.N = N;
    g.K = K;
    g.A.ptr = const_cast<float*>(A);
    g.A.slot_stride = a_slot;
    g.A.ld = lda;
    g.a_mn = a_mn != 0;
    g.B.ptr = const_cast<float*>(B);
    g.B.slot_stride = b_slot;
    g.B.ld = ldb;
    g.b_mn = b_mn != 0;
    g.ep.kind = EPI_STORE;
    g.ep.out1.ptr = Cp;
    g.ep.out1.slot_stride = c_slot;
    g.ep.out1.ld = ldc;
    if (bias) {
      g.ep.bias.ptr = const_cast<float*>(bias);
      g.ep.bias.slot_stride = 0;
    }
    float* hl = nullptr;
    int* dflag = nullptr;
    MGLP_CUDA(cudaMalloc(&dflag, sizeof(int)));
    MGLP_CUDA(cudaMemset(dflag, 0, sizeof(int)));
    g.range_flag = dflag;
    float* ahl = nullptr;
    float* bmn = nullptr;
    float* amn = nullptr;
    if (b_presplit == 8 && engine == 0 && a_mn) {
      // A MN-major ([K][M] rows) handed over pre-split (GemmArgs::a_mn_hl)
      if (M % 32) throw ValidationError("test_gemm: pre-split MN-major A needs M % 32 == 0");
      MGLP_CUDA(cudaMalloc(&amn, (size_t)G * K * M * sizeof(float)));
      launch_pack_hl(A, a_slot, lda, amn, (long long)K * M, M, G, K, M, false, 0);
      g.A.ptr = amn;
      g.A.slot_stride = (long long)K * M;
      g.A.ld = M;
      g.a_mn_hl = true;
    }
    if (b_presplit == 4 && engine == 0 && b_mn) {
      // B MN-major ([K][N] rows) handed over pre-split row by row: the
      // converters regroup instead of splitting (GemmArgs::b_mn_hl)
      if (N % 32) throw ValidationError("test_gemm: pre-split MN-major B needs N % 32 == 0");
      MGLP_CUDA(cudaMalloc(&bmn, (size_t)G * K * N * sizeof(float)));
      launch_pack_hl(B, b_slot, ldb, bmn, (long long)K * N, N, G, K, N, false, 0);
      g.B.ptr = bmn;
      g.B.slot_stride = (long long)K * N;
      g.B.ld = N;
      g.b_mn_hl = true;
    } else if (b_presplit && b_presplit != 8 && engine == 0) {
      const long long kp = pack_hl_cols(K);
      MGLP_CUDA(cudaMalloc(&hl, (size_t)G * N * kp * sizeof(float)));
      launch_pack_hl(B, b_slot, ldb, hl, (long long)N * kp, (int)kp, G, N, K, b_mn != 0, 0);
      g.Bhl.ptr = hl;
      g.Bhl.slot_stride = (long long)N * kp;
      g.Bhl.ld = (int)kp;
      if ((b_presplit & 2) && !a_mn) {  // A pre-split too: the converter-free mainloop
        MGLP_CUDA(cudaMalloc(&ahl, (size_t)G * M * kp * sizeof(float)));
        launch_pack_hl(A, a_slot, lda, ahl, (long long)M * kp, (int)kp, G, M, K, false, 0);
        g.Ahl.ptr = ahl;
        g.Ahl.slot_stride = (long long)M * kp;
        g.Ahl.ld = (int)kp;
      }
    }
    if (engine == 0)
      launch_gemm_tc(g, nullptr, 0);
    else
      launch_gemm_simt(g, nullptr, 0);
    MGLP_CUDA(cudaGetLastError());
    MGLP_CUDA(cudaDeviceSynchronize());
    if (hl) cudaFree(hl);
    if (ahl) cudaFree(ahl);
    if (bmn) cudaFree(bmn);
    if (amn) cudaFree(amn);
    int flag = 0;
    MGLP_CUDA(cudaMemcpy(&flag, dflag, sizeof(int), cudaMemcpyDeviceToHost));
    cudaFree(dflag);
    if (range_flag) *range_flag = flag;
  });
}

// ---- test / bench hook: the fused tcgen05 attention (attn_tc.cu) ----
namespace {
AttnArgs attn_args(int B, int H, int sq, int skv, int dh, int causal, const float* Q, const float* K,
                   const float* V, int ld, float* O, float* P, const float* dO, float* dQ, float* dK,
                   float* dV) {
  auto heads = [&](const float* p, int s, int ldm) {
    Mat m;
    m.ptr = const_cast<float*>(p);
    m.ld = ldm;
    m.bstride = (long long)s * ldm;
    m.hstride = dh;
    return m;
  };
  AttnArgs a;
  a.G = 1;
  a.Bb = B;
  a.H = H;
  a.sq = sq;
  a.skv = skv;
  a.dh = dh;
  a.causal = causal;
  a.scale = (float)(1.0 / std::sqrt((double)dh));
  a.Q = heads(Q, sq, ld);
  a.K = heads(K, skv, ld);
  a.V = heads(V, skv, ld);
  a.O = heads(O, sq, ld);
  const int ldp = (skv + 3) & ~3;
  a.P.ptr = P;
  a.P.ld = ldp;
  a.P.hstride = (long long)sq * ldp;
  a.P.bstride = (long long)H * sq * ldp;
  if (dO) {
    a.dO = heads(dO, sq, ld);
    a.dQ = heads(dQ, sq, ld);
    a.dK = heads(dK, skv, ld);
    a.dV = heads(dV, skv, ld);
  }
  return a;
}
}  // namespace

mglp_status mglp_test_attention(int B, int H, int sq, int skv, int dh, int causal, const float* Q,
                                const float* K, const float* V, int ld, float* O, float* P,
                                const float* dO, float* dQ, float* dK, float* dV,
                                int* range_flag) {
  return guard([&] {
    need(Q, "Q");
    need(K, "K");
    need(V, "V");
    need(O, "O");
    need(P, "P");
    const int p_hl = (causal >> 1) & 1;  // bit 1: P kept pre-split (s = 128)
    const int hs = (causal >> 2) & 1;    // bit 2: Q, K, V, dO head-split pre-split
    const int flash = (causal >> 3) & 1;  // bit 3 (long, with bit 2): single-pass backward
    causal &= 1;
    AttnArgs a = attn_args(B, H, sq, skv, dh, causal, Q, K, V, ld, O, P, dO, dQ, dK, dV);
    a.p_hl = p_hl;
    a.qkv_hs = hs;
    // the long backward's row dot reads fp32 dO; the single-pass one pre-split dO
    a.do_hs = hs && ((sq <= 128 && skv <= 128) || flash);
    float* dsbuf = nullptr;
    if (hs && flash && dO) {  // the dS tile-pair store of the single-pass backward
      const long long per_head = (long long)((sq + 63) / 64) * ((skv + 127) / 128) * 8192;
      MGLP_CUDA(cudaMalloc(&dsbuf, (size_t)B * H * per_head * sizeof(float)));
      a.dS.ptr = dsbuf;
      a.dS.hstride = per_head;
      a.dS.bstride = (long long)H * per_head;
    }
    const bool bwd = dO != nullptr;
    const bool shortp = attn_tc_supported(a, bwd);
    if (!shortp && !attn_long_supported(a, bwd))
      throw ValidationError(
          "fused attention: unsupported shape (sq, skv <= 128 and multiples of 8, or 128..512; dh 32 "
          "or 64)");
    int* dflag = nullptr;
    MGLP_CUDA(cudaMalloc(&dflag, sizeof(int)));
    MGLP_CUDA(cudaMemset(dflag, 0, sizeof(int)));
    a.range_flag = dflag;
    if (shortp) {
      launch_attn_fwd(a, nullptr, 0);
      if (bwd) launch_attn_bwd(a, nullptr, 0);
    } else {
      // long form: P receives the per-row (max, 1/sum) statistics instead
      launch_attn_fwd_long(a, nullptr, 0);
      if (bwd) launch_attn_bwd_long(a, nullptr, 0);
    }
    MGLP_CUDA(cudaDeviceSynchronize());
    if (dsbuf) cudaFree(dsbuf);
    int flag = 0;
    MGLP_CUDA(cudaMemcpy(&flag, dflag, sizeof(int), cudaMemcpyDeviceToHost));
    cudaFree(dflag);
    if (range_flag) *range_flag = flag;
  });
}

mglp_status mglp_bench_attention(int G, int B, int H, int s, int dh, int causal, int backward,
                                 int reps, float* ms_per_launch) {
  return guard([&] {
    const int d = H * dh, ld = 3 * d;
    const long long ntok = (long long)G * B * s;
    float *qkv = nullptr, *O = nullptr, *P = nullptr, *dO = nullptr, *dqkv = nullptr;
    const int ldp = (s + 3) & ~3;
    const long long np = (long long)G * B * H * s * ldp;
    MGLP_CUDA(cudaMalloc(&qkv, ntok * ld * sizeof(float)));
    MGLP_CUDA(cudaMalloc(&dqkv, ntok * ld * sizeof(float)));
    MGLP_CUDA(cudaMalloc(&O, ntok * d * sizeof(float)));
    MGLP_CUDA(cudaMalloc(&dO, ntok * d * sizeof(float)));
    MGLP_CUDA(cudaMalloc(&P, np * sizeof(float)));
    MGLP_CUDA(cudaMemset(qkv, 0x3c, ntok * ld * sizeof(float)));
    MGLP_CUDA(cudaMemset(dO, 0x3c, ntok * d * sizeof(float)));
    AttnArgs a = attn_args(B, H, s, s, dh, causal, qkv, qkv + d, qkv + 2 * d, ld, O, P,
                           backward ? dO : nullptr, dqkv, dqkv + d, dqkv + 2 * d);
    a.G = G;
    a.O.ld = d;
    a.O.bstride = (long long)s * d;
    a.dO.ld = d;
    a.dO.bstride = (long long)s * d;
    for (Mat* m : {&a.Q, &a.K, &a.V, &a.dQ, &a.dK, &a.dV}) m->slot_stride = (long long)B * s * ld;
    for (Mat* m : {&a.O, &a.dO}) m->slot_stride = (long long)B * s * d;
    a.P.slot_stride = (long long)B * H * s * ldp;
    // backward: 0 forward (P / row statistics stored), 1 backward,
    // 2 forward without P (s <= 128), 3 as 2 with O written pre-split only;
    // + 4: Q, K, V, dO head-split pre-split (dh = 64)
    const int mode = backward & 3;
    a.qkv_hs = (backward >> 2) & 1;
    const bool flash = ((backward >> 3) & 1) && a.qkv_hs && s > 128;
    a.do_hs = a.qkv_hs && (s <= 128 || flash);
    float* dsbuf = nullptr;
    if (flash) {
      const long long per_head = (long long)((s + 63) / 64) * ((s + 127) / 128) * 8192;
      MGLP_CUDA(cudaMalloc(&dsbuf, (size_t)G * B * H * per_head * sizeof(float)));
      a.dS.ptr = dsbuf;
      a.dS.hstride = per_head;
      a.dS.bstride = (long long)H * per_head;
      a.dS.slot_stride = (long long)B * H * per_head;
    }
    backward = mode == 1;
    const bool shortp = attn_tc_supported(a, backward != 0);
    if (!shortp && !attn_long_supported(a, backward != 0))
      throw ValidationError("bench_attention: unsupported shape");
    if (mode >= 2 && shortp) a.P = Mat{};
    if (mode == 3) {
      a.Ohl = a.O;
      a.O = Mat{};
    }
    cudaEvent_t e0, e1;
    MGLP_CUDA(cudaEventCreate(&e0));
    MGLP_CUDA(cudaEventCreate(&e1));
    auto run = [&] {
      if (shortp) {
        if (backward)
          launch_attn_bwd(a, nullptr, 0);
        else
          launch_attn_fwd(a, nullptr, 0);
      } else {
        if (backward)
          launch_attn_bwd_long(a, nullptr, 0);
        else
          launch_attn_fwd_long(a, nullptr, 0);
      }
    };
    run();
    run();
    MGLP_CUDA(cudaEventRecord(e0, 0));
    for (int i = 0; i < reps; ++i) run();
    MGLP_CUDA(cudaEventRecord(e1, 0));
    MGLP_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    MGLP_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *ms_per_launch = ms / reps;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    for (float* p : {qkv, O, P, dO, dqkv, dsbuf}) cudaFree(p);
  });
}

// ---- GEMM micro-benchmark (tools/gemm_bench.py) ----
mglp_status mglp_bench_gemm(int G, int M, int N, int K, int a_mn, int b_mn, int b_presplit,
                            int epi, int reps, float* ms_per_launch) {
  return guard([&] {
    float* ahl = nullptr;
    float *A = nullptr, *B = nullptr, *Cm = nullptr, *hl = nullptr, *C2 = nullptr,
          *bias = nullptr;
    const long long na = (long long)G * M * K, nb = (long long)G * N * K,
                    nc = (long long)G * M * N;
    MGLP_CUDA(cudaMalloc(&A, na * sizeof(float)));
    MGLP_CUDA(cudaMalloc(&B, nb * sizeof(float)));
    MGLP_CUDA(cudaMalloc(&Cm, nc * sizeof(float)));
    MGLP_CUDA(cudaMemset(A, 0x3c, na * sizeof(float)));
    MGLP_CUDA(cudaMemset(B, 0x3c, nb * sizeof(float)));
    GemmArgs g;
    g.G = G;
    g.M = M;
    g.N = N;
    g.K = K;
    g.A.ptr = A;
    g.A.slot_stride = (long long)M * K;
    g.A.ld = a_mn ? M : K;
    g.a_mn = a_mn != 0;
    g.B.ptr = B;
    g.B.slot_stride = (long long)N * K;
    g.B.ld = b_mn ? N : K;
    g.b_mn = b_mn != 0;
    g.ep.kind = EPI_STORE;
    g.ep.out1.ptr = Cm;
    g.ep.out1.slot_stride = (long long)M * N;
    g.ep.out1.ld = N;
    if (epi == EPI_BIAS_GELU || epi == EPI_GELU_BWD) {
      MGLP_CUDA(cudaMalloc(&C2, nc * sizeof(float)));
      MGLP_CUDA(cudaMalloc(&bias, (size_t)N * sizeof(float)));
      MGLP_CUDA(cudaMemset(C2, 0, nc * sizeof(float)));
      MGLP_CUDA(cudaMemset(bias, 0, (size_t)N * sizeof(float)));
      g.ep.kind = epi;
      Mat m2 = g.ep.out1;
      m2.ptr = C2;
      if (epi == EPI_BIAS_GELU) {
        g.ep.out2 = m2;
        g.ep.bias.ptr = bias;
      } else {
        g.ep.aux = m2;
      }
    }
    if (b_presplit) {
      const long long kp = pack_hl_cols(K);
      MGLP_CUDA(cudaMalloc(&hl, (size_t)G * N * kp * sizeof(float)));
      launch_pack_hl(B, g.B.slot_stride, g.B.ld, hl, (long long)N * kp, (int)kp, G, N, K,
                     b_mn != 0, 0);
      g.Bhl.ptr = hl;
      g.Bhl.slot_stride = (long long)N * kp;
      g.Bhl.ld = (int)kp;
      if ((b_presplit & 2) && !a_mn) {
        MGLP_CUDA(cudaMalloc(&ahl, (size_t)G * M * kp * sizeof(float)));
        launch_pack_hl(A, g.A.slot_stride, g.A.ld, ahl, (long long)M * kp, (int)kp, G, M, K,
                       false, 0);
        g.Ahl.ptr = ahl;
        g.Ahl.slot_stride = (long long)M * kp;
        g.Ahl.ld = (int)kp;
      }
    }
    cudaEvent_t e0, e1;
    MGLP_CUDA(cudaEventCreate(&e0));
    MGLP_CUDA(cudaEventCreate(&e1));
    launch_gemm_tc(g, nullptr, 0);
    MGLP_CUDA(cudaEventRecord(e0, 0));
    for (int r = 0; r < reps; ++r) launch_gemm_tc(g, nullptr, 0);
    MGLP_CUDA(cudaEventRecord(e1, 0));
    MGLP_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    MGLP_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *ms_per_launch = ms / reps;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    for (float* p : {ahl, A, B, Cm, hl, C2, bias})
      if (p) cudaFree(p);
  });
}

// ---- training edge ---------------------------------------------------------------
struct mglp_trainer {
  std::unique_ptr<Trainer> t;
};

mglp_status mglp_trainer_create(const mglp_stack_desc* stack, const mglp_solve_config* solve,
                                const mglp_task_desc* task, const mglp_opt_desc* opt, int vocab,
                                int max_seq, int batch_size, unsigned long long seed, int device,
                                mglp_trainer** out) {
  return guard([&] {
    need(stack, "stack");
    need(solve, "solve");
    need(task, "task");
    need(opt, "opt");
    need(out, "out");
    TaskDesc td;
    td.kind = task->kind;
    td.vocab = task->vocab;
    td.seq_len = task->seq_len;
    td.train_size = task->train_size;
    td.val_size = task->val_size;
    td.seed = task->seed;
    OptDesc od;
    od.kind = opt->kind;
    od.lr = opt->lr;
    od.beta1 = opt->beta1;
    od.beta2 = opt->beta2;
    od.eps = opt->eps;
    od.weight_decay = opt->weight_decay;
    od.momentum = opt->momentum;
    auto* h = new mglp_trainer;
    try {
      h->t = std::make_unique<Trainer>(to_stack(stack), to_solve(solve), vocab, max_seq, td, od,
                                       batch_size, seed, device);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

mglp_status mglp_trainer_destroy(mglp_trainer* t) {
  return guard([&] { delete t; });
}

static Trainer& tr(mglp_trainer* t) {
  if (!t || !t->t) throw ValidationError("null trainer");
  return *t->t;
}

mglp_status mglp_trainer_update(mglp_trainer* t, long long k, int parallel, int apply,
                                double* loss) {
  return guard([&] {
    const double l = tr(t).update(k, parallel != 0, apply != 0);
    if (loss) *loss = l;
  });
}

mglp_status mglp_trainer_monitor_attach(mglp_trainer* t, double threshold, int policy_switch,
                                       int max_iter_cap) {
  return guard([&] { tr(t).engine().monitor_attach(threshold, policy_switch, max_iter_cap); });
}

mglp_status mglp_trainer_update_probe(mglp_trainer* t, long long k, int use_probe_gradient,
                                      double* loss, int* fwd_iters, int* bwd_iters,
                                      double* fwd_factor, double* bwd_factor, int* decision,
                                      int* switched) {
  return guard([&] {
    const ProbeOutcome o = tr(t).update_probe(k, use_probe_gradient != 0);
    if (loss) *loss = o.loss;
    if (fwd_iters) *fwd_iters = o.fwd_iters;
    if (bwd_iters) *bwd_iters = o.bwd_iters;
    if (fwd_factor) *fwd_factor = o.fwd_factor;
    if (bwd_factor) *bwd_factor = o.bwd_factor;
    if (decision) *decision = o.decision;
    if (switched) *switched = o.switched;
  });
}

mglp_status mglp_trainer_last_factors(mglp_trainer* t, double* fwd_factor, double* bwd_factor,
                                      int* fwd_iters, int* bwd_iters) {
  return guard([&] {
    const MonitorSummary& m = tr(t).engine().monitor_read();
    if (fwd_factor) *fwd_factor = m.trace_ff;
    if (bwd_factor) *bwd_factor = m.trace_bf;
    if (fwd_iters) *fwd_iters = m.used[0];
    if (bwd_iters) *bwd_iters = m.used[1];
  });
}

mglp_status mglp_trainer_monitor_reports(mglp_trainer* t, long long* batch, double* fwd_factor,
                                        double* bwd_factor, int* decision, int cap, int* n) {
  return guard([&] {
    const int k = tr(t).engine().monitor_reports(batch, fwd_factor, bwd_factor, decision, cap);
    if (n) *n = k;
  });
}

mglp_status mglp_trainer_evaluate(mglp_trainer* t, double* accuracy) {
  return guard([&] {
    need(accuracy, "accuracy");
    *accuracy = tr(t).evaluate();
  });
}

mglp_status mglp_trainer_num_params(mglp_trainer* t, long long* n) {
  return guard([&] {
    need(n, "n");
    *n = tr(t).num_params();
  });
}

mglp_status mglp_trainer_get_params(mglp_trainer* t, double* flat) {
  return guard([&] {
    need(flat, "flat");
    tr(t).get_params(flat);
  });
}

mglp_status mglp_trainer_set_params(mglp_trainer* t, const double* flat) {
  return guard([&] {
    need(flat, "flat");
    tr(t).set_params(flat);
  });
}

mglp_status mglp_trainer_get_grads(mglp_trainer* t, double* flat) {
  return guard([&] {
    need(flat, "flat");
    tr(t).get_grads(flat);
  });
}

mglp_status mglp_trainer_read_logits(mglp_trainer* t, float* out) {
  return guard([&] {
    need(out, "out");
    tr(t).read_logits(out);
  });
}

mglp_status mglp_trainer_read_batch(mglp_trainer* t, int split, long long start, int* src,
                                    int* tgt_in, int* tgt_out) {
  return guard([&] {
    need(src, "src");
    need(tgt_out, "tgt_out");
    tr(t).read_batch(split, start, src, tgt_in, tgt_out);
  });
}

mglp_status mglp_trainer_get_iters(mglp_trainer* t, int* fwd_iters, int* bwd_iters) {
  return guard([&] {
    const SolveCfg& c = tr(t).engine().config();
    if (fwd_iters) *fwd_iters = c.fwd_iters;
    if (bwd_iters) *bwd_iters = c.bwd_iters;
  });
}

mglp_status mglp_trainer_set_iters(mglp_trainer* t, int fwd_iters, int bwd_iters) {
  return guard([&] {
    if (fwd_iters < 1 || bwd_iters < 1) throw ValidationError("iterations must be >= 1");
    Engine& en = tr(t).engine();
    if (!en.monitor_on()) en.drop_graph();
    en.set_budget(fwd_iters, bwd_iters);
  });
}

mglp_status mglp_trainer_snapshot(mglp_trainer* t) {
  return guard([&] { tr(t).engine().snapshot(); });
}

mglp_status mglp_trainer_restore(mglp_trainer* t) {
  return guard([&] { tr(t).engine().restore(); });
}

mglp_status mglp_trainer_trace(mglp_trainer* t, int fwd, double* out, int cap, int* n,
                               int* converged) {
  return guard([&] {
    std::vector<double> trace;
    bool conv = false;
    tr(t).engine().read_trace(fwd != 0, &trace, &conv);
    const int m = (int)std::min<size_t>(trace.size(), (size_t)std::max(cap, 0));
    if (out) std::copy(trace.begin(), trace.begin() + m, out);
    if (n) *n = (int)trace.size();
    if (converged) *converged = conv ? 1 : 0;
  });
}

mglp_status mglp_trainer_save_checkpoint(mglp_trainer* t, long long batch, const char* echo,
                                         long long echo_len, char* out, long long cap,
                                         long long* len) {
  return guard([&] {
    need(len, "len");
    const std::string blob =
        tr(t).save_checkpoint(batch, echo ? std::string(echo, (size_t)echo_len) : std::string());
    *len = (long long)blob.size();
    if (out && (long long)blob.size() <= cap) std::memcpy(out, blob.data(), blob.size());
  });
}

mglp_status mglp_trainer_load_checkpoint(mglp_trainer* t, const char* blob, long long len,
                                         long long* batch, char* echo, long long echo_cap,
                                         long long* echo_len, int* has_optimizer) {
  return guard([&] {
    need(blob, "blob");
    const CheckpointMeta m = tr(t).load_checkpoint(std::string(blob, (size_t)len));
    if (batch) *batch = m.batch;
    if (echo_len) *echo_len = (long long)m.config_echo.size();
    if (echo && (long long)m.config_echo.size() <= echo_cap)
      std::memcpy(echo, m.config_echo.data(), m.config_echo.size());
    if (has_optimizer) *has_optimizer = m.has_optimizer ? 1 : 0;
  });
}

}  // extern "C"
