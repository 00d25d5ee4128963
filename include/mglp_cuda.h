/* mglp_cuda.h -- C-ABI drop-in boundary for the layer-parallel (MGRIT) hot path.
 *
 * The reference (mglp, /root/reference/proj) exposes this path as C++
 * classes, not an FFI: LayerStack (blocks.hpp:120-175), SolveConfig /
 * LayerParallelEngine (adjoint.hpp:70-219) and the controller free functions
 * (controller.hpp:63-105). Each entry point below replaces one of those
 * members; the file:line of the replaced interface is given per function.
 * Plain pointers and sizes only -- no torch, no C++ types.
 *
 * States cross the boundary as flat float64 arrays in the reference's
 * State{x, y} layout (blocks.hpp:70-73): x [batch, s_x, d] followed by
 * y [batch, s_y, d] (y absent unless the stack is encoder-decoder).
 * Parameters and gradients are flat float64 arrays in visit_params order
 * (blocks.cpp:627-646). On the device everything is fp32 with 3-pass
 * fp16-split tensor-core GEMMs (~22-bit operands, fp32 accumulation);
 * results agree with the f64 reference to ~1e-5 relative.
 *
 * Status codes mirror the reference's error taxonomy (errors.hpp:25-35,
 * tools/main.cpp:244-252): 0 ok, 1 ValidationError (bad input / config),
 * 2 ContractViolation (broken invariant, CUDA failure). mglp_last_error()
 * returns the message of the last failing call on this thread.
 *
 * Threading: one engine per host thread, as in the reference.
 */
#ifndef MGLP_CUDA_H_
#define MGLP_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int mglp_status;
#define MGLP_OK 0
#define MGLP_VALIDATION_ERROR 1
#define MGLP_CONTRACT_VIOLATION 2

/* ModelKind (blocks.hpp:98) */
#define MGLP_ENCODER 0
#define MGLP_DECODER_ONLY 1
#define MGLP_ENCODER_DECODER 2

/* InitialGuess (mgrit.hpp:30) */
#define MGLP_GUESS_BROADCAST 0
#define MGLP_GUESS_ZERO 1
#define MGLP_GUESS_WARM 2

/* StackConfig (blocks.hpp:100-114) */
typedef struct {
  int kind;
  int d, heads, ffn;
  int n_enc, n_dec;
  int buffer_open, buffer_close;
  double ln_eps;
  double base_h;
  double dropout; /* frozen per-batch masks: mglp_engine_refresh_dropout / _set_dropout_masks */
  double init_std;
  int depth_scaled_init;
} mglp_stack_desc;

/* SolveConfig (adjoint.hpp:70-79) */
typedef struct {
  int coarsen, levels;
  int fwd_iters, bwd_iters;
  double fwd_tol, bwd_tol;
  int cold_guess;
  int warm_start;
} mglp_solve_config;

typedef struct mglp_engine mglp_engine;

const char* mglp_last_error(void);
/* library build string (arch, precision mode) */
const char* mglp_version(void);

/* LayerParallelEngine(const LayerStack&, Executor&, SolveConfig)
 * (adjoint.hpp:101-108) + LayerStack(StackConfig, seed) shape checks
 * (blocks.cpp:385-419). Parameters start at zero: call
 * mglp_engine_init_params or mglp_engine_set_params. */
mglp_status mglp_engine_create(const mglp_stack_desc* stack, const mglp_solve_config* solve,
                               int device, mglp_engine** out);
mglp_status mglp_engine_destroy(mglp_engine* e);

/* LayerStack accessors (blocks.hpp:125-130) */
mglp_status mglp_engine_info(mglp_engine* e, int* total_layers, int* interior_begin,
                             int* interior_end, long long* num_params);
mglp_status mglp_engine_step_size(mglp_engine* e, int layer, double* h);

/* LayerStack(cfg, seed) parameter initialisation (blocks.cpp:432-449);
 * bit-identical f64 values. flat_out (nullable) receives them. */
mglp_status mglp_engine_init_params(mglp_engine* e, unsigned long long seed, double* flat_out);
/* params() write / read in visit_params order (blocks.cpp:627-655) */
mglp_status mglp_engine_set_params(mglp_engine* e, const double* flat, long long n);
mglp_status mglp_engine_get_params(mglp_engine* e, double* flat, long long n);

/* config() (adjoint.hpp:110-111) */
mglp_status mglp_engine_get_config(mglp_engine* e, mglp_solve_config* cfg);
mglp_status mglp_engine_set_config(mglp_engine* e, const mglp_solve_config* cfg);

/* ForwardOutcome forward(const State& z0) (adjoint.hpp:113-137).
 * traj_out (nullable): (total_layers+1) states. trace_out: up to max_trace
 * residual norms; *n_trace gets the count, *converged the flag. */
mglp_status mglp_engine_forward(mglp_engine* e, int batch, int s_x, int s_y, const double* z0,
                                double* traj_out, double* trace_out, int max_trace,
                                int* n_trace, int* converged);

/* BackwardOutcome backward(traj, lambda_N, grads*) (adjoint.hpp:139-183).
 * traj_in == NULL reuses the device-resident trajectory of the last forward
 * (the common case; no host copy). grads_accum (nullable) is ACCUMULATED
 * (+=), like the reference's caller-owned grads. */
mglp_status mglp_engine_backward(mglp_engine* e, int batch, int s_x, int s_y,
                                 const double* traj_in, const double* lam_n, double* lam0_out,
                                 double* grads_accum, double* trace_out, int max_trace,
                                 int* n_trace, int* converged);

/* mglp_engine_backward with the parameter gradients kept in the engine's
 * device slab (zeroed, then this call's gradients; scaled by h as the
 * reference's) for a device optimizer or a later mglp_engine_get_grads /
 * _get_grads_layers -- the host sees lambda_0 and the trace only. This is
 * the boundary a device-resident training step uses (the reference's
 * Trainer::run_update hands its grads straight to the optimizer, training.cpp:224-239). */
mglp_status mglp_engine_backward_keep_grads(mglp_engine* e, int batch, int s_x, int s_y,
                                            const double* traj_in, const double* lam_n,
                                            double* lam0_out, double* trace_out, int max_trace,
                                            int* n_trace, int* converged);

/* WarmSnapshot snapshot() / restore() / reset() (adjoint.hpp:187-206).
 * The engine keeps ONE snapshot slot: snapshot_id returns the id of the
 * snapshot just taken, restore_id(id) fails with status 1 if that snapshot
 * was overwritten (a later snapshot or a shape change); restore() restores
 * whatever the slot holds. */
mglp_status mglp_engine_snapshot(mglp_engine* e);
mglp_status mglp_engine_restore(mglp_engine* e);
mglp_status mglp_engine_snapshot_id(mglp_engine* e, long long* id);
mglp_status mglp_engine_restore_id(mglp_engine* e, long long id);
mglp_status mglp_engine_reset(mglp_engine* e);
/* The forward solver's warm states := the device trajectory currently held
 * (e.g. after mglp_serial_forward): the next warm-guess forward starts there.
 * (Serial sweeps and uploaded trajectories otherwise never touch the
 * solver's warm states, as in the reference.) */
mglp_status mglp_engine_seed_forward_from_traj(mglp_engine* e);

/* serial_forward / serial_adjoint (blocks.cpp:659-682). lam_all_out
 * (nullable) receives lambda at every time point. */
mglp_status mglp_serial_forward(mglp_engine* e, int batch, int s_x, int s_y, const double* z0,
                                double* traj_out);
mglp_status mglp_serial_adjoint(mglp_engine* e, int batch, int s_x, int s_y,
                                const double* traj_in, const double* lam_n, double* lam_all_out,
                                double* grads_accum);

/* LayerStack::step / adjoint_step (blocks.cpp:509-514, 566-574) for one layer */
mglp_status mglp_stack_step(mglp_engine* e, int layer, double dt, int batch, int s_x, int s_y,
                            const double* z, double* out);
mglp_status mglp_stack_adjoint_step(mglp_engine* e, int layer, double dt, int batch, int s_x,
                                    int s_y, const double* z, const double* lam,
                                    double* grads_accum, double gscale, double* out);

/* ---- device-resident hot path (inputs already in HBM; no host sync) ----
 * Pointers are device fp32 buffers of state_elems() floats (x then y).
 * These are what bench.py times; mglp_engine_stream() is the CUDA stream
 * every launch goes to. */
mglp_status mglp_engine_set_shape(mglp_engine* e, int batch, int s_x, int s_y,
                                  long long* state_elems);
mglp_status mglp_engine_stream(mglp_engine* e, void** cuda_stream);
mglp_status mglp_engine_forward_device(mglp_engine* e, const float* z0_dev);
mglp_status mglp_engine_backward_device(mglp_engine* e, const float* lam_n_dev,
                                        float* lam0_dev, int want_grads);
mglp_status mglp_serial_forward_device(mglp_engine* e, const float* z0_dev);
mglp_status mglp_serial_adjoint_device(mglp_engine* e, const float* lam_n_dev, float* lam0_dev,
                                       int want_grads);
/* CUDA graph of one whole step (forward_device + backward_device on these
 * fixed buffers, current config); replay is a single graph launch. The
 * solve's stopping rule runs on the device, so the captured step is exact. */
mglp_status mglp_engine_graph_capture(mglp_engine* e, const float* z0_dev, const float* lam_n_dev,
                                      float* lam0_dev, int want_grads);
mglp_status mglp_engine_graph_replay(mglp_engine* e);
mglp_status mglp_engine_zero_grads(mglp_engine* e);
/* flat (visit_params order) += device gradient bank */
mglp_status mglp_engine_get_grads(mglp_engine* e, double* flat, long long n);
/* flat (n = the parameter count of layers [layer_lo, layer_hi), visit_params
 * order) += those layers' gradients: per-layer-block download (a rank's
 * owned block; full-depth parity checks without a whole-model host copy) */
mglp_status mglp_engine_get_grads_layers(mglp_engine* e, int layer_lo, int layer_hi,
                                         double* flat, long long n);
/* PhaseTrace of the last forward (which=0) or backward (which=1) solve */
mglp_status mglp_engine_trace(mglp_engine* e, int which, double* trace_out, int max_trace,
                              int* n_trace, int* converged);
/* device pointer of the trajectory (total_layers+1 states) */
/* copies time points [first, first+count) of the device trajectory (fp32,
 * state_elems floats per point, padding included) to dst (host or device) */
mglp_status mglp_engine_read_traj(mglp_engine* e, int first, int count, float* dst);
mglp_status mglp_engine_traj_device(mglp_engine* e, float** traj);
mglp_status mglp_engine_sync(mglp_engine* e);
/* hot-path kernel launches issued since the last call (then reset) */
mglp_status mglp_engine_take_launch_count(mglp_engine* e, long long* n);

/* per-kernel-class device timing for roofline reporting: when enabled, every
 * launch is bracketed by CUDA events on the engine stream. Classes: 0 tensor
 * core GEMM, 1 attention, 2 LayerNorm rows. Reading returns per class the
 * summed device ms, algorithmic FLOPs, algorithmic bytes and launch count
 * since profiling was (re)enabled. */
mglp_status mglp_engine_profile(mglp_engine* e, int enable);
mglp_status mglp_engine_profile_read(mglp_engine* e, double* ms, double* flops, double* bytes,
                                     long long* launches);
/* per-launch rows (8 doubles each: class, M, N, K, batch, flops, ms, variant; variant
 * for GEMMs = epilogue kind + 16 A pre-split + 32 B pre-split + 64 A MN-major +
 * 128 B MN-major, -1 otherwise) */
mglp_status mglp_engine_profile_dump(mglp_engine* e, double* rows, int max_rows, int* n);

/* ---- multi-GPU: layer blocks over ranks ----
 * Rank r of P owns the contiguous block of coarse intervals
 * [r*C/P, (r+1)*C/P) (C = N/c_f; P must divide the interval count of every
 * level): its layers' parameters, activation cache and gradients. Boundary
 * states move by NCCL send/recv over NVLink. One process per GPU: rank 0
 * calls mglp_nccl_unique_id and shares the 128 bytes (e.g. via
 * torch.distributed); every rank then calls mglp_engine_create_dist. The
 * device-resident entry points (…_device) then run the distributed solve;
 * lambda_0 is produced on rank 0, traces are identical on every rank. */
mglp_status mglp_nccl_unique_id(void* id128);
mglp_status mglp_engine_create_dist(const mglp_stack_desc* stack, const mglp_solve_config* solve,
                                    int device, int rank, int world, const void* id128,
                                    mglp_engine** out);
/* rank, world and the owned interior layer range [layer_lo, layer_hi) */
mglp_status mglp_engine_rank_info(mglp_engine* e, int* rank, int* world, int* layer_lo,
                                  int* layer_hi);
/* LayerStack::masks() set explicitly (a reference-side stack's frozen masks,
 * blocks.cpp:576-599): keep[(layer * 3 + site) * max(B*s_x, B*s_y) * d + i]
 * = 1 keeps element i of that layer's site (0 attention out phi1, 1 MLP out
 * phi2, 2 cross-attention out phi3 -- decoder layers only), 0 drops it; the
 * kept values are scaled by 1 / (1 - dropout) as in the reference. */
mglp_status mglp_engine_set_dropout_masks(mglp_engine* e, int batch, int s_x, int s_y,
                                          const unsigned char* keep);

/* Device memory this engine holds (parameters, pre-split weights, gradients,
 * activation caches, trajectory, solver levels, scratch): on a P-rank engine
 * the per-layer and per-time-point buffers are mapped only under the rank's
 * own block (CUDA virtual memory; the rest of the virtual range faults), so
 * this is about 1/P of the single-rank figure plus the shared scratch. */
mglp_status mglp_engine_memory(mglp_engine* e, long long* bytes);

/* The communicator behind a multi-rank engine: *backend 0 = none (one GPU),
 * 1 = NCCL, 2 = in-process loopback; *nranks = the rank count the backend
 * itself reports (ncclCommCount), recorded by bench.py next to n_gpus. */
mglp_status mglp_engine_comm_info(mglp_engine* e, int* backend, int* nranks);

/* Test support: P virtual ranks as P engines on ONE device exchanging through
 * device buffers (same partitioned control flow as NCCL). run_fwd_bwd runs
 * forward_device + backward_device on all P engines concurrently (one host
 * thread each); lam0_dev is written by rank 0. */
mglp_status mglp_loopback_create(const mglp_stack_desc* stack, const mglp_solve_config* solve,
                                 int device, int world, mglp_engine** engines);
mglp_status mglp_loopback_run_fwd_bwd(mglp_engine** engines, int world, const float* z0_dev,
                                      const float* lam_n_dev, float* lam0_dev, int want_grads);

/* ---- gradient-bias monitor on the device (controller.hpp:32-166) ----
 * attach: InexactnessMonitor(IndicatorConfig{threshold, policy, cap}); the
 * engine's fwd/bwd iteration budgets (SolveConfig::fwd_iters / bwd_iters)
 * move into device memory and every solve runs the DEVICE budget (the host
 * issues an upper bound of cycles; surplus cycles are no-ops on the device).
 * probe(1/0): ProbeScope begin / end -- both budgets doubled for one batch
 * (controller.hpp:88-105), on the device.
 * mglp_monitor_record: InexactnessMonitor::record(batch, ...)
 * as ONE kernel on the engine stream: f = last_pair_factor of the forward /
 * adjoint traces the last solves left in device memory, decision = decide(f)
 * (0 keep, 1 increase iterations, 2 switch to serial), budgets doubled
 * (capped) on increase, the switch flag set on switch, the report logged.
 * No allocation, no host round trip; with decision == NULL it is fully
 * asynchronous (and graph-capturable); otherwise it synchronises to return
 * the decision. mglp_engine_monitor_read synchronises and returns the
 * device state (last report, budgets now, budgets the last solves used);
 * _reports copies the report log (oldest first, up to 1024 kept).
 * mglp_engine_capture_cycles(n): a CUDA graph captured next issues n cycles
 * per solve, gated by the device budget, so a monitor decision changes the
 * replayed budget without recapture; a budget above n makes the trace read
 * fail (status 2) instead of silently truncating. */
mglp_status mglp_engine_monitor_attach(mglp_engine* e, double threshold, int policy_switch,
                                      int max_iter_cap);
mglp_status mglp_engine_monitor_probe(mglp_engine* e, int begin);
mglp_status mglp_monitor_record(mglp_engine* e, long long batch, int* decision);
mglp_status mglp_engine_monitor_read(mglp_engine* e, int* switched, int* decision,
                                    double* fwd_factor, double* bwd_factor, int* fwd_iters,
                                    int* bwd_iters, int* used_fwd, int* used_bwd);
mglp_status mglp_engine_monitor_reports(mglp_engine* e, long long* batch, double* fwd_factor,
                                       double* bwd_factor, int* decision, int cap, int* n);
mglp_status mglp_engine_capture_cycles(mglp_engine* e, int cycles);

/* Host helper: out[i] = scale * rng::gaussian(seed, a, b, i) (rng.hpp:70-79),
 * bit-identical to the reference (same libm); the reference bench's z0 draw
 * is (seed, kTestOnly=6, 7) with scale 0.5 (tools/main.cpp:121-128). */
mglp_status mglp_rng_gaussian_fill(unsigned long long seed, unsigned long long a,
                                   unsigned long long b, double scale, double* out, long long n);

/* ---- test hook: one GEMM family on device buffers ----
 * C_g[M,N] = A_g . B_g^T (+ bias), g < G; A_g at A + g*a_slot (row stride
 * lda; [M,K] or, if a_mn, [K,M]); B likewise ([N,K] or [K,N]); C at
 * C + g*c_slot, row stride ldc. engine 0 = tcgen05 fp16x3 split (the
 * product kernel), 1 = fp32 CUDA-core reference. b_presplit exercises the
 * pre-split (hi|lo) weight path of the tensor-core kernel (bit 1 set: a
 * K-major A is pre-split too -- the converter-free mainloop); b_presplit = 4
 * with b_mn hands B's [K][N] rows over pre-split instead (the weight-gradient
 * operand form: the converters regroup, no split); b_presplit = 8 with a_mn
 * does the same for A. range_flag
 * (nullable) receives 1 if a finite operand overflowed the fp16 split
 * range. Synchronous. */
mglp_status mglp_test_gemm(int G, int M, int N, int K, const float* A, long long a_slot, int lda,
                           int a_mn, const float* B, long long b_slot, int ldb, int b_mn,
                           int b_presplit, const float* bias, float* C, long long c_slot, int ldc,
                           int engine, int* range_flag);

/* ---- frozen dropout masks: LayerStack::refresh_dropout / clear_dropout
 * (blocks.cpp:576-599). refresh sets the shape and generates, on the device,
 * the masks of batch `batch_index` for every layer and site from the
 * reference's counter streams (bit-identical keep / drop decisions); they
 * apply to every following step / adjoint step / solve of that shape until
 * cleared or refreshed. No-ops when the stack's dropout is <= 0. */
mglp_status mglp_engine_refresh_dropout(mglp_engine* e, unsigned long long seed,
                                        unsigned long long batch_index, int batch, int s_x,
                                        int s_y);
mglp_status mglp_engine_clear_dropout(mglp_engine* e);

/* ---- Lipschitz probe (lipschitz.cpp:53-149, estimate_lipschitz /
 * estimate_stack) on the device: for each layer in `layers` (NULL: every
 * layer, n_layers ignored) the max over `samples` draws of
 * ||F(x + delta) - F(x)|| / ||delta|| of the layer's residual map F, x =
 * input_scale * N(.), delta = delta_scale * N(.) over one [1, seq_len, d]
 * sequence (the reference's rng streams kProbeInput / kProbeDelta, folded
 * per layer). estimates: one double per probed layer. Synchronous. */
mglp_status mglp_engine_lipschitz(mglp_engine* e, int samples, double delta_scale,
                                  double input_scale, int seq_len, unsigned long long seed,
                                  const int* layers, int n_layers, double* estimates);

/* ---- test hook: the fused tcgen05 attention (attn_tc.cu) on device buffers ----
 * Q, K, V (and dO, dQ, dK, dV, O) are [B][s][ld] token rows with head h at
 * column h*dh (the qkv layout of the layer); P is [B][H][sq][pad4(skv)].
 * Forward always; with dO set, also the backward (dQ, dK, dV overwritten).
 * sq, skv <= 128 and multiples of 8 (attn_tc.cu), or 128 <= sq, skv <= 512
 * (attn_long.cu: P then receives the per-row (max, 1/sum) statistics, [sq][2]
 * per head, instead of the probabilities); dh 32 or 64 (else status 1).
 * causal bit 0: causal mask; bit 1 (sq = skv = 128 only): P is kept in the
 * pre-split form the engine uses at s = 128 (the forward's hi|lo' tiles, 64
 * KiB per head; not probabilities); bit 2 (dh = 64, s <= 128): Q, K, V and dO
 * are given in the head-split pre-split form the engine's GEMMs write (per
 * 64 columns: 64 fp16 hi, 64 fp16 lo' = fp16((x - hi) 2^11)). The reference's attention /
 * vjp_attention (blocks.cpp:142-236). Synchronous. */
mglp_status mglp_test_attention(int B, int H, int sq, int skv, int dh, int causal, const float* Q,
                                const float* K, const float* V, int ld, float* O, float* P,
                                const float* dO, float* dQ, float* dK, float* dV,
                                int* range_flag);

/* ---- micro-benchmark: `reps` launches of the fused attention over G x B x H
 * heads of length s (forward, or backward when `backward`), device-timed. */
mglp_status mglp_bench_attention(int G, int B, int H, int s, int dh, int causal, int backward /* 0 fwd, 1 bwd, 2 fwd no P, 3 fwd no P, O pre-split */,
                                 int reps, float* ms_per_launch);

/* ---- micro-benchmark: `reps` launches of one tensor-core GEMM family
 * (epilogue kind epi: 0 store, 2 bias+GELU (two outputs), 4 GELU-backward;
 * device-resident synthetic operands), device-timed. */
mglp_status mglp_bench_gemm(int G, int M, int N, int K, int a_mn, int b_mn, int b_presplit,
                            int epi, int reps, float* ms_per_launch);

/* ---- training edge: the reference's Trainer::run_update on the device ----
 * (training.cpp:230-268): make_batch (tasks.cpp:45-89, bit-exact tokens),
 * Model::embed / logits / cross_entropy / head_backward / embed_backward
 * (model.cpp:133-275) and Optimizer::step (optimizer.cpp:43-88, f64 master
 * parameters and moments), around the layer-parallel engine. Parameters are
 * flat float64 arrays in Model::param_tensors order (model.cpp:74-92). */

/* TaskSpec (tasks.hpp:24-42); kind 0 copy_sequence, 1 token_classification,
 * 2 tiny_translation */
typedef struct {
  int kind;
  int vocab, seq_len, train_size, val_size;
  unsigned long long seed;
} mglp_task_desc;

/* OptConfig (optimizer.hpp:24-34); kind 0 sgd, 1 adam, 2 adamw */
typedef struct {
  int kind;
  double lr, beta1, beta2, eps, weight_decay, momentum;
} mglp_opt_desc;

typedef struct mglp_trainer mglp_trainer;

/* Trainer(task, ModelConfig{stack, vocab, max_seq}, TrainConfig) +
 * Model(mcfg, seed) init (training.cpp:74-90, model.cpp:50-72) */
mglp_status mglp_trainer_create(const mglp_stack_desc* stack, const mglp_solve_config* solve,
                                const mglp_task_desc* task, const mglp_opt_desc* opt, int vocab,
                                int max_seq, int batch_size, unsigned long long seed, int device,
                                mglp_trainer** out);
mglp_status mglp_trainer_destroy(mglp_trainer* t);
/* run_update(k, parallel, apply) (training.cpp:230-268): loss of batch k */
mglp_status mglp_trainer_update(mglp_trainer* t, long long k, int parallel, int apply,
                                double* loss);
/* probe_batch(k) (training.cpp:244-276) with the engine's device monitor
 * (mglp_trainer_monitor_attach first): ProbeScope on the device budgets, the
 * update (use_probe_gradient: the doubled run IS the update; else a
 * measurement-only run behind a warm-state snapshot, then the nominal update
 * at the decided budget), record() on the device. Outputs: the row's loss,
 * budgets and factors, the decision and the switch flag. */
mglp_status mglp_trainer_monitor_attach(mglp_trainer* t, double threshold, int policy_switch,
                                       int max_iter_cap);
mglp_status mglp_trainer_update_probe(mglp_trainer* t, long long k, int use_probe_gradient,
                                      double* loss, int* fwd_iters, int* bwd_iters,
                                      double* fwd_factor, double* bwd_factor, int* decision,
                                      int* switched);
/* last_pair_factor of the last parallel update's traces and the budgets it
 * ran with, evaluated on the device (monitor attached) */
mglp_status mglp_trainer_last_factors(mglp_trainer* t, double* fwd_factor, double* bwd_factor,
                                      int* fwd_iters, int* bwd_iters);
mglp_status mglp_trainer_monitor_reports(mglp_trainer* t, long long* batch, double* fwd_factor,
                                        double* bwd_factor, int* decision, int cap, int* n);
/* evaluate() (training.cpp:296-310): validation token accuracy */
mglp_status mglp_trainer_evaluate(mglp_trainer* t, double* accuracy);
mglp_status mglp_trainer_num_params(mglp_trainer* t, long long* n);
mglp_status mglp_trainer_get_params(mglp_trainer* t, double* flat);
mglp_status mglp_trainer_set_params(mglp_trainer* t, const double* flat);
/* gradients of the last update (zeroed at the start of every update) */
mglp_status mglp_trainer_get_grads(mglp_trainer* t, double* flat);
/* logits of the last update / evaluation batch, [batch*seq][vocab] */
mglp_status mglp_trainer_read_logits(mglp_trainer* t, float* out);
/* test hook: make_batch(task, split, start, batch) on the device
 * (tasks.cpp:45-89); tgt_in may be NULL for single-stream tasks */
mglp_status mglp_trainer_read_batch(mglp_trainer* t, int split, long long start, int* src,
                                    int* tgt_in, int* tgt_out);
/* the engine's SolveConfig iteration budget (engine_->config(),
 * training.cpp:118-119, controller.hpp:126-147) and its warm snapshot */
mglp_status mglp_trainer_get_iters(mglp_trainer* t, int* fwd_iters, int* bwd_iters);
mglp_status mglp_trainer_set_iters(mglp_trainer* t, int fwd_iters, int bwd_iters);
mglp_status mglp_trainer_snapshot(mglp_trainer* t);
mglp_status mglp_trainer_restore(mglp_trainer* t);
/* residual-norm trace of the last forward (fwd = 1) / adjoint solve */
mglp_status mglp_trainer_trace(mglp_trainer* t, int fwd, double* out, int cap, int* n,
                               int* converged);
/* MGLP v1 checkpoint (checkpoint.cpp:88-180): save writes *len bytes into
 * out when cap suffices (always reports *len); load overwrites parameters and
 * optimizer state and reports the stored batch counter and config echo. */
mglp_status mglp_trainer_save_checkpoint(mglp_trainer* t, long long batch, const char* echo,
                                         long long echo_len, char* out, long long cap,
                                         long long* len);
mglp_status mglp_trainer_load_checkpoint(mglp_trainer* t, const char* blob, long long len,
                                         long long* batch, char* echo, long long echo_cap,
                                         long long* echo_len, int* has_optimizer);

#ifdef __cplusplus
}
#endif

#endif /* MGLP_CUDA_H_ */
