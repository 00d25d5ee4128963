// Launch wrappers for the hot-path kernels. All take a `const int* active`
// solve-control flag (nullable): when *active == 0 the kernel returns
// immediately, which is how a solve that converged (or went non-finite)
// mid-way stops without a host round trip (mgrit.hpp:252-259).
#pragma once

#include "common.cuh"

namespace mglp {

// ---- LayerNorm (tensor.cpp:239-308) -----------------------------------------
struct LnFwdArgs {
  int G = 1, rows = 0, d = 0;
  float eps = 1e-5f;
  Mat x, out, stats;  // stats: [rows][2] = (mean, rstd); out nullable
  Mat gain, bias;     // slot = layer
  Mat out_hl;         // optional: out pre-split (hi|lo' rows) for the next GEMM
  int* range_flag = nullptr;
};
void launch_ln_fwd(const LnFwdArgs& a, const int* active, cudaStream_t s);

// L = LNbwd(x, up); out1 = addA ? addA + L : L; out2 = addB + L;
// optional combine of F = out1 into the solver state.
struct LnBwdArgs {
  int G = 1, rows = 0, d = 0;
  Mat x, stats, up, gain;
  Mat addA, addB, out1, out2;
  Combine cmb;
  DropMask drop2;  // out2 = (addB + L) * mask: the VJP through a dropout site
  Mat out2_hl;     // optional: out2 pre-split (hi|lo' rows) for the next dgrad GEMM
  int* range_flag = nullptr;
};
void launch_ln_bwd(const LnBwdArgs& a, const int* active, cudaStream_t s);
int ln_bwd_blocks(int rows);

// Parameter-gradient column sums (deterministic, fixed order):
//   dbias[j] += gscale * sum_r up[r][j]
//   dgain[j] += gscale * sum_r up[r][j] * xhat[r][j]   (if x given)
struct ColRedArgs {
  int G = 1, rows = 0, cols = 0;
  Mat up, x, stats;
  Mat dgain, dbias;  // slot = layer
  float gscale = 1.f;
  const float* gscale_mul = nullptr;  // optional device factor (EpiArgs::gscale_mul)
  // optional f64 scratch (>= G * kColRedChunks * cols * 2 doubles): enables the
  // two-stage row-chunked form (fixed-order partials, then an ordered sum)
  double* partials = nullptr;
  long long partials_cap = 0;
  // up rows pre-split (hi|lo' per 32-column chunk; value = hi + 2^-11 lo')
  int up_hl = 0;
};
constexpr int kColRedChunks = 8;
void launch_colred(const ColRedArgs& a, const int* active, cudaStream_t s);

// Row softmax of attention scores S [rows][ncols] in place (scale, causal
// mask by query index row % sq); with dS set, the VJP dS = P (dP - sum dP P)
// in place over dS, where S then holds P.
struct SoftmaxArgs {
  int G = 1;
  long long rows = 0;
  int ncols = 0, sq = 1, causal = 0;
  float scale = 1.f;
  Mat S, dS;
};
void launch_softmax(const SoftmaxArgs& a, const int* active, cudaStream_t s);

// ---- state algebra (blocks.cpp:25-79; mgrit.hpp:199-223) --------------------
// Passive-stream / elementwise combine: F = Fsrc ? Fsrc : 0 over n elements
// (the stream a layer does not advance gets exactly dt*0, blocks.cpp:487,491).
struct ElemCombineArgs {
  int G = 1;
  long long n = 0;
  Mat F;  // nullable
  Combine cmb;
};
void launch_elem_combine(const ElemCombineArgs& a, const int* active, cudaStream_t s);
int elem_combine_blocks(long long n);

// dst_g = src_g
void launch_copy(int G, long long n, Mat dst, Mat src, const int* active, cudaStream_t s);
// dst_g[r][c] = src_g[r][c] * mask(r, c)  (rows x d; hadamard with a dropout site)
void launch_mask_copy(int G, int rows, int d, Mat dst, Mat src, const DropMask& m,
                      const int* active, cudaStream_t s);
// dst_g = dst_g + (a_g - b_g)     (correct_from, mgrit.hpp:219-221)
void launch_correct(int G, long long n, Mat dst, Mat a, Mat b, const int* active,
                    cudaStream_t s);
void launch_zero(int G, long long n, Mat dst, const int* active, cudaStream_t s);

// ---- solve control ------------------------------------------------------------
constexpr int kMaxTrace = 256;
struct SolveCtrl {
  int active;
  int n_trace;
  int converged;
  int cycles_run;
  double pending;
  double trace[kMaxTrace];
  int budget;     // cycles this solve may run (the host loop or the device budget)
  int truncated;  // the device budget asked for more cycles than the host loop issued
};
// budget_dev == nullptr: budget = host_cycles (the host loop count); else the
// solve's budget is the device-resident *budget_dev (the gradient-bias
// monitor's, controller.hpp:126-147), capped at host_cycles (truncated = 1
// if it asked for more)
void launch_ctrl_begin(SolveCtrl* c, int host_cycles, const int* budget_dev, cudaStream_t s);

// ---- gradient-bias monitor on the device (controller.hpp:63-155) ----------------
// InexactnessMonitor state, the live iteration budgets the solves read, and
// the report log, all in device memory: record() runs as one kernel on the
// engine stream right after a probe's solves (no host round trip, capturable).
constexpr int kMonReports = 1024;
struct MonitorDev {
  double threshold;
  int policy_switch, cap;
  int switched, n_reports;
  int budget[2];  // [fwd, bwd] SolveConfig::fwd_iters / bwd_iters
  int saved[2];   // ProbeScope
  int last_decision, pad;
  double last_ff, last_bf;
  long long rep_batch[kMonReports];
  double rep_ff[kMonReports], rep_bf[kMonReports];
  int rep_dec[kMonReports];
};
// what the host mirrors after a step (pinned, copied asynchronously)
struct MonitorSummary {
  int switched, n_reports, last_decision, pad;
  int budget[2];  // budgets now
  int used[2];    // budgets the last forward / adjoint solve ran with
  double last_ff, last_bf;  // factors of the last record()
  double trace_ff, trace_bf;  // last_pair_factor of the last solves' traces
};
void launch_monitor_init(MonitorDev* m, double threshold, int policy_switch, int cap, int fwd,
                         int bwd, cudaStream_t s);
void launch_monitor_set_budget(MonitorDev* m, int fwd, int bwd, cudaStream_t s);
// ProbeScope (controller.hpp:88-105): begin doubles both budgets, end restores
void launch_monitor_probe(MonitorDev* m, int begin, cudaStream_t s);
// record (controller.hpp:126-147) from the traces in f / b when batch >= 0;
// always refreshes *out
void launch_monitor_record(MonitorDev* m, const SolveCtrl* f, const SolveCtrl* b,
                           long long batch, MonitorSummary* out, cudaStream_t s);

// Exact power-of-two scaling of the adjoint. The adjoint
// (Phi^T, the parameter pass, the residual norms) is linear in lambda, so the
// engine runs it on 2^k lambda_N with max|2^k lambda_N| in [1, 2) and undoes
// the factor exactly where values leave the solve: lambda_0, the gradient
// accumulation (gscale * 2^-k), the residual trace (norm * 2^-k). With every
// value a normal number the result is bitwise that of the unscaled adjoint;
// lambda_N of O(1e-5..1e-8) (a mean-token cross entropy over many tokens)
// no longer lands in the fp16 split's subnormal range, and |lambda| >= 65520
// no longer overflows it. A zero or non-finite lambda_N keeps k = 0.
struct LamScale {
  unsigned int amax_bits;  // max |lambda_N| as float bits (non-negative: uint order = float order)
  float up;                // 2^k
  float down;              // 2^-k
  int k;
  double down_d;           // 2^-k
  int k_state;             // k of the adjoint solver's stored states (its warm start)
  int pad;
};
// s->amax_bits = 0; then max |x| over n floats (deterministic atomicMax)
void launch_lam_amax(const float* x, long long n, LamScale* sc, cudaStream_t s);
// warm start: also fold in max |x| * 2^-k_state over n floats (the stored
// adjoint states in their true scale), so the rescaled warm guess cannot
// overflow when lambda_N drops by binades between solves
void launch_lam_amax_warm(const float* x, long long n, LamScale* sc, cudaStream_t s);
// multi-rank max of amax_bits: out[0] = (double)amax_bits (exact), gathered
// over ranks by the caller, then amax_bits = max_r in[r]
void launch_lam_bits_to_f64(const LamScale* sc, double* out, cudaStream_t s);
void launch_lam_bits_max(const double* in, int n, LamScale* sc, cudaStream_t s);
// dst = src * 2^(+k) (dir > 0; also publishes up/down/k) or * 2^-k (dir < 0)
void launch_lam_scale(const float* src, float* dst, long long n, LamScale* sc, int dir,
                      cudaStream_t s);
// warm-start states stored at k_state, this solve runs at k: dst *= 2^(k - k_state)
// (no-op when equal)
void launch_lam_rescale(int G, long long n, Mat dst, const LamScale* sc, cudaStream_t s);
// k_state := k (the adjoint solver's states now hold this solve's scaling)
void launch_lam_commit(LamScale* sc, cudaStream_t s);
// trace entry = sqrt(sum of the per-interval partials [n_chunks][S]), measured
// mid-cycle (mgrit.hpp:235-238)
void launch_trace_record(SolveCtrl* c, const double* partials, int n_chunks, int S, int per_rank,
                         bool reversed, cudaStream_t s, const LamScale* sc = nullptr);
// end of one V-cycle: push the trace, stop on non-finite / converged (mgrit.hpp:252-259)
void launch_cycle_end(SolveCtrl* c, double tol, cudaStream_t s);

// ---- GEMM -------------------------------------------------------------------
// Reference fp32 CUDA-core GEMM: test oracle for the tensor-core path only.
void launch_gemm_simt(const GemmArgs& a, const int* active, cudaStream_t s);
int gemm_simt_blocks(const GemmArgs& a);
// Parity-grade tcgen05 (kind::f16, 3-pass fp16 hi/lo split) GEMM.
void launch_gemm_tc(const GemmArgs& a, const int* active, cudaStream_t s);
int gemm_tc_blocks(const GemmArgs& a);
// Pre-splits a family of G matrices into the hi|lo' form GemmArgs::Bhl
// expects: dst row r = per 32-wide K block [32 fp16 hi | 32 fp16 lo'], K
// zero-padded to pack_hl_cols(K) (floats per row). transpose: B = src^T
// (src is [K][rows]).
long long pack_hl_cols(int K);
void launch_pack_hl(const float* src, long long src_slot, int src_ld, float* dst,
                    long long dst_slot, int dst_ld, int G, int rows, int K, bool transpose,
                    cudaStream_t s, int* range_flag = nullptr);

// ---- fused attention (attn_tc.cu), sq, skv <= 128, dh in {32, 64} -------------
// One CTA per (member g, batch b, head h); operands address (g, b, h) through
// Mat::at(g, b, h). Forward: O = softmax(Q K^T * scale [causal]) V, P stored
// when P is set. Backward (P required): dQ = scale dS K, dK = scale dS^T Q,
// dV = P^T dO with dS = P (dO V^T - rowsum(...)).
struct AttnArgs {
  int G = 1, Bb = 1, H = 1, sq = 0, skv = 0, dh = 0, causal = 0;
  float scale = 1.f;
  Mat Q, K, V, O, P;
  Mat dO, dQ, dK, dV;
  Mat Ohl;  // forward, optional: O pre-split (hi|lo' rows) for the O-projection
  Mat dQhl, dKhl, dVhl;  // backward, optional: pre-split gradients for the QKV dgrad
  // s = 128 fused path (attn_tc.cu): P is kept in its pre-split form, the
  // forward's hi|lo' MMA operand tiles (64 KiB per problem, exactly the fp32
  // P slot), bulk-copied out by the forward and back in by the backward
  int p_hl = 0;
  // long backward, optional (s multiples of 128): the dK/dV kernel stores each
  // (query block, key block) dS tile pre-split (64 KiB) here, P-slot strides,
  // and the dQ kernel reads them instead of recomputing S, P and dP
  Mat dS;
  // Q, K, V (qkv_hs) and dO (do_hs) written by their producer GEMMs in the
  // head-split pre-split form (common.cuh st_hs4; dh = 64): TMA'd straight
  // into the operand tiles, no fp32 staging or conversion in the kernel
  int qkv_hs = 0, do_hs = 0;
  int pingpong = 1;  // s <= 128 backward: alternate the dO / V region (launch_attn_bwd)
  int* range_flag = nullptr;
};
bool attn_tc_supported(const AttnArgs& a, bool backward);
void launch_attn_fwd(const AttnArgs& a, const int* active, cudaStream_t s);
void launch_attn_bwd(const AttnArgs& a, const int* active, cudaStream_t s);
// 128 <= sq, skv <= 512 (attn_long.cu): P is not stored; the forward writes
// per-row (max, 1/sum) statistics at P.at(g, b, h) ([sq][2]) and the backward
// (which also needs O for the softmax-VJP row constant dO . O) recomputes P.
bool attn_long_supported(const AttnArgs& a, bool backward);
void launch_attn_fwd_long(const AttnArgs& a, const int* active, cudaStream_t s);
void launch_attn_bwd_long(const AttnArgs& a, const int* active, cudaStream_t s);
// 128 < sq, skv <= 512 with head-split pre-split operands (qkv_hs, dh = 64;
// attn_flash.cu): single-pass online softmax, P~ kept in TMEM; same P-slot row
// statistics (max, 1/sum) as the long form
bool attn_flash_supported(const AttnArgs& a, bool backward);
void launch_attn_fwd_flash(const AttnArgs& a, const int* active, cudaStream_t s);
// backward (qkv_hs and do_hs, fp32 O, AttnArgs::dS): t_q row dot, dK / dV per
// 128-key block storing the dS tiles, dQ per 128-query block
void launch_attn_bwd_flash(const AttnArgs& a, const int* active, cudaStream_t s);

}  // namespace mglp
