// CudaLayerParallelEngine: the B200 implementation behind the C-ABI
// (include/mglp_cuda.h). It re-expresses the reference's LayerParallelEngine
// (adjoint.hpp:99-219) + MgritSolver (mgrit.hpp:58-303) + LayerStack
// (blocks.hpp:120-175) as device-resident state and batched kernel launches:
// every relaxation sweep over the N/c_f coarse intervals is ONE family of
// launches (G = number of intervals) instead of N/c_f executor tasks.
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace mglp {

struct StackDesc {
  int kind = 0;  // 0 encoder, 1 decoder-only (causal), 2 encoder-decoder
  int d = 32, heads = 2, ffn = 64, n_enc = 8, n_dec = 0;
  int buffer_open = 0, buffer_close = 0;
  double ln_eps = 1e-5, base_h = 1.0, init_std = 0.02;
  int depth_scaled_init = 0;
  double dropout = 0.0;
};

struct SolveCfg {
  int coarsen = 2, levels = 2, fwd_iters = 2, bwd_iters = 1;
  double fwd_tol = 0.0, bwd_tol = 0.0;
  int cold_guess = 0;  // 0 broadcast, 1 zero, 2 warm
  int warm_start = 1;
};

// Point-to-point transport between the ranks that own consecutive layer
// blocks (NCCL over NVLink in production; an in-process loopback in tests).
class Transport {
 public:
  virtual ~Transport() = default;
  virtual int rank() const = 0;
  virtual int size() const = 0;
  virtual void send(const float* buf, size_t n, int peer, cudaStream_t s) = 0;
  virtual void recv(float* buf, size_t n, int peer, cudaStream_t s) = 0;
  // gathers `n` doubles from every rank into out[rank*n .. ]
  virtual void allgather(const double* in, double* out, size_t n, cudaStream_t s) = 0;
  // root's buf -> every rank's buf (n floats)
  virtual void bcast(float* buf, size_t n, int root, cudaStream_t s) = 0;
  virtual void group_start() {}
  virtual void group_end() {}
  // 1 NCCL, 2 loopback; and the rank count the backend itself reports
  // (ncclCommCount for NCCL) -- bench.py records it next to n_gpus
  virtual int backend() const = 0;
  virtual int backend_nranks() const { return size(); }
};

// out[i] = scale * gaussian(seed, a, b, i), multithreaded, bit-identical to rng.hpp
void rng_gaussian_fill(uint64_t seed, uint64_t a, uint64_t b, double scale, double* out,
                       long long n);

class Engine {
 public:
  // tr == nullptr (or a 1-rank transport): single GPU. Otherwise this engine
  // owns rank tr->rank()'s block of coarse intervals.
  Engine(const StackDesc& sd, const SolveCfg& cfg, int device, std::shared_ptr<Transport> tr);
  int rank() const { return rank_; }
  int world() const { return world_; }
  Transport* transport() const { return tr_.get(); }
  // owned interior layer range [lo, hi) (interior indices)
  void owned_layers(int* lo, int* hi) const {
    *lo = fwd_.p_lo.empty() ? 0 : fwd_.p_lo[0];
    *hi = fwd_.p_hi.empty() ? N_ : fwd_.p_hi[0];
  }
  ~Engine();

  // ---- LayerStack surface ----
  long long num_params() const { return n_params_flat_; }
  int total_layers() const { return total_; }
  int interior_begin() const { return ib_; }
  int interior_end() const { return ie_; }
  double step_size(int layer) const { return h_[layer]; }
  void init_params(uint64_t seed, std::vector<double>* flat_out);
  void set_params(const double* flat);
  void get_params(double* flat) const;
  void get_grads(double* flat_accum) const;  // flat += device grads
  // flat (covering layers [lo, hi) only, visit_params order) += their grads
  void get_grads_range(int lo, int hi, double* flat_accum) const;
  // pinned double-buffered staging of the gradient download (get_grads_range)
  mutable float* grad_pin_ = nullptr;
  mutable long long grad_pin_layers_ = 0;
  long long flat_offset(int layer) const;  // first flat index of `layer`
  void zero_grads();
  // device parameter / gradient slabs (fp32, layer-major, kernel layout) and
  // the host mapping between that layout and the flat visit_params order
  // (blocks.cpp:627-646): the trainer's optimizer runs over whole slabs
  float* params_dev() const { return P_; }
  float* grads_dev() const { return Gr_; }
  long long slab_elems() const { return (long long)total_ * layer_stride_; }
  void flat_to_slab(const double* flat, double* slab) const;  // slab zero-filled first
  void slab_to_flat(const double* slab, double* flat) const;
  // after P_ changed on the device: re-derive the pre-split GEMM weights
  void params_updated();
  long long y_offset() const { return y_off_; }
  int batch() const { return B_; }

  // ---- frozen dropout masks (blocks.cpp:576-599) ----
  // refresh: the masks of batch `batch_index` (per layer and site, generated
  // on the fly from the reference's counter streams); clear: no masks (the
  // exact map, as for evaluation). No-ops when the stack's dropout is 0.
  void refresh_dropout(uint64_t seed, uint64_t batch_index);
  void clear_dropout();
  // explicit masks (a reference LayerStack's masks(), blocks.cpp:576-599):
  // keep bytes [total][3 sites][max(Tx, Ty) * d], site 2 on decoder layers only
  void set_dropout_masks(const unsigned char* keep_host);
  bool dropout_active() const { return drop_on_; }

  // ---- shape ----
  // eval-only engines (the Lipschitz probe) skip the per-layer activation
  // caches and trajectory storage: they only run residual_device
  void set_eval_only(bool on) {
    eval_only_ = on;
    if (on) Gmax_ = 2;  // families of at most two evaluations (x, x + delta)
  }
  void set_shape(int batch, int s_x, int s_y);
  long long state_elems() const { return state_n_; }
  int width() const { return sd_.d; }
  SolveCtrl* ctrl(bool fwd) const { return fwd ? fwd_.ctrl : bwd_.ctrl; }

  // ---- LayerParallelEngine surface ----
  SolveCfg& config() { return cfg_; }
  const SolveCfg& config() const { return cfg_; }
  void forward_device(const float* z0_dev);
  void backward_device(const float* lamN_dev, float* lam0_dev, bool want_grads,
                       bool traj_is_current);
  void read_trace(bool fwd, std::vector<double>* trace, bool* converged);
  // WarmSnapshot (adjoint.hpp:187-206): one slot per engine; snapshot()
  // returns its id, restore(id) refuses an id that has been overwritten
  long long snapshot();
  void restore(long long id = -1);
  void reset() { first_fwd_ = first_bwd_ = true; }
  void invalidate_linearization() { std::fill(cache_valid_.begin(), cache_valid_.end(), 0); }
  // The forward solver's level-0 states ARE the trajectory window
  // traj[ib..ie] (no copy per solve). Anything else that writes traj_ -- a
  // serial sweep, evaluation, an uploaded trajectory -- first calls this: the
  // warm window moves to a stash and the next forward solve brings it back,
  // so the solver's warm start never sees another trajectory (the reference
  // keeps serial_forward's output apart from the engine's solver states,
  // blocks.cpp:659-666, adjoint.hpp:113-137).
  void displace_forward_window();
  // the forward solver's warm states := the current device trajectory (e.g.
  // the serial sweep's): seeds the next warm-guess solve with it (the
  // fixed-point self-test of SURVEY 8(c))
  void seed_forward_from_traj();
  // fp16-split range flag: throws ContractViolation (and clears the flag) if
  // a GEMM operand or pre-split producer saw |x| >= 65520 since the last
  // check. Synchronises the engine stream; host-facing entry points call it.
  void check_range();
  int* range_flag() const { return range_flag_; }

  // ---- gradient-bias monitor on the device (controller.hpp:63-155) ----
  // attach: the solves' iteration budgets move into device memory
  // (MonitorDev::budget) and every solve runs the device budget; record()
  // evaluates last_pair_factor + decide + the budget / switch update as one
  // kernel from the traces the solves left on the device -- no host round
  // trip, no allocation, capturable. The host keeps an upper bound of the
  // device budget to size its cycle loop (exact after monitor_read(), which
  // synchronises and copies the small summary; surplus cycles are no-ops).
  void monitor_attach(double threshold, int policy_switch, int cap);
  bool monitor_on() const { return mon_ != nullptr; }
  void monitor_probe(bool begin);        // ProbeScope on the device budgets
  void monitor_record(long long batch);  // batch < 0: refresh the summary only
  const MonitorSummary& monitor_read();  // synchronises; host budgets := device budgets
  int monitor_reports(long long* batch, double* ff, double* bf, int* dec, int cap);
  void set_budget(int fwd_iters, int bwd_iters);  // host-side budget change -> device
  // graph capture with a monitor: the host issues `n` cycles per solve and
  // the device budget gates them (0: the host bound)
  void set_capture_cycles(int n) { capture_cycles_ = n; }

  // CUDA graph of one full training-step solve (forward_device +
  // backward_device on fixed device buffers). Every host decision of the
  // step is shape/config-static and the solve's stopping rule lives on the
  // device (SolveCtrl), so the whole step is capturable; replay = one launch.
  void capture_step(const float* z0_dev, const float* lamN_dev, float* lam0_dev, bool want_grads);
  void replay_step();
  void drop_graph();
  bool has_graph() const { return graph_exec_ != nullptr; }

  // F(z_g) of one layer for a family of G input states (LayerStack::residual,
  // blocks.cpp:466-514, without the step or any solver combine): the map the
  // Lipschitz probe differentiates (lipschitz.cpp:120-129)
  void residual_device(int layer, const float* z, int G, float* F);
  const StackDesc& stack_desc() const { return sd_; }
  int n_split() const { return n_split_; }

  // serial reference sweeps on device (blocks.cpp:659-682)
  void serial_forward_device(const float* z0_dev);
  void serial_adjoint_device(const float* lamN_dev, float* lam0_dev, bool want_grads);

  // device-resident trajectory, slot i = time point i (total+1 slots)
  float* traj_dev() const { return traj_; }
  // lambda at every time point of the last serial adjoint, SCALED by 2^k
  // (lam_scale_dev()->up); lam_unscale() returns 2^-k (synchronises)
  float* lam_all_dev() const { return lam_all_; }
  const LamScale* lam_scale_dev() const { return lam_sc_; }
  double lam_unscale() const;
  cudaStream_t stream() const { return stream_; }
  int device() const { return device_; }
  // number of hot-path kernel launches issued since the last reset_launch_count()
  long long launch_count() const { return launches_; }
  void reset_launch_count() { launches_ = 0; }

  // per-kernel-class device timing (CUDA events around every launch of the
  // class on the engine stream); used by bench.py for the roofline, never in
  // the timed region.
  enum ProfClass { PROF_GEMM = 0, PROF_ATTN = 1, PROF_ROW = 2, PROF_NCLASS = 3 };
  void set_profiling(bool on);
  void read_profile(double* ms, double* flops, double* bytes, long long* launches);
  // one row per profiled launch: class, M, N, K, batch, flops, ms
  int dump_profile(double* out, int max_rows);
  // test hooks: one Phi / Phi^T application on the device
  void step_device(int layer, double dt, const float* z, float* out);
  void adjoint_step_device(int layer, double dt, const float* z, const float* lam, float* out,
                           bool want_grads, double gscale);

 private:
  // ----- parameter layout -----
  struct Piece {
    long long flat_off, dev_off, n;
  };
  struct LayerLayout {
    bool decoder = false;
    // device offsets (floats) within one layer's slab
    long long ln1_g, ln1_b, w_qkv, b_qkv, w_o, b_o, ln2_g, ln2_b, w_in, b_in, w_out, b_out;
    long long ln3_g, ln3_b, w_cq, b_cq, w_ckv, b_ckv, w_co, b_co;
    long long size = 0;
    std::vector<Piece> pieces;  // flat (visit_params) <-> device
    long long flat_size = 0;
    // weight matrices in the pre-split hi|lo' form of the tensor-core GEMM
    // (gemm_tc.cu): W [rows][cols] as a K-major B operand (forward, K = cols)
    // and W^T (dgrad, K = rows), offsets within one layer of Whl_
    struct WPack {
      long long p_off;
      int rows, cols;
      long long n_off, t_off;
    };
    std::vector<WPack> wpack;
    long long hl_size = 0;
  };
  void build_layouts();

  // ----- activation arena layout (per slot) -----
  struct ActLayout {
    long long n1, qkv, ctx, P, a1, u, n2, h, g, st1, st2;              // encoder / self
    long long n3, u3, cq, ckv, cctx, cP, ybar, st3;                    // decoder cross
    long long size = 0;
  };
  struct BwdLayout {
    long long dh, dn2, du, da1, dctx, dqkv, dn1, dP;                   // encoder / self
    long long dybar, dy, dcctx, dcq, dckv, dn3, dxe, dP2;              // decoder
    long long upm = 0, dcpre = 0;  // dropout: masked upstream of the MLP / cross-attention branch
    long long size = 0;
  };

  // a reference to G activation slots (cache: slot = layer; scratch: slot = g)
  struct ActRef {
    float* base;
    long long stride;
    int slot0, step;
  };

  // ----- Phi / Phi^T evaluation families -----
  struct EvalSpec {
    int G = 1;
    int layer0 = 0, layer_step = 1;  // absolute layer of member g
    float dt = 0.f;
    Mat in;      // input states (full State rows)
    ActRef act;  // where forward activations go / come from
    Combine cmb; // z/out/base/phib/rho/v are full-State families; mode
    bool want_grads = false;
    float gscale = 0.f;
    Mat lam;     // adjoint: upstream state family
    // adjoint: where the dgrad-chain intermediates (dh, dn2, da1, dqkv, dn1,
    // ...) live -- null = backward scratch (slot g); the per-layer backward
    // cache (slot = layer) when captured for the parameter pass
    ActRef bact{nullptr, 0, 0, 1};
    bool wgrad_only = false;  // intermediates already in bact: only form dW, db
    bool keep_act = false;    // scratch activations are read by a following adjoint
    bool residual_only = false;  // out = F(z) (the combine starts from a zero state)
    const float* gscale_mul = nullptr;  // device factor of gscale (LamScale::down)
  };
  void check_family_writes(const EvalSpec& e, bool adjoint) const;
  void eval_forward(const EvalSpec& e);
  void eval_adjoint(const EvalSpec& e);
  void encoder_forward(const EvalSpec& e, int Rx, bool causal, Mat xin, Mat yin_passive);
  void decoder_forward(const EvalSpec& e);
  void encoder_adjoint(const EvalSpec& e, bool causal);
  void decoder_adjoint(const EvalSpec& e);
  void gemm(GemmArgs g);
  // attention of a family as tcgen05 GEMMs per (batch, head):
  // S = Q.K^T, P = softmax(S/sqrt(dh)), O = P.V (blocks.cpp:142-170) and the
  // VJP (blocks.cpp:172-236). Q/K/V/O are token-major [tokens][ld] column
  // slices (head h at columns h*dh); P is [B][H][sq][skv] per member.
  // Ohl (optional): also write O pre-split for the O-projection (returns
  // whether it did; O itself is then skipped unless keep_p)
  // qkv_hs: Q, K, V were written head-split pre-split (attn_hs) by their GEMMs
  bool attention_fwd(int G, Mat Q, Mat K, Mat V, Mat O, Mat P, int sq, int skv, bool causal,
                     bool keep_p, Mat Ohl = Mat{}, bool qkv_hs = false);
  // the attention operands of an (sq, skv) problem travel head-split
  // pre-split (AttnArgs::qkv_hs / do_hs): the QKV (cross Q / KV) GEMMs and the
  // O-projection dgrad write them so for the fused s <= 128 kernels, dh = 64.
  // A function of the shape only (forward and backward agree);
  // MGLP_NO_ATTN_HS=1 keeps them fp32.
  // grad: the dO operand of the backward (fused s <= 128 kernels only)
  bool attn_hs(int sq, int skv, bool grad = false) const;
  // the family's pre-split activation buffer `which` (0: [rows][d] LN outputs,
  // 1: [rows][cols <= max(d, ffn)] attention O / GELU output; hi|lo' rows, the
  // next forward GEMM's A operand); empty when unavailable
  Mat hl_mat(int G, int which, int cols) const;
  bool p_hl_ok(int sq, int skv, const Mat& P) const;
  Mat dgrad_hl(int G, int which, int cols) const;
  // kept linearisations store their LN and GELU outputs (n1, n2, n3, g)
  // pre-split only (the forward GEMMs and the weight gradients read them so)
  bool cache_hl() const {
#ifdef MGLP_GEMM_SIMT
    return false;  // the SIMT GEMMs read fp32 operands only
#else
    return hlscr_ != nullptr && !cache_hl_off();
#endif
  }
  static bool cache_hl_off();  // MGLP_NO_CACHE_HL=1: cache fp32 + transient pre-split copies
  Mat pack_upstream(int G, int rows, const Mat& up);
  // the activations of this evaluation are the linearization the adjoint
  // reads (cache), not per-evaluation scratch
  bool keep_lin(const EvalSpec& e) const { return e.act.base != scratch_ || e.keep_act; }
  // dQhl/dKhl/dVhl (optional): also write the gradients pre-split for the
  // QKV dgrad (returns whether it did; the fp32 ones are then skipped unless
  // keep32)
  bool attention_bwd(int G, Mat Q, Mat K, Mat V, Mat P, Mat O, Mat dO, Mat dP, Mat dQ, Mat dK, Mat dV,
                     int sq, int skv, bool causal, Mat dQhl = Mat{}, Mat dKhl = Mat{},
                     Mat dVhl = Mat{}, bool keep32 = true, bool qkv_hs = false,
                     bool do_hs = false);
  int gemm_blocks(const GemmArgs& g) const;
  Mat act_mat(const ActRef& r, long long off, int ld) const;
  Mat bwd_mat(const EvalSpec& e, long long off, int ld) const;
  Mat par(long long off, int ld, int layer0, int step) const;
  // pre-split weight W at P_ offset `off` of layout L as the GEMM B operand:
  // forward (B = W, K = in) or, transposed, dgrad (B = W^T, K = out)
  Mat par_hl(const LayerLayout& L, long long off, int layer0, int step, bool transposed) const;
  void repack_weights();
  Mat grad(long long off, int ld, int layer0, int step) const;

  // ----- MGRIT solver (mgrit.hpp) -----
  struct Level {
    int n = 0;
    float* v = nullptr;   // n+1 states
    float* rho = nullptr; // n+1 (level > 0)
    float* phib = nullptr;
    // base of level l aliases v of level l-1 at stride c_f
  };
  struct Solver {
    bool adjoint = false;
    int tpos = 0;                 // this rank's position in the solver's time order
    std::vector<Level> lv;
    std::vector<int> p_lo, p_hi;  // per level: owned points (p_lo, p_hi]; p_lo is a ghost
    SolveCtrl* ctrl = nullptr;
    double* partials = nullptr;   // [n_chunks][slots_per_chunk] residual-norm partials
    double* gathered = nullptr;   // all ranks' partials (world > 1)
    int n_chunks = 0, slots_per_chunk = 0;
  };
  int rank_at(const Solver& s, int tpos) const;
  void exchange_ghost(Solver& s, int level);
  bool owns_layer(int l) const;
  Mat lv_v(const Solver& s, int l, int slot0, int step) const;
  Mat lv_base(const Solver& s, int l, int slot0, int step) const;
  Mat lv_rho(const Solver& s, int l, int slot0, int step) const;
  Mat lv_phib(const Solver& s, int l, int slot0, int step) const;
  void sys_eval(Solver& s, int level, int k0, int kstep, int G, Mat in, Combine cmb,
                bool capture);
  void relax_family(Solver& s, int level, int j0, int jstep, int G, bool capture);
  void f_relax(Solver& s, int level, bool capture);
  void c_relax(Solver& s, int level);
  void residual_c_rows(Solver& s, int level, bool capture);
  void restrict_to(Solver& s, int level);
  void correct_from(Solver& s, int level);
  void exact_solve(Solver& s, int level);
  void descend(Solver& s, int level);
  void v_cycle(Solver& s, double tol, bool first);
  void solve(Solver& s, int iters, double tol);
  void alloc_solver(Solver& s, bool adjoint);
  void free_solver(Solver& s);
  void ensure_linearization();

  // ----- members -----
  StackDesc sd_;
  SolveCfg cfg_;
  bool eval_only_ = false;
  unsigned char* drop_masks_ = nullptr;  // device [total][3][drop_slot_] keep bytes
  long long drop_slot_ = 0;
  bool drop_on_ = false;
  DropMask dmask(int site, int layer0, int layer_step) const;
  int device_ = 0;
  std::shared_ptr<Transport> tr_;
  cudaStream_t stream_ = nullptr;
  int total_ = 0, n_split_ = 0, ib_ = 0, ie_ = 0, N_ = 0;
  bool causal_ = false;
  std::vector<double> h_;
  std::vector<LayerLayout> lay_;  // [0]=encoder kind, [1]=decoder kind
  long long layer_stride_ = 0;
  long long n_params_flat_ = 0;
  float* P_ = nullptr;     // fp32 params
  float* Whl_ = nullptr;   // pre-split weights (LayerLayout::wpack), hl_stride_ floats per layer
  long long hl_stride_ = 0;
  int* range_flag_ = nullptr;  // device: a GEMM operand overflowed fp16 (gemm_tc.cu)
  LamScale* lam_sc_ = nullptr;  // device: the adjoint's exact 2^k scaling of lambda_N
  LamScale* snap_sc_ = nullptr;
  double* lam_gather_ = nullptr;
  MonitorDev* mon_ = nullptr;
  MonitorSummary* mon_host_ = nullptr;  // pinned mirror
  MonitorSummary* mon_sum_ = nullptr;   // device summary
  int bound_[2] = {0, 0};               // host upper bound of the device budgets
  int capture_cycles_ = 0;
  int bound_saved_[2] = {0, 0};
  int mon_cap_ = 1;
  int host_cycles(int which) const;  // [2 * world] per-rank maxima (multi-rank warm scaling)  // the scaling stored with the snapshot's adjoint states
  float* Gr_ = nullptr;    // fp32 grads
  // shape
  int B_ = 0, sx_ = 0, sy_ = 0, Tx_ = 0, Ty_ = 0;
  long long state_n_ = 0, x_off_ = 0, y_off_ = 0;
  ActLayout al_;
  BwdLayout bl_;
  int Gmax_ = 1;
  float* scratch_ = nullptr;  // Gmax forward activation slots
  // pre-split forward GEMM A operands (LN outputs, attention O, GELU output):
  // two buffers per member ([max(Tx,Ty)][d] and [max(Tx,Ty)][max(d,ffn)]),
  // alternating stage by stage so a GEMM never writes the buffer it reads
  float* hlscr_ = nullptr;
  long long hl_slot_ = 0;
  int hl_cap_ = 0;
  int hl_w1_ = 0;  // row width (floats) of buffer 1
  float* cache_ = nullptr;    // total_ forward activation slots (slot = layer)
  float* bscratch_ = nullptr; // Gmax backward slots
  double* colred_part_ = nullptr;  // f64 column-sum partials (rowops.cu colred)
  long long colred_cap_ = 0;
  float* bcache_ = nullptr;   // total_ backward slots (slot = layer), for the parameter pass
  std::vector<char> bcache_valid_;
  float* traj_ = nullptr;     // total_+1 states
  float* lam_all_ = nullptr;  // total_+1 states (serial adjoint)
  float* zero_state_ = nullptr;
  Solver fwd_, bwd_;
  std::vector<char> cache_valid_;
  bool first_fwd_ = true, first_bwd_ = true;
  // snapshot
  float* snap_fwd_ = nullptr;
  float* snap_bwd_ = nullptr;
  long long snap_id_ = 0;       // id of the snapshot in the slot (0: none)
  bool snap_empty_ = false;     // taken before any shape / solve: flags only
  long long snap_seq_ = 0;
  float* fwd_stash_ = nullptr;  // displaced forward warm window (N+1 states)
  bool fwd_displaced_ = false;
  bool snap_first_fwd_ = true, snap_first_bwd_ = true;
  long long launches_ = 0;
  cudaGraphExec_t graph_exec_ = nullptr;
  long long graph_launches_ = 0;  // hot-path kernels inside the captured step
  const int* active_ = nullptr;  // current solve-control flag
  int part_off_ln_ = 0, part_off_elem_ = 0;  // partial-slot offsets within an interval
  int rank_ = 0, world_ = 1;
  // ----- per-rank memory -----
  // slot ranges [a, b) this rank reads or writes: on a P-rank engine the
  // per-layer and per-time-point buffers keep their global indexing, but
  // physical HBM is mapped only under these slots (vmm.cu); 1 rank: all
  using Ranges = std::vector<std::pair<long long, long long>>;
  Ranges lay_r_;   // layers: parameters, gradients, pre-split weights, activation caches
  Ranges traj_r_;  // trajectory time points (the forward level-0 window + buffers)
  Ranges lam_r_;   // the buffer layers' adjoint points
  Ranges win_r_;   // the forward level-0 window [0, N] (traj_r_ - ib)
  Ranges bwd0_r_;  // the adjoint level-0 window [0, N]
  std::vector<Ranges> lvl_r_[2];  // coarse levels l >= 1 of the forward / adjoint solver
  size_t hbm_bytes_ = 0;          // device memory this engine holds (mapped)
  void build_ranges();
  float* dalloc(long long slot_elems, long long nslots, const Ranges& r);
  void dfree(float*& p);
  void dmemset(float* p, long long slot_elems, const Ranges& r);
  void dcopy(float* dst, const float* src, long long slot_elems, const Ranges& r,
             long long first = 0);
  static Ranges clip(const Ranges& r, long long lo, long long hi);

 public:
  size_t hbm_bytes() const { return hbm_bytes_; }
  bool owns_layer_slot(int l) const;
  // every time point of [first, first + count) is held by this rank
  bool holds_points(int first, int count) const;

 private:
  struct ProfRec {
    cudaEvent_t a, b;
    int cls;
    double flops, bytes;
    std::vector<int> shape;
  };
  std::vector<int> prof_shape_{0, 0, 0, 0};
  bool profiling_ = false;
  std::vector<ProfRec> prof_;
  std::vector<cudaEvent_t> ev_pool_;
  size_t ev_used_ = 0;
  cudaEvent_t prof_event();
  template <class F>
  void timed(int cls, double flops, double bytes, F&& launch) {
    if (!profiling_) {
      launch();
      return;
    }
    ProfRec r{prof_event(), prof_event(), cls, flops, bytes, prof_shape_};
    prof_shape_ = {0, 0, 0, 0, -1};
    cudaEventRecord(r.a, stream_);
    launch();
    cudaEventRecord(r.b, stream_);
    prof_.push_back(r);
  }
};

// Lipschitz probe (probe.cu; lipschitz.cpp:53-149): per requested layer the
// max over `samples` draws of ||F(x + delta) - F(x)|| / ||delta||.
void lipschitz_probe(const Engine& src, int samples, double delta_scale, double input_scale,
                     int seq_len, uint64_t seed, const std::vector<int>& layers,
                     std::vector<double>* est);

}  // namespace mglp
