// Device training step around the layer-parallel engine: the reference's
// Trainer::run_update (training.cpp:230-268) with every tensor op on the B200
// -- synthetic batches (tasks.cpp:45-89, integer-exact), embedding
// (model.cpp:133-164), head logits / cross-entropy / head backward
// (model.cpp:166-248), embedding backward (model.cpp:250-275) and the
// optimizer (optimizer.cpp:43-88) -- plus evaluation (training.cpp:296-310)
// and the MGLP v1 checkpoint wire format (checkpoint.cpp:88-180).
//
// Parameters: the optimizer keeps f64 master copies of every parameter (the
// stack in the engine's slab layout, the head in its own slab) together with
// the Adam moments, and writes the fp32 copies the kernels read after each
// step -- the reference's parameters are f64 (tensor.hpp:32-88).
#pragma once

#include <memory>
#include <string>
#include <vector>

#include "engine.h"

namespace mglp {

struct TaskDesc {
  int kind = 0;  // 0 copy_sequence, 1 token_classification, 2 tiny_translation
  int vocab = 16, seq_len = 8, train_size = 256, val_size = 64;
  uint64_t seed = 1;
};

struct OptDesc {
  int kind = 2;  // 0 sgd, 1 adam, 2 adamw (optimizer.hpp:24)
  double lr = 1e-3, beta1 = 0.9, beta2 = 0.999, eps = 1e-8, weight_decay = 0.01,
         momentum = 0.0;
};

struct CheckpointMeta {
  uint32_t version = 0;
  std::string config_echo;
  long long batch = 0;
  bool has_optimizer = false;
};

// one indicator probe batch (training.cpp:244-276), decided on the device
struct ProbeOutcome {
  double loss = 0.0;
  int fwd_iters = 0, bwd_iters = 0;  // the row's budgets
  double fwd_factor = 0.0, bwd_factor = 0.0;
  int decision = 0, switched = 0;
};

class Trainer {
 public:
  Trainer(const StackDesc& sd, const SolveCfg& solve, int vocab, int max_seq, const TaskDesc& task,
          const OptDesc& opt, int batch_size, uint64_t seed, int device);
  ~Trainer();

  Engine& engine() { return *eng_; }

  // one optimizer step's worth of work (run_update): batch k of the train
  // split; parallel = layer-parallel engine, else the serial sweeps; apply =
  // take the optimizer step. Returns the mean cross-entropy loss.
  double update(long long k, bool parallel, bool apply);
  // probe_batch (training.cpp:244-276) with the engine's device monitor
  // (attached first): ProbeScope, the update (the doubled run IS the update
  // with use_probe_gradient, else a measurement-only run behind a warm-state
  // snapshot followed by the nominal update), record() on the device
  ProbeOutcome update_probe(long long k, bool use_probe_gradient);
  // token accuracy on the validation split through the serial forward
  double evaluate();
  // logits of the last update's final state ([B*seq][vocab])
  void read_logits(float* out) const;
  // test hook: the device batch (src, tgt_in, tgt_out), [B*seq] each
  void read_batch(int split, long long start, int* src, int* tin, int* tout);

  // flat parameters / optimizer state in Model::param_tensors order
  long long num_params() const { return n_flat_; }
  void get_params(double* flat) const;
  void set_params(const double* flat);
  void get_grads(double* flat) const;  // gradients of the last update
  long long opt_steps() const { return t_; }
  std::string save_checkpoint(long long batch, const std::string& echo) const;
  CheckpointMeta load_checkpoint(const std::string& blob);
  // tensor shapes in param_tensors order (rank, dims...)
  const std::vector<std::vector<long long>>& shapes() const { return shapes_; }

 private:
  struct HeadLayout {
    long long tok, pos, tok_out, pos_out, lnf_g, lnf_b, w, b, size;
  };
  void init_head(uint64_t seed, std::vector<double>* flat_head);
  void head_to_flat(const double* slab, double* flat) const;
  void flat_to_head(const double* flat, double* slab) const;
  void sync_fp32();  // masters -> fp32 copies (+ repack)
  void make_batch(int split, long long start);
  void embed();
  double head_forward_loss(const float* final_state, bool want_dlogits);
  void head_backward(const float* final_state);
  void embed_backward(const float* lam0);
  void optimizer_step();
  int correct_predictions();

  StackDesc sd_;
  TaskDesc task_;
  OptDesc opt_;
  uint64_t seed_ = 0;  // TrainConfig::seed: model init and dropout streams
  int V_, S_, B_, T_, d_, ldv_;
  bool two_stream_;
  std::unique_ptr<Engine> eng_;
  cudaStream_t s_;
  HeadLayout hl_{};
  long long n_flat_ = 0, n_stack_flat_ = 0, n_head_flat_ = 0;
  std::vector<std::vector<long long>> shapes_;
  // device buffers
  float* H32_ = nullptr;    // head params fp32
  float* HG_ = nullptr;     // head grads fp32
  float* Whl_ = nullptr;    // head.w pre-split: [V][pad32(d)] then w^T [d][pad32(V)]
  double* P64_ = nullptr;   // stack master (engine slab layout)
  double* H64_ = nullptr;   // head master
  double *Pm_ = nullptr, *Pv_ = nullptr, *Hm_ = nullptr, *Hv_ = nullptr;
  int *src_ = nullptr, *tin_ = nullptr, *tout_ = nullptr;
  int *perm_ = nullptr, *offs_ = nullptr, *hits_ = nullptr;
  float *z0_ = nullptr, *lamN_ = nullptr, *lam0_ = nullptr;
  float *n_ = nullptr, *stats_ = nullptr, *logits_ = nullptr, *dl_ = nullptr, *dn_ = nullptr;
  double *row_loss_ = nullptr, *loss_ = nullptr;
  long long t_ = 0;  // optimizer steps taken
};

}  // namespace mglp
