// swap_trainer: runs the reference's own run_training (training.cpp:348-360,
// compiled with the CudaLayerParallelEngine swap) on a configuration given
// on the command line and writes the metrics CSV, the final MGLP v1 state
// and, if the run switched, the handover state -- for tests/test_integration.py
// to compare with the stock engine (oracle/_ref).
//
//   swap_trainer <out_prefix> kind task d heads ffn n_enc n_dec vocab seq
//                train val batch epochs mode cf levels fwd bwd probe thr policy
//                cap use_probe_grad val_every dropout
#include <execinfo.h>
#include <unistd.h>

#include <csignal>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <string>

#include "mglp/training.hpp"

using namespace mglp;

static void on_fault(int sig) {
  void* frames[64];
  const int n = backtrace(frames, 64);
  std::fprintf(stderr, "signal %d\n", sig);
  backtrace_symbols_fd(frames, n, STDERR_FILENO);
  std::_Exit(128 + sig);
}

int main(int argc, char** argv) {
  std::signal(SIGSEGV, on_fault);
  if (argc != 27) {
    std::fprintf(stderr, "usage: see swap_trainer.cpp (%d args)\n", argc);
    return 64;
  }
  int a = 2;
  auto I = [&] { return std::atoi(argv[a++]); };
  auto D = [&] { return std::atof(argv[a++]); };
  const std::string out = argv[1];
  ModelConfig mc;
  mc.stack.kind = static_cast<ModelKind>(I());
  TaskSpec task;
  task.kind = static_cast<TaskKind>(I());
  mc.stack.d = I();
  mc.stack.heads = I();
  mc.stack.ffn = I();
  mc.stack.n_enc = I();
  mc.stack.n_dec = I();
  task.vocab = mc.vocab = I();
  task.seq_len = mc.max_seq = I();
  task.train_size = I();
  task.val_size = I();
  TrainConfig tc;
  tc.batch_size = I();
  tc.epochs = I();
  tc.mode = static_cast<TrainMode>(I());
  tc.solve.coarsen = I();
  tc.solve.levels = I();
  tc.solve.fwd_iters = I();
  tc.solve.bwd_iters = I();
  tc.indicator.probe_period = I();
  tc.indicator.threshold = D();
  tc.indicator.policy = static_cast<IndicatorPolicy>(I());
  tc.indicator.max_iter_cap = I();
  tc.indicator.use_probe_gradient = I() != 0;
  tc.val_every = I();
  mc.stack.dropout = D();
  try {
    const TrainResult r = run_training(task, mc, tc);
    std::ofstream(out + ".csv") << r.csv;
    std::ofstream(out + ".state", std::ios::binary) << r.final_state;
    std::ofstream(out + ".switch", std::ios::binary) << r.switch_state;
    std::printf("switched %d switch_batch %lld rows %zu\n", r.switched ? 1 : 0, r.switch_batch,
                r.rows.size());
  } catch (const ValidationError& e) {
    std::fprintf(stderr, "ValidationError: %s\n", e.what());
    return 1;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 2;
  }
  return 0;
}
