// Transports between the ranks that own consecutive layer blocks.
//
//  * NcclTransport: one process per GPU, NCCL point-to-point over NVLink /
//    NVSwitch (ncclSend/ncclRecv in a group for the ghost exchange,
//    ncclAllGather for the residual-norm partials, ncclBroadcast for the
//    adjoint initial condition). libnccl.so.2 is dlopen'ed on first use (the
//    one torch already loaded, when present), so single-GPU use of the
//    library has no NCCL dependency.
//  * LoopbackTransport: P "virtual ranks" as P engines on one device, one
//    host thread each, exchanging through device buffers with CUDA events --
//    exercises the exact partitioned control flow of the multi-GPU solve on a
//    single GPU (tests/test_dist.py).
#include <dlfcn.h>

#include <condition_variable>
#include <deque>
#include <map>
#include <mutex>

#include "transport.h"

namespace mglp {

// ---- NCCL (subset of nccl.h, ABI-stable since 2.x) ----------------------------
namespace {
typedef struct ncclComm* ncclComm_t;
typedef int ncclResult_t;
enum { kNcclFloat32 = 7, kNcclFloat64 = 8 };

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(NcclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, NcclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, int, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommCount)(ncclComm_t, int*) = nullptr;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* n : names) {
      api.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (!api.h) return;
    auto sym = [](const char* s) { return dlsym(api.h, s); };
    api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
    api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
    api.Send = (decltype(api.Send))sym("ncclSend");
    api.Recv = (decltype(api.Recv))sym("ncclRecv");
    api.AllGather = (decltype(api.AllGather))sym("ncclAllGather");
    api.Broadcast = (decltype(api.Broadcast))sym("ncclBroadcast");
    api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
    api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
    api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
    api.CommCount = (decltype(api.CommCount))sym("ncclCommCount");
  });
  if (!api.h || !api.CommInitRank || !api.Send || !api.Recv || !api.AllGather)
    throw ContractViolation("NCCL (libnccl.so.2) could not be loaded for a multi-GPU engine");
  return api;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r != 0) {
    const char* msg = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
    throw ContractViolation(std::string("NCCL ") + what + ": " + msg);
  }
}

class NcclTransport final : public Transport {
 public:
  NcclTransport(int rank, int world, const NcclUniqueId& id, int device)
      : rank_(rank), world_(world) {
    MGLP_CUDA(cudaSetDevice(device));
    nccl_check(nccl().CommInitRank(&comm_, world, id, rank), "CommInitRank");
  }
  ~NcclTransport() override {
    if (comm_) nccl().CommDestroy(comm_);
  }
  int rank() const override { return rank_; }
  int size() const override { return world_; }
  void send(const float* buf, size_t n, int peer, cudaStream_t s) override {
    nccl_check(nccl().Send(buf, n, kNcclFloat32, peer, comm_, s), "Send");
  }
  void recv(float* buf, size_t n, int peer, cudaStream_t s) override {
    nccl_check(nccl().Recv(buf, n, kNcclFloat32, peer, comm_, s), "Recv");
  }
  void allgather(const double* in, double* out, size_t n, cudaStream_t s) override {
    nccl_check(nccl().AllGather(in, out, n, kNcclFloat64, comm_, s), "AllGather");
  }
  void bcast(float* buf, size_t n, int root, cudaStream_t s) override {
    nccl_check(nccl().Broadcast(buf, buf, n, kNcclFloat32, root, comm_, s), "Broadcast");
  }
  void group_start() override { nccl_check(nccl().GroupStart(), "GroupStart"); }
  void group_end() override { nccl_check(nccl().GroupEnd(), "GroupEnd"); }
  int backend() const override { return 1; }
  int backend_nranks() const override {
    int n = -1;
    if (nccl().CommCount) nccl_check(nccl().CommCount(comm_, &n), "CommCount");
    return n;
  }

 private:
  int rank_, world_;
  ncclComm_t comm_ = nullptr;
};

// ---- in-process loopback ---------------------------------------------------------
struct Msg {
  void* staging;
  cudaEvent_t ready;
};

class LoopbackTransport;

}  // namespace

class LoopbackHub {
 public:
  explicit LoopbackHub(int world) : world_(world) {}
  int world() const { return world_; }
  void post(int src, int dst, const void* buf, size_t bytes, cudaStream_t s) {
    Msg m;
    MGLP_CUDA(cudaMallocAsync(&m.staging, bytes, s));
    MGLP_CUDA(cudaMemcpyAsync(m.staging, buf, bytes, cudaMemcpyDeviceToDevice, s));
    MGLP_CUDA(cudaEventCreateWithFlags(&m.ready, cudaEventDisableTiming));
    MGLP_CUDA(cudaEventRecord(m.ready, s));
    {
      std::lock_guard<std::mutex> lk(mu_);
      box_[{src, dst}].push_back(m);
    }
    cv_.notify_all();
  }
  void take(int src, int dst, void* buf, size_t bytes, cudaStream_t s) {
    Msg m;
    {
      std::unique_lock<std::mutex> lk(mu_);
      auto& q = box_[{src, dst}];
      cv_.wait(lk, [&] { return !q.empty(); });
      m = q.front();
      q.pop_front();
    }
    MGLP_CUDA(cudaStreamWaitEvent(s, m.ready, 0));
    MGLP_CUDA(cudaMemcpyAsync(buf, m.staging, bytes, cudaMemcpyDeviceToDevice, s));
    MGLP_CUDA(cudaFreeAsync(m.staging, s));
    MGLP_CUDA(cudaEventDestroy(m.ready));
  }

 private:
  int world_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::map<std::pair<int, int>, std::deque<Msg>> box_;
};

namespace {
class LoopbackTransport final : public Transport {
 public:
  LoopbackTransport(std::shared_ptr<LoopbackHub> hub, int rank) : hub_(std::move(hub)), rank_(rank) {}
  int rank() const override { return rank_; }
  int size() const override { return hub_->world(); }
  int backend() const override { return 2; }
  void send(const float* buf, size_t n, int peer, cudaStream_t s) override {
    hub_->post(rank_, peer, buf, n * sizeof(float), s);
  }
  void recv(float* buf, size_t n, int peer, cudaStream_t s) override {
    hub_->take(peer, rank_, buf, n * sizeof(float), s);
  }
  void allgather(const double* in, double* out, size_t n, cudaStream_t s) override {
    const int P = size();
    for (int r = 0; r < P; ++r)
      if (r != rank_) hub_->post(rank_, r, in, n * sizeof(double), s);
    MGLP_CUDA(cudaMemcpyAsync(out + (size_t)rank_ * n, in, n * sizeof(double),
                              cudaMemcpyDeviceToDevice, s));
    for (int r = 0; r < P; ++r)
      if (r != rank_) hub_->take(r, rank_, out + (size_t)r * n, n * sizeof(double), s);
  }
  void bcast(float* buf, size_t n, int root, cudaStream_t s) override {
    if (rank_ == root) {
      for (int r = 0; r < size(); ++r)
        if (r != root) hub_->post(root, r, buf, n * sizeof(float), s);
    } else {
      hub_->take(root, rank_, buf, n * sizeof(float), s);
    }
  }

 private:
  std::shared_ptr<LoopbackHub> hub_;
  int rank_;
};
}  // namespace

void nccl_unique_id(NcclUniqueId* id) {
  nccl_check(nccl().GetUniqueId(id), "GetUniqueId");
}

std::shared_ptr<Transport> make_nccl_transport(int rank, int world, const NcclUniqueId& id,
                                               int device) {
  return std::make_shared<NcclTransport>(rank, world, id, device);
}

std::shared_ptr<LoopbackHub> make_loopback_hub(int world) {
  return std::make_shared<LoopbackHub>(world);
}

std::shared_ptr<Transport> make_loopback_transport(std::shared_ptr<LoopbackHub> hub, int rank) {
  return std::make_shared<LoopbackTransport>(std::move(hub), rank);
}

}  // namespace mglp
