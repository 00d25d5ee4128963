// Factories for the rank-to-rank transports (see transport.cu).
#pragma once

#include <memory>

#include "engine.h"

namespace mglp {

struct NcclUniqueId {
  char internal[128];
};

void nccl_unique_id(NcclUniqueId* id);
std::shared_ptr<Transport> make_nccl_transport(int rank, int world, const NcclUniqueId& id,
                                               int device);

class LoopbackHub;
std::shared_ptr<LoopbackHub> make_loopback_hub(int world);
std::shared_ptr<Transport> make_loopback_transport(std::shared_ptr<LoopbackHub> hub, int rank);

}  // namespace mglp
