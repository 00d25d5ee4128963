// swap_engine.hpp -- the maintainer's one-line change, as a build step.
//
// The reference Trainer (proj/src/training.cpp:71-307) holds
//     std::optional<LayerParallelEngine> engine_;
// and calls forward / backward / config / snapshot / restore on it. Swapping
// in the B200 engine is a change of that one type. To show it works on the
// UNMODIFIED source, integration/Makefile compiles training.cpp with
//     -include integration/swap_engine.hpp
// which includes adjoint.hpp first (its include guard then makes the
// translation unit's own #include a no-op), declares CudaLayerParallelEngine,
// and renames the type for the rest of training.cpp.
#pragma once
#include "mglp/adjoint.hpp"
#include "mglp_cuda_engine.hpp"
#define LayerParallelEngine CudaLayerParallelEngine
