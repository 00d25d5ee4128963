// Partially backed device buffers (vmm.cu): the whole virtual range is
// reserved, physical memory is mapped only under the byte ranges given
// (rounded out to the allocation granularity).
#pragma once

#include <cstddef>
#include <utility>
#include <vector>

#include "common.cuh"

namespace mglp {

void* partial_alloc(int device, size_t bytes, std::vector<std::pair<size_t, size_t>> ranges,
                    size_t* mapped_bytes);
// false if p was not made by partial_alloc
bool partial_free(void* p);

}  // namespace mglp
