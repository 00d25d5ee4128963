// Partially backed device buffers for the layer-partitioned engine
// (SURVEY 8(e)): a rank of a P-rank engine reserves the whole virtual range
// of a per-layer / per-time-point buffer (so every index computation stays
// the global one) but maps physical HBM only under the slots it owns, with
// the CUDA virtual memory API (cuMemAddressReserve / cuMemCreate / cuMemMap).
// A stray access to another rank's slot is an illegal-address fault, not a
// silent read of stale data, and per-rank memory shrinks with P.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <map>
#include <mutex>

#include "vmm.h"

namespace mglp {

namespace {

struct Api {
  PFN_cuMemAddressReserve_v10020 reserve = nullptr;
  PFN_cuMemAddressFree_v10020 addr_free = nullptr;
  PFN_cuMemCreate_v10020 create = nullptr;
  PFN_cuMemRelease_v10020 release = nullptr;
  PFN_cuMemMap_v10020 map = nullptr;
  PFN_cuMemUnmap_v10020 unmap = nullptr;
  PFN_cuMemSetAccess_v10020 access = nullptr;
  PFN_cuMemGetAllocationGranularity_v10020 gran = nullptr;
};

template <class T>
void sym(const char* name, T* out) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || fn == nullptr)
    throw ContractViolation(std::string("CUDA driver entry point unavailable: ") + name);
  *out = reinterpret_cast<T>(fn);
}

Api& api() {
  static Api a;
  static std::once_flag once;
  std::call_once(once, [] {
    sym("cuMemAddressReserve", &a.reserve);
    sym("cuMemAddressFree", &a.addr_free);
    sym("cuMemCreate", &a.create);
    sym("cuMemRelease", &a.release);
    sym("cuMemMap", &a.map);
    sym("cuMemUnmap", &a.unmap);
    sym("cuMemSetAccess", &a.access);
    sym("cuMemGetAllocationGranularity", &a.gran);
  });
  return a;
}

void drv(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS)
    throw ContractViolation(std::string("CUDA VMM ") + what + " failed (" + std::to_string((int)r) +
                            ")");
}

struct Rec {
  CUdeviceptr va = 0;
  size_t va_size = 0;
  std::vector<std::pair<size_t, size_t>> chunks;  // mapped [offset, size)
  std::vector<CUmemGenericAllocationHandle> handles;
};

std::mutex g_mu;
std::map<void*, Rec> g_recs;

}  // namespace

void* partial_alloc(int device, size_t bytes, std::vector<std::pair<size_t, size_t>> ranges,
                    size_t* mapped_bytes) {
  Api& A = api();
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  size_t g = 0;
  drv(A.gran(&g, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "granularity");
  const size_t va_size = (bytes + g - 1) / g * g;
  Rec r;
  r.va_size = va_size;
  drv(A.reserve(&r.va, va_size, g, 0, 0), "reserve");
  // granularity-aligned, merged chunks covering every requested byte range
  std::vector<std::pair<size_t, size_t>> iv;
  for (const auto& x : ranges) {
    if (x.second <= x.first) continue;
    const size_t a = x.first / g * g;
    const size_t b = std::min(va_size, (x.second + g - 1) / g * g);
    iv.push_back({a, b});
  }
  std::sort(iv.begin(), iv.end());
  std::vector<std::pair<size_t, size_t>> merged;
  for (const auto& x : iv) {
    if (!merged.empty() && x.first <= merged.back().second)
      merged.back().second = std::max(merged.back().second, x.second);
    else
      merged.push_back(x);
  }
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  size_t total = 0;
  try {
    for (const auto& m : merged) {
      const size_t sz = m.second - m.first;
      CUmemGenericAllocationHandle h;
      drv(A.create(&h, sz, &prop, 0), "create");
      r.handles.push_back(h);
      drv(A.map(r.va + m.first, sz, 0, h, 0), "map");
      r.chunks.push_back({m.first, sz});
      drv(A.access(r.va + m.first, sz, &acc, 1), "set access");
      total += sz;
    }
  } catch (...) {
    for (const auto& c : r.chunks) A.unmap(r.va + c.first, c.second);
    for (auto h : r.handles) A.release(h);
    A.addr_free(r.va, r.va_size);
    throw;
  }
  if (mapped_bytes) *mapped_bytes = total;
  void* p = reinterpret_cast<void*>(r.va);
  std::lock_guard<std::mutex> lk(g_mu);
  g_recs[p] = std::move(r);
  return p;
}

bool partial_free(void* p) {
  Rec r;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_recs.find(p);
    if (it == g_recs.end()) return false;
    r = std::move(it->second);
    g_recs.erase(it);
  }
  Api& A = api();
  for (const auto& c : r.chunks) A.unmap(r.va + c.first, c.second);
  for (auto h : r.handles) A.release(h);
  A.addr_free(r.va, r.va_size);
  return true;
}

}  // namespace mglp
