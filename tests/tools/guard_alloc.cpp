// Test infrastructure (not part of the product): a PyTorch pluggable CUDA
// allocator that ends every allocation at a guard page.  Each tensor gets its
// own virtual range: the bytes it needs rounded up to the allocation
// granularity are mapped, the granule after them is reserved but left
// unmapped, and the returned pointer is placed so the tensor's last byte sits
// within 256 bytes of the unmapped granule (the pointer stays 256-byte
// aligned; SSM_GUARD_ALIGN=16 puts it within 16 bytes).  A kernel that reads
// or writes past that slack at the end of any tensor faults at once instead
// of silently touching a neighbour -- a bounds check for a GPU pool without
// compute-sanitizer.  SSM_GUARD_SIDE=front moves the unmapped granule in
// front of the tensor instead (reads before its start fault).  No caching: free
// synchronises the device, then unmaps and releases the range.
//
// Build: g++ -O2 -shared -fPIC tests/tools/guard_alloc.cpp -I$CUDA/include -L$CUDA/lib64/stubs -lcuda
// Use (before the first CUDA allocation):
//   torch.cuda.memory.change_current_allocator(torch.cuda.memory.CUDAPluggableAllocator(
//       path, "guard_malloc", "guard_free"))
#include <cuda.h>

#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

namespace {

struct Range {
  CUdeviceptr va;
  CUdeviceptr va_mapped;
  size_t reserved;
  size_t mapped;
  CUmemGenericAllocationHandle h;
};

std::mutex g_mu;
std::unordered_map<uintptr_t, Range> g_live;

bool ok(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return true;
  const char* s = nullptr;
  cuGetErrorString(r, &s);
  std::fprintf(stderr, "guard_alloc: %s failed: %s\n", what, s ? s : "?");
  return false;
}

}  // namespace

extern "C" void* guard_malloc(ssize_t size, int device, void* /*stream*/) {
  if (size <= 0) size = 1;
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  size_t gran = 0;
  if (!ok(cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM), "granularity"))
    return nullptr;
  const size_t mapped = (static_cast<size_t>(size) + gran - 1) / gran * gran;
  Range r{0, 0, mapped + gran, mapped, 0};
  if (!ok(cuMemAddressReserve(&r.va, r.reserved, 0, 0, 0), "reserve")) return nullptr;
  if (!ok(cuMemCreate(&r.h, mapped, &prop, 0), "create")) {
    cuMemAddressFree(r.va, r.reserved);
    return nullptr;
  }
  // SSM_GUARD_SIDE=front: the unmapped granule precedes the tensor (under-reads fault)
  static const bool front = [] {
    const char* e = std::getenv("SSM_GUARD_SIDE");
    return e && e[0] == 'f';
  }();
  const CUdeviceptr mva = front ? r.va + gran : r.va;
  if (!ok(cuMemMap(mva, mapped, 0, r.h, 0), "map")) {
    cuMemRelease(r.h);
    cuMemAddressFree(r.va, r.reserved);
    return nullptr;
  }
  CUmemAccessDesc acc = {};
  acc.location = prop.location;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if (!ok(cuMemSetAccess(mva, mapped, &acc, 1), "access")) {
    cuMemUnmap(mva, mapped);
    cuMemRelease(r.h);
    cuMemAddressFree(r.va, r.reserved);
    return nullptr;
  }
  r.va_mapped = mva;
  const uintptr_t end = static_cast<uintptr_t>(mva) + mapped;
  static const uintptr_t align = [] {
    const char* e = std::getenv("SSM_GUARD_ALIGN");  // 256 by default; 16 tightens the check
    const long v = e ? std::strtol(e, nullptr, 10) : 256;
    return static_cast<uintptr_t>(v >= 16 && (v & (v - 1)) == 0 ? v : 256);
  }();
  const uintptr_t p = front ? static_cast<uintptr_t>(mva) : (end - static_cast<uintptr_t>(size)) & ~(align - 1);
  std::lock_guard<std::mutex> lk(g_mu);
  g_live[p] = r;
  return reinterpret_cast<void*>(p);
}

extern "C" void guard_free(void* ptr, ssize_t /*size*/, int /*device*/, void* /*stream*/) {
  Range r;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_live.find(reinterpret_cast<uintptr_t>(ptr));
    if (it == g_live.end()) return;
    r = it->second;
    g_live.erase(it);
  }
  cuCtxSynchronize();  // no kernel may still use the range
  cuMemUnmap(r.va_mapped, r.mapped);
  cuMemRelease(r.h);
  cuMemAddressFree(r.va, r.reserved);
}
