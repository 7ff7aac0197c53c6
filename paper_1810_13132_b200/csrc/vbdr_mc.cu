// vbdr_mc.cu -- a device buffer bound to a multicast (NVLS) object on the
// calling process's device, for vbdr_slide_multicast (include/vbdr.h).
//
// On a multi-GPU node the ranks' state buffers are bound to one multicast
// object whose handle is exported to every rank (torch symmetric memory does
// that: paper_1810_13132_b200.NvlsMerge).  vbdr_mc_alloc builds the one-device
// case in-process -- the same driver calls without the export -- so the
// multicast slide can run, and be checked against the oracle, on one GPU: a
// multimem load then reduces over the single member, a multimem store or red
// reaches the single copy.  The driver API is reached through
// cudaGetDriverEntryPoint, so the library does not link libcuda directly.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <map>
#include <mutex>

#include "../../include/vbdr.h"

namespace {

struct Driver {
  CUresult (*getDevice)(CUdevice *) = nullptr;
  CUresult (*mcGetGran)(size_t *, const CUmulticastObjectProp *, CUmulticastGranularity_flags) = nullptr;
  CUresult (*mcCreate)(CUmemGenericAllocationHandle *, const CUmulticastObjectProp *) = nullptr;
  CUresult (*mcAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
  CUresult (*mcBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t,
                        size_t, unsigned long long) = nullptr;
  CUresult (*mcUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
  CUresult (*memGetGran)(size_t *, const CUmemAllocationProp *, CUmemAllocationGranularity_flags) = nullptr;
  CUresult (*memCreate)(CUmemGenericAllocationHandle *, size_t, const CUmemAllocationProp *,
                        unsigned long long) = nullptr;
  CUresult (*memRelease)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*addrReserve)(CUdeviceptr *, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*addrFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*memMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle,
                     unsigned long long) = nullptr;
  CUresult (*memUnmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*setAccess)(CUdeviceptr, size_t, const CUmemAccessDesc *, size_t) = nullptr;
  CUresult (*errName)(CUresult, const char **) = nullptr;
  bool ok = false;
};

template <typename F>
bool entry(const char *name, F *fn) {
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p)
    return false;
  *fn = reinterpret_cast<F>(p);
  return true;
}

const Driver &drv() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    d.ok = entry("cuCtxGetDevice", &d.getDevice) &&
           entry("cuMulticastGetGranularity", &d.mcGetGran) &&
           entry("cuMulticastCreate", &d.mcCreate) && entry("cuMulticastAddDevice", &d.mcAddDevice) &&
           entry("cuMulticastBindMem", &d.mcBindMem) && entry("cuMulticastUnbind", &d.mcUnbind) &&
           entry("cuMemGetAllocationGranularity", &d.memGetGran) &&
           entry("cuMemCreate", &d.memCreate) && entry("cuMemRelease", &d.memRelease) &&
           entry("cuMemAddressReserve", &d.addrReserve) && entry("cuMemAddressFree", &d.addrFree) &&
           entry("cuMemMap", &d.memMap) && entry("cuMemUnmap", &d.memUnmap) &&
           entry("cuMemSetAccess", &d.setAccess) && entry("cuGetErrorName", &d.errName);
  });
  return d;
}

struct McAlloc {
  CUmemGenericAllocationHandle mem = 0, mc = 0;
  CUdeviceptr uc = 0, mcva = 0;
  size_t size = 0;
  CUdevice dev = 0;
};
std::mutex g_mu;
thread_local char g_err[256] = "";

bool step(const Driver &d, CUresult r, const char *what, unsigned ht) {
  if (r == CUDA_SUCCESS) return true;
  const char *name = "?";
  if (d.errName) d.errName(r, &name);
  snprintf(g_err, sizeof g_err, "%s failed: %s (%d), multicast handle types 0x%x", what, name,
           (int)r, ht);
  return false;
}
std::map<uintptr_t, McAlloc> g_allocs;  // by unicast address

void release(const Driver &d, McAlloc &a) {
  if (a.mcva) {
    d.memUnmap(a.mcva, a.size);
    d.addrFree(a.mcva, a.size);
  }
  if (a.uc) {
    d.memUnmap(a.uc, a.size);
    d.addrFree(a.uc, a.size);
  }
  if (a.mc && a.mem) d.mcUnbind(a.mc, a.dev, 0, a.size);
  if (a.mem) d.memRelease(a.mem);
  if (a.mc) d.memRelease(a.mc);
}

}  // namespace

extern "C" {

vbdr_status vbdr_mc_alloc(uint64_t bytes, void **d_uc, void **d_mc, uint64_t *granted) {
  if (!bytes || !d_uc || !d_mc || !granted) return VBDR_EINVAL;
  *d_uc = *d_mc = nullptr;
  *granted = 0;
  const Driver &d = drv();
  if (!d.ok) {
    snprintf(g_err, sizeof g_err, "driver entry points for multicast not found");
    return VBDR_ECUDA;
  }
  cudaFree(nullptr);  // make sure the runtime's primary context is current
  // handle types: none first (one process), then the exportable kinds some
  // drivers require for any multicast object
  const unsigned kinds[] = {0u, (unsigned)CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
                            (unsigned)CU_MEM_HANDLE_TYPE_FABRIC};
  for (unsigned ht : kinds) {
    McAlloc a;
    if (!step(d, d.getDevice(&a.dev), "cuCtxGetDevice", ht)) return VBDR_ECUDA;
    CUmulticastObjectProp mp{};
    mp.numDevices = 1;
    mp.handleTypes = ht;
    mp.size = bytes;
    size_t g1 = 0, g2 = 0;
    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = a.dev;
    prop.requestedHandleTypes = (CUmemAllocationHandleType)ht;
    if (!step(d, d.mcGetGran(&g1, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED), "cuMulticastGetGranularity", ht) ||
        !step(d, d.memGetGran(&g2, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED), "cuMemGetAllocationGranularity", ht))
      continue;
    const size_t gran = g1 > g2 ? g1 : g2;
    a.size = (bytes + gran - 1) / gran * gran;
    mp.size = a.size;
    CUmemAccessDesc acc{};
    acc.location = prop.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    const bool ok =
        step(d, d.mcCreate(&a.mc, &mp), "cuMulticastCreate", ht) &&
        step(d, d.mcAddDevice(a.mc, a.dev), "cuMulticastAddDevice", ht) &&
        step(d, d.memCreate(&a.mem, a.size, &prop, 0), "cuMemCreate", ht) &&
        step(d, d.mcBindMem(a.mc, 0, a.mem, 0, a.size, 0), "cuMulticastBindMem", ht) &&
        step(d, d.addrReserve(&a.uc, a.size, gran, 0, 0), "cuMemAddressReserve", ht) &&
        step(d, d.memMap(a.uc, a.size, 0, a.mem, 0), "cuMemMap (unicast)", ht) &&
        step(d, d.setAccess(a.uc, a.size, &acc, 1), "cuMemSetAccess (unicast)", ht) &&
        step(d, d.addrReserve(&a.mcva, a.size, gran, 0, 0), "cuMemAddressReserve (mc)", ht) &&
        step(d, d.memMap(a.mcva, a.size, 0, a.mc, 0), "cuMemMap (multicast)", ht) &&
        step(d, d.setAccess(a.mcva, a.size, &acc, 1), "cuMemSetAccess (multicast)", ht);
    if (!ok) {
      release(d, a);
      continue;
    }
    *d_uc = reinterpret_cast<void *>(a.uc);
    *d_mc = reinterpret_cast<void *>(a.mcva);
    *granted = a.size;
    std::lock_guard<std::mutex> lk(g_mu);
    g_allocs[(uintptr_t)a.uc] = a;
    g_err[0] = 0;
    return VBDR_OK;
  }
  return VBDR_ECUDA;
}

const char *vbdr_mc_last_error(void) { return g_err; }

vbdr_status vbdr_mc_free(void *d_uc) {
  const Driver &d = drv();
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_allocs.find((uintptr_t)d_uc);
  if (it == g_allocs.end() || !d.ok) return VBDR_EINVAL;
  cudaDeviceSynchronize();
  release(d, it->second);
  g_allocs.erase(it);
  return VBDR_OK;
}

}  // extern "C"
