// cm_mc.cpp -- NVLink SHARP (NVLS) multicast buffers for the a8 key reduction.
//
// The a8 step is a MIN over ranks of the per-budget keys.  Instead of a separate NCCL all-reduce
// after every call, the fused kernel's reduce step can issue multimem.red.min straight into a
// multicast address (cm_eval_args.best_key_mc): the NVSwitch applies the
// MIN to every participating GPU's replica, so when all ranks' calls are done every rank holds
// the global keys.  This file is the host plumbing: a multicast object (cuMulticastCreate), one
// physical allocation per GPU bound to it, mapped twice -- a unicast view (plain loads, the
// filter read and the final read) and the multicast view (multimem.red).  One process per GPU:
// rank 0 creates the object and exports it as a POSIX file descriptor; the others import it
// (the descriptor travels over a Unix socket, paper_1910_02653_b200/dist.py); every rank adds
// its device, then (after all have) binds and maps.
//
// Driver entry points come through the runtime (cudaGetDriverEntryPoint): no -lcuda link.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "cm.h"

namespace {
thread_local std::string g_mc_err;
cm_status mc_fail(cm_status s, const std::string& msg) {
  g_mc_err = msg;
  return s;
}

template <class F>
F entry(const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(p);
}

struct Driver {
  decltype(&cuMulticastCreate) mc_create = entry<decltype(&cuMulticastCreate)>("cuMulticastCreate");
  decltype(&cuMulticastGetGranularity) mc_gran = entry<decltype(&cuMulticastGetGranularity)>("cuMulticastGetGranularity");
  decltype(&cuMulticastAddDevice) mc_add = entry<decltype(&cuMulticastAddDevice)>("cuMulticastAddDevice");
  decltype(&cuMulticastBindMem) mc_bind = entry<decltype(&cuMulticastBindMem)>("cuMulticastBindMem");
  decltype(&cuMulticastUnbind) mc_unbind = entry<decltype(&cuMulticastUnbind)>("cuMulticastUnbind");
  decltype(&cuMemCreate) mem_create = entry<decltype(&cuMemCreate)>("cuMemCreate");
  decltype(&cuMemGetAllocationGranularity) mem_gran =
      entry<decltype(&cuMemGetAllocationGranularity)>("cuMemGetAllocationGranularity");
  decltype(&cuMemAddressReserve) va_reserve = entry<decltype(&cuMemAddressReserve)>("cuMemAddressReserve");
  decltype(&cuMemAddressFree) va_free = entry<decltype(&cuMemAddressFree)>("cuMemAddressFree");
  decltype(&cuMemMap) map = entry<decltype(&cuMemMap)>("cuMemMap");
  decltype(&cuMemUnmap) unmap = entry<decltype(&cuMemUnmap)>("cuMemUnmap");
  decltype(&cuMemSetAccess) set_access = entry<decltype(&cuMemSetAccess)>("cuMemSetAccess");
  decltype(&cuMemRelease) release = entry<decltype(&cuMemRelease)>("cuMemRelease");
  decltype(&cuMemExportToShareableHandle) export_h =
      entry<decltype(&cuMemExportToShareableHandle)>("cuMemExportToShareableHandle");
  decltype(&cuMemImportFromShareableHandle) import_h =
      entry<decltype(&cuMemImportFromShareableHandle)>("cuMemImportFromShareableHandle");
  decltype(&cuDeviceGet) dev_get = entry<decltype(&cuDeviceGet)>("cuDeviceGet");
  decltype(&cuDeviceGetAttribute) dev_attr = entry<decltype(&cuDeviceGetAttribute)>("cuDeviceGetAttribute");
  bool ok() const {
    return mc_create && mc_gran && mc_add && mc_bind && mc_unbind && mem_create && mem_gran && va_reserve && va_free &&
           map && unmap && set_access && release && export_h && import_h && dev_get && dev_attr;
  }
};
const Driver& drv() {
  static const Driver d;
  return d;
}

cm_status cu_fail(CUresult r, const char* where) {
  return mc_fail(CM_ECUDA, std::string(where) + ": CUresult " + std::to_string((int)r));
}

cm_status current_device(CUdevice* dev, int* ordinal) {
  if (cudaGetDevice(ordinal) != cudaSuccess) return mc_fail(CM_ECUDA, "cudaGetDevice failed");
  cudaFree(nullptr);                                                // make the primary context current
  const CUresult r = drv().dev_get(dev, *ordinal);
  return r == CUDA_SUCCESS ? CM_OK : cu_fail(r, "cuDeviceGet");
}
}  // namespace

struct cm_mc {
  CUmemGenericAllocationHandle mc = 0;   // the multicast object
  CUmemGenericAllocationHandle mem = 0;  // this GPU's physical replica
  CUdeviceptr uc = 0, mcva = 0;          // unicast and multicast views of the replica
  size_t size = 0;                       // bytes, rounded up to the multicast granularity
  int device = -1;
  int handle_type = 0;                   // CUmemAllocationHandleType the object was created with
  bool added = false, bound = false;
};

extern "C" {

const char* cm_mc_last_error(void) { return g_mc_err.c_str(); }

int32_t cm_mc_supported(void) {
  if (!drv().ok()) return 0;
  CUdevice dev;
  int ord;
  if (current_device(&dev, &ord) != CM_OK) return 0;
  int v = 0;
  if (drv().dev_attr(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev) != CUDA_SUCCESS) return 0;
  return v ? 1 : 0;
}

cm_status cm_mc_create(int64_t bytes, int32_t n_devices, cm_mc** out) {
  if (!out || bytes <= 0 || n_devices < 1) return mc_fail(CM_EINVAL, "bad arguments");
  *out = nullptr;
  if (!drv().ok()) return mc_fail(CM_ECUDA, "multicast driver entry points unavailable");
  CUdevice dev;
  int ord;
  cm_status st = current_device(&dev, &ord);
  if (st != CM_OK) return st;
  // size: a multiple of both the multicast and the physical allocation granularity (minimum)
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = ord;
  size_t ag = 0;
  CUresult r = drv().mem_gran(&ag, &ap, CU_MEM_ALLOC_GRANULARITY_MINIMUM);
  if (r != CUDA_SUCCESS) return cu_fail(r, "cuMemGetAllocationGranularity");
  CUmulticastObjectProp prop = {};
  prop.numDevices = (unsigned)n_devices;
  prop.size = (size_t)bytes;
  // a team: exportable as a POSIX fd (the other ranks import it).  A team of one needs no
  // export; it takes the first handle type the driver accepts (measured on the B200 boxes: only
  // FABRIC -- POSIX fd and none give CUDA_ERROR_INVALID_VALUE there)
  const CUmemAllocationHandleType team[] = {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR};
  const CUmemAllocationHandleType solo[] = {CU_MEM_HANDLE_TYPE_FABRIC, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
                                            CU_MEM_HANDLE_TYPE_NONE};
  const int n_ht = n_devices > 1 ? 1 : 3;
  for (int i = 0; i < n_ht; ++i) {
    const CUmemAllocationHandleType ht = n_devices > 1 ? team[i] : solo[i];
    prop.handleTypes = ht;
    size_t mg = 0;
    r = drv().mc_gran(&mg, &prop, CU_MULTICAST_GRANULARITY_MINIMUM);
    if (r != CUDA_SUCCESS) continue;
    size_t g = mg;
    while (g % ag) g += mg;                                         // lcm (both powers of two in practice)
    prop.size = ((size_t)bytes + g - 1) / g * g;
    CUmemGenericAllocationHandle h = 0;
    r = drv().mc_create(&h, &prop);
    if (r == CUDA_SUCCESS) {
      cm_mc* m = new cm_mc;
      m->mc = h;
      m->size = prop.size;
      m->handle_type = (int)ht;
      *out = m;
      return CM_OK;
    }
  }
  return mc_fail(CM_ECUDA, "cuMulticastCreate: CUresult " + std::to_string((int)r) + " for every handle type (size " +
                               std::to_string(prop.size) + ", alloc granularity " + std::to_string(ag) + ")");
}

cm_status cm_mc_export_fd(const cm_mc* m, int32_t* fd) {
  if (!m || !fd) return mc_fail(CM_EINVAL, "bad arguments");
  int h = -1;
  const CUresult r = drv().export_h(&h, m->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
  if (r != CUDA_SUCCESS) return cu_fail(r, "cuMemExportToShareableHandle");
  *fd = h;
  return CM_OK;
}

cm_status cm_mc_import_fd(int32_t fd, int64_t bytes, cm_mc** out) {
  if (!out || fd < 0 || bytes <= 0) return mc_fail(CM_EINVAL, "bad arguments");
  *out = nullptr;
  if (!drv().ok()) return mc_fail(CM_ECUDA, "multicast driver entry points unavailable");
  cm_mc* m = new cm_mc;
  m->size = (size_t)bytes;
  const CUresult r = drv().import_h(&m->mc, reinterpret_cast<void*>((uintptr_t)fd),
                                    CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
  if (r != CUDA_SUCCESS) {
    delete m;
    return cu_fail(r, "cuMemImportFromShareableHandle");
  }
  *out = m;
  return CM_OK;
}

int64_t cm_mc_size(const cm_mc* m) { return m ? (int64_t)m->size : -1; }

int32_t cm_mc_handle_type(const cm_mc* m) { return m ? m->handle_type : -1; }

cm_status cm_mc_add_device(cm_mc* m) {
  if (!m || m->added) return mc_fail(CM_EINVAL, "NULL or device already added");
  CUdevice dev;
  const cm_status s = current_device(&dev, &m->device);
  if (s != CM_OK) return s;
  const CUresult r = drv().mc_add(m->mc, dev);
  if (r != CUDA_SUCCESS) return cu_fail(r, "cuMulticastAddDevice");
  m->added = true;
  return CM_OK;
}

cm_status cm_mc_bind(cm_mc* m, void** uc_ptr, void** mc_ptr) {
  if (!m || !uc_ptr || !mc_ptr || !m->added || m->bound) return mc_fail(CM_EINVAL, "bad arguments or state");
  const Driver& d = drv();
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = m->device;
  size_t g = 0;
  CUresult r = d.mem_gran(&g, &ap, CU_MEM_ALLOC_GRANULARITY_MINIMUM);
  if (r != CUDA_SUCCESS) return cu_fail(r, "cuMemGetAllocationGranularity");
  if (m->size % g) return mc_fail(CM_EINVAL, "multicast size not a multiple of the allocation granularity");
  if ((r = d.mem_create(&m->mem, m->size, &ap, 0)) != CUDA_SUCCESS) return cu_fail(r, "cuMemCreate");
  if ((r = d.mc_bind(m->mc, 0, m->mem, 0, m->size, 0)) != CUDA_SUCCESS) return cu_fail(r, "cuMulticastBindMem");
  m->bound = true;
  CUmemAccessDesc acc = {};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = m->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if ((r = d.va_reserve(&m->uc, m->size, 0, 0, 0)) != CUDA_SUCCESS) return cu_fail(r, "cuMemAddressReserve");
  if ((r = d.map(m->uc, m->size, 0, m->mem, 0)) != CUDA_SUCCESS) return cu_fail(r, "cuMemMap (unicast)");
  if ((r = d.set_access(m->uc, m->size, &acc, 1)) != CUDA_SUCCESS) return cu_fail(r, "cuMemSetAccess (unicast)");
  if ((r = d.va_reserve(&m->mcva, m->size, 0, 0, 0)) != CUDA_SUCCESS) return cu_fail(r, "cuMemAddressReserve");
  if ((r = d.map(m->mcva, m->size, 0, m->mc, 0)) != CUDA_SUCCESS) return cu_fail(r, "cuMemMap (multicast)");
  if ((r = d.set_access(m->mcva, m->size, &acc, 1)) != CUDA_SUCCESS) return cu_fail(r, "cuMemSetAccess (multicast)");
  *uc_ptr = reinterpret_cast<void*>(m->uc);
  *mc_ptr = reinterpret_cast<void*>(m->mcva);
  return CM_OK;
}

void cm_mc_destroy(cm_mc* m) {
  if (!m) return;
  const Driver& d = drv();
  if (d.ok()) {
    cudaDeviceSynchronize();
    if (m->mcva) {
      d.unmap(m->mcva, m->size);
      d.va_free(m->mcva, m->size);
    }
    if (m->uc) {
      d.unmap(m->uc, m->size);
      d.va_free(m->uc, m->size);
    }
    if (m->bound) {
      CUdevice dev;
      if (d.dev_get(&dev, m->device) == CUDA_SUCCESS) d.mc_unbind(m->mc, dev, 0, m->size);
    }
    if (m->mem) d.release(m->mem);
    if (m->mc) d.release(m->mc);
  }
  delete m;
}

}  // extern "C"
