#!/usr/bin/env python
"""Probe cuMulticastCreate parameter combinations on this box (diagnostic, not product code)."""
import json
from cuda.bindings import driver as cu
import torch

torch.cuda.init()
torch.zeros(1, device="cuda")
cu.cuInit(0)
err, dev = cu.cuDeviceGet(0)
out = {}
for name in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED"):
    try:
        e, v = cu.cuDeviceGetAttribute(getattr(cu.CUdevice_attribute, name), dev)
        out[name] = (str(e), int(v))
    except Exception as ex:
        out[name] = repr(ex)
HT = {"fabric": cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_FABRIC,
      "posix": cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
      "none": cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_NONE}
res = []
for nd in (1, 2):
    for hn, ht in HT.items():
        for size in (2 << 20, 64 << 20, 512 << 20):
            p = cu.CUmulticastObjectProp()
            p.numDevices = nd
            p.size = size
            p.handleTypes = ht
            p.flags = 0
            eg, g = cu.cuMulticastGetGranularity(p, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_MINIMUM)
            ec, h = cu.cuMulticastCreate(p)
            ok = ec == cu.CUresult.CUDA_SUCCESS
            eadd = None
            if ok:
                eadd = str(cu.cuMulticastAddDevice(h, dev)[0])
                cu.cuMemRelease(h)
            res.append({"nd": nd, "ht": hn, "size": size, "gran": (str(eg), int(g) if g is not None else None),
                        "create": str(ec), "add": eadd})
out["combos"] = res
print(json.dumps(out, indent=1))
