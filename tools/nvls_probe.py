#!/usr/bin/env python
"""Probe: can this box give an NVLink-SHARP multicast address (NVLS) for the
per-budget keys?  Checks CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED and torch symmetric memory's
multicast pointer at world size 1.  Measurement tool, not product code.

    python tools/nvls_probe.py
"""
import json
import os

import torch
import torch.distributed as dist

out = {}
try:
    from cuda.bindings import driver as cu
    cu.cuInit(0)
    err, dev = cu.cuDeviceGet(0)
    err, v = cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
    out["multicast_supported_attr"] = int(v)
    out["attr_err"] = str(err)
except Exception as ex:  # pragma: no cover
    out["attr_error"] = repr(ex)
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29577")
try:
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    import torch.distributed._symmetric_memory as symm
    out["backend"] = str(symm.get_backend(torch.device("cuda", 0))) if hasattr(symm, "get_backend") else None
    t = symm.empty(64, dtype=torch.int64, device="cuda")
    h = symm.rendezvous(t, dist.group.WORLD.group_name)
    out["multicast_ptr"] = int(getattr(h, "multicast_ptr", 0) or 0)
    out["buffer_ptr"] = int(t.data_ptr())
    out["world"] = int(h.world_size)
    out["has_multicast"] = bool(out["multicast_ptr"])
except Exception as ex:  # pragma: no cover
    out["symm_error"] = repr(ex)[:400]
print(json.dumps(out))
try:
    dist.destroy_process_group()
except Exception:
    pass
