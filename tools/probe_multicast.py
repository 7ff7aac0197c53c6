"""Probe NVLS / multicast support on the GPU box (one GPU): the device
attribute, and whether torch symmetric memory hands out a multicast pointer
for a one-rank group (what a multimem.ld_reduce kernel needs)."""
import json
import os
import sys

out = {}
try:
    from cuda.bindings import driver as cu
    cu.cuInit(0)
    err, dev = cu.cuDeviceGet(0)
    for name in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED",
                 "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
                 "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED"):
        attr = getattr(cu.CUdevice_attribute, name, None)
        if attr is not None:
            e, v = cu.cuDeviceGetAttribute(attr, dev)
            out[name] = (str(e), v)
except Exception as ex:  # noqa: BLE001
    out["driver_error"] = repr(ex)

try:
    import torch
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    t = symm.empty(1 << 20, dtype=torch.uint8, device="cuda")
    h = symm.rendezvous(t, dist.group.WORLD)
    out["symm_world"] = h.world_size
    out["symm_buffer_ptr0"] = int(h.buffer_ptrs[0])
    mc = getattr(h, "multicast_ptr", None)
    out["symm_multicast_ptr"] = int(mc) if mc is not None else None
    out["has_multicast_support"] = bool(symm.is_nvshmem_available()) if hasattr(symm, "is_nvshmem_available") else None
    dist.destroy_process_group()
except Exception as ex:  # noqa: BLE001
    out["symm_error"] = repr(ex)[:400]

print(json.dumps(out, indent=1))
sys.stdout.flush()
