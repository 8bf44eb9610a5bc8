"""Probe multicast / symmetric-memory support on the box (1 GPU)."""
import os
import sys

import torch

print("torch", torch.__version__)
try:
    from cuda.bindings import driver as cu
except Exception:
    try:
        from cuda import cuda as cu
    except Exception as e:
        cu = None
        print("no cuda-python", e)
if cu is not None:
    cu.cuInit(0)
    err, dev = cu.cuDeviceGet(0)
    for name in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED",
                 "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED"):
        attr = getattr(cu.CUdevice_attribute, name, None)
        if attr is not None:
            print(name, cu.cuDeviceGetAttribute(attr, dev))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
import torch.distributed as dist
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
try:
    import torch.distributed._symmetric_memory as symm
    t = symm.empty(1024, dtype=torch.float32, device="cuda")
    h = symm.rendezvous(t, dist.group.WORLD.group_name)
    print("symm handle", type(h), "multicast_ptr", getattr(h, "multicast_ptr", None),
          "world", h.world_size)
except Exception as e:
    print("symm failed:", repr(e)[:300])
dist.destroy_process_group()
