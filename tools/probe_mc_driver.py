"""Probe: single-device multicast object via the driver API (cuda-python)."""
import ctypes

import torch
from cuda.bindings import driver as cu


def ok(r):
    if isinstance(r, tuple):
        err, *rest = r
    else:
        err, rest = r, []
    assert err == cu.CUresult.CUDA_SUCCESS, err
    return rest[0] if len(rest) == 1 else rest


torch.cuda.init()
ok(cu.cuInit(0))
dev = ok(cu.cuDeviceGet(0))
ctx = ok(cu.cuDevicePrimaryCtxRetain(dev))
ok(cu.cuCtxSetCurrent(ctx))
H = cu.CUmemAllocationHandleType
for nd, ht in ((1, H.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR), (2, H.CU_MEM_HANDLE_TYPE_NONE),
               (2, H.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR), (2, H.CU_MEM_HANDLE_TYPE_FABRIC),
               (1, H.CU_MEM_HANDLE_TYPE_FABRIC | H.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR)):
    prop = cu.CUmulticastObjectProp()
    prop.numDevices = nd
    prop.size = 2 << 20
    prop.handleTypes = ht
    r = cu.cuMulticastGetGranularity(prop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
    print("granularity", ht, r)
    r = cu.cuMulticastCreate(prop)
    print("create", nd, ht, r[0])
    if r[0] != cu.CUresult.CUDA_SUCCESS:
        continue
    mc = r[1]
    print("add device", cu.cuMulticastAddDevice(mc, dev))
    aprop = cu.CUmemAllocationProp()
    aprop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    aprop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    aprop.location.id = 0
    aprop.requestedHandleTypes = ht
    r = cu.cuMemCreate(2 << 20, aprop, 0)
    print("memcreate", r[0])
    mem = r[1]
    print("bind", cu.cuMulticastBindMem(mc, 0, mem, 0, 2 << 20, 0))
    va = ok(cu.cuMemAddressReserve(2 << 20, 2 << 20, 0, 0))
    print("map mc", cu.cuMemMap(va, 2 << 20, 0, mc, 0))
    acc = cu.CUmemAccessDesc()
    acc.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    acc.location.id = 0
    acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
    print("access", cu.cuMemSetAccess(va, 2 << 20, [acc], 1))
    print("mc va", hex(int(va)))
