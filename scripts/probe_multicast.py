#!/usr/bin/env python
"""Probe: can this box build an NVLS multicast object over ONE GPU (CUDA driver API), so that a
multimem.red epilogue can be tested on a single B200?  Prints each step's status (no state kept)."""
import ctypes

import cuda.bindings.driver as cu


def ck(r, what):
    err = r[0] if isinstance(r, tuple) else r
    print(f"{what}: {err}")
    if err != cu.CUresult.CUDA_SUCCESS:
        raise SystemExit(1)
    return r[1] if isinstance(r, tuple) and len(r) > 1 else None


ck(cu.cuInit(0), "cuInit")
dev = ck(cu.cuDeviceGet(0), "cuDeviceGet")
ctx = ck(cu.cuDevicePrimaryCtxRetain(dev), "retain")
ck(cu.cuCtxSetCurrent(ctx), "setcurrent")
sup = ck(cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev), "attr multicast")
print("multicast supported:", sup)
prop = cu.CUmulticastObjectProp()
prop.numDevices = 1
prop.handleTypes = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
gran = ck(cu.cuMulticastGetGranularity(prop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED), "granularity")
print("granularity", gran)
size = max(int(gran), 2 << 20)
prop.size = size
mc = ck(cu.cuMulticastCreate(prop), "cuMulticastCreate")
ck(cu.cuMulticastAddDevice(mc, dev), "cuMulticastAddDevice")
ap = cu.CUmemAllocationProp()
ap.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
ap.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
ap.location.id = 0
ap.requestedHandleTypes = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
mem = ck(cu.cuMemCreate(size, ap, 0), "cuMemCreate")
ck(cu.cuMulticastBindMem(mc, 0, mem, 0, size, 0), "cuMulticastBindMem")
va = ck(cu.cuMemAddressReserve(size, 0, 0, 0), "reserve mc va")
ck(cu.cuMemMap(va, size, 0, mc, 0), "map mc")
acc = cu.CUmemAccessDesc()
acc.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
acc.location.id = 0
acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
ck(cu.cuMemSetAccess(va, size, [acc], 1), "set access mc")
print("multicast VA", hex(int(va)))
print("OK: single-GPU multicast object works")
