"""Multicast (NVLS) probe v2: cuMulticastCreate with 1 device under each handle type."""
from cuda.bindings import driver as cu
def ck(r):
    e = r[0] if isinstance(r, tuple) else r
    return e, (r[1:] if isinstance(r, tuple) else None)
cu.cuInit(0)
_, (dev,) = ck(cu.cuDeviceGet(0))
_, (ctx,) = ck(cu.cuDevicePrimaryCtxRetain(dev)); cu.cuCtxSetCurrent(ctx)
for name in ("CU_MEM_HANDLE_TYPE_NONE", "CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR", "CU_MEM_HANDLE_TYPE_FABRIC"):
    prop = cu.CUmulticastObjectProp()
    prop.numDevices = 1
    prop.handleTypes = getattr(cu.CUmemAllocationHandleType, name)
    e, g = ck(cu.cuMulticastGetGranularity(prop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_MINIMUM))
    print(name, "granularity", e, g)
    prop.size = g[0] if g else (2 << 20)
    e, mc = ck(cu.cuMulticastCreate(prop))
    print(name, "create", e)
    if mc:
        e2, _ = ck(cu.cuMulticastAddDevice(mc[0], dev))
        print(name, "add device", e2)
