"""Probe multicast (NVLS) support on the box: device attribute + a 1-device multicast object."""
import os, subprocess
print(subprocess.run(["nvidia-smi", "-L"], capture_output=True, text=True).stdout)
print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout)
print("CUDA_VISIBLE_DEVICES", os.environ.get("CUDA_VISIBLE_DEVICES"))
from cuda.bindings import driver as cu
def ck(r):
    e = r[0] if isinstance(r, tuple) else r
    if e != cu.CUresult.CUDA_SUCCESS:
        raise RuntimeError(str(e))
    return r[1:] if isinstance(r, tuple) and len(r) > 1 else None
ck(cu.cuInit(0))
(dev,) = ck(cu.cuDeviceGet(0))
for a in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
          "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED"):
    try:
        print(a, ck(cu.cuDeviceGetAttribute(getattr(cu.CUdevice_attribute, a), dev)))
    except Exception as ex:
        print(a, "ERR", ex)
(ctx,) = ck(cu.cuDevicePrimaryCtxRetain(dev)); ck(cu.cuCtxSetCurrent(ctx))
prop = cu.CUmulticastObjectProp()
prop.numDevices = 1
prop.size = 2 << 20
prop.handleTypes = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
try:
    (g,) = ck(cu.cuMulticastGetGranularity(prop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
    print("mc granularity", g)
    (mc,) = ck(cu.cuMulticastCreate(prop))
    ck(cu.cuMulticastAddDevice(mc, dev))
    print("multicast object created + device added OK")
except Exception as ex:
    print("multicast ERR", ex)
