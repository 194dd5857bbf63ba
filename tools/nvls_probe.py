"""Probe NVSwitch multicast support per device (CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED)
and the multicast granularity, through cuda-python."""
from cuda.bindings import driver as cu
import sys
err, = cu.cuInit(0)
n = cu.cuDeviceGetCount()[1]
for d in range(n):
    dev = cu.cuDeviceGet(d)[1]
    r = cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
    f = cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev)
    p = cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED, dev)
    print("dev", d, "multicast", r, "fabric", f, "posix_fd", p)
ctx = cu.cuDevicePrimaryCtxRetain(cu.cuDeviceGet(0)[1])[1]
cu.cuCtxSetCurrent(ctx)
prop = cu.CUmulticastObjectProp()
prop.numDevices = n
prop.size = 2 << 20
prop.handleTypes = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
print("gran", cu.cuMulticastGetGranularity(prop, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
res = cu.cuMulticastCreate(prop)
print("create", res)
