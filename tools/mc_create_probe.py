"""Probe: can a one-device multicast object be created on this box?"""
import torch
from cuda.bindings import driver as drv

torch.zeros(1, device="cuda:0")
drv.cuInit(0)
_, dev = drv.cuDeviceGet(0)
print("multicast supported:", drv.cuDeviceGetAttribute(drv.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev))
print("fabric handle supported:", drv.cuDeviceGetAttribute(drv.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev))
H = drv.CUmemAllocationHandleType
for name, ht in (("none", 0), ("posix_fd", H.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR), ("fabric", H.CU_MEM_HANDLE_TYPE_FABRIC)):
    for nd in (1, 2):
        mp = drv.CUmulticastObjectProp()
        mp.numDevices = nd
        mp.handleTypes = ht
        mp.size = 2 << 20
        g = drv.cuMulticastGetGranularity(mp, drv.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
        mp.size = max(int(g[1]) if g[0] == drv.CUresult.CUDA_SUCCESS else 2 << 20, 2 << 20)
        r = drv.cuMulticastCreate(mp)
        print(name, "numDevices", nd, "granularity", g, "create", r[0])
