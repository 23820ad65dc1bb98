"""Probe NVLS multicast object creation on this box (every handle type x granularity; tools only)."""
import torch
from cuda.bindings import driver as drv
torch.cuda.init(); torch.zeros(1, device="cuda")
print("cuInit", drv.cuInit(0))
err, dev = drv.cuDeviceGet(0)
for a in ["CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED", "CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED"]:
    try: print(a, drv.cuDeviceGetAttribute(getattr(drv.CUdevice_attribute, a), dev))
    except Exception as e: print(a, "ERR", e)
print("driver", drv.cuDriverGetVersion())
for ht_name in ["CU_MEM_HANDLE_TYPE_NONE", "CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR", "CU_MEM_HANDLE_TYPE_FABRIC"]:
    ht = getattr(drv.CUmemAllocationHandleType, ht_name)
    for flagname in ["CU_MULTICAST_GRANULARITY_MINIMUM", "CU_MULTICAST_GRANULARITY_RECOMMENDED"]:
        p = drv.CUmulticastObjectProp(); p.numDevices = 1; p.handleTypes = ht; p.size = 1 << 21
        r = drv.cuMulticastGetGranularity(p, getattr(drv.CUmulticastGranularity_flags, flagname))
        print(ht_name, flagname, "gran", r)
        if r[0] == drv.CUresult.CUDA_SUCCESS:
            g = r[1]; p.size = max(g, 1 << 21) // g * g
            c = drv.cuMulticastCreate(p)
            print("   create size", p.size, c[0])
            if c[0] == drv.CUresult.CUDA_SUCCESS:
                print("   adddev", drv.cuMulticastAddDevice(c[1], dev))
                drv.cuMemRelease(c[1])
