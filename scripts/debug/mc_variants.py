from cuda.bindings import driver as cu
cu.cuInit(0)
_, dev = cu.cuDeviceGet(0)
_, ctx = cu.cuDevicePrimaryCtxRetain(dev)
cu.cuCtxSetCurrent(ctx)
for nd in (1, 2):
    for ht in ("CU_MEM_HANDLE_TYPE_FABRIC", "CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR", "CU_MEM_HANDLE_TYPE_NONE"):
        p = cu.CUmulticastObjectProp()
        p.numDevices = nd
        p.size = 2 << 20
        p.handleTypes = getattr(cu.CUmemAllocationHandleType, ht)
        r, g = cu.cuMulticastGetGranularity(p, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
        p.size = ((2 << 20) + g - 1) // g * g
        r2, h = cu.cuMulticastCreate(p)
        print(nd, ht, "gran", r, g, "create", r2)
