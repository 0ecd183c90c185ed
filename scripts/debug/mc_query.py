from cuda import cuda
cuda.cuInit(0)
err, dev = cuda.cuDeviceGet(0)
for name in ["CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED", "CU_DEVICE_ATTRIBUTE_VIRTUAL_MEMORY_MANAGEMENT_SUPPORTED"]:
    a = getattr(cuda.CUdevice_attribute, name)
    print(name, cuda.cuDeviceGetAttribute(a, dev))
