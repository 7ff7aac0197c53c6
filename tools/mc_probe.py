"""Probe one-device multicast-object creation on the GPU box (cuda-python
driver API): which handle types / sizes cuMulticastCreate accepts."""
from cuda.bindings import driver as cu

cu.cuInit(0)
_, dev = cu.cuDeviceGet(0)
_, ctx = cu.cuDevicePrimaryCtxRetain(dev)
cu.cuCtxSetCurrent(ctx)
for name in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED",):
    print(name, cu.cuDeviceGetAttribute(getattr(cu.CUdevice_attribute, name), dev))
for nd in (1, 2):
    for ht in (0, 1, 8):
        mp = cu.CUmulticastObjectProp()
        mp.numDevices = nd
        mp.handleTypes = ht
        mp.size = 1 << 21
        e, g = cu.cuMulticastGetGranularity(mp, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
        e2, gmin = cu.cuMulticastGetGranularity(mp, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_MINIMUM)
        for size in (g if g else 1 << 21, 1 << 29):
            mp.size = size
            r, h = cu.cuMulticastCreate(mp)
            print(f"numDevices={nd} handleTypes={ht} gran={g} ({e}) min={gmin} size={size}: create={r}")
            if r == cu.CUresult.CUDA_SUCCESS:
                print("  add:", cu.cuMulticastAddDevice(h, dev))
                cu.cuMemRelease(h)
