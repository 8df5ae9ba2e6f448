"""Device L2 persistence limits (cudaDevAttrMaxPersistingL2CacheSize, max access-policy window)."""
import torch
from cuda.bindings import runtime as rt
for name in ["cudaDevAttrL2CacheSize", "cudaDevAttrMaxPersistingL2CacheSize", "cudaDevAttrMaxAccessPolicyWindowSize"]:
    err, v = rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, name), 0)
    print(name, err, v)
