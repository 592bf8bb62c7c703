"""Time a prototype specialized pass kernel (cubin) on a 24-qubit state."""
import ctypes
import json
import sys

import numpy as np
import torch
import cuda.bindings.driver as cu

cubin = open(sys.argv[1], "rb").read()
js = json.load(open(sys.argv[2]))
nops = len(js["ops"])
x = torch.randn(2 << 24, dtype=torch.float64, device="cuda")
cu.cuInit(0)
err, mod = cu.cuModuleLoadData(cubin)
assert err == cu.CUresult.CUDA_SUCCESS, err
err, fn = cu.cuModuleGetFunction(mod, b"kpass")
cu.cuFuncSetAttribute(fn, cu.CUfunction_attribute.CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES, 65536)
size = (8 + nops * 64 + 15) // 16 * 16
P = np.zeros(size, dtype=np.uint8)
m = np.zeros((nops, 8))
for o, op in enumerate(js["ops"]):
    m[o] = op["m"]
P[8:8 + nops * 64] = np.frombuffer(m.tobytes(), dtype=np.uint8)
ptr = ctypes.c_uint64(x.data_ptr())
args = (ctypes.c_void_p * 2)(P.ctypes.data, ctypes.addressof(ptr))
stream = torch.cuda.current_stream().cuda_stream
def launch():
    r = cu.cuLaunchKernel(fn, 4096, 1, 1, 256, 1, 1, 65536, stream, ctypes.addressof(args), 0)
    assert r[0] == cu.CUresult.CUDA_SUCCESS, r
for _ in range(3):
    launch()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    launch()
e1.record()
torch.cuda.synchronize()
print(json.dumps({"kernel_us": e0.elapsed_time(e1) * 1000 / 20}))
