"""Is torch pinned memory seen as page-locked by the driver, and how fast is
the library's H2D from it vs pageable memory?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from cuda.bindings import driver as cu
torch.cuda.init()
x = torch.empty(2_270_000 // 4, dtype=torch.int32).pin_memory()
a = x.numpy()
err, mt = cu.cuPointerGetAttribute(cu.CUpointer_attribute.CU_POINTER_ATTRIBUTE_MEMORY_TYPE, a.ctypes.data)
print("driver sees memory type:", err, mt)
d = torch.empty_like(x, device="cuda")
for name, src in (("pinned", x), ("pageable", torch.from_numpy(np.array(a)))):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(20):
        d.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    print(name, "torch H2D GB/s", 20 * x.numel() * 4 / (time.perf_counter() - t) / 1e9)
