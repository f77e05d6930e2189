"""H2D of one bench batch (S=4096, 6-D gamma_k: ~2.3 MB in 4 arrays) from
pinned and pageable host memory, timed with CUDA events."""
import numpy as np
import torch

sizes = [(4096, np.float64), (140_000, np.int32), (140_000, np.int32), (140_000, np.float64)]
for mode in ("pinned", "pageable"):
    hs = []
    for n, dt in sizes:
        t = torch.from_numpy(np.ones(n, dt))
        hs.append(t.pin_memory() if mode == "pinned" else t)
    ds = [torch.empty_like(h, device="cuda") for h in hs]
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for h, d in zip(hs, ds):
            d.copy_(h, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        nb = sum(h.numel() * h.element_size() for h in hs)
        ms = e0.elapsed_time(e1)
        print(f"{mode}: {nb / 1e6:.2f} MB in {ms * 1e3:.1f} us = {nb / ms / 1e6:.1f} GB/s")
big = torch.ones(256 << 20, dtype=torch.uint8).pin_memory()
dbig = torch.empty_like(big, device="cuda")
for rep in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); dbig.copy_(big, non_blocking=True); e1.record(); torch.cuda.synchronize()
    print(f"pinned 256 MB: {256 * 1.048576 / e0.elapsed_time(e1):.1f} GB/s")
