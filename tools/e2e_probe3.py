"""Round-trip latency of a small kernel + host wait, and of an 8-byte D2H to
pinned memory, alone and while a 112 MB D2H / H2D runs on another stream."""
import sys
import time
import torch
s = torch.cuda.current_stream()
cs = torch.cuda.Stream()
big_d = torch.empty(112_500_000 // 8, dtype=torch.float64, device="cuda")
big_h = torch.empty(112_500_000 // 8, dtype=torch.float64).pin_memory()
small_d = torch.zeros(1, dtype=torch.float64, device="cuda")
small_h = torch.zeros(1, dtype=torch.float64).pin_memory()


def rt_kernel(n=200):
    t = time.perf_counter()
    for _ in range(n):
        small_d.add_(1.0)
        s.synchronize()
    return (time.perf_counter() - t) / n * 1e6


def rt_d2h(n=200):
    t = time.perf_counter()
    for _ in range(n):
        small_d.add_(1.0)
        small_h.copy_(small_d, non_blocking=True)
        s.synchronize()
    return (time.perf_counter() - t) / n * 1e6


for label, fn in (("kernel+sync", rt_kernel), ("kernel+8B d2h+sync", rt_d2h)):
    fn(20)
    base = fn()
    res = {}
    for kind in ("d2h", "h2d"):
        torch.cuda.synchronize()
        with torch.cuda.stream(cs):
            for _ in range(40):
                if kind == "d2h":
                    big_h.copy_(big_d, non_blocking=True)
                else:
                    big_d.copy_(big_h, non_blocking=True)
        res[kind] = fn(100)
        torch.cuda.synchronize()
    print(f"{label:22s} alone {base:7.1f} us   under big D2H {res['d2h']:8.1f} us   "
          f"under big H2D {res['h2d']:8.1f} us")
