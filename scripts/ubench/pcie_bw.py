"""PCIe copy bandwidth of this box (pinned host <-> HBM), one direction and both at once."""
import torch

n = 256 * 1024 * 1024
h1 = torch.empty(n, dtype=torch.uint8).pin_memory()
h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
d1 = torch.empty(n, dtype=torch.uint8, device="cuda")
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 5


def h2d():
    with torch.cuda.stream(s1):
        d1.copy_(h1, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)


def d2h():
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)


def both():
    h2d()
    d2h()


for name, fn, b in (("H2D", h2d, n), ("D2H", d2h, n), ("H2D+D2H concurrent", both, 2 * n)):
    ms = timed(fn)
    print(f"{name:20s} {ms:7.3f} ms  {b / ms / 1e6:7.1f} GB/s")
